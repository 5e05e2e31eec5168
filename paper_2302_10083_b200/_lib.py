"""ctypes binding of libdqmc.so (the C ABI declared in include/dqmc.h).

The shared library is built in-tree by __graft_entry__.build() and must be
present: there is no CPU fallback. Loading fails loudly if it is missing, and
every call that needs a GPU raises if no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdqmc.so")

DQMC_OK = 0
DQMC_ERR_INVALID = 1
DQMC_ERR_RESOURCE = 2
DQMC_ERR_CUDA = 3
DQMC_ERR_NODEVICE = 4

FLAG_KEEP_BITMAP = 1
FLAG_TIMING = 2
FLAG_COUNT_ONLY = 4
FLAG_ASYNC = 8

IN_WORDS = 0
IN_U8 = 1

# every symbol include/dqmc.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "dqmc_abi_version",
    "dqmc_last_error",
    "dqmc_device_count",
    "dqmc_set_device",
    "dqmc_block_bits",
    "dqmc_state_bytes",
    "dqmc_device_bytes",
    "dqmc_primes_tt",
    "dqmc_primes_u8",
    "dqmc_free_result",
    "dqmc_submit_tt",
    "dqmc_submit_u8",
    "dqmc_collect",
    "dqmc_host_threads",
    "dqmc_widen_host",
    "dqmc_primes_device",
    "dqmc_last_timings",
    "dqmc_last_pass_bytes",
    "dqmc_bitmap_device",
    "dqmc_bitmap_download",
    "dqmc_gen3_device",
    "dqmc_gen3_range_device",
    "dqmc_gen3_host",
    "dqmc_gen_sbox_device",
    "dqmc_gen_sbox_host",
    "dqmc_ipc_get",
    "dqmc_ipc_open",
    "dqmc_ipc_close",
    "dqmc_order_by_weight",
    "dqmc_merge_device",
    "dqmc_reduce_low_device",
    "dqmc_extract_kills_device",
    "dqmc_bitop_batch_device",
    "dqmc_bitop_device",
    "dqmc_plan",
    "dqmc_release",
    "dqmc_engine_generation",
    "dqmc_engine_enter",
    "dqmc_engine_exit",
    "dqmc_gather_threshold",
    "dqmc_last_gather",
    "dqmc_launch_count",
    "dqmc_sparse_primes_tt",
    "dqmc_state_create",
    "dqmc_state_free",
    "dqmc_state_info",
    "dqmc_state_load_tt",
    "dqmc_state_set_words",
    "dqmc_state_get_words",
    "dqmc_state_run_pass",
    "dqmc_state_run_merge_reduce",
    "dqmc_state_padding_zero",
    "dqmc_state_extract",
    "dqmc_state_equal",
    "dqmc_state_copy",
)


class DqmcResult(ctypes.Structure):
    _fields_ = [
        ("count", ctypes.c_int64),
        ("ranks", ctypes.POINTER(ctypes.c_int64)),
        ("_owner", ctypes.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libdqmc.so once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
            )
        L = ctypes.CDLL(LIB_PATH)
        i32, i64, u32, u64, vp, dbl = (
            ctypes.c_int,
            ctypes.c_int64,
            ctypes.c_uint32,
            ctypes.c_uint64,
            ctypes.c_void_p,
            ctypes.c_double,
        )
        sig = {
            "dqmc_abi_version": (i32, []),
            "dqmc_last_error": (ctypes.c_char_p, []),
            "dqmc_device_count": (i32, []),
            "dqmc_set_device": (i32, [i32]),
            "dqmc_block_bits": (u64, [i32]),
            "dqmc_state_bytes": (u64, [i32, i32]),
            "dqmc_device_bytes": (u64, [i32]),
            "dqmc_primes_tt": (i32, [vp, i32, i32, u64, u32, ctypes.POINTER(DqmcResult)]),
            "dqmc_primes_u8": (i32, [vp, i32, i32, u64, u32, ctypes.POINTER(DqmcResult)]),
            "dqmc_free_result": (None, [ctypes.POINTER(DqmcResult)]),
            "dqmc_submit_tt": (i32, [vp, i32, u32, ctypes.POINTER(ctypes.c_int64)]),
            "dqmc_submit_u8": (i32, [vp, i32, u32, ctypes.POINTER(ctypes.c_int64)]),
            "dqmc_collect": (i32, [ctypes.c_int64, ctypes.POINTER(DqmcResult)]),
            "dqmc_host_threads": (i32, [i32]),
            "dqmc_widen_host": (None, [vp, vp, vp, i64, i64, i64, i64, i64, i64]),
            "dqmc_primes_device": (i32, [vp, i32, i32, vp, i64, ctypes.POINTER(ctypes.c_int64), u32, vp]),
            "dqmc_last_timings": (i32, [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float), i32]),
            "dqmc_last_pass_bytes": (i32, [ctypes.POINTER(ctypes.c_uint64), i32]),
            "dqmc_bitmap_device": (i32, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_uint64)]),
            "dqmc_bitmap_download": (i32, [vp, u64]),
            "dqmc_state_create": (i32, [i32, i32, u64, ctypes.POINTER(ctypes.c_void_p)]),
            "dqmc_state_free": (None, [vp]),
            "dqmc_state_info": (i32, [vp, ctypes.POINTER(ctypes.c_int64)]),
            "dqmc_state_load_tt": (i32, [vp, vp]),
            "dqmc_state_set_words": (i32, [vp, vp, u64]),
            "dqmc_state_get_words": (i32, [vp, vp, u64]),
            "dqmc_state_run_pass": (i32, [vp, i32, vp, i32, vp]),
            "dqmc_state_run_merge_reduce": (i32, [vp]),
            "dqmc_state_padding_zero": (i32, [vp, ctypes.POINTER(ctypes.c_int)]),
            "dqmc_state_extract": (i32, [vp, vp, i64, ctypes.POINTER(ctypes.c_int64)]),
            "dqmc_state_equal": (i32, [vp, vp, ctypes.POINTER(ctypes.c_int)]),
            "dqmc_state_copy": (i32, [vp, ctypes.POINTER(ctypes.c_void_p)]),
            "dqmc_gen3_device": (i32, [vp, i32, dbl, dbl, u64, vp]),
            "dqmc_gen3_range_device": (i32, [vp, i64, i64, dbl, dbl, u64, vp]),
            "dqmc_gen3_host": (i32, [vp, i32, dbl, dbl, u64]),
            "dqmc_gen_sbox_device": (i32, [vp, u64, vp]),
            "dqmc_gen_sbox_host": (i32, [vp, u64]),
            "dqmc_ipc_get": (i32, [vp, vp, ctypes.POINTER(ctypes.c_uint64)]),
            "dqmc_ipc_open": (i32, [vp, ctypes.POINTER(ctypes.c_void_p)]),
            "dqmc_ipc_close": (i32, [vp]),
            "dqmc_order_by_weight": (i32, [vp, i64, i32, vp]),
            "dqmc_merge_device": (i32, [vp, i32, i32, vp, vp]),
            "dqmc_reduce_low_device": (i32, [vp, i32, i64, vp]),
            "dqmc_extract_kills_device": (i32, [vp, i32, i64, vp, vp, vp, i64, vp, vp, ctypes.POINTER(ctypes.c_int64),
                                                u32, vp]),
            "dqmc_bitop_batch_device": (i32, [vp, i64, u64, i32, vp]),
            "dqmc_bitop_device": (i32, [vp, vp, vp, u64, i32, vp]),
            "dqmc_plan": (i32, [i32, ctypes.POINTER(ctypes.c_int64), i32]),
            "dqmc_release": (None, []),
            "dqmc_engine_generation": (u64, []),
            "dqmc_engine_enter": (i32, [vp]),
            "dqmc_engine_exit": (i32, [vp]),
            "dqmc_gather_threshold": (i32, [i32]),
            "dqmc_launch_count": (u64, []),
            "dqmc_last_gather": (i32, [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_int)]),
            "dqmc_sparse_primes_tt": (i32, [vp, i32, u64, ctypes.POINTER(DqmcResult)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
        return _lib


def last_error() -> str:
    msg = load().dqmc_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a status code to the reference's exception types (errors.py)."""
    if rc == DQMC_OK:
        return
    msg = last_error()
    if rc == DQMC_ERR_INVALID:
        raise ValueError(msg)
    if rc == DQMC_ERR_RESOURCE:
        raise errors.ResourceLimitError(msg)
    if rc == DQMC_ERR_NODEVICE:
        raise RuntimeError(f"CUDA device required: {msg}")
    raise RuntimeError(f"libdqmc CUDA error: {msg}")


def result_to_array(res: DqmcResult) -> np.ndarray:
    """Zero-copy int64 view of a pinned result; freed when the array dies."""
    L = load()
    count = int(res.count)
    if count == 0 or not res.ranks:
        L.dqmc_free_result(ctypes.byref(res))
        return np.zeros(0, dtype=np.int64)
    addr = ctypes.cast(res.ranks, ctypes.c_void_p).value
    base_t = ctypes.c_int64 * count

    class _PinnedRanks(base_t):  # owns the pinned buffer; frees it on collection
        _res = res

        def __del__(self, _free=L.dqmc_free_result, _res=res):
            _free(ctypes.byref(_res))

    buf = _PinnedRanks.from_address(addr)
    return np.frombuffer(buf, dtype=np.int64)


def timings() -> list[tuple[str, float, int]]:
    """(kernel name, ms, algorithmic bytes) of each pass of the last timed call."""
    L = load()
    k = L.dqmc_last_timings(None, None, 0)
    names = (ctypes.c_char_p * max(1, k))()
    ms = (ctypes.c_float * max(1, k))()
    by = (ctypes.c_uint64 * max(1, k))()
    L.dqmc_last_timings(names, ms, k)
    L.dqmc_last_pass_bytes(by, k)
    return [(names[i].decode(), float(ms[i]), int(by[i])) for i in range(k)]


def plan(n: int) -> dict:
    """The engine's pass plan for n variables (host logic; no GPU needed)."""
    out = (ctypes.c_int64 * 32)()
    k = load().dqmc_plan(n, out, 32)
    if k != 32:
        raise ValueError(f"no plan for n={n}")
    v = [int(x) for x in out]
    return dict(
        ne=v[0], H=v[1], g=v[2], T=v[3], m=v[4], r=v[5:13], a=v[13:21],
        ib_C=v[21], ib_E=v[22], ib_D=v[23:31], rank_sub=v[31],
    )
