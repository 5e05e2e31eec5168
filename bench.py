#!/usr/bin/env python
"""Benchmark of the dense prime-implicant path (BASELINE.json metric).

Metric: ternary cells per second, 3^n / t, for "all prime implicants at n"
(BASELINE.json `metric`). Workload at N=1: BASELINE config 4 — n=24, 2^24
uint8 values i.i.d. P(on)=0.75, P(dc)=0.05, rest off, seed 3; the largest
configuration that fits one GPU (config 5, n=27, needs 1 TB). Seeded synthetic
inputs from the reference's frozen generator.

  value  device-resident: the uint8 table is generated in HBM before the
         timed region; a step = the whole engine (pack, merge passes, reduce
         passes, compaction of all prime ranks into an HBM int64 buffer).
  e2e    the public host API with a pinned host input and the int64 rank array
         returned on the host: H2D of the table and D2H of every rank inside
         each timed step. Headline: a batch of max(K, 30) calls through
         stream_prime_ranks (three in flight, call i's D2H overlapping call
         i+1's passes; the batch fills and drains once); single_call: one
         synchronous prime_ranks_from_values call.
  roofline  the dominant kernel's algorithmic bytes per launch / its
         CUDA-event duration vs MEASURED_PEAKS.json hbm_gbs.
  configs  BASELINE configs 1-3 (n = 10, 16, 20): wall time to all prime
         implicants through the drop-in call (t_api: host table -> host int64
         ranks) and device-resident (t_device), each with the CPU times beside
         it: the oracle port on 1 thread and on all threads, and the reference
         package itself (implicants.dense_prime_ranks, 1 thread) when it is
         installed in baseline/_ref.
  next_rows  SURVEY.md §8(f) rows against the reference's own code: the GPU
         sparse engine (f4) at low density, the device DenseState path (f2),
         the on-device generator (f3).
  cpu_baseline  the oracle port (C restatement of the reference's dense
         engine, all host threads) on a bounded sample of the same workload,
         with the host CPU model and core count, the reference package's own
         time at n=21 as a cross-check of the port, and the one-off 1-thread
         n=24 measurement (profiles/r2_cpu_n24.json, tools/cpu_n24.py).

--impl reference times the reference's CPU path (the oracle port, all host
threads) on the SAME workload as our arm: full n=24 config-4 calls, one per
step (the step count is capped by a time budget; see run_reference).
Under torchrun (N>1) the engine runs sharded on the top log2(N) variables
(paper_2302_10083_b200.sharded); the reference arm runs on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = dict(n=24, p_on=0.75, p_dc=0.05, seed=3)  # BASELINE config 4
WORKLOAD_NAME = "BASELINE config 4: n=24, P(on)=0.75, P(dc)=0.05, seed 3, all primes as int64 ranks"
E2E_MIN_CALLS = 30  # calls per timed job-stream batch (fill + drain amortised)
METRIC = "ternary cells/s to all prime implicants"
UNIT = "cells/s"


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak_gbs():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region, in
    process through NVML (the data nvidia-smi's clocks query reports; spawning
    nvidia-smi itself stalled the GPU for ~100 ms per call on these boxes)."""

    def __init__(self, device: int, interval: float = 0.05):
        self.device = device
        self.interval = interval
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, mx, rs))
            except Exception:
                pass
            self._stop.wait(self.interval)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["NVML unavailable"]}
        nv = self._nv
        names = {
            "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
            "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
            "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
            "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
        }
        reasons = sorted({k for _, _, r in self.samples for k, bit in names.items() if r & bit})
        return {
            "sm_mhz": statistics.median(s[0] for s in self.samples),
            "sm_max_mhz": max(s[1] for s in self.samples),
            "reasons": reasons,
            "samples": len(self.samples),
            "source": "NVML (nvmlDeviceGetClockInfo / GetCurrentClocksEventReasons)",
        }


def cpu_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem = None
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable"):
                    mem = int(line.split()[1]) * 1024
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "mem_available_bytes": mem}


def config_values_cpu(cfg: int):
    """uint8 values of a BASELINE config from the oracle's generator (CPU leg)."""
    from oracle import gen as G

    return G.config_values(cfg)


def cpu_port_run(n: int, threads: int = 0, values=None) -> tuple[float, int, int]:
    """Oracle port (C restatement of dense.py) on the host cores: (seconds, primes, threads)."""
    from oracle import gen as G
    from oracle import oracle as O

    O.build()
    t = O.set_threads(threads if threads > 0 else (os.cpu_count() or 1))
    v = values if values is not None else G.gen3(n, WORKLOAD["p_on"], WORKLOAD["p_dc"], WORKLOAD["seed"])
    w = G.values_to_words(v)
    t0 = time.perf_counter()
    r = O.dense_prime_ranks(w, n)
    dt = time.perf_counter() - t0
    if values is None:
        _PORT_PRIMES[n] = len(r)
    return dt, len(r), t


_PORT_PRIMES: dict = {}  # n -> prime count of the last port run on the config-4 distribution
REF_PKG = os.path.join(REPO, "baseline", "_ref")
_REF_TIMER = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(1, sys.argv[2])
from implicants import TruthTable, dense_prime_ranks, sparse_prime_ranks
from implicants.dense import extract_ranks, load
from oracle import gen as G


def state_path(tt):  # load -> run_merge_reduce -> extract_ranks (dense.py:317-397)
    st = load(tt)
    st.run_merge_reduce()
    return extract_ranks(st)


ENG = {"dense": dense_prime_ranks, "sparse": sparse_prime_ranks, "state": state_path}
out = {}
for spec in json.loads(sys.argv[3]):
    if "density" in spec:
        n = spec["n"]
        tt = TruthTable(n, G.random_words(n, spec["density"], spec["seed"]))
    else:
        v = G.config_values(spec["cfg"], spec.get("n"))
        n = len(v).bit_length() - 1
        tt = TruthTable.from_bools(n, v != 0)
    f = ENG[spec.get("engine", "dense")]
    best, cnt = None, 0
    for _ in range(spec["reps"]):
        t0 = time.perf_counter()
        r = f(tt)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        cnt = len(r)
    out[spec["key"]] = {"n": n, "seconds": best, "primes": cnt}
print(json.dumps(out))
"""


def reference_numpy_times(specs: list[dict]) -> dict | None:
    """implicants.dense_prime_ranks itself (the reference package, NumPy, one
    thread as it is written) from baseline/_ref, in a subprocess: min over reps
    of perf_counter around the call only (bench.py:125,136-158 of the
    reference). None when the package is not installed there."""
    import subprocess

    if not os.path.isdir(os.path.join(REF_PKG, "implicants")):
        return None
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-c", _REF_TIMER, REF_PKG, REPO, json.dumps(specs)], env=env,
                       capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        return {"error": r.stderr.strip().splitlines()[-1] if r.stderr.strip() else f"rc={r.returncode}"}
    return json.loads(r.stdout.strip().splitlines()[-1])


def one_thread_n24():
    """The one-off 1-thread n=24 measurement of the port (tools/cpu_n24.py)."""
    try:
        with open(os.path.join(REPO, "profiles", "r2_cpu_n24.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


REF_STEP_BUDGET_S = 300.0  # timed reference steps stop once this much CPU time has elapsed


def run_reference(args):
    """The reference arm: the reference's CPU path for this workload — the
    oracle port (C restatement of dense.py; the reference itself is Python
    and is timed beside it in our arm's configs/cpu_baseline) — on all host
    threads, on OUR arm's workload (full n=24 config-4 calls, same metric).
    One warm-up call at most (a CPU call has nothing to warm beyond the page
    cache), then up to --steps timed calls, stopping early once
    REF_STEP_BUDGET_S has elapsed (steps = the calls actually timed)."""
    rank, world, _ = dist_info()
    if rank != 0:
        return 0
    n = args.n
    info = cpu_info()
    from oracle import gen as G

    v = G.gen3(n, WORKLOAD["p_on"], WORKLOAD["p_dc"], WORKLOAD["seed"])
    for _ in range(min(args.warmup, 1)):
        cpu_port_run(n, values=v)
    times, cnt, thr = [], 0, 1
    t_start = time.perf_counter()
    for _ in range(args.steps):
        dt, cnt, thr = cpu_port_run(n, values=v)
        times.append(dt)
        if time.perf_counter() - t_start > REF_STEP_BUDGET_S:
            break
    t = sum(times) / len(times)
    value = 3**n / t
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": len(times),
        "steps_requested": args.steps,
        "warmup": min(args.warmup, 1),
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded frozen generator, SURVEY.md §8(d))",
        "config": {"workload": WORKLOAD_NAME, "n": n, "primes": cnt, "same_config": n == WORKLOAD["n"]},
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": thr,
            "kind": "port",
            "sample": f"the full n={n} config-4 call per step ({3**n} cells, {cnt} primes); "
                      f"{len(times)} timed calls (budget {REF_STEP_BUDGET_S:.0f} s)",
            **info,
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def load_ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu summary, if any."""
    p = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get("kernels", {}).get(kernel)
        if e and e.get("n") == WORKLOAD["n"]:
            return e.get("dram_bytes")
    except Exception:
        pass
    return None


def cpu_port_primes(n: int) -> int | None:
    return _PORT_PRIMES.get(n)


def bench_configs(args, pkg, device, _lib) -> dict:
    """Configs 1-3: t_api = dense_prime_ranks(TruthTable) host to host (the
    reference's clock placement, bench.py:136-138 of the reference), and
    t_device = device-resident table to device ranks; min over reps. Beside
    them the CPU: oracle port on 1 thread and on all threads, and the
    reference package (NumPy, 1 thread) if installed in baseline/_ref."""
    import torch

    from paper_2302_10083_b200 import configs as C

    reps = {1: 20, 2: 10, 3: 5}
    out = {}
    for cfg in (1, 2, 3):
        n = C.CONFIGS[cfg]["n"]
        vd = C.config_values_device(cfg)
        hv = vd.cpu().numpy()
        tt = pkg.TruthTable.from_values(n, hv)
        r = pkg.dense_prime_ranks(tt)  # warm (sizes the engine for n)
        primes = len(r)
        t_api = []
        for _ in range(reps[cfg]):
            t0 = time.perf_counter()
            r = pkg.dense_prime_ranks(tt)
            t_api.append(time.perf_counter() - t0)
        assert len(r) == primes
        outd = torch.empty(primes + 1024, dtype=torch.int64, device=vd.device)
        device.dense_prime_ranks_device(vd, n, out=outd)
        t_dev = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(reps[cfg]):
            torch.cuda.synchronize()
            e0.record()
            device.dense_prime_ranks_device(vd, n, out=outd)
            e1.record()
            torch.cuda.synchronize()
            t_dev.append(e0.elapsed_time(e1) / 1e3)
        d = {"n": n, "primes": primes, "t_api_ms": min(t_api) * 1e3, "t_device_ms": min(t_dev) * 1e3,
             "cells_per_s_api": 3**n / min(t_api), "cells_per_s_device": 3**n / min(t_dev)}
        if not args.no_cpu:
            v = config_values_cpu(cfg)
            dt1, c1, _ = cpu_port_run(n, threads=1, values=v)
            dta, ca, tha = cpu_port_run(n, values=v)
            d["cpu_port_primes_match"] = c1 == ca == primes
            d["cpu_port_1thread_ms"] = dt1 * 1e3
            d["cpu_port_all_ms"] = dta * 1e3
            d["cpu_port_threads"] = tha
        out[str(cfg)] = d
    if not args.no_cpu:
        ref = reference_numpy_times([{"key": str(c), "cfg": c, "reps": {1: 5, 2: 3, 3: 1}[c]} for c in (1, 2, 3)])
        for c in ("1", "2", "3"):
            if ref is None:
                out[c]["reference_numpy_ms"] = None
            elif c in ref:
                out[c]["reference_numpy_ms"] = ref[c]["seconds"] * 1e3
                out[c]["reference_numpy_primes_match"] = ref[c]["primes"] == out[c]["primes"]
            else:
                out[c]["reference_numpy_ms"] = ref
    out["note"] = ("t_api: dense_prime_ranks(TruthTable) host to host; t_device: device-resident table to "
                   "device ranks (CUDA events); CPU: oracle port (C restatement, 1 thread / all threads) and "
                   "the reference package itself (implicants.dense_prime_ranks, NumPy, 1 thread) from "
                   "baseline/_ref; min over reps")
    return out


def bench_next_rows(args, pkg, device) -> dict:
    """SURVEY.md §8(f) rows beside the reference's own implementation of each
    (NumPy, 1 thread, baseline/_ref; min over reps, perf_counter around the
    call only): f4 the sparse engine at low density, f2 the DenseState path
    (load -> run_merge_reduce -> extract_ranks), f3 the input generator."""
    import torch

    from oracle import gen as G
    from paper_2302_10083_b200 import state as ST

    out = {}
    cases = [("f4_sparse_n20_d0.1", 20, 0.1, 1), ("f4_sparse_n18_d0.3", 18, 0.3, 2)]
    specs = []
    for key, n, d, seed in cases:
        tt = pkg.TruthTable(n, G.random_words(n, d, seed))
        r = pkg.sparse_prime_ranks(tt)  # warm
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            r = pkg.sparse_prime_ranks(tt)
            ts.append(time.perf_counter() - t0)
        td = []
        for _ in range(5):
            t0 = time.perf_counter()
            rd = pkg.dense_prime_ranks(tt)
            td.append(time.perf_counter() - t0)
        out[key] = {"n": n, "density": d, "primes": len(r), "gpu_sparse_ms": min(ts) * 1e3,
                    "gpu_dense_ms": min(td) * 1e3, "sparse_equals_dense": bool(np.array_equal(r, rd))}
        specs.append({"key": key, "n": n, "density": d, "seed": seed, "reps": 1, "engine": "sparse"})
    # f2: the layer-by-layer DenseState on the device (mirror off), config 2
    v = config_values_cpu(2)
    tt2 = pkg.TruthTable.from_values(16, v)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        st = ST.load(tt2, mirror=False)
        st.run_merge_reduce()
        r = ST.extract_ranks(st)
        ts.append(time.perf_counter() - t0)
        del st
    out["f2_state_config2"] = {"n": 16, "primes": len(r), "gpu_state_ms": min(ts[1:]) * 1e3}
    specs.append({"key": "f2_state_config2", "cfg": 2, "reps": 2, "engine": "state"})
    # f3: the frozen generator, config-4 size, on the device vs the NumPy restatement
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    vd = device.gen3_device(24, 0.75, 0.05, 3)
    e0.record()
    for _ in range(5):
        vd = device.gen3_device(24, 0.75, 0.05, 3)
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.gen3(24, 0.75, 0.05, 3)
    tcpu = time.perf_counter() - t0
    out["f3_generator_n24"] = {"values": 1 << 24, "gpu_ms": e0.elapsed_time(e1) / 5,
                               "numpy_ms": tcpu * 1e3, "note": "oracle/gen.py restatement of ttio.py:331-378"}
    ref = reference_numpy_times(specs) if not args.no_cpu else None
    for sp in specs:
        k = sp["key"]
        if isinstance(ref, dict) and k in ref:
            out[k]["reference_numpy_ms"] = ref[k]["seconds"] * 1e3
            out[k]["reference_primes_match"] = ref[k]["primes"] == out[k]["primes"]
        else:
            out[k]["reference_numpy_ms"] = ref if isinstance(ref, dict) else None
    return out


def run_engine_bench(args):
    import torch

    from paper_2302_10083_b200 import _lib, device
    import paper_2302_10083_b200 as pkg

    rank, world, local = dist_info()
    n = args.n
    if world > 1:
        from paper_2302_10083_b200 import sharded

        return sharded.bench_main(args, {**WORKLOAD, "name": WORKLOAD_NAME + "; sharded on the top log2(N) variables"},
                                  METRIC, UNIT, clock_sampler=ClockSampler)
    torch.cuda.set_device(local)

    dev = torch.device(f"cuda:{local}")
    values = device.gen3_device(n, WORKLOAD["p_on"], WORKLOAD["p_dc"], WORKLOAD["seed"], device=local)
    torch.cuda.synchronize()
    # size the device output once (untimed)
    out = torch.empty(1, dtype=torch.int64, device=dev)
    r, cnt = device.dense_prime_ranks_device(values, n, out=None)
    out = torch.empty(int(cnt * 1.02) + 1024, dtype=torch.int64, device=dev)
    del r
    for _ in range(args.warmup):
        device.dense_prime_ranks_device(values, n, out=out)
    torch.cuda.synchronize()

    # ---- value: device-resident, CUDA events on the launching stream (no per-pass
    #      timing). Stream-ordered calls (DQMC_FLAG_ASYNC): the K steps queue back
    #      to back, so a host-side stall cannot idle the GPU between steps.
    stream = torch.cuda.current_stream(dev)
    cnt_dev = torch.zeros(args.steps, dtype=torch.int64, device=dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        launches0 = int(_lib.load().dqmc_launch_count())
        ev0.record(stream)
        for i in range(args.steps):
            device.enqueue_prime_ranks(values, n, out, cnt_dev[i : i + 1])
        ev1.record(stream)
        torch.cuda.synchronize()
        # the library counts its own kernel launches (dqmc_launch_count)
        timed_launches = int(_lib.load().dqmc_launch_count()) - launches0
    assert cnt_dev.eq(cnt).all().item(), cnt_dev.tolist()
    t_step = ev0.elapsed_time(ev1) / 1e3 / args.steps
    value = 3**n / t_step

    # ---- per-pass breakdown (CUDA events around every pass, separate loop)
    pass_times: dict[str, list[float]] = {}
    pass_bytes: dict[str, int] = {}
    launches = 0
    for _ in range(args.steps):
        device.dense_prime_ranks_device(values, n, out=out, timing=True)
        tl = _lib.timings()
        # + the uint8 -> bit packing kernel and the async count publish (CUB's
        # scan kernels inside the k_scan_tiles mark are library launches, not counted)
        launches += len(tl) + 2
        for name, ms, by in tl:
            pass_times.setdefault(name, []).append(ms)
            pass_bytes[name] = by

    # dominant kernel (largest share of the step)
    tot = {k: sum(v) for k, v in pass_times.items()}
    dom = max(tot, key=tot.get)
    launches_per_step = {k: len(v) / args.steps for k, v in pass_times.items()}
    dom_ms = tot[dom] / len(pass_times[dom])
    peak, peak_kind = measured_peak_gbs()
    achieved = pass_bytes[dom] / (dom_ms / 1e3) / 1e9
    all_bytes = sum(pass_bytes.values())
    all_ms = sum(tot.values()) / args.steps

    # ---- e2e: public host API, pinned input, ranks back to the host
    host_vals = torch.empty(1 << n, dtype=torch.uint8, pin_memory=True)
    host_vals.copy_(values.cpu())
    hv = host_vals.numpy()
    for _ in range(max(1, args.warmup)):
        res = pkg.prime_ranks_from_values(hv)
        del res
    # single synchronous drop-in call: dense_prime_ranks(tt) on the reference's
    # TruthTable layout (host uint64 words in, host int64 ranks out)
    tt = pkg.TruthTable.from_values(n, hv)
    for _ in range(max(1, args.warmup)):
        del_ = pkg.dense_prime_ranks(tt)
        del del_
    e2e_times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pkg.dense_prime_ranks(tt)
        e2e_times.append(time.perf_counter() - t0)
        assert len(res) == cnt
        del res
    t_single = sum(e2e_times) / len(e2e_times)
    # the headline e2e: K calls through the job stream (dqmc_submit_u8 /
    # dqmc_collect, three in flight). Every step still copies its table from pinned
    # host memory and its full rank array back to the host inside the timed
    # region; call i's D2H overlaps call i+1's passes.
    # The stream fills (the first call's passes) and drains (the last call's
    # D2H) once per batch, so the batch is at least E2E_MIN_CALLS calls long.
    for r in pkg.stream_prime_ranks([hv] * 3):  # warm the job slots for this n
        del r
    n_stream = max(args.steps, E2E_MIN_CALLS)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = 0
    for r in pkg.stream_prime_ranks([hv] * n_stream):
        assert len(r) == cnt
        got += 1
        del r
    t_e2e = (time.perf_counter() - t0) / got

    # ---- BASELINE configs 1-3: wall time to all primes at n (the metric's
    #      second half), GPU beside the CPU
    configs = bench_configs(args, pkg, device, _lib)
    next_rows = bench_next_rows(args, pkg, device)

    # ---- CPU baseline: oracle port on a bounded sample (rank 0, N=1)
    cpu = None
    if not args.no_cpu:
        dt, ccnt, thr = cpu_port_run(args.cpu_sample_n)
        cpu = {
            "value": 3**args.cpu_sample_n / dt,
            "unit": UNIT,
            "cores": thr,
            "kind": "port",
            "sample": f"n={args.cpu_sample_n} of the config-4 distribution ({3**args.cpu_sample_n} cells, "
                      f"{ccnt} primes), one run",
            **cpu_info(),
        }
        ref = reference_numpy_times([{"key": "n21", "cfg": 4, "n": 21, "reps": 1}])
        if ref and "n21" in ref:
            r21 = ref["n21"]
            cpu["reference_numpy_n21"] = {**r21, "cells_per_s": 3**21 / r21["seconds"], "threads": 1,
                                          "primes_match_port": r21["primes"] == cpu_port_primes(21)}
        elif ref is not None:
            cpu["reference_numpy_n21"] = ref
        cpu["one_thread_n24"] = one_thread_n24()

    traffic = load_ncu_traffic(dom)
    # how the plan finished the state (include/dqmc.h, dqmc_last_gather): sparse states skip
    # the read+write pass D and gather the lower group's parents in the final stage
    import ctypes

    nzb, totb, gath = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
    L = _lib.load()
    if L.dqmc_last_gather(ctypes.byref(nzb), ctypes.byref(totb), ctypes.byref(gath)) == 0:
        finish = {"kind": "gather" if gath.value else "pass_d", "nonzero_blocks": nzb.value,
                  "blocks": totb.value, "threshold_permille": int(L.dqmc_gather_threshold(-1))}
    else:
        finish = None
    # the whole step against the floor of reading the table and writing + reading the state once
    floor_ms = ((1 << n) / 8 + 2 * pkg.state_bytes(n, 5)) / (peak * 1e9) * 1e3
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded frozen generator, SURVEY.md §8(d)); generated on device",
        "config": {
            "workload": WORKLOAD_NAME,
            "n": n,
            "cells": 3**n,
            "primes": cnt,
            "state_bytes": pkg.state_bytes(n, 5),
            "l2": "no flush needed: the 37 GB state is far larger than the 126 MB L2",
            "plan": _lib.plan(n),
        },
        "e2e": {
            "value": 3**n / t_e2e,
            "unit": UNIT,
            "ms_per_step": t_e2e * 1e3,
            "h2d_bytes_per_step": int(1 << n),
            # results of 4M+ ranks cross PCIe packed: 4-byte tile offsets + the tiles' int64
            # positions (3^(n-12) tiles) + the count; the host threads widen them to int64 ranks
            "d2h_bytes_per_step": int(cnt * 4 + 3 ** max(0, n - 12) * 8 + 8) if cnt >= (1 << 22) else int(cnt * 8 + 8),
            "result_bytes_per_step": int(cnt * 8),
            "transfer": "packed (uint32 tile offsets over PCIe, widened to int64 ranks by the library's host "
                        "thread pool inside the timed region)" if cnt >= (1 << 22) else "int64 ranks",
            "api": "paper_2302_10083_b200.stream_prime_ranks (C ABI dqmc_submit_u8 / dqmc_collect), "
                   "three calls in flight, pinned input",
            "calls": n_stream,
            "single_call": {
                "value": 3**n / t_single,
                "ms": t_single * 1e3,
                "api": "paper_2302_10083_b200.dense_prime_ranks(TruthTable) (C ABI dqmc_primes_tt), the drop-in call",
            },
        },
        "roofline": {
            "bound": "hbm",
            "kernel": dom,
            "achieved": achieved,
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": achieved / peak,
            "frac_of_nominal_8000_gbs": achieved / 8000.0,  # also vs the 8 TB/s nominal
            "traffic": traffic,
            "algorithmic_bytes_per_launch": pass_bytes[dom],
            "ms_per_launch": dom_ms,
        },
        "passes": {
            k: {"ms": tot[k] / len(pass_times[k]), "bytes": pass_bytes[k],
                "gbs": pass_bytes[k] / (tot[k] / len(pass_times[k]) / 1e3) / 1e9,
                "launches_per_step": launches_per_step[k]}
            for k in tot
        },
        "all_passes_gbs": all_bytes / (all_ms / 1e3) / 1e9,
        "all_passes_bytes": all_bytes,
        "finish": finish,
        "step_floor": {"ms": floor_ms, "what": "truth table read + state written once and read once, at the measured "
                       "copy peak", "step_over_floor": t_step * 1e3 / floor_ms},
        "gpu_launches": timed_launches,
        "gpu_launches_what": "libdqmc's own kernels launched inside the timed region of `value` (counted by the "
                             "library, dqmc_launch_count); CUB's scan kernels are library launches and not counted",
        "clocks": clk.summary(),
        "configs": configs,
        "next_rows": next_rows,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nvars", dest="n", type=int, default=WORKLOAD["n"], help="variable count (default: config 4, n=24)")
    ap.add_argument("--cpu-sample-n", type=int, default=21)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="print the sharded plan's per-rank device byte budget for --gpus/--nvars and exit")
    args = ap.parse_args()
    if args.dry_run:
        from paper_2302_10083_b200 import sharded

        k = max(1, args.gpus).bit_length() - 1
        print(json.dumps(sharded.dry_run(args.n, k)), flush=True)
        return 0
    if args.impl == "reference":
        return run_reference(args)
    return run_engine_bench(args)


if __name__ == "__main__":
    sys.exit(main())
