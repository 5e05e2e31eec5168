// dqmc_shard.cu — building blocks of the sharded multi-GPU path.
//
// One process per GPU; the top k variables select the GPU and the next m
// split every top block into super-blocks that are owned by an interleaved
// rule (paper_2302_10083_b200/sharded.py). The block-level
// MERGE of the top axes (dense.py:174-212, merge_triple dense.py:46-48) is a
// bitwise AND of two super-blocks, one of them read in place from a peer
// GPU's memory over NVLink (CUDA IPC), a whole level per launch; the REDUCE
// of the low axes runs over all of a rank's super-blocks at once, and the
// REDUCE of the top axes clears the OR of up to kMaxKill parent super-blocks,
// read the same way inside the final pass (reduce_triple dense.py:51-53,
// formula oracle.py:77-80).
#include "dqmc_internal.cuh"

namespace dqmc {
namespace {

// dst = a & b (op 0) or a | b (op 1), 16 B per thread: the top-axis block
// ANDs of the sharded path (M_t = AND over completions) and kill accumulation.
__global__ void k_bitop(uint4 *__restrict__ dst, const uint4 *__restrict__ a, const uint4 *__restrict__ b, int64_t n16,
                        int op) {
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4 x = __ldcs(a + i), y = __ldcs(b + i);
        dst[i] = op == 0 ? make_uint4(x.x & y.x, x.y & y.y, x.z & y.z, x.w & y.w)
                         : make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w);
    }
}

__global__ void k_bitop_batch(const uint64_t *__restrict__ jobs, int64_t n16, int op) {
    const uint64_t *j = jobs + 3 * (int64_t)blockIdx.y;
    uint4 *dst = reinterpret_cast<uint4 *>(j[0]);
    const uint4 *a = reinterpret_cast<const uint4 *>(j[1]);
    const uint4 *b = reinterpret_cast<const uint4 *>(j[2]);
    const int64_t stride = gridDim.x * (int64_t)blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
        const uint4 x = __ldcs(a + i), y = __ldcs(b + i);
        dst[i] = op == 0 ? make_uint4(x.x & y.x, x.y & y.y, x.z & y.z, x.w & y.w)
                         : make_uint4(x.x | y.x, x.y | y.y, x.z | y.z, x.w | y.w);
    }
}

}  // namespace
}  // namespace dqmc

using namespace dqmc;

extern "C" {

int dqmc_ipc_get(const void *dev_ptr, void *handle_out, uint64_t *offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    int rc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if (!g_eng.addr_range) {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
            if (!fn || q != cudaDriverEntryPointSuccess) return set_err(DQMC_ERR_CUDA, "cuMemGetAddressRange unavailable");
            g_eng.addr_range = (AddrRangeFn)fn;
        }
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUresult r = g_eng.addr_range(&base, &size, (CUdeviceptr)dev_ptr);
    if (r != CUDA_SUCCESS) return set_err(DQMC_ERR_INVALID, "not a device allocation: " + std::to_string((int)r));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void *)base));
    memcpy(handle_out, &h, sizeof h);
    *offset_out = (uint64_t)((CUdeviceptr)dev_ptr - base);
    return DQMC_OK;
}

int dqmc_ipc_open(const void *handle, void **base_out) {
    if (!handle || !base_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    int rc;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    CK(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
    return DQMC_OK;
}

int dqmc_ipc_close(void *base) {
    if (!base) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    CK(cudaIpcCloseMemHandle(base));
    return DQMC_OK;
}

int dqmc_merge_device(const void *input_dev, int in_kind, int n, uint32_t *state_out, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (n < 5) return set_err(DQMC_ERR_INVALID, "dqmc_merge_device needs n >= 5 (h=5 layout)");
    if (!input_dev || !state_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const Plan p = make_plan(n, false);  // caller-owned state in the reference layout
    const uint32_t *tt32 = nullptr;
    if ((rc = engine_begin(s))) return rc;
    if ((rc = input_words(input_dev, in_kind, n, &tt32, s))) return rc;
    Timer tm{false, s};
    if ((rc = run_merge(p, tt32, state_out, true, tm, s))) return rc;
    return engine_done(s);
}

// REDUCE of the strided groups (and their in-block axes) of nslots
// consecutive super-blocks, in place: passes C/D as reduce-only, batched over
// the slots. The C0 and remaining in-block axes are reduced inside the
// extract pass, on the tile in shared memory. A parent read as a kill source
// may be reduced along any subset of its low axes: a parent cell cleared by
// one of its own low parents implies the cell's own low parent along that
// axis is an implicant, so the cell dies anyway.
int dqmc_reduce_low_device(uint32_t *arena, int n, int64_t nslots, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (n < 5) return set_err(DQMC_ERR_INVALID, "dqmc_reduce_low_device needs n >= 5 (h=5 layout)");
    if (!arena || nslots < 1) return set_err(DQMC_ERR_INVALID, "null arena or no slots");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const Plan p = make_plan(n, false);     // caller-owned states in the reference layout
    if (p.T == 0) return DQMC_OK;           // one tile per state: the extract pass does everything
    Timer tm{false, s};
    if ((rc = engine_begin(s))) return rc;
    if ((rc = run_reduce(p, arena, false, tm, s, nslots))) return rc;
    return engine_done(s);
}

// Primes of nslots super-blocks after dqmc_reduce_low_device: every tile
// finishes its low REDUCE in shared memory (the C0 axes and the remaining
// in-block axes), clears the OR of its slot's parent super-blocks (kill_tab:
// nslots x 8 device addresses, null padded; local or IPC peer memory) and
// emits its ranks (+ rank_add[slot]). Ranks go out in slot order;
// slot_start/slot_count (device, nslots each) give each slot's range;
// *total_out the sum (host).
int dqmc_extract_kills_device(const uint32_t *arena, int n, int64_t nslots, const uint64_t *kill_tab,
                              const int64_t *rank_add, int64_t *ranks_dev, int64_t ranks_cap, int64_t *slot_start,
                              int64_t *slot_count, int64_t *total_out, uint32_t flags, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (n < 5) return set_err(DQMC_ERR_INVALID, "dqmc_extract_kills_device needs n >= 5 (h=5 layout)");
    if (!arena || nslots < 1 || !kill_tab || !rank_add || !slot_start || !slot_count || !total_out)
        return set_err(DQMC_ERR_INVALID, "null pointer argument");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const Plan p = make_plan(n, false);
    const bool count_only = (flags & DQMC_FLAG_COUNT_ONLY) != 0 || ranks_dev == nullptr;
    Timer tm{(flags & DQMC_FLAG_TIMING) != 0, s};
    if ((rc = engine_begin(s))) return rc;
    tm.begin();
    FinalOpts fo;
    fo.nbatch = nslots;
    fo.kill_tab = kill_tab;
    fo.rank_add_tab = rank_add;
    fo.slot_start = slot_start;
    fo.slot_count = slot_count;
    if ((rc = run_final_retry(p, nullptr, arena, p.ib_E, 0, ranks_dev, ranks_cap, count_only, fo, total_out, tm, s)))
        return rc;
    if ((rc = engine_done(s))) return rc;
    tm.finish();
    return DQMC_OK;
}

// dst_j = a_j & b_j (op 0) or a_j | b_j (op 1) for njobs (dst, a, b) address
// triples in device memory, nbytes each: one launch for a whole merge level
// of the sharded path (a or b may be peer memory).
int dqmc_bitop_batch_device(const uint64_t *jobs_dev, int64_t njobs, uint64_t nbytes, int op, void *stream) {
    int rc;
    if (!jobs_dev || njobs < 0 || njobs > 65535 || (nbytes % 16) || (op != 0 && op != 1))
        return set_err(DQMC_ERR_INVALID, "bitop batch: null jobs, bad count, size not a multiple of 16, or bad op");
    if (njobs == 0 || nbytes == 0) return DQMC_OK;
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n16 = (int64_t)(nbytes / 16);
    const int64_t want = ((int64_t)g_eng.num_sms * 16 + njobs - 1) / njobs;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (n16 + 255) / 256));
    k_bitop_batch<<<dim3(gx, (unsigned)njobs), 256, 0, s>>>(jobs_dev, n16, op);
    CK_LAUNCH();
    return DQMC_OK;
}

int dqmc_bitop_device(uint32_t *dst, const uint32_t *a, const uint32_t *b, uint64_t nbytes, int op, void *stream) {
    int rc;
    if (!dst || !a || !b || (nbytes % 16) || (op != 0 && op != 1))
        return set_err(DQMC_ERR_INVALID, "bitop: null pointer, size not a multiple of 16, or bad op");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    const int64_t n16 = (int64_t)(nbytes / 16);
    const int grid = (int)std::min<int64_t>((n16 + 255) / 256, 148ll * 16);
    if (n16) k_bitop<<<grid, 256, 0, s>>>((uint4 *)dst, (const uint4 *)a, (const uint4 *)b, n16, op);
    CK_LAUNCH();
    return DQMC_OK;
}


}  // extern "C"
