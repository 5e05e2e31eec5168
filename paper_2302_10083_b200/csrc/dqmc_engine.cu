// dqmc_engine.cu — the pass plan, the engine workspace and the C ABI of the
// dense path (include/dqmc.h): dqmc_primes_tt/u8 replace dense_prime_ranks
// (/root/reference/pkg/src/implicants/dense.py:405-418), with load()'s
// validation and memory-cap refusal (dense.py:340-373) and the reference's
// output contract (int64 ranks, unique, ascending; dense.py:395-397).
#include "dqmc_internal.cuh"

namespace dqmc {

thread_local std::string g_err;
const bool g_debug = getenv("DQMC_DEBUG") != nullptr;  // sync + report after every pass
std::mutex g_mu;
Engine g_eng;
std::atomic<uint64_t> g_launches{0};

// padded: each C0 tile of 3^g blocks is stored at a pitch rounded up to a
// multiple of 4 blocks (128 B; 2187 -> 2188 blocks at g = 7) so that every
// 128-B row piece the strided passes move is 128-B aligned (TMA load+store of
// misaligned 32-B-granular rows measured 24% slower, tools/probes/layout_probe.cu).
// The pad block is zero and stays zero (MERGE: 0 & 0, REDUCE: 0 & ~x). Only the
// fused single-GPU plan uses it; the bitmap-keeping and sharded entry points
// keep the reference layout (dense.py:1-23).
Plan make_plan(int n, bool padded) {
    Plan p;
    p.n = n;
    p.ne = n < 5 ? 5 : n;
    p.rank_sub = n < 5 ? (243 - pow3l(n)) : 0;
    p.H = p.ne - 5;
    p.g = std::min(p.H, kC0Max);
    p.T = p.H - p.g;
    p.nblocks = pow3l(p.H);
    p.pitch = pow3l(p.g);
    if (padded && p.T > 0) p.pitch = (p.pitch + kRowBlocks - 1) / kRowBlocks * kRowBlocks;
    p.sbytes = (uint64_t)pow3l(p.T) * (uint64_t)p.pitch * 32;
    if (p.T > 0) {
        p.m = (p.T + kGroupMax - 1) / kGroupMax;
        int a = p.g;
        for (int k = 0; k < p.m; k++) {
            const int rk = p.T / p.m + (k < p.T % p.m ? 1 : 0);
            p.r[k] = rk;
            p.a[k] = a;
            a += rk;
        }
    }
    // piece-major group 0: the state is stored as [upper digits][piece x of the
    // C0 tile][group-0 row][128 B] instead of [upper][group-0 row][C0 tile], so
    // the tile of pass D (group 0 reduce, the read+write pass) is one
    // contiguous 93 KB range instead of 729 pieces 70 KB apart, and pass E reads
    // its C0 tile as pieces 93 KB apart (tools/probes/layout_probe.cu: in-place
    // R+W of contiguous tiles 11.8 vs 15.6 ms; the E read 5.9 vs 5.1 ms).
    // Groups above 0 see the same rows/columns as before (columns enumerate the
    // pieces). Needs one 128-B column per tile (3^6 rows) and a separate D pass.
    p.pm = padded && p.T > 0 && p.m >= 2 && p.r[0] == kGroupMax;
    // distribute the five in-block REDUCE axes over the passes that hold whole
    // blocks: pass C (write-only) takes axes 1 and 4, the read+write passes D
    // share the rest, the final pass E takes none when a D pass exists (it is
    // latency-bound by the C0 axes + compaction). With the sparse skip, D runs
    // at the HBM copy rate with three axes (n = 24: C 9.8 / D 11.6 ms; axes
    // 1 / 2-5 gave 10.8 / 12.5, 1-2 / 3-5 10.0 / 11.5, none / all 11.9 / 11.8
    // — tools/ab_ib.sh).
    if (p.T == 0) {
        p.ib_E = 31u;
    } else if (p.m == 1) {
        p.ib_C = 3u;   // axes 1,2
        p.ib_E = 28u;  // axes 3,4,5
    } else {
        p.ib_C = 9u;
        const int rest[3] = {1, 2, 4};  // 0-based axes 2, 3, 5
        int i = 0;
        const int nd = p.m - 1;
        for (int q = 0; q < nd; q++) {
            const int take = (3 - i) / (nd - q);
            for (int c = 0; c < take; c++) p.ib_D[p.m - 2 - q] |= 1u << rest[i++];
        }
    }
    // zero-skip flags (n = 24: groups 6 + 6, piece-major, one column per C
    // tile): ~15% of D items and ~18% of E tiles are all zero at config 4
    // (tools/sparsity.py) and are skipped without touching HBM
    p.nz = p.pm && p.m == 2 && p.r[1] == kGroupMax && p.ib_C != 0;
    return p;
}


int ensure_device() {
    if (g_eng.device >= 0) return DQMC_OK;
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0)
        return set_err(DQMC_ERR_NODEVICE, "no CUDA device visible: libdqmc has no CPU fallback");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaSetDevice(dev));
    g_eng.device = dev;
    CK(cudaStreamCreateWithFlags(&g_eng.stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&g_eng.alloc, 256));
    CK(cudaStreamCreateWithFlags(&g_eng.stream2, cudaStreamNonBlocking));
    for (int i = 0; i < 16; i++) CK(cudaEventCreateWithFlags(&g_eng.chunk_ev[i], cudaEventDisableTiming));
    for (int i = 0; i < 16; i++) CK(cudaEventCreateWithFlags(&g_eng.copy_ev[i], cudaEventDisableTiming));
    CK(cudaMalloc(&g_eng.chunk_base, 17 * sizeof(int64_t)));
    CK(cudaHostAlloc((void **)&g_eng.hbase, 17 * sizeof(int64_t), cudaHostAllocMapped));
    CK(cudaMalloc(&g_eng.total, 256));
    CK(cudaEventCreateWithFlags(&g_eng.last_use, cudaEventDisableTiming));
    return DQMC_OK;
}

int ensure_attrs() {
    if (g_eng.attrs_set) return DQMC_OK;
    int rc;
    if ((rc = merge_set_attrs()) || (rc = reduce_set_attrs()) || (rc = final_set_attrs())) return rc;
    CK(cudaDeviceGetAttribute(&g_eng.num_sms, cudaDevAttrMultiProcessorCount, g_eng.device));
    g_eng.attrs_set = true;
    return DQMC_OK;
}


// Entry points that touch the engine workspace on different streams (the
// host API stream, a caller's stream, a graph replay) are ordered through one
// event: wait for the previous user, record after the last enqueue. Inside a
// stream capture the wait/record would reference work outside the graph, so
// they are skipped there; dqmc_engine_acquire/release order the replays.
int engine_begin(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return DQMC_OK;
    CK(cudaStreamWaitEvent(s, g_eng.last_use, 0));
    return DQMC_OK;
}

int engine_done(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return DQMC_OK;
    CK(cudaEventRecord(g_eng.last_use, s));
    return DQMC_OK;
}

int ensure_encode() {
    if (!g_eng.encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return set_err(DQMC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        g_eng.encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    return DQMC_OK;
}

uint64_t state_bytes_ref(int n, int h) {
    // dense.py:56-63
    uint64_t used = (uint64_t)pow3l(h), b = 1;
    while (b < used) b <<= 1;
    if (b < 64) b = 64;
    return (uint64_t)pow3l(n - h) * b / 8;
}

void note_held(const Plan &p, bool keep);

uint64_t engine_device_bytes(const Plan &p, bool keep) {
    if (p.T == 0 && !keep) return 0;
    return p.sbytes + (uint64_t)pow3l(p.T) * 20;
}

// Run the whole single-GPU plan on a device-resident 32-bit truth table.
int run_plan(const Plan &p, const uint32_t *tt32, int64_t *ranks, int64_t cap, int64_t *count, uint32_t flags,
             cudaStream_t s) {
    int64_t *count_dev = (flags & DQMC_FLAG_ASYNC) ? count : nullptr;  // async: count is a device pointer
    Timer tm{(flags & DQMC_FLAG_TIMING) != 0 && !count_dev, s};
    const bool keep = (flags & DQMC_FLAG_KEEP_BITMAP) != 0;
    const bool count_only = (flags & DQMC_FLAG_COUNT_ONLY) != 0 || ranks == nullptr;
    int rc;
    const uint64_t S = (uint64_t)p.nblocks * 32;
    if (p.T > 0 || keep) {
        if ((rc = grow(g_eng.state, g_eng.state_cap, std::max<uint64_t>(S, p.sbytes), 1))) return rc;
    }
    tm.begin();
    int64_t total = 0;
    FinalOpts fo;
    fo.bitmap_out = keep ? g_eng.state : nullptr;
    fo.count_dev = count_dev;
    if (p.T > 0) {
        if ((rc = run_merge(p, tt32, g_eng.state, false, tm, s))) return rc;
        if ((rc = run_reduce(p, g_eng.state, true, tm, s))) return rc;
        if ((rc = run_final_retry(p, nullptr, g_eng.state, p.ib_E, -p.rank_sub, ranks, cap, count_only, fo, &total, tm,
                                  s)))
            return rc;
        if ((rc = nz_account(p, tm, s))) return rc;
    } else {
        if ((rc = run_final_retry(p, tt32, nullptr, p.ib_E, -p.rank_sub, ranks, cap, count_only, fo, &total, tm, s)))
            return rc;
    }
    tm.finish();
    if (!count_dev) *count = total;
    note_held(p, keep);
    g_eng.state_n = keep ? p.n : -1;
    return DQMC_OK;
}

// total device pass (input conversion + plan)
int primes_device_impl(const void *in, int kind, int n, int64_t *ranks, int64_t cap, int64_t *count,
                       uint32_t flags, cudaStream_t s) {
    const Plan p = make_plan(n, !(flags & DQMC_FLAG_KEEP_BITMAP));
    const uint32_t *tt32 = nullptr;
    int rc;
    if ((rc = engine_begin(s))) return rc;
    if ((rc = input_words(in, kind, n, &tt32, s))) return rc;
    if ((rc = run_plan(p, tt32, ranks, cap, count, flags, s))) return rc;
    return engine_done(s);
}

int validate(int n, int h) {
    if (n < 1 || n > 31) return set_err(DQMC_ERR_INVALID, "variable count must be in 1..31, got " + std::to_string(n));
    if (h != 0 && (h < 1 || h > n))
        return set_err(DQMC_ERR_INVALID,
                       "split must be in 1.." + std::to_string(n) + ", got " + std::to_string(h));
    return DQMC_OK;
}

// dense.py:358-364: refuse before allocating, message names the bytes.
// Steady state (the engine already holds the buffers of a call this size, so
// nothing will be allocated) skips the free-memory query: cudaMemGetInfo is a
// driver round trip measured at p99 12 ms / max 110 ms on these boxes, which
// idled the GPU between back-to-back calls.
int check_cap(int n, int h, uint64_t mem_cap, uint64_t device_need) {
    const int hh = h == 0 ? std::min(n, 5) : h;
    const uint64_t need = state_bytes_ref(n, hh);
    const uint64_t bb = (uint64_t)state_bytes_ref(hh, hh) * 8;
    char buf[512];
    auto refuse = [&](uint64_t cap) {
        snprintf(buf, sizeof buf,
                 "dense state needs %llu bytes (%lld blocks of %llu bits), exceeding the cap of %llu bytes",
                 (unsigned long long)need, (long long)pow3l(n - hh), (unsigned long long)bb,
                 (unsigned long long)cap);
        return set_err(DQMC_ERR_RESOURCE, buf);
    };
    if (mem_cap != 0 && need > mem_cap) return refuse(mem_cap);
    if (device_need <= g_eng.held_need && need <= g_eng.state_cap) return DQMC_OK;
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    if (mem_cap == 0) {
        const uint64_t cap = (uint64_t)((double)(fr + g_eng.state_cap + g_eng.ranks_cap * 8) * 0.75);
        if (need > cap) return refuse(cap);
    }
    const uint64_t have = (uint64_t)fr + g_eng.state_cap;
    if (device_need > have) {
        snprintf(buf, sizeof buf, "device state needs %llu bytes, only %llu bytes of device memory are free",
                 (unsigned long long)device_need, (unsigned long long)have);
        return set_err(DQMC_ERR_RESOURCE, buf);
    }
    return DQMC_OK;
}

// a call of this plan finished: its buffers are held until dqmc_release
void note_held(const Plan &p, bool keep) { g_eng.held_need = std::max(g_eng.held_need, engine_device_bytes(p, keep)); }

int alloc_pinned(size_t entries, PinnedBuf &out) {
    // reuse the smallest cached buffer that fits
    int best = -1;
    for (size_t i = 0; i < g_eng.free_pinned.size(); i++)
        if (g_eng.free_pinned[i].cap >= entries && (best < 0 || g_eng.free_pinned[i].cap < g_eng.free_pinned[best].cap))
            best = (int)i;
    if (best >= 0) {
        out = g_eng.free_pinned[best];
        g_eng.free_pinned.erase(g_eng.free_pinned.begin() + best);
        return DQMC_OK;
    }
    size_t want = std::max<size_t>(entries, 1024);
    int64_t *p = nullptr;
    cudaError_t e = cudaHostAlloc((void **)&p, want * 8, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        char buf[160];
        snprintf(buf, sizeof buf, "pinned host allocation of %llu bytes failed", (unsigned long long)(want * 8));
        return set_err(DQMC_ERR_RESOURCE, buf);
    }
    out.ptr = p;
    out.cap = want;
    return DQMC_OK;
}

int grow_pinned(void **ptr, size_t &cap, size_t need, size_t elem) {
    if (*ptr && need <= cap) return DQMC_OK;
    if (*ptr) {
        cudaFreeHost(*ptr);
        *ptr = nullptr;
        cap = 0;
    }
    const size_t want = std::max<size_t>(need, 1024);
    cudaError_t e = cudaHostAlloc(ptr, want * elem, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        *ptr = nullptr;
        char buf[160];
        snprintf(buf, sizeof buf, "pinned host allocation of %llu bytes failed", (unsigned long long)(want * elem));
        return set_err(DQMC_ERR_RESOURCE, buf);
    }
    cap = want;
    return DQMC_OK;
}

int primes_host_impl(const void *host_in, int kind, int n, int h, uint64_t mem_cap, uint32_t flags,
                     dqmc_result_t *out) {
    if (!out) return set_err(DQMC_ERR_INVALID, "null result pointer");
    out->count = 0;
    out->ranks = nullptr;
    out->_owner = nullptr;
    int rc;
    if ((rc = validate(n, h))) return rc;
    if (!host_in) return set_err(DQMC_ERR_INVALID, "null input pointer");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    const Plan p = make_plan(n, !(flags & DQMC_FLAG_KEEP_BITMAP));
    if ((rc = check_cap(n, h, mem_cap, engine_device_bytes(p, flags & DQMC_FLAG_KEEP_BITMAP)))) return rc;
    cudaStream_t s = g_eng.stream;
    // H2D of the input (pageable source; small relative to the state)
    const size_t in_bytes = kind == DQMC_IN_U8 ? ((size_t)1 << n) : (size_t)std::max<int64_t>(1, (1ll << n) / 64) * 8;
    if ((rc = grow(g_eng.in_tmp, g_eng.in_tmp_cap, std::max<size_t>(in_bytes, 8), 1))) return rc;
    if ((rc = engine_begin(s))) return rc;
    CK(cudaMemcpyAsync(g_eng.in_tmp, host_in, in_bytes, cudaMemcpyHostToDevice, s));
    const bool count_only = (flags & DQMC_FLAG_COUNT_ONLY) != 0;
    // the chunked final stage overlaps the packed rank D2H (4-byte tile
    // offsets) and the host's widening to int64 with the last chunks' compute;
    // it pays one host round trip per chunk (16), so it only runs when the
    // hinted output is large enough for the overlap to win (>= 4M ranks =
    // 32 MB; config 2's 0.4M ranks: 0.79 -> ~0.3 ms per call)
    const bool pipelined = !count_only && !(flags & (DQMC_FLAG_KEEP_BITMAP | DQMC_FLAG_TIMING)) && p.T > 0 &&
                           g_eng.hint_n == n && g_eng.hint_count >= kPackedMinRanks;
    if (pipelined) {
        // merge/reduce passes, then the chunked final stage straight into pinned host memory
        g_eng.state_n = -1;  // the state is overwritten in the plan's own layout
        const uint32_t *tt32 = nullptr;
        if ((rc = input_words(g_eng.in_tmp, kind, n, &tt32, s))) return rc;
        if ((rc = grow(g_eng.state, g_eng.state_cap, (size_t)p.sbytes, 1))) return rc;
        Timer tm{false, s};
        if ((rc = run_merge(p, tt32, g_eng.state, false, tm, s))) return rc;
        if ((rc = run_reduce(p, g_eng.state, true, tm, s))) return rc;
        PinnedBuf pb;
        if ((rc = alloc_pinned((size_t)((double)g_eng.hint_count * 1.02) + 4096, pb))) return rc;
        int64_t count = 0;
        bool ok = true;
        if ((rc = run_final_pipelined(p, g_eng.state, pb.ptr, (int64_t)pb.cap, &count, &ok, s))) return rc;
        if (!ok) {  // the output outgrew the hinted buffer: rerun the stage into a larger one
            g_eng.free_pinned.push_back(pb);
            if ((rc = alloc_pinned((size_t)count, pb))) return rc;
            if ((rc = run_final_pipelined(p, g_eng.state, pb.ptr, (int64_t)pb.cap, &count, &ok, s))) return rc;
        }
        if ((rc = engine_done(s))) return rc;
        g_eng.hint_count = count;
        out->count = count;
        if (count > 0) {
            out->ranks = pb.ptr;
            out->_owner = new PinnedBuf(pb);
        } else {
            g_eng.free_pinned.push_back(pb);
        }
        return DQMC_OK;
    }
    if (!count_only && g_eng.ranks_cap == 0) {
        if ((rc = grow(g_eng.ranks, g_eng.ranks_cap, (size_t)1 << 20, 8))) return rc;
    }
    int64_t count = 0;
    if ((rc = primes_device_impl(g_eng.in_tmp, kind, n, count_only ? nullptr : g_eng.ranks, (int64_t)g_eng.ranks_cap,
                                 &count, flags, s)))
        return rc;
    if (!count_only && (size_t)count > g_eng.ranks_cap) {
        // grow the output and run again (only the count was exact)
        if ((rc = grow(g_eng.ranks, g_eng.ranks_cap, (size_t)((double)count * 1.05) + 1024, 8))) return rc;
        if ((rc = primes_device_impl(g_eng.in_tmp, kind, n, g_eng.ranks, (int64_t)g_eng.ranks_cap, &count, flags, s)))
            return rc;
    }
    out->count = count;
    if (!count_only) {
        g_eng.hint_n = n;
        g_eng.hint_count = count;
    }
    if (!count_only && count > 0) {
        PinnedBuf pb;
        if ((rc = alloc_pinned((size_t)count, pb))) return rc;
        CK(cudaMemcpyAsync(pb.ptr, g_eng.ranks, (size_t)count * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        PinnedBuf *owner = new PinnedBuf(pb);
        out->ranks = pb.ptr;
        out->_owner = owner;
    }
    return DQMC_OK;
}

// Host-API jobs, up to kJobSlots (3) in flight: submit queues the H2D of the table, every pass
// and the final stage on the engine stream and returns; collect waits for the
// job's final stage, then copies its ranks to pinned host memory on the copy
// stream while the engine stream already runs the next job. A stream of calls
// thus overlaps call i's D2H with call i+1's passes. The first job of an n (no
// count hint yet to size the outputs) runs synchronously inside submit.
int submit_impl(const void *host_in, int kind, int n, uint32_t flags, int64_t *job_out) {
    if (!job_out) return set_err(DQMC_ERR_INVALID, "null job pointer");
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!host_in) return set_err(DQMC_ERR_INVALID, "null input pointer");
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if ((rc = ensure_device())) return rc;
        if ((rc = ensure_attrs())) return rc;
        if (g_eng.jobs.size() >= (size_t)kJobSlots)
            return set_err(DQMC_ERR_INVALID, "three jobs outstanding: collect the oldest first");
        const Plan p = make_plan(n);
        const bool async = !(flags & (DQMC_FLAG_COUNT_ONLY | DQMC_FLAG_KEEP_BITMAP | DQMC_FLAG_TIMING)) && p.T > 0 &&
                           g_eng.hint_n == n && g_eng.hint_count > 0;
        if (async) {
            if ((rc = check_cap(n, 0, 0, engine_device_bytes(p, false)))) return rc;
            const int64_t id = g_eng.next_job++;
            const int slot = (int)(id % kJobSlots);
            if (!g_eng.jcount_host)
                CK(cudaHostAlloc((void **)&g_eng.jcount_host, kJobSlots * sizeof(int64_t), cudaHostAllocDefault));
            if (!g_eng.jev[slot]) CK(cudaEventCreateWithFlags(&g_eng.jev[slot], cudaEventDisableTiming));
            const size_t in_bytes =
                kind == DQMC_IN_U8 ? ((size_t)1 << n) : (size_t)std::max<int64_t>(1, (1ll << n) / 64) * 8;
            if ((rc = grow(g_eng.jin[slot], g_eng.jin_cap[slot], std::max<size_t>(in_bytes, 8), 1))) return rc;
            const size_t want = (size_t)((double)g_eng.hint_count * 1.05) + 4096;
            // large results stay packed in the slot (4-byte tile offsets in rank order)
            const bool packed = g_eng.hint_count >= kPackedMinRanks;
            const int64_t ntiles = pow3l(p.T);
            if ((rc = grow(g_eng.jranks[slot], g_eng.jranks_cap[slot], packed ? (want + 1) / 2 : want, 8))) return rc;
            if (packed && (rc = grow(g_eng.jpos[slot], g_eng.jpos_cap[slot], (size_t)ntiles, 8))) return rc;
            g_eng.scratch_want = std::max(g_eng.scratch_want, want);
            if ((rc = grow(g_eng.state, g_eng.state_cap, (size_t)p.sbytes, 1))) return rc;
            cudaStream_t s = g_eng.stream;
            g_eng.state_n = -1;  // the state is overwritten in the plan's own layout
            if ((rc = engine_begin(s))) return rc;
            CK(cudaMemcpyAsync(g_eng.jin[slot], host_in, in_bytes, cudaMemcpyHostToDevice, s));
            const uint32_t *tt32 = nullptr;
            if ((rc = input_words(g_eng.jin[slot], kind, n, &tt32, s))) return rc;
            Timer tm{false, s};
            if ((rc = run_merge(p, tt32, g_eng.state, false, tm, s))) return rc;
            if ((rc = run_reduce(p, g_eng.state, true, tm, s))) return rc;
            int64_t unused = 0;
            int64_t *cdev = g_eng.total + 8 + slot;  // device count of this slot (-(count+1): outputs too small)
            FinalOpts fo;
            fo.count_dev = cdev;
            if (packed) fo.packed32 = (uint32_t *)g_eng.jranks[slot];
            if ((rc = run_final(p, nullptr, g_eng.state, p.ib_E, -p.rank_sub, packed ? nullptr : g_eng.jranks[slot],
                                (int64_t)g_eng.jranks_cap[slot] * (packed ? 2 : 1), false, fo, &unused, tm, s)))
                return rc;
            if (packed)  // the next job's final stage rewrites the engine's tile positions
                CK(cudaMemcpyAsync(g_eng.jpos[slot], g_eng.tile_pos, (size_t)ntiles * 8, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(g_eng.jcount_host + slot, cdev, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            CK(cudaEventRecord(g_eng.jev[slot], s));
            if ((rc = engine_done(s))) return rc;
            Job j;
            j.id = id;
            j.slot = slot;
            j.in = host_in;
            j.kind = kind;
            j.n = n;
            j.flags = flags;
            j.packed = packed;
            j.ntiles = ntiles;
            j.tile_cells = pow3l(p.g) * 243;
            j.rank_add = -p.rank_sub;
            g_eng.jobs.push_back(j);
            *job_out = id;
            return DQMC_OK;
        }
    }
    dqmc_result_t res{};
    if ((rc = primes_host_impl(host_in, kind, n, 0, 0, flags, &res))) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    Job j;
    j.id = g_eng.next_job++;
    j.res = res;
    g_eng.jobs.push_back(j);
    *job_out = j.id;
    return DQMC_OK;
}

// A packed job's result: the tile positions first (they say where every
// tile's offsets lie), then the offsets in 16 chunks of about equal size on
// the copy stream; each chunk is widened to int64 ranks by the host threads
// as soon as it has landed, while the copy engine moves the next one.
static int collect_packed(const Job &j, int64_t c, int64_t *host) {
    int rc;
    if ((rc = grow_pinned((void **)&g_eng.stage32, g_eng.stage32_cap, (size_t)c, 4))) return rc;
    if ((rc = grow_pinned((void **)&g_eng.stage_pos, g_eng.stage_pos_cap, (size_t)j.ntiles, 8))) return rc;
    const uint32_t *dev32 = (const uint32_t *)g_eng.jranks[j.slot];
    int64_t *pos = g_eng.stage_pos;
    cudaStream_t s2 = g_eng.stream2;
    CK(cudaMemcpyAsync(pos, g_eng.jpos[j.slot], (size_t)j.ntiles * 8, cudaMemcpyDeviceToHost, s2));
    CK(cudaStreamSynchronize(s2));
    const int K = (int)std::min<int64_t>(16, j.ntiles);
    int64_t tb[17], at[17];  // chunk k: tiles [tb[k], tb[k+1]), entries [at[k], at[k+1])
    for (int k = 0; k <= K; k++) {
        tb[k] = k == 0 ? 0 : (k == K ? j.ntiles : std::lower_bound(pos, pos + j.ntiles, c / K * k) - pos);
        at[k] = tb[k] < j.ntiles ? pos[tb[k]] : c;
    }
    for (int k = 0; k < K; k++) {
        if (at[k + 1] > at[k])
            CK(cudaMemcpyAsync(g_eng.stage32 + at[k], dev32 + at[k], (size_t)(at[k + 1] - at[k]) * 4,
                               cudaMemcpyDeviceToHost, s2));
        CK(cudaEventRecord(g_eng.copy_ev[k], s2));
    }
    for (int k = 0; k < K; k++) {
        CK(cudaEventSynchronize(g_eng.copy_ev[k]));
        host_widen(g_eng.stage32, host, pos + tb[k], 0, at[k + 1], tb[k], tb[k + 1], j.tile_cells, j.rank_add);
    }
    return DQMC_OK;
}

int collect_impl(int64_t job, dqmc_result_t *out) {
    if (!out) return set_err(DQMC_ERR_INVALID, "null result pointer");
    out->count = 0;
    out->ranks = nullptr;
    out->_owner = nullptr;
    std::unique_lock<std::mutex> lk(g_mu);
    if (g_eng.jobs.empty() || g_eng.jobs.front().id != job)
        return set_err(DQMC_ERR_INVALID, "unknown job, or jobs collected out of submission order");
    const Job j = g_eng.jobs.front();
    g_eng.jobs.pop_front();
    if (j.slot < 0) {
        *out = j.res;
        return DQMC_OK;
    }
    CK(cudaEventSynchronize(g_eng.jev[j.slot]));
    const int64_t c = g_eng.jcount_host[j.slot];
    if (c < 0) {  // the hinted output was too small: run this job again, synchronously
        g_eng.hint_count = -c - 1;
        g_eng.scratch_want = std::max(g_eng.scratch_want, (size_t)((double)(-c - 1) * 1.05) + 4096);
        lk.unlock();
        return primes_host_impl(j.in, j.kind, j.n, 0, 0, j.flags, out);
    }
    g_eng.hint_count = c;
    if (c > 0) {
        PinnedBuf pb;
        int rc;
        if ((rc = alloc_pinned((size_t)c, pb))) return rc;
        if (j.packed) {
            if ((rc = collect_packed(j, c, pb.ptr))) {
                g_eng.free_pinned.push_back(pb);
                return rc;
            }
        } else {
            CK(cudaMemcpyAsync(pb.ptr, g_eng.jranks[j.slot], (size_t)c * 8, cudaMemcpyDeviceToHost, g_eng.stream2));
            CK(cudaStreamSynchronize(g_eng.stream2));
        }
        out->count = c;
        out->ranks = pb.ptr;
        out->_owner = new PinnedBuf(pb);
    }
    return DQMC_OK;
}
}  // namespace dqmc

using namespace dqmc;

// ---------------------------------------------------------------------------
// C ABI

// shared error channel of the state API (dqmc_state.cu); not part of the ABI
extern "C" __attribute__((visibility("hidden"))) void dqmc_internal_set_error(const char *m) { g_err = m; }

extern "C" {

int dqmc_abi_version(void) { return DQMC_ABI_VERSION; }

const char *dqmc_last_error(void) { return g_err.c_str(); }

int dqmc_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return c;
}

int dqmc_set_device(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_eng.device == device) return DQMC_OK;
    if (g_eng.device >= 0) return set_err(DQMC_ERR_INVALID, "device already selected; call dqmc_release first");
    CK(cudaSetDevice(device));
    return DQMC_OK;
}

uint64_t dqmc_block_bits(int h) { return state_bytes_ref(h, h) * 8; }

uint64_t dqmc_state_bytes(int n, int h) { return state_bytes_ref(n, h); }

uint64_t dqmc_device_bytes(int n) {
    if (n < 1 || n > 31) return 0;
    return engine_device_bytes(make_plan(n), false);
}

int dqmc_primes_tt(const uint64_t *tt_words, int n, int h, uint64_t mem_cap, uint32_t flags, dqmc_result_t *out) {
    return primes_host_impl(tt_words, DQMC_IN_WORDS, n, h, mem_cap, flags, out);
}

int dqmc_primes_u8(const uint8_t *values, int n, int h, uint64_t mem_cap, uint32_t flags, dqmc_result_t *out) {
    return primes_host_impl(values, DQMC_IN_U8, n, h, mem_cap, flags, out);
}

int dqmc_host_threads(int n) { return host_widen_threads(n); }

void dqmc_widen_host(const uint32_t *off32, int64_t *out, const int64_t *pos, int64_t add, int64_t end, int64_t t0,
                     int64_t t1, int64_t tile_cells, int64_t rank_add) {
    host_widen(off32, out, pos, add, end, t0, t1, tile_cells, rank_add);
}

void dqmc_free_result(dqmc_result_t *res) {
    if (!res) return;
    if (res->_owner) {
        std::lock_guard<std::mutex> lk(g_mu);
        PinnedBuf *pb = (PinnedBuf *)res->_owner;
        g_eng.free_pinned.push_back(*pb);
        // keep at most two cached pinned buffers
        while (g_eng.free_pinned.size() > 2) {
            auto it = std::min_element(g_eng.free_pinned.begin(), g_eng.free_pinned.end(),
                                       [](const PinnedBuf &a, const PinnedBuf &b) { return a.cap < b.cap; });
            cudaFreeHost(it->ptr);
            g_eng.free_pinned.erase(it);
        }
        delete pb;
    }
    res->_owner = nullptr;
    res->ranks = nullptr;
    res->count = 0;
}

int dqmc_primes_device(const void *input_dev, int in_kind, int n, int64_t *ranks_dev, int64_t ranks_cap,
                       int64_t *count_out, uint32_t flags, void *stream) {
    int rc;
    if ((rc = validate(n, 0))) return rc;
    if (!input_dev || !count_out) return set_err(DQMC_ERR_INVALID, "null pointer argument");
    if (in_kind != DQMC_IN_WORDS && in_kind != DQMC_IN_U8) return set_err(DQMC_ERR_INVALID, "bad input kind");
    std::lock_guard<std::mutex> lk(g_mu);
    if ((rc = ensure_device())) return rc;
    if ((rc = ensure_attrs())) return rc;
    const Plan p = make_plan(n, !(flags & DQMC_FLAG_KEEP_BITMAP));
    if ((rc = check_cap(n, 0, 0, engine_device_bytes(p, flags & DQMC_FLAG_KEEP_BITMAP)))) return rc;
    cudaStream_t s = (cudaStream_t)stream;  // 0 = the legacy default stream (CUDA convention)
    if (!ranks_dev) flags |= DQMC_FLAG_COUNT_ONLY;
    return primes_device_impl(input_dev, in_kind, n, ranks_dev, ranks_cap, count_out, flags, s);
}

int dqmc_last_timings(const char **names, float *ms, int max) {
    const int k = (int)g_eng.pass_ms.size();
    for (int i = 0; i < k && i < max; i++) {
        if (names) names[i] = g_eng.pass_names[i].c_str();
        if (ms) ms[i] = g_eng.pass_ms[i];
    }
    return k;
}

int dqmc_last_pass_bytes(uint64_t *bytes, int max) {
    const int k = (int)g_eng.pass_bytes.size();
    for (int i = 0; i < k && i < max; i++) bytes[i] = g_eng.pass_bytes[i];
    return k;
}

int dqmc_bitmap_device(void **ptr, uint64_t *bytes) {
    if (g_eng.state_n < 0) return set_err(DQMC_ERR_INVALID, "no bitmap held: run with DQMC_FLAG_KEEP_BITMAP");
    const Plan p = make_plan(g_eng.state_n, false);
    if (ptr) *ptr = g_eng.state;
    if (bytes) *bytes = (uint64_t)p.nblocks * 32;
    return DQMC_OK;
}

int dqmc_bitmap_download(void *host, uint64_t bytes) {
    if (g_eng.state_n < 0) return set_err(DQMC_ERR_INVALID, "no bitmap held: run with DQMC_FLAG_KEEP_BITMAP");
    const Plan p = make_plan(g_eng.state_n, false);
    const uint64_t need = (uint64_t)p.nblocks * 32;
    if (bytes < need) return set_err(DQMC_ERR_INVALID, "host buffer too small");
    CK(cudaMemcpy(host, g_eng.state, need, cudaMemcpyDeviceToHost));
    return DQMC_OK;
}

int dqmc_submit_tt(const uint64_t *tt_words, int n, uint32_t flags, int64_t *job) {
    return submit_impl(tt_words, DQMC_IN_WORDS, n, flags, job);
}

int dqmc_submit_u8(const uint8_t *values, int n, uint32_t flags, int64_t *job) {
    return submit_impl(values, DQMC_IN_U8, n, flags, job);
}

int dqmc_collect(int64_t job, dqmc_result_t *out) { return collect_impl(job, out); }

int dqmc_plan(int n, int64_t *out, int max) {
    if (n < 1 || n > 31 || !out) return 0;
    const Plan p = make_plan(n);
    int64_t v[32];
    int k = 0;
    v[k++] = p.ne;
    v[k++] = p.H;
    v[k++] = p.g;
    v[k++] = p.T;
    v[k++] = p.m;
    for (int i = 0; i < 8; i++) v[k++] = p.r[i];
    for (int i = 0; i < 8; i++) v[k++] = p.a[i];
    v[k++] = p.ib_C;
    v[k++] = p.ib_E;
    for (int i = 0; i < 8; i++) v[k++] = p.ib_D[i];
    v[k++] = p.rank_sub;
    const int w = std::min(k, max);
    for (int i = 0; i < w; i++) out[i] = v[i];
    return w;
}

void dqmc_release(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_eng.device < 0) return;
    cudaDeviceSynchronize();  // nothing in flight may still use the workspace
    sparse_release();
    cudaFree(g_eng.state);
    cudaFree(g_eng.tile_base);
    cudaFree(g_eng.tile_pos);
    cudaFree(g_eng.tile_cnt);
    cudaFree(g_eng.scratch);
    cudaFree(g_eng.tile_rank0);
    cudaFree(g_eng.alloc);
    cudaFree(g_eng.cub_tmp);
    cudaFree(g_eng.total);
    cudaFree(g_eng.tt_tmp);
    cudaFree(g_eng.in_tmp);
    cudaFree(g_eng.ranks);
    cudaFree(g_eng.nzflags);
    for (auto &b : g_eng.free_pinned) cudaFreeHost(b.ptr);
    if (g_eng.stream) cudaStreamDestroy(g_eng.stream);
    if (g_eng.stream2) cudaStreamDestroy(g_eng.stream2);
    for (int i = 0; i < 16; i++) {
        if (g_eng.chunk_ev[i]) cudaEventDestroy(g_eng.chunk_ev[i]);
        if (g_eng.copy_ev[i]) cudaEventDestroy(g_eng.copy_ev[i]);
    }
    if (g_eng.stage32) cudaFreeHost(g_eng.stage32);
    if (g_eng.stage_pos) cudaFreeHost(g_eng.stage_pos);
    cudaFree(g_eng.chunk_base);
    if (g_eng.hbase) cudaFreeHost(g_eng.hbase);
    for (int i = 0; i < kJobSlots; i++) {
        cudaFree(g_eng.jin[i]);
        cudaFree(g_eng.jranks[i]);
        cudaFree(g_eng.jpos[i]);
        if (g_eng.jev[i]) cudaEventDestroy(g_eng.jev[i]);
    }
    if (g_eng.jcount_host) cudaFreeHost(g_eng.jcount_host);
    if (g_eng.last_use) cudaEventDestroy(g_eng.last_use);
    const uint64_t gen = g_eng.generation;
    g_eng = Engine();
    g_eng.generation = gen + 1;  // every pointer a captured graph holds is gone
}

uint64_t dqmc_engine_generation(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    return g_eng.generation;
}

int dqmc_engine_enter(void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc;
    if ((rc = ensure_device())) return rc;
    return engine_begin((cudaStream_t)stream);
}

int dqmc_engine_exit(void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    int rc;
    if ((rc = ensure_device())) return rc;
    return engine_done((cudaStream_t)stream);
}

uint64_t dqmc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int dqmc_gather_threshold(int permille) {
    std::lock_guard<std::mutex> lk(g_mu);
    const int prev = g_eng.gather_permille;
    if (permille >= 0) g_eng.gather_permille = std::min(permille, 1000);
    return prev;
}

int dqmc_last_gather(int64_t *nonzero_blocks, int64_t *total_blocks, int *gathered) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_eng.gather_n < 0 || !g_eng.nzflags) return set_err(DQMC_ERR_INVALID, "no call of the two-group plan has run");
    const Plan p = make_plan(g_eng.gather_n);
    const size_t npiece = (size_t)(p.pitch / kRowBlocks), nr = (size_t)pow3l(p.r[0]);
    unsigned long long c = 0;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&c, g_eng.nzflags + nz_count_offset(npiece, nr), 8, cudaMemcpyDeviceToHost));
    if (nonzero_blocks) *nonzero_blocks = (int64_t)c;
    if (total_blocks) *total_blocks = p.nblocks;
    if (gathered) *gathered = c <= g_eng.gather_limit_last;
    return DQMC_OK;
}

}  // extern "C"
