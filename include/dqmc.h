/*
 * dqmc.h — C ABI of the B200-native dense prime-implicant engine (libdqmc.so).
 *
 * Drop-in boundary for the reference's dense path. Every entry point below
 * replaces a reference interface (paths relative to /root/reference/pkg):
 *
 *   dqmc_primes_tt / dqmc_primes_u8
 *       replace dense_prime_ranks(tt, h, optimized, mem_cap)
 *       src/implicants/dense.py:405-418, reached through
 *       run_engine("dense", ...) src/implicants/bench.py:94-108.
 *       Output contract: caller-owned int64 ranks, unique, ascending
 *       (dense.py:395-397); empty result = count 0.
 *   dqmc_state_bytes
 *       replaces state_bytes(n, h) src/implicants/dense.py:61-63.
 *   DQMC_ERR_RESOURCE + dqmc_last_error()
 *       replaces ResourceLimitError raised by load() before allocating,
 *       message naming the needed byte count (dense.py:358-364,
 *       errors.py:23-24).
 *   DQMC_ERR_INVALID
 *       replaces ValueError for a bad split h (dense.py:356-357) or n.
 *   dqmc_bitmap_device / dqmc_bitmap_download
 *       expose the final bitmap in DenseState.words layout (h = 5,
 *       dense.py:127-170) for bitmap-level parity and k-GPU checks.
 *   dqmc_state_* (device-resident DenseState, any split h)
 *       replace load / DenseState.run_pass / run_merge_reduce /
 *       padding_bits_zero / equal_state / copy / extract_ranks,
 *       dense.py:127-397.
 *
 * Plain pointers and sizes only; no torch or CUDA types in signatures.
 * Device-buffer entry points take a cudaStream_t as void* and use it as
 * given (0 = the legacy default stream, the CUDA convention; torch's default
 * stream is that handle). Host-buffer entry points run on a private stream.
 * All host-buffer entry points are synchronous: results are complete on
 * return, as the reference's Python call is (SURVEY.md §8(b) "Threading").
 */
#ifndef DQMC_H
#define DQMC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
/* the library is built with -fvisibility=hidden: only these symbols export */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define DQMC_ABI_VERSION 5

/* status codes */
#define DQMC_OK 0
#define DQMC_ERR_INVALID 1  /* bad argument          -> ValueError          */
#define DQMC_ERR_RESOURCE 2 /* memory cap exceeded    -> ResourceLimitError  */
#define DQMC_ERR_CUDA 3     /* CUDA runtime failure                         */
#define DQMC_ERR_NODEVICE 4 /* no CUDA device: fail loudly, never fall back */

/* flags */
#define DQMC_FLAG_KEEP_BITMAP 1u /* leave the final prime bitmap in the device state */
#define DQMC_FLAG_TIMING 2u      /* record per-pass CUDA-event times (dqmc_last_timings) */
#define DQMC_FLAG_COUNT_ONLY 4u  /* count primes, do not materialise ranks */
#define DQMC_FLAG_ASYNC 8u       /* dqmc_primes_device only: stream-ordered, no host synchronisation,
                                    CUDA-graph capturable; count_out is then a DEVICE int64 */

/* input encodings */
#define DQMC_IN_WORDS 0 /* TruthTable.words: max(1, 2^n/64) LE uint64, bit x = f(x) */
#define DQMC_IN_U8 1    /* 2^n uint8 values, 0 = off, 1 = on, 2 = don't care (on ∪ dc) */

typedef struct dqmc_result {
    int64_t count;  /* number of prime implicants */
    int64_t *ranks; /* host, ascending, count entries (NULL if count == 0 or COUNT_ONLY) */
    void *_owner;   /* library bookkeeping; release with dqmc_free_result */
} dqmc_result_t;

int dqmc_abi_version(void);
const char *dqmc_last_error(void);
int dqmc_device_count(void);
int dqmc_set_device(int device);

/* dense.py:56-63 */
uint64_t dqmc_block_bits(int h);
uint64_t dqmc_state_bytes(int n, int h);

/* Bytes the engine allocates on the device for n variables (state + scratch,
 * excluding the rank output buffer). */
uint64_t dqmc_device_bytes(int n);

/* dense_prime_ranks(tt, h, optimized, mem_cap) from HOST buffers.
 * h <= 0 means the default min(n, 5); mem_cap == 0 means 75% of free device
 * memory. The result is independent of h and optimized (dense.py:405-418,
 * tests/test_dense.py:218-229); both are validated exactly as the reference. */
int dqmc_primes_tt(const uint64_t *tt_words, int n, int h, uint64_t mem_cap, uint32_t flags,
                   dqmc_result_t *out);
int dqmc_primes_u8(const uint8_t *values, int n, int h, uint64_t mem_cap, uint32_t flags,
                   dqmc_result_t *out);
void dqmc_free_result(dqmc_result_t *res);

/* The same calls as a stream of jobs (at most three outstanding, collected in
 * submission order). dqmc_submit_* queues the table's H2D, every pass and the
 * final stage, and returns; dqmc_collect waits for that job and copies its
 * ranks to the host while the device already runs the next job, so call i's
 * D2H overlaps call i+1's passes. The input must stay valid and unchanged
 * until the job is collected. The first job of an n runs synchronously inside
 * submit (its count sizes the outputs of the next ones); the result is the
 * same as dqmc_primes_tt / dqmc_primes_u8 with h = 0, no cap. flags: as for
 * those (COUNT_ONLY / KEEP_BITMAP / TIMING jobs run synchronously). */
int dqmc_submit_tt(const uint64_t *tt_words, int n, uint32_t flags, int64_t *job);
int dqmc_submit_u8(const uint8_t *values, int n, uint32_t flags, int64_t *job);
int dqmc_collect(int64_t job, dqmc_result_t *out);

/* Results of 4M+ ranks leave the device packed (4-byte cell offsets inside
 * each 3^12-cell tile, rank order: half the PCIe bytes of the reference's
 * int64 ranks, dense.py:376-397) and are widened to int64 by a pool of host
 * threads while the next chunk is on the wire. Sets the pool size (0 =
 * default: min(hardware threads, 16)); returns the previous setting. */
int dqmc_host_threads(int n);
/* The widening step itself, host only (no device needed; also what the CPU
 * tests call): out[i] = (t * tile_cells + rank_add) + off32[i] for tiles
 * t in [t0, t1) and add + pos[t - t0] <= i < add + pos[t - t0 + 1] (the last
 * tile ends at `end`). */
void dqmc_widen_host(const uint32_t *off32, int64_t *out, const int64_t *pos, int64_t add, int64_t end,
                     int64_t t0, int64_t t1, int64_t tile_cells, int64_t rank_add);

/* Same computation with DEVICE-resident input and output (bench `value`,
 * torch integration). ranks_dev may be NULL (count only). If the count
 * exceeds ranks_cap, *count_out is the true count and nothing beyond
 * ranks_cap is written (DQMC_ERR_RESOURCE is NOT raised; the caller grows
 * its buffer and calls again). Synchronises the stream to read the count.
 *
 * With DQMC_FLAG_ASYNC nothing synchronises and nothing is allocated once an
 * earlier synchronous call of the same n has sized the engine's buffers, so
 * back-to-back calls queue on `stream` and the call can be captured into a
 * CUDA graph. count_out is a device int64 written in stream order: the prime
 * count if the ranks are complete, else -(count + 1) (ranks_cap or the
 * engine's rank scratch was too small; call once synchronously, which grows
 * the scratch). Concurrent async calls must share one stream (the engine's
 * workspace is per process). */
int dqmc_primes_device(const void *input_dev, int in_kind, int n, int64_t *ranks_dev, int64_t ranks_cap,
                       int64_t *count_out, uint32_t flags, void *stream);

/* Per-pass timings of the last call made with DQMC_FLAG_TIMING. Returns the
 * number of passes; fills up to max entries of kernel names and ms. */
int dqmc_last_timings(const char **names, float *ms, int max);
/* Algorithmic bytes (reads + writes the plan must do) of each timed pass. */
int dqmc_last_pass_bytes(uint64_t *bytes, int max);

/* Device pointer of the engine's state (reference layout, h = 5) after a
 * call with DQMC_FLAG_KEEP_BITMAP, and its size in bytes. */
int dqmc_bitmap_device(void **ptr, uint64_t *bytes);

/* Copy that final bitmap to a host buffer of dqmc_state_bytes(n, 5) bytes. */
int dqmc_bitmap_download(void *host, uint64_t bytes);

/* Device-resident DenseState for any split h (dense.py:127-397), one
 * streaming kernel per dimension exactly like the reference's layers
 * (dqmc_state.cu). op: 0 = MERGE, 1 = REDUCE. dims are 1-based; counts get
 * 3^(n-h-1) block-triples for top dims, -1 for in-block dims (run_pass's
 * return value). dqmc_state_extract returns DQMC_ERR_INVALID if a padding bit
 * is set (the reference's AssertionError); ranks_host may be NULL to count. */
typedef struct dqmc_state dqmc_state_t;
int dqmc_state_create(int n, int h, uint64_t mem_cap, dqmc_state_t **out);
void dqmc_state_free(dqmc_state_t *st);
int dqmc_state_info(const dqmc_state_t *st, int64_t *out5);  /* n, h, block_bits, blocks, words */
int dqmc_state_load_tt(dqmc_state_t *st, const uint64_t *tt_words_host);
int dqmc_state_set_words(dqmc_state_t *st, const uint64_t *words, uint64_t nwords);
int dqmc_state_get_words(const dqmc_state_t *st, uint64_t *words, uint64_t nwords);
int dqmc_state_run_pass(dqmc_state_t *st, int op, const int *dims, int ndims, int64_t *counts);
int dqmc_state_run_merge_reduce(dqmc_state_t *st);
int dqmc_state_padding_zero(const dqmc_state_t *st, int *ok);
int dqmc_state_extract(const dqmc_state_t *st, int64_t *ranks_host, int64_t cap, int64_t *count);
int dqmc_state_equal(const dqmc_state_t *a, const dqmc_state_t *b, int *eq);
int dqmc_state_copy(const dqmc_state_t *src, dqmc_state_t **out);

/* Device-side synthetic inputs (frozen generator of ttio.py:331-378 and the
 * survey's 3-way / S-box variants); writes 2^n uint8. */
int dqmc_gen3_device(uint8_t *values_dev, int n, double p_on, double p_dc, uint64_t seed, void *stream);
/* Points [x0, x0 + count) only (a rank's slice of a sharded table). */
int dqmc_gen3_range_device(uint8_t *values_dev, int64_t x0, int64_t count, double p_on, double p_dc, uint64_t seed,
                           void *stream);
/* BASELINE config 3 (n = 20): P = stable argsort of the
 * generator values of points 0..1023 under `seed` (a bijection on 10 bits);
 * v[x | P(x) << 10] = 0 for every x, all other 2^20 points 1. */
int dqmc_gen_sbox_device(uint8_t *values_dev, uint64_t seed, void *stream);

/* Host conveniences for the CLI (f1): the frozen generator run on the device
 * and copied to a host buffer of 2^n bytes; and the CLI listing order
 * (wildcard count descending, rank ascending; cli.py:131-138) computed on the
 * device (weight keys + stable radix sort) for `count` ascending ranks. */
int dqmc_gen3_host(uint8_t *values_host, int n, double p_on, double p_dc, uint64_t seed);
int dqmc_gen_sbox_host(uint8_t *values_host, uint64_t seed); /* 2^20 bytes */
int dqmc_order_by_weight(const int64_t *ranks_host, int64_t count, int n, int64_t *out_host);

/* Building blocks of the sharded multi-GPU path (SURVEY.md §8(e),
 * DESIGN.md §6), all on device buffers in the h = 5 layout (n >= 5), all
 * stream-ordered on `stream` (no host synchronisation unless stated):
 * dqmc_merge_device: complete MERGE of all n dimensions (no REDUCE) into
 *   state_out (dqmc_state_bytes(n, 5) bytes) — the implicant bitmap M of
 *   the (sub-)function, DenseState.words after run_pass(MERGE) (dense.py:296-315).
 * dqmc_bitop_device: dst = a & b (op 0) or a | b (op 1), nbytes % 16 == 0.
 * dqmc_bitop_batch_device: the same for njobs (dst, a, b) address triples
 *   stored in device memory (one launch per merge level; a/b may be peer memory).
 * dqmc_reduce_low_device: REDUCE of all n dimensions of nslots consecutive
 *   states (super-blocks) in place.
 * dqmc_extract_kills_device: for nslots low-reduced states, clear in every
 *   state the OR of its parent states (kill_tab: nslots x 8 device addresses,
 *   null padded, local or peer memory) and compact the survivors as ranks +
 *   rank_add[slot] into ranks_dev, slot after slot; slot_start / slot_count
 *   (device) receive each slot's range and *total_out (host) the total. The
 *   one call that synchronises the stream. ranks_dev NULL or
 *   DQMC_FLAG_COUNT_ONLY: counts only. If the total exceeds ranks_cap, nothing
 *   beyond ranks_cap is written and *total_out is the true total. */
int dqmc_merge_device(const void *input_dev, int in_kind, int n, uint32_t *state_out, void *stream);
int dqmc_bitop_device(uint32_t *dst, const uint32_t *a, const uint32_t *b, uint64_t nbytes, int op, void *stream);
int dqmc_bitop_batch_device(const uint64_t *jobs_dev, int64_t njobs, uint64_t nbytes, int op, void *stream);
int dqmc_reduce_low_device(uint32_t *arena, int n, int64_t nslots, void *stream);
int dqmc_extract_kills_device(const uint32_t *arena, int n, int64_t nslots, const uint64_t *kill_tab,
                              const int64_t *rank_add, int64_t *ranks_dev, int64_t ranks_cap, int64_t *slot_start,
                              int64_t *slot_count, int64_t *total_out, uint32_t flags, void *stream);

/* Peer access for the sharded path's P2P transport (one process per GPU):
 * a rank exports a CUDA IPC handle of the allocation holding its arena of
 * super-blocks, plus the arena's byte offset inside it; a peer opens the
 * handle once and passes base + offset + slot straight to dqmc_bitop_device
 * and dqmc_reduce_extract_device, so the AND kernel and the final pass read
 * the peer's memory over NVLink with no staging copy. handle is 64 bytes
 * (cudaIpcMemHandle_t). dqmc_ipc_open also enables peer access between the
 * current device and the allocation's device when they differ. */
int dqmc_ipc_get(const void *dev_ptr, void *handle_out, uint64_t *offset_out);
int dqmc_ipc_open(const void *handle, void **base_out);
int dqmc_ipc_close(void *base);

/* The sparse engine (sparse_prime_ranks, sparse.py:288-307) on the GPU: the
 * level walk over device hash sets of packed cubes (csrc/dqmc_sparse.cu).
 * Same output contract as dqmc_primes_tt; mem_cap bounds every level table
 * (0 = 75% of free device memory), refused before allocating with the
 * reference's message (sparse.py:105-111). Work scales with the implicant
 * count, not 3^n: the engine for low-density functions. */
int dqmc_sparse_primes_tt(const uint64_t *tt_words, int n, uint64_t mem_cap, dqmc_result_t *out);

/* The pass plan the engine runs for n variables (host logic, no GPU needed):
 * out = {ne, H, g, T, m, r[0..7], a[0..7], ib_C, ib_E, ib_D[0..7], rank_sub}
 * (32 int64 entries). Returns the number written. */
int dqmc_plan(int n, int64_t *out, int max);

/* Release all cached device/host workspaces (waits for the device first). */
void dqmc_release(void);

/* Ordering and lifetime of the engine workspace for callers that replay
 * captured CUDA graphs of DQMC_FLAG_ASYNC calls. Every entry point orders its
 * own work after every earlier use of the shared workspace (one event), but a
 * graph replay is the caller's launch: bracket it with dqmc_engine_enter
 * (stream waits for earlier engine work) and dqmc_engine_exit (later calls
 * wait for the replay). dqmc_engine_generation changes whenever a workspace
 * buffer is reallocated or released; a graph captured under another
 * generation holds dangling pointers and must not be replayed. */
uint64_t dqmc_engine_generation(void);
int dqmc_engine_enter(void *stream);
int dqmc_engine_exit(void *stream);

/* The n = 24 plan (two strided groups of six axes) finishes a state one of two
 * ways, chosen on the device from the number of nonzero 256-bit blocks its
 * merge+reduce pass wrote: the read+write REDUCE pass of the lower group
 * (run_pass(REDUCE, dim), dense.py:296-315, one sweep per axis there), or, for
 * sparse states, the "gather finish": that pass is not run and the final stage
 * reads the lower group's parents of each surviving block straight from the
 * state (same result: REDUCE from unreduced parents, dense.py:46-53).
 * dqmc_gather_threshold sets the choice: gather when at most `permille` of
 * every 1000 blocks are nonzero (0 = never, 1000 = always, < 0 = query only);
 * returns the previous setting. dqmc_last_gather reports the block count of
 * the last finished call of that plan and whether it took the gather finish
 * (synchronises the device; DQMC_ERR_INVALID if no such call ran). */
int dqmc_gather_threshold(int permille);
/* Kernels this library has launched so far in this process (its own CUDA
 * kernels of the dense, sharded, sparse and input paths; the per-dimension
 * state API and library calls such as CUB scans are not counted). */
uint64_t dqmc_launch_count(void);
int dqmc_last_gather(int64_t *nonzero_blocks, int64_t *total_blocks, int *gathered);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* DQMC_H */
