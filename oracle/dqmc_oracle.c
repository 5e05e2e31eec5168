/*
 * dqmc_oracle.c — CPU restatement of the reference DenseQMC engine.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product): linked by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs. The product path (paper_2302_10083_b200, libdqmc.so) never
 * loads this file.
 *
 * It restates /root/reference/pkg/src/implicants/dense.py line by line in C,
 * with OpenMP over the independent triples/blocks the reference already
 * declares independent:
 *   block_bits_for / state_bytes ........ dense.py:56-63
 *   _digit_masks ......................... dense.py:70-88
 *   DenseState._top_dim .................. dense.py:174-212
 *   DenseState._bottom_dim_optimized ..... dense.py:216-243
 *   DenseState._bottom_dim_reference ..... dense.py:245-280
 *   DenseState.run_pass .................. dense.py:296-315
 *   DenseState.run_merge_reduce .......... dense.py:317-337
 *   load (+ index_to_rank) ............... dense.py:340-373, ternary.py:120-126
 *   extract_ranks ........................ dense.py:376-397
 *   padding_bits_zero .................... dense.py:154-160
 * State layout is identical to DenseState.words: block a occupies words
 * [a*wpb, (a+1)*wpb), bit b of block a is rank a*3^h + b, padding zero.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OP_MERGE 0
#define OP_REDUCE 1

static int64_t pow3(int k) {
    int64_t r = 1;
    while (k-- > 0) r *= 3;
    return r;
}

/* dense.py:56-58 */
int64_t oracle_block_bits(int h) {
    int64_t used = pow3(h), b = 1;
    while (b < used) b <<= 1;
    return b < 64 ? 64 : b;
}

/* dense.py:61-63 */
int64_t oracle_state_bytes(int n, int h) { return pow3(n - h) * oracle_block_bits(h) / 8; }

int oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

/* dense.py:70-88 — masks[(d*h + (i-1))*wpb + w] selects in-block bits whose
 * digit i equals d; padding positions are zero in every mask. */
static uint64_t *digit_masks(int h) {
    int64_t bb = oracle_block_bits(h), wpb = bb / 64, used = pow3(h);
    uint64_t *m = (uint64_t *)calloc((size_t)(3 * h * wpb), sizeof(uint64_t));
    for (int i = 1; i <= h; i++) {
        int64_t p3 = pow3(i - 1);
        for (int64_t pos = 0; pos < used; pos++) {
            int d = (int)((pos / p3) % 3);
            m[((int64_t)d * h + (i - 1)) * wpb + pos / 64] |= 1ULL << (pos % 64);
        }
    }
    return m;
}

/* multiword shifts inside one block (little-endian word stream, zero fill) */
static void shl_block(const uint64_t *src, uint64_t *dst, int64_t wpb, int64_t bits) {
    int64_t q = bits / 64, r = bits % 64;
    for (int64_t k = wpb - 1; k >= 0; k--) {
        uint64_t v = 0;
        if (k - q >= 0) {
            v = src[k - q] << r;
            if (r && k - q - 1 >= 0) v |= src[k - q - 1] >> (64 - r);
        }
        dst[k] = v;
    }
}

static void shr_block(const uint64_t *src, uint64_t *dst, int64_t wpb, int64_t bits) {
    int64_t q = bits / 64, r = bits % 64;
    for (int64_t k = 0; k < wpb; k++) {
        uint64_t v = 0;
        if (k + q < wpb) {
            v = src[k + q] >> r;
            if (r && k + q + 1 < wpb) v |= src[k + q + 1] << (64 - r);
        }
        dst[k] = v;
    }
}

/* dense.py:216-243, applied block by block (the flat-chunk shifts of the
 * reference leak only onto masked-off positions, dense.py:219-222, so the
 * per-block form is identical). */
static void bottom_dim_opt(uint64_t *v, int64_t wpb, const uint64_t *masks, int h, int i, int op,
                           uint64_t *t1, uint64_t *t2) {
    int64_t d = pow3(i - 1);
    const uint64_t *m0 = masks + ((int64_t)0 * h + (i - 1)) * wpb;
    const uint64_t *m1 = masks + ((int64_t)1 * h + (i - 1)) * wpb;
    const uint64_t *m2 = masks + ((int64_t)2 * h + (i - 1)) * wpb;
    if (op == OP_MERGE) {
        /* u |= s & t : v |= (v << 2d) & (v << d) & digit2 */
        shl_block(v, t1, wpb, 2 * d);
        shl_block(v, t2, wpb, d);
        for (int64_t k = 0; k < wpb; k++) v[k] |= t1[k] & t2[k] & m2[k];
    } else {
        /* s &= ~u, t &= ~u : v &= ~(((v >> 2d) & digit0) | ((v >> d) & digit1)) */
        shr_block(v, t1, wpb, 2 * d);
        shr_block(v, t2, wpb, d);
        for (int64_t k = 0; k < wpb; k++) v[k] &= ~((t1[k] & m0[k]) | (t2[k] & m1[k]));
    }
}

/* dense.py:245-280: literal shift-right / mask / op / recompose form */
static void bottom_dim_ref(uint64_t *v, int64_t wpb, const uint64_t *masks, int h, int i, int op,
                           uint64_t *s, uint64_t *t, uint64_t *u, uint64_t *tmp) {
    int64_t d = pow3(i - 1);
    const uint64_t *mu = masks + ((int64_t)0 * h + (i - 1)) * wpb; /* digit-0 selector */
    shr_block(v, s, wpb, 0);
    shr_block(v, t, wpb, d);
    shr_block(v, u, wpb, 2 * d);
    for (int64_t k = 0; k < wpb; k++) { s[k] &= mu[k]; t[k] &= mu[k]; u[k] &= mu[k]; }
    for (int64_t k = 0; k < wpb; k++) {
        if (op == OP_MERGE) {
            u[k] |= s[k] & t[k];                       /* merge_triple, dense.py:46-48 */
        } else {
            s[k] &= ~u[k]; t[k] &= ~u[k];             /* reduce_triple, dense.py:51-53 */
        }
    }
    for (int64_t k = 0; k < wpb; k++) v[k] = s[k];
    shl_block(t, tmp, wpb, d);
    for (int64_t k = 0; k < wpb; k++) v[k] |= tmp[k];
    shl_block(u, tmp, wpb, 2 * d);
    for (int64_t k = 0; k < wpb; k++) v[k] |= tmp[k];
}

/* dense.py:174-212: top dimension i (1-based above the split) */
int64_t oracle_top_dim(uint64_t *words, int n, int h, int i, int op) {
    int64_t wpb = oracle_block_bits(h) / 64;
    int64_t nw = pow3(n - h) * wpb;
    int64_t inner = pow3(i - 1) * wpb;
    int64_t groups = nw / (3 * inner);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t g = 0; g < groups; g++) {
        for (int64_t c = 0; c < inner; c++) {
            uint64_t *s = words + g * 3 * inner + c;
            uint64_t *t = s + inner;
            uint64_t *u = t + inner;
            if (op == OP_MERGE) {
                *u |= *s & *t;
            } else {
                uint64_t nu = ~*u;
                *s &= nu;
                *t &= nu;
            }
        }
    }
    return groups * inner / wpb; /* block-triple count, 3^(n-h-1) */
}

/* dense.py:282-292: one bottom dimension over every block */
void oracle_bottom_dim(uint64_t *words, int n, int h, int i, int op, int optimized) {
    int64_t wpb = oracle_block_bits(h) / 64;
    int64_t blocks = pow3(n - h);
    uint64_t *masks = digit_masks(h);
#pragma omp parallel
    {
        uint64_t *buf = (uint64_t *)malloc((size_t)(4 * wpb) * sizeof(uint64_t));
#pragma omp for schedule(static)
        for (int64_t a = 0; a < blocks; a++) {
            uint64_t *v = words + a * wpb;
            if (optimized)
                bottom_dim_opt(v, wpb, masks, h, i, op, buf, buf + wpb);
            else
                bottom_dim_ref(v, wpb, masks, h, i, op, buf, buf + wpb, buf + 2 * wpb, buf + 3 * wpb);
        }
        free(buf);
    }
    free(masks);
}

/* dense.py:296-315: dims processed in the given order (1-based). Returns 0,
 * or -1 on a bad op / dimension (the reference raises ValueError). */
int oracle_run_pass(uint64_t *words, int n, int h, int op, const int *dims, int ndims, int optimized,
                    int64_t *counts) {
    if (op != OP_MERGE && op != OP_REDUCE) return -1;
    for (int k = 0; k < ndims; k++)
        if (dims[k] < 1 || dims[k] > n) return -1;
    for (int k = 0; k < ndims; k++) {
        int dim = dims[k];
        if (dim > h) {
            int64_t c = oracle_top_dim(words, n, h, dim - h, op);
            if (counts) counts[k] = c;
        } else {
            oracle_bottom_dim(words, n, h, dim, op, optimized);
            if (counts) counts[k] = -1;
        }
    }
    return 0;
}

/* dense.py:317-337: top merges, per-block bottom merges then reduces, top reduces */
void oracle_run_merge_reduce(uint64_t *words, int n, int h) {
    int64_t wpb = oracle_block_bits(h) / 64;
    int64_t blocks = pow3(n - h);
    for (int i = 1; i <= n - h; i++) oracle_top_dim(words, n, h, i, OP_MERGE);
    uint64_t *masks = digit_masks(h);
#pragma omp parallel
    {
        uint64_t *buf = (uint64_t *)malloc((size_t)(2 * wpb) * sizeof(uint64_t));
#pragma omp for schedule(static)
        for (int64_t a = 0; a < blocks; a++) {
            uint64_t *v = words + a * wpb;
            for (int i = 1; i <= h; i++) bottom_dim_opt(v, wpb, masks, h, i, OP_MERGE, buf, buf + wpb);
            for (int i = 1; i <= h; i++) bottom_dim_opt(v, wpb, masks, h, i, OP_REDUCE, buf, buf + wpb);
        }
        free(buf);
    }
    free(masks);
    for (int i = 1; i <= n - h; i++) oracle_top_dim(words, n, h, i, OP_REDUCE);
}

/* ternary.py:120-126: binary point index -> ternary rank of the 0/1 string */
static int64_t index_to_rank(uint64_t x, int n) {
    int64_t r = 0, p = 1;
    for (int i = 0; i < n; i++, p *= 3)
        if ((x >> i) & 1) r += p;
    return r;
}

/* dense.py:340-373 (without the memory-cap check, done by the caller):
 * words must hold state_bytes(n,h)/8 zeroed uint64. tt has max(1, 2^n/64) words. */
void oracle_load(const uint64_t *tt, int n, int h, uint64_t *words) {
    int64_t bb = oracle_block_bits(h), used = pow3(h);
    int64_t npts = (int64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < npts; x++) {
        if ((tt[x >> 6] >> (x & 63)) & 1) {
            int64_t r = index_to_rank((uint64_t)x, n);
            int64_t block = r / used, bit = r % used;
            int64_t flat = block * bb + bit;
            __atomic_fetch_or(&words[flat >> 6], 1ULL << (flat & 63), __ATOMIC_RELAXED);
        }
    }
}

/* dense.py:154-160 */
int oracle_padding_bits_zero(const uint64_t *words, int n, int h) {
    int64_t bb = oracle_block_bits(h), wpb = bb / 64, used = pow3(h), blocks = pow3(n - h);
    int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
    for (int64_t a = 0; a < blocks; a++) {
        for (int64_t k = 0; k < wpb; k++) {
            uint64_t w = words[a * wpb + k];
            int64_t lo = k * 64;
            uint64_t pad;
            if (lo >= used) pad = ~0ULL;
            else if (lo + 64 <= used) pad = 0;
            else pad = ~0ULL << (used - lo);
            if (w & pad) bad = 1;
        }
    }
    return !bad;
}

/* dense.py:376-397: ranks of set bits, ascending (memory order = rank order).
 * Returns the count; writes ranks if out != NULL (must hold count entries).
 * Returns -2 if a padding bit is set (the reference raises AssertionError). */
int64_t oracle_extract(const uint64_t *words, int n, int h, int64_t *out) {
    int64_t bb = oracle_block_bits(h), wpb = bb / 64, used = pow3(h);
    int64_t nw = pow3(n - h) * wpb;
    if (!oracle_padding_bits_zero(words, n, h)) return -2;
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    int64_t *part = (int64_t *)calloc((size_t)nt + 1, sizeof(int64_t));
    int team = 1;
#pragma omp parallel num_threads(nt)
    {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        int64_t lo = nw * t / T, hi = nw * (t + 1) / T, c = 0;
        for (int64_t w = lo; w < hi; w++) c += __builtin_popcountll(words[w]);
        part[t + 1] = c;
#pragma omp barrier
#pragma omp single
        {
            team = T;
            for (int k = 0; k < T; k++) part[k + 1] += part[k];
        }
        if (out) {
            int64_t o = part[t];
            for (int64_t w = lo; w < hi; w++) {
                uint64_t v = words[w];
                while (v) {
                    int b = __builtin_ctzll(v);
                    v &= v - 1;
                    int64_t flat = w * 64 + b;
                    out[o++] = (flat / bb) * used + (flat % bb);
                }
            }
        }
    }
    int64_t total = part[team];
    free(part);
    return total;
}

/* dense.py:405-418 end to end. *out is malloc'ed (caller frees with
 * oracle_free). Returns the prime count, -1 bad h, -3 allocation failure. */
int64_t oracle_dense_prime_ranks(const uint64_t *tt, int n, int h, int optimized, int64_t **out) {
    *out = NULL;
    if (h < 1 || h > n) return -1;
    int64_t nwords = oracle_state_bytes(n, h) / 8;
    uint64_t *words = (uint64_t *)calloc((size_t)nwords, sizeof(uint64_t));
    if (!words) return -3;
    oracle_load(tt, n, h, words);
    if (optimized) {
        oracle_run_merge_reduce(words, n, h);
    } else {
        int *dims = (int *)malloc(sizeof(int) * (size_t)n);
        int k = 0;
        for (int d = h + 1; d <= n; d++) dims[k++] = d; /* default order, dense.py:306 */
        for (int d = 1; d <= h; d++) dims[k++] = d;
        oracle_run_pass(words, n, h, OP_MERGE, dims, n, 0, NULL);
        oracle_run_pass(words, n, h, OP_REDUCE, dims, n, 0, NULL);
        free(dims);
    }
    int64_t cnt = oracle_extract(words, n, h, NULL);
    if (cnt < 0) { free(words); return cnt; }
    int64_t *r = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt > 0 ? cnt : 1));
    if (!r) { free(words); return -3; }
    oracle_extract(words, n, h, r);
    free(words);
    *out = r;
    return cnt;
}

void oracle_free(void *p) { free(p); }
