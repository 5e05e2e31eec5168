// dqmc_device.cuh — register-level building blocks of the sm_100a kernels.
//
// Layout (identical to the reference DenseState with h = 5, dense.py:1-23,
// 56-63): the 3^n ternary cells are 3^(n-5) blocks of 256 bits (8 x u32);
// bit b of block a is the cube of rank a*243 + b; bits 243..255 are padding
// and stay zero. Block digit k (k = 0 .. n-6) is variable 6+k.
//
// Two kinds of axes:
//  * in-block axes 1..5 (shift distance 3^(i-1) bits inside a block) — done
//    with funnel shifts + LOP3 on a block held in 8 registers;
//  * block axes — a triple of blocks at distance 3^k blocks; done word-wise
//    on small ternary sub-cubes held in registers (cube_merge / cube_reduce).
#pragma once
#include <stdint.h>

namespace dqmc {

__host__ __device__ constexpr int pow3i(int k) {
    int r = 1;
    for (int i = 0; i < k; i++) r *= 3;
    return r;
}

template <int K>
struct P3 {
    static constexpr int v = pow3i(K);
};

// ---------------------------------------------------------------------------
// block-axis sub-cubes: v[idx], idx = sum_i d_i 3^i, d_i in {0,1,2=*}

// MERGE (dense.py:46-48 merge_triple, applied axis by axis as the top layer of
// dense.py:174-212): star slot := s & t.  Assignment instead of |= is exact
// because every cell's value is final at the step of its last star axis and
// is then computed from two cells that are already final (SURVEY.md App. B.1:
// star cells are empty before their axis is merged).
template <int K>
__device__ __forceinline__ void cube_merge(uint32_t (&v)[P3<K>::v]) {
#pragma unroll
    for (int i = 0; i < K; i++) {
        const int s = pow3i(i);
#pragma unroll
        for (int idx = 0; idx < P3<K>::v; idx++) {
            if ((idx / s) % 3 == 0) v[idx + 2 * s] = v[idx] & v[idx + s];
        }
    }
}

// REDUCE (dense.py:51-53 reduce_triple): s &= ~u, t &= ~u, axis by axis,
// in place (any order is exact: SURVEY.md App. B.2).
template <int K>
__device__ __forceinline__ void cube_reduce(uint32_t (&v)[P3<K>::v]) {
#pragma unroll
    for (int i = 0; i < K; i++) {
        const int s = pow3i(i);
#pragma unroll
        for (int idx = 0; idx < P3<K>::v; idx++) {
            if ((idx / s) % 3 == 0) {
                const uint32_t nu = ~v[idx + 2 * s];
                v[idx] &= nu;
                v[idx + s] &= nu;
            }
        }
    }
}

// number of fixed (0/1) digits among the K digits of idx
__host__ __device__ constexpr int fixed_digits(int idx, int K) {
    int f = 0;
    for (int i = 0; i < K; i++) {
        if (idx % 3 != 2) f++;
        idx /= 3;
    }
    return f;
}

// REDUCE of all K axes as ONE parallel step (every kill read from the state
// at step start): P(c) = M(c) & ~OR_{fixed axes i} M(c[i->*]). Done in place
// by visiting cells from most fixed digits to fewest, so every parent (one
// more star) is read before it is itself reduced. ~40% fewer LOP3 than the
// axis-by-axis form; exact by the parallel-step argument.
template <int K>
__device__ __forceinline__ void cube_reduce_par(uint32_t (&v)[P3<K>::v]) {
    constexpr int N = P3<K>::v;
#pragma unroll
    for (int f = K; f >= 1; f--) {
#pragma unroll
        for (int idx = 0; idx < N; idx++) {
            if (fixed_digits(idx, K) == f) {
                uint32_t kill = 0;
#pragma unroll
                for (int i = 0; i < K; i++) {
                    const int s = pow3i(i);
                    const int d = (idx / s) % 3;
                    if (d != 2) kill |= v[idx + (2 - d) * s];
                }
                v[idx] &= ~kill;
            }
        }
    }
}

// ternary index of the binary pattern b (bit k of b -> digit k)
__host__ __device__ constexpr int bin_to_tern(int b) {
    int r = 0, p = 1;
    for (int i = 0; i < 8; i++) {
        if ((b >> i) & 1) r += p;
        p *= 3;
    }
    return r;
}

// does ternary index idx (K digits) contain a star digit?
__host__ __device__ constexpr bool has_star(int idx, int K) {
    for (int i = 0; i < K; i++) {
        if (idx % 3 == 2) return true;
        idx /= 3;
    }
    return false;
}

// ---------------------------------------------------------------------------
// in-block axes (dense.py:216-243 _bottom_dim_optimized / _digit_masks 70-88)

// 32-bit word k of the in-block digit mask: bits p < 243 whose digit `axis`
// (0-based, distance 3^axis) equals d.
__host__ __device__ constexpr uint32_t digit_mask(int axis, int d, int k) {
    uint32_t m = 0;
    for (int b = 0; b < 32; b++) {
        int p = 32 * k + b;
        if (p < 243 && (p / pow3i(axis)) % 3 == d) m |= (1u << b);
    }
    return m;
}

// word K of (v >> S) over the 256-bit block (zero fill from above)
template <int S, int K>
__device__ __forceinline__ uint32_t shr_word(const uint32_t (&v)[8]) {
    constexpr int q = S / 32, r = S % 32;
    const uint32_t lo = (K + q < 8) ? v[(K + q) & 7] : 0u;
    const uint32_t hi = (K + q + 1 < 8) ? v[(K + q + 1) & 7] : 0u;
    if (r == 0) return lo;
    return __funnelshift_r(lo, hi, r);
}

// word K of (v << S) over the 256-bit block (zero fill from below)
template <int S, int K>
__device__ __forceinline__ uint32_t shl_word(const uint32_t (&v)[8]) {
    constexpr int q = S / 32, r = S % 32;
    const uint32_t hi = (K - q >= 0) ? v[(K - q) & 7] : 0u;
    const uint32_t lo = (K - q - 1 >= 0) ? v[(K - q - 1) & 7] : 0u;
    if (r == 0) return hi;
    return __funnelshift_l(lo, hi, r);
}

// Kill mask of in-block axis A (0-based): a cell with digit 0 (1) is killed
// when its star parent at +2d (+d) is set: kill |= ((v>>2d) & M0) | ((v>>d) & M1).
template <int A, int K = 0>
__device__ __forceinline__ void inblock_kill(const uint32_t (&v)[8], uint32_t (&kill)[8]) {
    if constexpr (K < 8) {
        constexpr int d = pow3i(A);
        constexpr uint32_t m0 = digit_mask(A, 0, K), m1 = digit_mask(A, 1, K);
        kill[K] |= (shr_word<2 * d, K>(v) & m0) | (shr_word<d, K>(v) & m1);
        inblock_kill<A, K + 1>(v, kill);
    }
}

// Reduce along the in-block axes selected by `mask` (bit A = axis A+1), all
// kills taken from the same input state (a parallel step; exact by the
// first-killing-axis argument of SURVEY.md App. B.2).
__device__ __forceinline__ void inblock_reduce(uint32_t (&v)[8], uint32_t mask) {
    uint32_t kill[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (mask & 1u) inblock_kill<0>(v, kill);
    if (mask & 2u) inblock_kill<1>(v, kill);
    if (mask & 4u) inblock_kill<2>(v, kill);
    if (mask & 8u) inblock_kill<3>(v, kill);
    if (mask & 16u) inblock_kill<4>(v, kill);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] &= ~kill[k];
}

template <int A, int K = 0>
__device__ __forceinline__ void and_shr(const uint32_t (&v)[8], uint32_t (&x)[8]) {
    if constexpr (K < 8) {
        x[K] = v[K] & shr_word<pow3i(A), K>(v);
        and_shr<A, K + 1>(v, x);
    }
}

template <int A, int K = 0>
__device__ __forceinline__ void or_shl_masked(const uint32_t (&x)[8], uint32_t (&v)[8]) {
    if constexpr (K < 8) {
        constexpr uint32_t m2 = digit_mask(A, 2, K);
        v[K] |= shl_word<2 * pow3i(A), K>(x) & m2;
        or_shl_masked<A, K + 1>(x, v);
    }
}

// In-block MERGE of axis A: u(c+2d) |= s(c) & t(c+d)  (dense.py:228-234)
template <int A>
__device__ __forceinline__ void inblock_merge_axis(uint32_t (&v)[8]) {
    uint32_t x[8];
    and_shr<A>(v, x);
    or_shl_masked<A>(x, v);
}

// All implicants of the 5-variable sub-function given by 32 truth-table bits:
// bit p of w is f(p), p = x1 + 2x2 + ... + 16x5. Spreads p to its ternary rank
// (index_to_rank, ternary.py:120-126) and merges the five in-block axes.
__device__ __forceinline__ void lm5(uint32_t w, uint32_t (&v)[8]) {
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const uint32_t b = (w >> (8 * q)) & 0xFFu;
        // bits (x1,x2,x3) -> positions x1 + 3x2 + 9x3
        const uint32_t s = (b & 0x3u) | ((b & 0xCu) << 1) | ((b & 0x30u) << 5) | ((b & 0xC0u) << 6);
        const int off = 27 * ((q & 1) + 3 * (q >> 1));  // (x4,x5) -> field x4 + 3x5
        const int wk = off / 32, sh = off % 32;
        v[wk] |= s << sh;
        if (sh > 18) v[wk + 1] |= s >> (32 - sh);
    }
    inblock_merge_axis<0>(v);
    inblock_merge_axis<1>(v);
    inblock_merge_axis<2>(v);
    inblock_merge_axis<3>(v);
    inblock_merge_axis<4>(v);
}

}  // namespace dqmc
