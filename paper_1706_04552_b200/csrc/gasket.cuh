// gasket.cuh -- shared device helpers for the sm_100a gasket kernels.
//
// Geometry (reference core.py:75-81, blockmap.py:34-108):
//   cell (x, y) of the n x n grid is a gasket member iff (x & (n-1-y)) == 0;
//   lambda(omega) for omega = (wx, wy) in the 3^floor(r_b/2) x 3^ceil(r_b/2)
//   rectangle sums, for mu = 1..r_b, the region offset of base-3 digit
//   beta_mu (odd mu: digit (mu-1)/2 of wy, even mu: digit mu/2-1 of wx):
//   beta = 0 -> (0,0), 1 -> (0,2^(mu-1)), 2 -> (2^(mu-1),2^(mu-1)).
//   Each level sets exactly one bit per axis, so lambda is a Morton-style
//   interleave of per-axis "digit != 0" (y) and "digit == 2" (x) bit masks.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gm {

enum Kind { KIND_CONST = 0, KIND_NSUM4 = 1, KIND_NSUM8 = 2, KIND_COUNT = 3 };
enum Strategy { STRAT_UNROLL = 0, STRAT_TABLE = 1, STRAT_SUBBOX = 2, STRAT_TUNED = 3 };
enum Mapping { MAP_BB = 0, MAP_LAMBDA = 1, MAP_BB_EXIT = 2, MAP_BB_VEC = 3 };

template <int C> struct CellT;
template <> struct CellT<1> { using T = uint8_t; };
template <> struct CellT<2> { using T = uint16_t; };
template <> struct CellT<4> { using T = uint32_t; };
template <> struct CellT<8> { using T = uint64_t; };

// Wrap-to-width arithmetic: the numba backend sums in 64-bit (int32 param
// sign-extended) and truncates on store (backends.py:127-141); modulo
// 2^(8C) the sign/zero extension of C<8 neighbours is irrelevant.
template <int C>
__device__ __forceinline__ uint64_t ld_cell(const void* base, int64_t idx) {
    using T = typename CellT<C>::T;
    return (uint64_t)__ldg(reinterpret_cast<const T*>(base) + idx);
}
template <int C>
__device__ __forceinline__ void st_cell(void* base, int64_t idx, uint64_t v) {
    using T = typename CellT<C>::T;
    reinterpret_cast<T*>(base)[idx] = (T)v;
}

// backends.py:127-141 _cell_value (+ our 8-neighbour extension, KIND_NSUM8).
template <int C, int KIND>
__device__ __forceinline__ uint64_t cell_value(const void* src, int64_t n, int64_t x, int64_t y,
                                               uint64_t param) {
    if (KIND == KIND_CONST) return param;
    uint64_t t = param;
    const int64_t i = y * n + x;
    const bool l = x > 0, r = x < n - 1, u = y > 0, d = y < n - 1;
    if (l) t += ld_cell<C>(src, i - 1);
    if (r) t += ld_cell<C>(src, i + 1);
    if (u) t += ld_cell<C>(src, i - n);
    if (d) t += ld_cell<C>(src, i + n);
    if (KIND == KIND_NSUM8) {
        if (u && l) t += ld_cell<C>(src, i - n - 1);
        if (u && r) t += ld_cell<C>(src, i - n + 1);
        if (d && l) t += ld_cell<C>(src, i + n - 1);
        if (d && r) t += ld_cell<C>(src, i + n + 1);
    }
    return t;
}

// One cell "op": a store of the kernel value, or (KIND_COUNT, coverage audit
// engine.py:214-258) an atomic increment of a uint32 per-cell counter.
template <int C, int KIND>
__device__ __forceinline__ void cell_op(void* grid, const void* src, int64_t n, int64_t x, int64_t y,
                                        uint64_t param) {
    if (KIND == KIND_COUNT) {
        atomicAdd(reinterpret_cast<unsigned int*>(grid) + (y * n + x), 1u);
    } else {
        st_cell<C>(grid, y * n + x, cell_value<C, KIND>(src, n, x, y, param));
    }
}

// ---------------------------------------------------------------------------
// lambda(omega), three ways.
// ---------------------------------------------------------------------------

// (1) Literal level loop with Python floor semantics on int64 (any input,
//     including out-of-rectangle and negative coordinates): blockmap.py:91-108.
__device__ __forceinline__ int64_t floordiv3(int64_t a) {
    return a >= 0 ? a / 3 : -((-(a + 1)) / 3) - 1;
}
__device__ __forceinline__ void lambda_loop64(int64_t wx, int64_t wy, int r_b, int64_t& lx, int64_t& ly) {
    uint64_t ax = 0, ay = 0;
    for (int mu = 1; mu <= r_b; ++mu) {
        int64_t q;
        int64_t region;
        if (mu & 1) { q = floordiv3(wy); region = wy - 3 * q; wy = q; }
        else        { q = floordiv3(wx); region = wx - 3 * q; wx = q; }
        const uint64_t dx = (uint64_t)(region >> 1);
        const uint64_t step = (mu - 1) < 64 ? (1ull << (mu - 1)) : 0ull;
        ax += dx * step;
        ay += (uint64_t)(region - (int64_t)dx) * step;
    }
    lx = (int64_t)ax;
    ly = (int64_t)ay;
}

// (2) Cooperative lambda, the paper's GPU scheme:
//     lane l owns level mu = l+1, extracts beta_mu, and the per-level offsets
//     (disjoint bits) are combined with one warp reduction (redux.sync.or).
//     `lanes` = participating lanes (<= 32, lanes 0..lanes-1 of the warp).
__device__ __forceinline__ void lambda_warp(uint32_t wx, uint32_t wy, int r_b, int lane, int lanes,
                                            const uint64_t* __restrict__ pow3_magic, uint32_t& lx,
                                            uint32_t& ly) {
    uint32_t px = 0, py = 0;
    for (int l = lane; l < r_b; l += lanes) {
        const uint32_t w = (l & 1) ? wx : wy;
        const int d = l >> 1;
        // w / 3^d exactly for w < 2^32 (magic = floor(2^64/3^d)+1, d >= 1).
        const uint32_t q = d == 0 ? w : (uint32_t)__umul64hi((uint64_t)w, __ldg(pow3_magic + d));
        const uint32_t beta = q % 3u;
        px |= (beta >> 1) << l;
        py |= (beta != 0u ? 1u : 0u) << l;
    }
    const unsigned mask = lanes >= 32 ? 0xffffffffu : ((1u << lanes) - 1u);
    lx = __reduce_or_sync(mask, px);
    ly = __reduce_or_sync(mask, py);
}

// (3) Table closed form for the tuned kernels: 5 base-3 digits per lookup.
//     tab[v] (v < 243) = nonzero-digit mask (bits 0..4) | two-digit mask << 8.
struct DigitTable {
    uint16_t e[243];
};
__device__ __forceinline__ void digit_table_init(uint16_t* tab) {
    for (int v = threadIdx.x + threadIdx.y * blockDim.x; v < 243; v += blockDim.x * blockDim.y) {
        int t = v;
        uint32_t nz = 0, two = 0;
        for (int i = 0; i < 5; ++i) {
            const int d = t % 3;
            t /= 3;
            nz |= (d != 0 ? 1u : 0u) << i;
            two |= (d == 2 ? 1u : 0u) << i;
        }
        tab[v] = (uint16_t)(nz | (two << 8));
    }
}
__device__ __forceinline__ uint32_t spread_even(uint32_t m) {  // 16 -> 32 bit interleave
    m &= 0xffffu;
    m = (m | (m << 8)) & 0x00ff00ffu;
    m = (m | (m << 4)) & 0x0f0f0f0fu;
    m = (m | (m << 2)) & 0x33333333u;
    m = (m | (m << 1)) & 0x55555555u;
    return m;
}

// Digit masks of w < 3^20 (four 5-digit chunks).
__device__ __forceinline__ void digit_masks(uint32_t w, const uint16_t* tab, uint32_t& nz, uint32_t& two) {
    uint32_t c0 = w % 243u; w /= 243u;
    uint32_t c1 = w % 243u; w /= 243u;
    uint32_t c2 = w % 243u; w /= 243u;
    uint32_t c3 = w;  // < 243 for w < 3^20
    const uint32_t e0 = tab[c0], e1 = tab[c1], e2 = tab[c2], e3 = tab[c3];
    nz = (e0 & 31u) | ((e1 & 31u) << 5) | ((e2 & 31u) << 10) | ((e3 & 31u) << 15);
    two = (e0 >> 8) | ((e1 >> 8) << 5) | ((e2 >> 8) << 10) | ((e3 >> 8) << 15);
}

// lambda(omega) exactly as defined (omega in the rectangle, r_b <= 32).
__device__ __forceinline__ void lambda_table(uint32_t wx, uint32_t wy, const uint16_t* tab, uint32_t& lx,
                                             uint32_t& ly) {
    uint32_t nzx, twx, nzy, twy;
    digit_masks(wx, tab, nzx, twx);
    digit_masks(wy, tab, nzy, twy);
    ly = spread_even(nzy) | (spread_even(nzx) << 1);
    lx = spread_even(twy) | (spread_even(twx) << 1);
}

// lambda composed with the digit-order linearisation of the rectangle:
// compact tile index c (base-3 digit i <-> level i+1).  Same image, same
// per-tile cell sets; consecutive c are spatially adjacent tiles.
__device__ __forceinline__ void lambda_digit_order(uint32_t c, const uint16_t* tab, uint32_t& lx, uint32_t& ly) {
    uint32_t nz, two;
    digit_masks(c, tab, nz, two);
    ly = nz;
    lx = two;
}

// Row-major order of the member tiles of a level-q gasket: tile k-th in the
// row-major enumeration (block row Y ascending, then column l ascending over the
// l that are bit-subsets of Y).  F(Y) = #member tiles in block rows < Y
//      = sum over set bits b of Y of 3^b * 2^popcount(Y >> (b+1)).
__device__ __forceinline__ uint32_t rows_before(uint32_t Y) {
    uint32_t f = 0, p3 = 1, above = __popc(Y);
    for (int b = 0; b < 20 && (Y >> b); ++b) {
        if ((Y >> b) & 1u) {
            --above;
            f += p3 << above;
        }
        p3 *= 3u;
    }
    return f;
}
__device__ __forceinline__ uint32_t pdep32(uint32_t i, uint32_t mask) {
    uint32_t out = 0;
    while (mask) {
        const uint32_t low = mask & (0u - mask);
        if (i & 1u) out |= low;
        i >>= 1;
        mask ^= low;
    }
    return out;
}
__device__ __forceinline__ void tile_rowmajor(uint32_t k, int q, uint32_t& l, uint32_t& Y) {
    uint32_t lo = 0, hi = 1u << q;  // largest Y with rows_before(Y) <= k
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (rows_before(mid) <= k) lo = mid; else hi = mid;
    }
    Y = lo;
    l = pdep32(k - rows_before(lo), lo);
}

// ---------------------------------------------------------------------------
// synthetic inputs (shared definition with oracle/gasket_oracle.c)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace gm
