// stencil_tb.cu -- T = 2 or 4 CA steps fused in one pass over memory (temporal
// blocking), for the multi-step CA driver (ca.py).
//
// A CA step is the reference's neighbour-sum launch with engine.launch's
// snapshot semantics (engine.py:201; backends.py:127-141 for 4 neighbours, our
// labelled 8-neighbour extension): state t+1 = param + sum of the in-grid
// neighbours of state t on gasket cells, state t elsewhere (off-gasket cells
// never change).  The single-step kernel (stencil2.cu) is bound by the DRAM
// access pattern of one read of the dilated gasket + one partial-line write
// per step; this kernel does that traffic once per T steps:
//
//   per lambda tile (TT x TT cells, rows one 128-byte line; CTAs in the row-major
//   tile order of stencil2.cu):
//   1. stage state t on rows -T..TT+T-1 (16-byte halo chunk each side) -- only the
//      chunks the phases read or the store blends (host-precomputed list) -- into
//      the S slot;
//   2. phases p = 1..T compute state t+p on the 4-byte words that phase p+1 reads
//      (the tile's own gasket words for p = T): the dependency cone of the tile,
//      shrinking by one cell per phase.  Ring words outside the tile belong to
//      neighbouring tiles and are computed redundantly (overlapped tiling) with the
//      exact global membership test (x & ~y) == 0 and in-grid, so ring words of
//      non-gasket neighbour tiles keep state t.
//      Only words that can hold gasket cells ("gsk", superset test modulo the tile)
//      are ever computed; every other word keeps state t, which stays in S.  Odd
//      phases read S and write their gsk words to I; even phases read gsk words
//      from I and the others from S, and write their gsk words back into S (no
//      phase reads the S gsk words it overwrites).  T is even: the result is in S.
//   3. every touched sector of the tile is stored whole from S (off-gasket cells are
//      state t: the CA invariant that both ping-pong buffers agree off the gasket).
// Work is per word, not per sector, and the tile's gasket words go in vertical runs
// of V rows.  Work lists are host-precomputed (tile-independent supersets).
// Arithmetic: the split-lane SIMD of stencil_common.cuh.  Results are bit-identical
// to T single steps (tests/test_gpu_parity.py).
#include <algorithm>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "gasket.cuh"
#include "launch.h"
#include "stencil_common.cuh"
#include "peer_epilogue.cuh"
#include "../../include/gasket_b200.h"

namespace gm {
namespace {

using namespace sc;

constexpr int ROWB = 128;
constexpr int PITCH = ROWB + 32;  // 16 B halo | 128 B row | 16 B halo (a 16 B pad: same speed)
constexpr int CHUNKS = 10;
constexpr int MAX_T = 6;
#ifndef TB_ONE_SLOT_FROM_T
#define TB_ONE_SLOT_FROM_T 6  // T = 6: one staging slot, 4 CTAs per SM (903 vs 916 us per launch; T = 4: 663 vs 652)
#endif

// Skewed row layout of the staged (S) and odd-phase (I) buffers: tile row r sits at
// buffer row idx = r + SHIFT, at byte idx * PITCH + 16 * ((r + 8) >> 2): 16 more bytes
// per 4-row quad (monotone, so rows never overlap).  The vertical-run work items of a
// warp come from several quads; with a plain 176-byte pitch a quad step moves the bank
// by 16, so items two quads apart with the same word collided.  The skew makes the
// quad step 20 banks: 8 consecutive quads land in 8 bank groups.  The skew of a tile
// row is the same in S and I, so the same word is `dS` bytes apart in the two.
constexpr int SKEW_BYTES = 16 * 36;  // >= 16 * (((TT + MAX_T - 1) + 8) >> 2) for TT <= 128
template <int SHIFT>
__device__ __host__ __forceinline__ int row_off(int idx) {
    return idx * PITCH + 16 * ((idx - SHIFT + 8) >> 2);  // tile row idx - SHIFT >= -8
}

template <int C, int T>
struct TB {
    static constexpr int V = 4 / C;
    static constexpr int TT = ROWB / C;
    static constexpr int SC = 32 / C;
    static constexpr int CC = 16 / C;          // cells per chunk
    static constexpr int SROWS = TT + 2 * T;   // state t rows -T .. TT+T-1
    static constexpr int IROWS = TT + 2 * T - 2;  // odd-phase results, rows -(T-1) .. TT+T-2
    static constexpr int SH_S = T, SH_I = T - 1;  // buffer row = tile row + SH
    // S slots are whole multiples of 128 bytes and I starts 32 bytes past one (IOFF): a word of
    // S and the same tile word in I (one row lower, SH_I = SH_S - 1) then sit in the same
    // bank, so the even phases' mixed S/I loads keep the conflict pattern of the odd phases
    // (sbuf - ibuf + PITCH == 0 mod 128)
    static constexpr int SBUF = (SROWS * PITCH + SKEW_BYTES + 127) / 128 * 128;
    static constexpr int IOFF = 32;
    static constexpr int IBUF = IROWS * PITCH + SKEW_BYTES;
    static constexpr int NTOUCH = 9 * SC;
    // 4/3 threads per touched sector: the store pass uses the first NTOUCH, the work
    // lists of the phases all of them.  With 16-bit work lists the CTA needs < 76 KB of
    // shared memory: 3 CTAs x 12 warps per SM for byte cells, which overlaps one CTA's
    // arithmetic with the others' memory phases better than 2 x 18 warps (n=2^17 NSUM8,
    // T = 2: 485 vs 549 us per pair)
    static constexpr int THREADS = (NTOUCH * 4 / 3 + 31) / 32 * 32;
};

// the work-list counts: staged chunks, the tile's runs (every phase), phase p's ring
// words at ring[p-1] .. ring[p] of the ring area
struct TbCounts {
    int ns = 0, ni = 0;
    int ring[MAX_T + 1] = {0, 0, 0, 0, 0, 0, 0};
};

// word k (cells (k-4)*V ..) of tile row r can hold gasket cells for some gasket
// neighbour tile: the superset test modulo the tile (r may be negative or >= TT)
template <int C>
__device__ __host__ __forceinline__ bool gsk_word(int r, int k) {
    constexpr int TT = ROWB / C, V = 4 / C;
    const uint32_t xm = (uint32_t)((k - 4) * V) & (TT - 1), rm = (uint32_t)r & (TT - 1);
    return (xm & ~rm) == 0;
}

// gasket cells of a word whose first cell is (x, y) (x a multiple of the word's
// cell count, so x + j = x | j): all-or-nothing on x, then the pattern of y's low bits
template <int C>
__device__ __forceinline__ uint32_t word_mask(int x, int y, int n) {
    const bool in = (unsigned)y < (unsigned)n && (unsigned)x < (unsigned)n && (x & ~y) == 0;
    return in ? member_mask<C>((uint32_t)y) : 0u;
}

template <int C, int T>
__device__ __forceinline__ const uint8_t* s_word(const uint8_t* sbuf, int r, int k) {
    return sbuf + row_off<TB<C, T>::SH_S>(r + TB<C, T>::SH_S) + 4 * k;
}
template <int C, int T>
__device__ __forceinline__ const uint8_t* i_word(const uint8_t* ibuf, int r, int k) {
    return ibuf + row_off<TB<C, T>::SH_I>(r + TB<C, T>::SH_I) + 4 * k;
}

// One word of state t+p at (tile row r, word k) from the 3 x 3 words around it.
// MIXED = false: all from S; MIXED = true: gsk words from I, the others from S.
template <int C, bool EIGHT, int T, bool MIXED>
__device__ __forceinline__ uint32_t word_sum(const uint8_t* ibuf, const uint8_t* sbuf, int r, int k, uint32_t pv,
                                             uint32_t& centre) {
    const int dS = (int)(sbuf - ibuf) + PITCH;
    uint32_t w[3][3];
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) {
        if constexpr (MIXED) {
            const uint8_t* row = i_word<C, T>(ibuf, r - 1 + rr, k);
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
                w[rr][cc] = *reinterpret_cast<const uint32_t*>(
                    row + 4 * (cc - 1) + (gsk_word<C>(r - 1 + rr, k - 1 + cc) ? 0 : dS));
        } else {
            const uint32_t* row = reinterpret_cast<const uint32_t*>(s_word<C, T>(sbuf, r - 1 + rr, k));
            w[rr][0] = row[-1];
            w[rr][1] = row[0];
            w[rr][2] = row[1];
        }
    }
    uint32_t o[1];
    sector_sums<C, EIGHT, 1>(w, pv, o);
    centre = w[1][1];
    return o[0];
}

// A vertical run of RUN = V words (word k of tile rows t0 .. t0+RUN-1, t0 a multiple of
// V) from the RUN+2 rows around it: row loads and lane splits are shared between the
// outputs.  Word k of a tile row holds gasket cells for a whole aligned run of V rows
// (its first cell k*V only constrains bits >= log2 V of the row), and the cell pattern
// of run row j is member_mask(j).  Rows t0 .. t0+RUN-1 also share one gsk pattern, so
// MIXED sources come in 3 row classes x 3 columns.
template <int C, bool EIGHT, int RUN, int T, bool MIXED>
__device__ __forceinline__ void vstrip(const uint8_t* ibuf, const uint8_t* sbuf, int t0, int k, uint32_t pv,
                                       uint32_t (&out)[RUN], uint32_t (&centre)[RUN]) {
    using S = TB<C, T>;
    const uint8_t* r1 = MIXED ? i_word<C, T>(ibuf, t0, k) : s_word<C, T>(sbuf, t0, k);  // tile row t0
    int sel[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if constexpr (MIXED) {
        const int dS = (int)(sbuf - ibuf) + PITCH;
        const uint32_t rm[3] = {(uint32_t)(t0 - 1) & (S::TT - 1), (uint32_t)t0, (uint32_t)(t0 + RUN) & (S::TT - 1)};
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            const uint32_t xm = (uint32_t)((k - 5 + cc) * S::V) & (S::TT - 1);
#pragma unroll
            for (int rc = 0; rc < 3; ++rc) sel[rc][cc] = (xm & ~rm[rc]) == 0 ? 0 : dS;
        }
    }
    uint32_t w[RUN + 2][3];
#pragma unroll
    for (int i = 0; i < RUN + 2; ++i) {
        const int rc = i == 0 ? 0 : i == RUN + 1 ? 2 : 1;
        // (RUN == 4: rows t0..t0+3 are one quad; one skew step before it and one after)
        const int roff = (RUN == 4) ? (i - 1) * PITCH + (i == 0 ? -16 : i == RUN + 1 ? 16 : 0)
                                    : row_off<0>(t0 - 1 + i) - row_off<0>(t0);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
            w[i][cc] = *reinterpret_cast<const uint32_t*>(r1 + roff + 4 * (cc - 1) + sel[rc][cc]);
    }
#pragma unroll
    for (int j = 0; j < RUN; ++j) {
        const uint32_t win[3][3] = {{w[j][0], w[j][1], w[j][2]},
                                    {w[j + 1][0], w[j + 1][1], w[j + 1][2]},
                                    {w[j + 2][0], w[j + 2][1], w[j + 2][2]}};
        uint32_t o[1];
        sector_sums<C, EIGHT, 1>(win, pv, o);
        out[j] = o[0];
        centre[j] = w[j + 1][1];
    }
}

template <int C, int KIND, int T, int NST>
__global__ void __launch_bounds__(TB<C, T>::THREADS)
    stencil_tb(uint8_t* __restrict__ grid, const uint8_t* __restrict__ src, int64_t n, uint32_t ntiles,
               uint64_t param, const uint32_t* __restrict__ order, const uint16_t* __restrict__ lists_g,
               TbCounts cnt, int flags, PeerEpilogue* epi, uint64_t wait_epoch, uint64_t signal_epoch,
               const int64_t* __restrict__ sg_off, int64_t pitch, uint32_t per) {
    using S = TB<C, T>;
    // NST = staging slots: 2 (tile idx+1 staged while idx computes) or 1 (staged after
    // tile idx is stored; a smaller CTA, so 4 instead of 3 share an SM)
    static_assert(NST == 1 || NST == 2, "one or two staging slots");
    static_assert(T % 2 == 0 && T <= MAX_T, "an even number of fused steps leaves the result in S");
    peer_prologue_wait(epi, wait_epoch);  // partitioned CA with the fused exchange only
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ibuf = smem + NST * S::SBUF + S::IOFF;
    // work lists: staged chunks as j * 16 + q (S row j, chunk q); runs as t0 * 64 + k
    // (first tile row, word k); ring words as (r + T) * 64 + k (tile row r, word k)
    uint16_t* slist = reinterpret_cast<uint16_t*>(ibuf + S::IBUF);
    const uint16_t* ilist = slist + cnt.ns;
    const int ns = cnt.ns, ni = cnt.ni;
    for (int i = threadIdx.x; i < ns + ni + cnt.ring[T]; i += S::THREADS) slist[i] = lists_g[i];
    __syncthreads();

    const bool v8 = (reinterpret_cast<uintptr_t>(grid) & 31u) == 0;
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(smem);
    const int64_t rowbytes = n * C;  // the global grid's row (bounds)
    const int64_t rowstride = pitch;  // the buffers' row pitch (addresses; tiled storage: its blocks')
    uint32_t pv;
    if constexpr (C == 1) pv = 0x00010001u * (uint32_t)(param & 0xffu);
    else if constexpr (C == 2) pv = (uint32_t)(param & 0xffffu);
    else pv = (uint32_t)param;

    // store-pass thread -> touched sector (t, g), as stencil2.cu
    const int e = threadIdx.x;
    int h, off;
    if (e < S::SC) { h = 0; off = 0; }
    else if (e < 3 * S::SC) { h = 1; off = S::SC; }
    else if (e < 5 * S::SC) { h = 2; off = 3 * S::SC; }
    else { h = 3; off = 5 * S::SC; }
    const int per_row = h == 0 ? 1 : h == 3 ? 4 : 2;
    const int t = h * S::SC + (e - off) / per_row;
    const int ii = (e - off) % per_row;
    const int g = h == 2 ? 2 * ii : ii;
    const bool active = e < S::NTOUCH;

    const uint32_t count = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
    auto tile_v = [&](uint32_t idx) { return idx < count ? __ldg(order + blockIdx.x + idx * gridDim.x) : 0u; };
    // byte offset of this CTA's tile #idx's sub-gasket block (tiled partition storage)
    auto tile_off = [&](uint32_t idx) -> int64_t {
        return sg_off != nullptr ? __ldg(sg_off + (blockIdx.x + idx * gridDim.x) / per) : 0;
    };
    auto tile_xy = [&](uint32_t v, int64_t& x0, int64_t& y0) {
        x0 = (int64_t)(v & 0xffffu) * S::TT;
        y0 = (int64_t)(v >> 16) * S::TT;
    };
    // design probes (scripts/variants.py): drop staging / arithmetic / stores
#ifdef GM_AB_VARIANTS
    const bool probe_noload = (flags & GM_FLAG_PROBE_NOLOAD) != 0;
#else
    constexpr bool probe_noload = false;  // design probe: A/B builds only
#endif
#ifdef GM_AB_VARIANTS
    const bool probe_nocompute = (flags & GM_FLAG_PROBE_NOCOMPUTE) != 0;
#else
    constexpr bool probe_nocompute = false;  // design probe: A/B builds only
#endif
#ifdef GM_AB_VARIANTS
    const bool probe_nostore = (flags & GM_FLAG_PROBE_NOSTORE) != 0;
#else
    constexpr bool probe_nostore = false;  // design probe: A/B builds only
#endif
    const bool fetch_line = (flags & GM_FLAG_FETCH_LINE) != 0;
    auto stage = [&](uint32_t idx, uint32_t v) {
        if (idx >= count || probe_noload) return;
        int64_t x0, y0;
        tile_xy(v, x0, y0);
        const uint32_t sb = smem0 + (idx % NST) * S::SBUF;
        const uint8_t* srct = src + tile_off(idx);
        const uint8_t* base = srct + (y0 - T) * rowstride + x0 * C - 16;  // staged (row -T, chunk 0)
        const bool interior = y0 >= T && y0 + S::TT + T <= n && x0 > 0 && x0 + S::TT < n;
        for (int i = threadIdx.x; i < ns; i += S::THREADS) {
            const uint32_t c = slist[i];
            const int j = (int)(c >> 4), q = (int)(c & 15u);
            const uint32_t so = sb + (uint32_t)(row_off<T>(j) + q * 16);
            if (interior) {
                cp_async16(so, base + (int64_t)j * rowstride + q * 16, 16, fetch_line);
            } else {
                const int64_t y = y0 + j - T;
                const int64_t xb = x0 * C + (q - 1) * 16;
                const bool in = y >= 0 && y < n && xb >= 0 && xb < rowbytes;
                cp_async16(so, in ? srct + y * rowstride + xb : src, in ? 16 : 0, fetch_line);
            }
        }
    };

    // When the next tile's staging starts matters (n=2^17 NSUM8, scripts/tb_ab.sh): for
    // T = 2 its order entry is loaded after the barrier, so the staging starts an L2
    // round trip after the previous tile's store burst (418 us per launch vs 440-458
    // with the entry loaded a tile ahead); for T = 4 the tile ahead wins (649 vs 671 us).
    constexpr bool AHEAD = T >= 4;
    uint32_t v_cur = tile_v(0), v_next = AHEAD ? tile_v(1) : 0u;
    stage(0, v_cur);
    cp_async_commit();
    for (uint32_t idx = 0; idx < count; ++idx) {
        const uint32_t v_after = AHEAD ? tile_v(idx + 2) : 0u;
        cp_async_wait<0>();
        __syncthreads();  // state t of tile idx staged; tile idx-1 fully stored (I and its S slot free)
        if constexpr (!AHEAD) v_next = tile_v(idx + 1);
        if constexpr (NST == 2) {
            stage(idx + 1, v_next);
            cp_async_commit();
        }
        int64_t x0, y0;
        tile_xy(v_cur, x0, y0);
        v_cur = v_next;
        v_next = v_after;
        uint8_t* sbuf = smem + (idx % NST) * S::SBUF;

        // ---- phases 1..T: item i < ni is a run of the tile's gasket words, the rest are
        //      phase p's ring words (exact global mask)
#pragma unroll
        for (int p = 1; p <= T; ++p) {  // (unrolled: each phase's code is specialised)
            const bool odd = (p & 1) != 0;
            const int nr = cnt.ring[p] - cnt.ring[p - 1];
            const uint16_t* rl = ilist + ni + cnt.ring[p - 1];
            for (int i = probe_nocompute ? ni + nr : threadIdx.x; i < ni + nr; i += S::THREADS) {
                if (i < ni) {
                    const int c = (int)ilist[i];
                    const int t0 = c >> 6, k = c & 63;
                    uint32_t sum[S::V], centre[S::V];
                    if (odd) vstrip<C, EIGHT, S::V, T, false>(ibuf, sbuf, t0, k, pv, sum, centre);
                    else vstrip<C, EIGHT, S::V, T, true>(ibuf, sbuf, t0, k, pv, sum, centre);
                    // odd phases write I, even phases S; rows t0 .. t0+V-1: one quad, one skew
                    uint32_t* dst = reinterpret_cast<uint32_t*>(
                        const_cast<uint8_t*>(odd ? i_word<C, T>(ibuf, t0, k) : s_word<C, T>(sbuf, t0, k)));
#pragma unroll
                    for (int j = 0; j < S::V; ++j) {
                        const uint32_t m = member_mask<C>((uint32_t)j);
                        dst[j * (PITCH / 4)] = (sum[j] & m) | (centre[j] & ~m);
                    }
                } else {
                    const int c = (int)rl[i - ni];
                    const int r = (c >> 6) - T, k = c & 63;
                    uint32_t centre;
                    const uint32_t sum = odd ? word_sum<C, EIGHT, T, false>(ibuf, sbuf, r, k, pv, centre)
                                             : word_sum<C, EIGHT, T, true>(ibuf, sbuf, r, k, pv, centre);
                    const uint32_t m = word_mask<C>((int)x0 + (k - 4) * S::V, (int)y0 + r, (int)n);
                    uint32_t* dst = reinterpret_cast<uint32_t*>(
                        const_cast<uint8_t*>(odd ? i_word<C, T>(ibuf, r, k) : s_word<C, T>(sbuf, r, k)));
                    *dst = (sum & m) | (centre & ~m);
                }
            }
            __syncthreads();
        }

        // ---- store: every touched sector whole (its S row now holds state t+T)
        if (active && !probe_nostore) {
            const int k0 = 4 + 8 * g;
            const uint32_t* srow = reinterpret_cast<const uint32_t*>(s_word<C, T>(sbuf, t, 0));
            const uint4 a = *reinterpret_cast<const uint4*>(srow + k0);
            const uint4 b = *reinterpret_cast<const uint4*>(srow + k0 + 4);
            const uint32_t out[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            st_sector(grid + tile_off(idx) + (y0 + t) * rowstride + x0 * C + g * 32, out, v8, false);
        }
        if constexpr (NST == 1) {  // the slot is free once every thread has read its sector
            __syncthreads();
            stage(idx + 1, v_cur);  // (v_cur already holds tile idx+1's order entry)
            cp_async_commit();
        }
    }
    cp_async_wait<0>();
    peer_epilogue_signal(grid, epi, signal_epoch);  // partitioned CA with the fused exchange only
}

// ---- host: the work lists (tile-independent supersets) ----------------------

// Reorder the list segment [b, e) of `v` so that the entries one warp instruction serves
// together fall on distinct shared-memory banks where the bank histogram allows: blocks of
// `blk` consecutive entries (the first block `first` entries long: where the segment starts
// inside a warp's 32 items), each filled round-robin over the keys with the most entries
// left.  Entries are independent work items (no order inside a list), so only the bank
// pattern changes (ncu, n=2^17 NSUM8, T = 6: 212 M shared wavefronts for 84 M ideal, most of
// it 2.5-way conflicts of the phases' loads/stores and 4.8-way of the staging copies).
template <class Key>
void spread_banks(std::vector<uint32_t>& v, size_t b, size_t e, Key key, int nkeys, int blk, int first) {
    std::vector<std::vector<uint32_t>> by(nkeys);
    for (size_t i = b; i < e; ++i) by[key(v[i])].push_back(v[i]);
    for (auto& q : by) std::reverse(q.begin(), q.end());  // (pop_back keeps the original order per key)
    std::vector<int> order(nkeys);
    size_t left = e - b, o = b;
    int size = first > 0 ? first : blk;
    while (left) {
        int cnt = 0;
        while (cnt < size && left) {
            for (int k = 0; k < nkeys; ++k) order[k] = k;
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return by[x].size() > by[y].size(); });
            for (int k : order) {
                if (cnt == size || by[k].empty()) break;
                v[o++] = by[k].back();
                by[k].pop_back();
                ++cnt;
                --left;
            }
        }
        size = blk;
    }
}

struct TbLists {
    uint16_t* lists = nullptr;  // [staged chunks | the tile's runs | ring words of phases 1..T]
    TbCounts cnt;
};

// The dependency cone of one tile, every neighbouring tile assumed a gasket tile (so
// the lists hold for every tile; the kernel's exact masks do the rest).  Cells are
// (c, r) in tile coordinates, c in [-CC, TT+CC), r in [-T, TT+T); word k of a row holds
// cells (k-4)*V .. (k-4)*V+V-1.  N_p = the cells whose state t+p must be right:
//   N_T     = the tile's touched sectors (stored whole);
//   W_p     = the gsk words holding a cell of N_p (computed at phase p: readers take
//             gsk words from phase p's output buffer); the other N_p cells are in
//             words that never change and are read from S (staged);
//   N_{p-1} = the N_p cells of W_p words and the neighbours of those that may be
//             gasket cells (a word's other cells may hold garbage: no reader uses
//             them, and the split-lane sums never carry between cells).
// Staged: N_0 (phase 1's inputs) and every N_p cell outside W_p words.
template <int C>
void build_lists(bool eight, int T, std::vector<uint32_t>& out, TbCounts& cnt) {
    constexpr int TT = ROWB / C, CC = 16 / C, V = 4 / C, SC = 32 / C;
    const int W = TT + 2 * CC, H = TT + 2 * T;
    auto mod = [&](int v) { return ((v % TT) + TT) % TT; };
    auto sup = [&](int c, int r) { return (mod(c) & ~mod(r)) == 0; };
    auto cell = [&](int c, int r) {
        if (c < -CC || c >= TT + CC || r < -T || r >= TT + T)
            throw std::runtime_error("stencil_tb: dependency cone outside the staged window");
        return (r + T) * W + (c + CC);
    };
    auto in_tile_word = [&](int r, int k) { return r >= 0 && r < TT && k >= 4 && k < 4 + TT / V; };
    std::vector<std::pair<int, int>> offs = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
    if (eight) offs.insert(offs.end(), {{1, 1}, {1, -1}, {-1, 1}, {-1, -1}});
    std::vector<char> N(W * H, 0), staged(W * H, 0);
    for (int r = 0; r < TT; ++r)
        for (int g = 0; g < ROWB / 32; ++g)
            if (((g * SC) & ~r) == 0)
                for (int c = g * SC; c < (g + 1) * SC; ++c) N[cell(c, r)] = 1;
    std::vector<std::vector<std::pair<int, int>>> ring(T + 1);
    for (int p = T; p >= 1; --p) {
        std::set<std::pair<int, int>> Wp;
        std::vector<char> prev(W * H, 0);
        for (int r = -T; r < TT + T; ++r)
            for (int c = -CC; c < TT + CC; ++c) {
                if (!N[cell(c, r)]) continue;
                const int k = (c + CC) / V;
                if (!gsk_word<C>(r, k)) {
                    staged[cell(c, r)] = 1;
                    continue;
                }
                Wp.insert({r, k});
                prev[cell(c, r)] = 1;
                if (sup(c, r))
                    for (auto [dx, dy] : offs) prev[cell(c + dx, r + dy)] = 1;
            }
        for (auto [r, k] : Wp)
            if (!in_tile_word(r, k)) ring[p].push_back({r, k});
        N.swap(prev);
    }
    for (int i = 0; i < W * H; ++i) staged[i] = staged[i] || N[i];
    out.clear();
    for (int r = -T; r < TT + T; ++r)
        for (int q = 0; q < CHUNKS; ++q) {
            bool any = false;
            for (int c = (q - 1) * CC; c < q * CC; ++c) any = any || staged[cell(c, r)];
            if (any) out.push_back((uint32_t)((r + T) * 16 + q));
        }
    cnt.ns = (int)out.size();
    // (the staging copies keep their row-major order: a cp.async fills shared memory once per
    // global sector it reads, so chunks of one row side by side beat any bank-aware order)
    auto roff = [&](int idx) { return idx * PITCH + 16 * ((idx - T + 8) >> 2); };  // row_off<T>: S row idx
    // the tile's gasket words, one entry per aligned run of V rows (every phase: every
    // N_p, p < T, holds all their cells)
    for (int t0 = 0; t0 < TT; t0 += V)
        for (int w = 0; w < TT / V; ++w)
            if (((w * V) & ~t0) == 0) out.push_back((uint32_t)(t0 * 64 + w + 4));
    cnt.ni = (int)out.size() - cnt.ns;
    // the runs: 32-bit loads/stores at word k of the run's rows; the bank of an entry is that
    // of its first word in S (I has the same pattern shifted)
    auto bank = [&](int r, int k) { return ((roff(r + T) >> 2) + k) & 31; };  // tile row r, word k
    spread_banks(out, cnt.ns, out.size(), [&](uint32_t c) { return bank((int)(c >> 6), (int)(c & 63u)); }, 32, 32, 0);
    cnt.ring[0] = 0;
    for (int p = 1; p <= MAX_T; ++p) {
        const size_t b0 = out.size();
        if (p <= T)
            for (auto [r, k] : ring[p]) out.push_back((uint32_t)((r + T) * 64 + k));
        // phase p's ring items follow the runs in the same thread loop: item ni + i
        spread_banks(out, b0, out.size(), [&](uint32_t c) { return bank((int)(c >> 6) - T, (int)(c & 63u)); }, 32, 32,
                     (32 - cnt.ni % 32) % 32);
        cnt.ring[p] = (int)out.size() - cnt.ns - cnt.ni;
    }
}

template <int C>
const TbLists* tb_lists(bool eight, int T) {
    static std::mutex mu;
    static std::map<std::tuple<int, bool, int>, TbLists> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(dev, eight, T);
    auto it = cache.find(key);
    if (it != cache.end()) return &it->second;
    std::vector<uint32_t> v;
    TbLists L;
    build_lists<C>(eight, T, v, L.cnt);
    std::vector<uint16_t> v16(v.begin(), v.end());  // every entry < 2^16
    if (cudaMalloc(&L.lists, v16.size() * 2) != cudaSuccess ||
        cudaMemcpy(L.lists, v16.data(), v16.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return &(cache[key] = L);
}

template <int C, int KIND, int T, int NST>
cudaError_t launch_ck(const LaunchArgs& a, int r_t) {
    using S = TB<C, T>;
    // tile range: the whole gasket, or (partitioned launches, gm_run_part_steps) the digit-order
    // sub-gasket range [sg_begin, sg_end) of level part_level; the order table groups
    // tiles by those sub-gaskets, so the range is a contiguous run of it
    uint32_t lo, hi;
    tile_range(a, r_t, lo, hi);
    if (hi == lo) return cudaSuccess;
    const uint32_t ntiles = hi - lo;
    const TbLists* L = tb_lists<C>(KIND == KIND_NSUM8, T);
    const uint32_t* order = rowmajor_table(r_t, order_level(a, r_t));
    if (order != nullptr) order += lo;
    if (L == nullptr || order == nullptr) return cudaErrorMemoryAllocation;
    const int entries = L->cnt.ns + L->cnt.ni + L->cnt.ring[T];
    const size_t smem = (size_t)NST * S::SBUF + S::IOFF + S::IBUF + 2 * (size_t)entries;
    auto* kern = stencil_tb<C, KIND, T, NST>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, smem);
    if (getenv("GASKET_DEBUG_OCC"))
        fprintf(stderr, "stencil_tb<C=%d,K=%d,T=%d>: %d CTAs/SM, smem %zu, lists %d+%d+%d\n", C, KIND, T, per_sm, smem,
                L->cnt.ns, L->cnt.ni, L->cnt.ring[T]);
    uint64_t blocks = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > ntiles) blocks = ntiles;
    kern<<<(unsigned)blocks, S::THREADS, smem, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid),
                                                          reinterpret_cast<const uint8_t*>(a.src), a.n, ntiles,
                                                          a.param, order, L->lists, L->cnt, a.flags,
                                                          reinterpret_cast<PeerEpilogue*>(a.peer_epi), a.wait_epoch,
                                                          a.signal_epoch, a.sg_off, row_pitch(a),
                                                          tiles_per_subgasket(a, r_t));
    note_launch();
    return cudaGetLastError();
}

template <int C, int T>
cudaError_t launch_c(const LaunchArgs& a, int r) {
    int k = 0;
    while ((1 << k) < TB<C, T>::TT) ++k;
    if (r - k > 15) return cudaErrorNotSupported;  // tile-order table limit
    constexpr int NST = T >= TB_ONE_SLOT_FROM_T ? 1 : 2;
    if (a.kind == KIND_NSUM4) return launch_ck<C, KIND_NSUM4, T, NST>(a, r - k);
    if (a.kind == KIND_NSUM8) return launch_ck<C, KIND_NSUM8, T, NST>(a, r - k);
    return cudaErrorNotSupported;
}

template <int T>
cudaError_t launch_t(const LaunchArgs& a) {
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    // the cone reaches T cells past the tile: it must fit the 16-byte halo chunks
    switch (a.cell_bytes) {
    case 1: if (a.n >= TB<1, T>::TT && T <= TB<1, T>::CC) return launch_c<1, T>(a, r); break;
    case 2: if (a.n >= TB<2, T>::TT && T <= TB<2, T>::CC) return launch_c<2, T>(a, r); break;
    case 4: if (a.n >= TB<4, T>::TT && T <= TB<4, T>::CC) return launch_c<4, T>(a, r); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace

// T fused CA steps (T = 2, 4 or 6): grid <- step^T(src); grid must equal src off the
// gasket.  cudaErrorNotSupported for other T, grids narrower than one tile, cell widths
// other than 1, 2, 4, and T = 6 on 4-byte cells (the cone outgrows the halo chunk).
cudaError_t launch_stencil_tb(const LaunchArgs& a, int steps) {
    if (steps == 2) return launch_t<2>(a);
    if (steps == 4) return launch_t<4>(a);
    if (steps == 6) return launch_t<6>(a);
    return cudaErrorNotSupported;
}
cudaError_t launch_stencil_tb2(const LaunchArgs& a) { return launch_stencil_tb(a, 2); }

}  // namespace gm
