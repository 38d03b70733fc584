// stencil_tb.cu -- two CA steps fused in one pass over memory (temporal
// blocking), for the multi-step CA driver (ca.py).
//
// A CA step is the reference's neighbour-sum launch with engine.launch's
// snapshot semantics (engine.py:201; backends.py:127-141 for 4 neighbours, our
// labelled 8-neighbour extension): state t+1 = param + sum of the in-grid
// neighbours of state t on gasket cells, state t elsewhere (off-gasket cells
// never change).  The single-step kernel (stencil2.cu) is bound by the DRAM
// access pattern of one read of the dilated gasket + one partial-line write
// per step; this kernel does that traffic once per TWO steps:
//
//   per lambda tile (TT x TT cells, rows one 128-byte line; CTAs in the row-major
//   tile order of stencil2.cu):
//   1. stage state t on rows -2..TT+1 (16-byte halo chunk each side) -- only the
//      chunks phase 1 or the off-gasket blend read (host-precomputed list);
//   2. phase 1: state t+1 on every 4-byte word of rows -1..TT holding a cell
//      that a gasket cell of the tile reads (its 4/8-neighbourhood and itself):
//      words that can hold gasket cells are computed (exact global membership
//      (x & ~y) == 0 and in-grid, so ring words of non-gasket neighbour tiles
//      stay state t), the others copied -- the ring belongs to neighbouring
//      tiles and is computed redundantly (overlapped tiling);
//   3. phase 2: state t+2 on the tile's words that hold gasket cells, written
//      over state t in the staging slot;
//   4. every touched sector stored whole, off-gasket cells from state t (the
//      CA invariant that both ping-pong buffers agree off the gasket).
// Work is per word, not per sector: only ~42% of a touched sector's words hold
// gasket cells, and the fused pass is arithmetic-heavy (two steps per tile).
// Work lists are host-precomputed (tile-independent supersets).  Arithmetic:
// the split-lane SIMD of stencil_common.cuh.  Results are bit-identical to two
// single steps (tests/test_gpu_parity.py).
#include <map>
#include <mutex>
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
constexpr int PITCH = ROWB + 48;  // 16 B halo | 128 B row | 16 B halo | 16 B pad
constexpr int CHUNKS = 10;

// Skewed row layout of the staged (S) and state-t+1 (I) buffers: the row of tile row r
// starts at idx * PITCH + 16 * ((r + 4) >> 2) (idx = buffer row, r = idx - SHIFT >= -4):
// 16 more bytes per 4-row quad (monotone, so rows never overlap).  The vertical-run
// work items of a warp come from several quads; with a plain 176-byte pitch a quad
// step moves the bank by 16, so items two quads apart with the same word collided.
// The skew makes the quad step 20 banks: 8 consecutive quads land in 8 bank groups.
constexpr int SKEW_BYTES = 16 * 36;  // >= 16 * (((TT + 1) + 4) >> 2) for TT <= 128
template <int SHIFT>
__device__ __host__ __forceinline__ int row_off(int idx) {
    return idx * PITCH + 16 * ((idx - SHIFT + 4) >> 2);
}

template <int C>
struct TB {
    static constexpr int V = 4 / C;
    static constexpr int TT = ROWB / C;
    static constexpr int SC = 32 / C;
    static constexpr int CC = 16 / C;          // cells per chunk
    static constexpr int SROWS = TT + 4;       // state-t rows -2 .. TT+1
    static constexpr int IROWS = TT + 2;       // state-t+1 rows -1 .. TT
    static constexpr int SBUF = SROWS * PITCH + SKEW_BYTES;
    static constexpr int IBUF = IROWS * PITCH + SKEW_BYTES;
    static constexpr int NTOUCH = 9 * SC;
    // 4/3 threads per touched sector: the store pass uses the first NTOUCH, the work
    // lists of phases 1-2 all of them.  With 16-bit work lists and no offset table the
    // CTA needs 73 KB of shared memory: 3 CTAs x 12 warps per SM for byte cells, which
    // overlaps one CTA's arithmetic with the others' memory phases better than
    // 2 x 18 warps (n=2^17 NSUM8: 485 vs 549 us per pair)
    static constexpr int THREADS = (NTOUCH * 4 / 3 + 31) / 32 * 32;
};

// gasket cells of a word whose first cell is (x, y) (x a multiple of the word's
// cell count, so x + j = x | j): all-or-nothing on x, then the pattern of y's low bits
template <int C>
__device__ __forceinline__ uint32_t word_mask(int x, int y, int n) {
    const bool in = (unsigned)y < (unsigned)n && (unsigned)x < (unsigned)n && (x & ~y) == 0;
    return in ? member_mask<C>((uint32_t)y) : 0u;
}

// word k (0..39, 4 halo words each side) of staged rows ji-1+0..2 -> one result word
template <int C, bool EIGHT, int SHIFT>
__device__ __forceinline__ uint32_t word_sum(const uint8_t* buf, int row0, int k, uint32_t pv, uint32_t& centre) {
    // rows row0 .. row0+2 of `buf` (skewed layout), word k
    uint32_t w[3][3];
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(buf + row_off<SHIFT>(row0 + rr));
        w[rr][0] = row[k - 1];
        w[rr][1] = row[k];
        w[rr][2] = row[k + 1];
    }
    uint32_t o[1];
    sector_sums<C, EIGHT, 1>(w, pv, o);
    centre = w[1][1];
    return o[0];
}

// A vertical run of RUN words (word k of RUN consecutive rows) from RUN+2 rows of `buf`
// starting at buffer row row0 (the row above the first output): row loads and lane splits
// are shared between the outputs.  Word k of a tile row holds gasket cells for a
// whole aligned run of V rows (its first cell k*V only constrains bits >= log2 V of
// the row), and the cell pattern of run row j is member_mask(j).
template <int C, bool EIGHT, int RUN, int SHIFT>
__device__ __forceinline__ void vstrip(const uint8_t* buf, int row0, int k, uint32_t pv, uint32_t (&out)[RUN],
                                       uint32_t (&centre)[RUN]) {
    uint32_t w[RUN + 2][3];
    // the run's rows are the last row of one quad, the V rows of the next, and the first
    // row of the one after (runs start at a tile row that is a multiple of V = 4 for
    // byte cells): offsets relative to the second row step by PITCH, plus one skew step
    // before it and one after the run
    const uint8_t* r1 = buf + row_off<SHIFT>(row0 + 1) + 4 * k;
#pragma unroll
    for (int i = 0; i < RUN + 2; ++i) {
        const int skew = (RUN == 4) ? (i == 0 ? -16 : i == RUN + 1 ? 16 : 0) : 0;
        const uint32_t* row = (RUN == 4) ? reinterpret_cast<const uint32_t*>(r1 + (i - 1) * PITCH + skew)
                                         : reinterpret_cast<const uint32_t*>(buf + row_off<SHIFT>(row0 + i)) + k;
        w[i][0] = row[-1];
        w[i][1] = row[0];
        w[i][2] = row[1];
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

// Phase 2's strip: state t+1 of tile rows t0-1 .. t0+RUN around word k.  Phase 1 wrote
// state t+1 into I only for the words that can hold gasket cells (superset test, the
// work lists' `gsk`); every other word has no gasket cell, so its state t+1 is its
// state t, read from the staged S slot instead (same skew for the same tile row, so the
// S address is the I address + dS).  Rows t0 .. t0+RUN-1 share one membership pattern
// (t0 is a multiple of V = RUN), so 3 row classes x 3 columns of sources.
template <int C, bool EIGHT, int RUN>
__device__ __forceinline__ void vstrip_p2(const uint8_t* ibuf, const uint8_t* sbuf, int t0, int k, uint32_t pv,
                                          uint32_t (&out)[RUN], uint32_t (&centre)[RUN]) {
    using S = TB<C>;
    const uint8_t* i1 = ibuf + row_off<1>(t0 + 1) + 4 * k;  // tile row t0, word k, in I
    const int dS = (int)(sbuf - ibuf) + PITCH;               // -> the same word in S
    const uint32_t rm[3] = {(uint32_t)(t0 - 1) & (S::TT - 1), (uint32_t)t0, (uint32_t)(t0 + RUN) & (S::TT - 1)};
    int sel[3][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const uint32_t xm = (uint32_t)((k - 5 + cc) * S::V) & (S::TT - 1);
#pragma unroll
        for (int rc = 0; rc < 3; ++rc) sel[rc][cc] = (xm & ~rm[rc]) == 0 ? 0 : dS;
    }
    uint32_t w[RUN + 2][3];
#pragma unroll
    for (int i = 0; i < RUN + 2; ++i) {
        const int rc = i == 0 ? 0 : i == RUN + 1 ? 2 : 1;
        // (RUN == 4: rows t0..t0+3 are one quad; one skew step before it and one after)
        const int roff = (RUN == 4) ? (i - 1) * PITCH + (i == 0 ? -16 : i == RUN + 1 ? 16 : 0)
                                    : row_off<1>(t0 + i) - row_off<1>(t0 + 1);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
            w[i][cc] = *reinterpret_cast<const uint32_t*>(i1 + roff + 4 * (cc - 1) + sel[rc][cc]);
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

template <int C, int KIND, int NST>
__global__ void __launch_bounds__(TB<C>::THREADS)
    stencil_tb2(uint8_t* __restrict__ grid, const uint8_t* __restrict__ src, int64_t n, uint32_t ntiles,
                uint64_t param, const uint32_t* __restrict__ order, const uint16_t* __restrict__ lists_g, int ns,
                int np1, int ng1, int ni1, int np2, int flags, PeerEpilogue* epi, uint64_t wait_epoch,
                uint64_t signal_epoch) {
    using S = TB<C>;
    peer_prologue_wait(epi, wait_epoch);  // partitioned CA with the fused exchange only
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ibuf = smem + NST * S::SBUF;          // state t+1, rows -1..TT
    // work lists: staged chunks as j * 16 + q (buffer row j, chunk q); phase-1/2 items as
    // row * 64 + k (buffer row, word k) -- offsets follow from the skewed row_off()
    uint16_t* slist = reinterpret_cast<uint16_t*>(ibuf + S::IBUF);
    uint16_t* p1list = slist + ns;                 // runs of inner gasket words, ring gasket words, copies
    uint16_t* p2list = p1list + np1;               // runs of the tile's gasket words
    const int64_t rowstride = n * C;
    for (int i = threadIdx.x; i < ns + np1 + np2; i += S::THREADS) {
        slist[i] = lists_g[i];
    }
    __syncthreads();

    const bool v8 = (reinterpret_cast<uintptr_t>(grid) & 31u) == 0;
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(smem);
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
    auto tile_xy = [&](uint32_t v, int64_t& x0, int64_t& y0) {
        x0 = (int64_t)(v & 0xffffu) * S::TT;
        y0 = (int64_t)(v >> 16) * S::TT;
    };
    // design probes (scripts/variants.py): drop staging / arithmetic / stores
    const bool probe_noload = (flags & GM_FLAG_PROBE_NOLOAD) != 0;
    const bool probe_nocompute = (flags & GM_FLAG_PROBE_NOCOMPUTE) != 0;
    const bool probe_nostore = (flags & GM_FLAG_PROBE_NOSTORE) != 0;
    const bool fetch_line = (flags & GM_FLAG_FETCH_LINE) != 0;
    auto stage = [&](uint32_t idx, uint32_t v) {
        if (idx >= count || probe_noload) return;
        int64_t x0, y0;
        tile_xy(v, x0, y0);
        const uint32_t sb = smem0 + (idx % NST) * S::SBUF;
        const uint8_t* base = src + (y0 - 2) * rowstride + x0 * C - 16;  // staged (row -2, chunk 0)
        const bool interior = y0 >= 2 && y0 + S::TT + 2 <= n && x0 > 0 && x0 + S::TT < n;
        for (int i = threadIdx.x; i < ns; i += S::THREADS) {
            const uint32_t c = slist[i];
            const int j = (int)(c >> 4), q = (int)(c & 15u);
            const uint32_t so = sb + (uint32_t)(row_off<2>(j) + q * 16);
            if (interior) {
                cp_async16(so, base + (int64_t)j * rowstride + q * 16, 16, fetch_line);
            } else {
                const int64_t y = y0 + j - 2;
                const int64_t xb = x0 * C + (q - 1) * 16;
                const bool in = y >= 0 && y < n && xb >= 0 && xb < rowstride;
                cp_async16(so, in ? src + y * rowstride + xb : src, in ? 16 : 0, fetch_line);
            }
        }
    };

    static_assert(NST == 2, "the tile-order registers below assume a 2-deep ring");
    // order entries are loaded one tile ahead of their use: the staging of tile idx+1
    // right after the barrier would otherwise wait on a global load every tile
    uint32_t v_cur = tile_v(0), v_next = tile_v(1);
    stage(0, v_cur);
    cp_async_commit();
    for (uint32_t idx = 0; idx < count; ++idx) {
        const uint32_t v_after = tile_v(idx + 2);
        cp_async_wait<NST - 2>();
        __syncthreads();  // state t of tile idx staged; tile idx-1 fully stored (I and its S slot free)
        stage(idx + 1, v_next);
        cp_async_commit();
        int64_t x0, y0;
        tile_xy(v_cur, x0, y0);
        v_cur = v_next;
        v_next = v_after;
        const uint8_t* sbuf = smem + (idx % NST) * S::SBUF;

        // ---- phase 1: state t+1 on rows -1..TT.  Item = ji * 64 + k: I row ji (tile row ji - 1,
        //      S rows ji .. ji+2), word k.
        //      [0, ni1): runs of V tile rows of a word holding gasket cells (first row);
        //      [ni1, np1): ring words that may hold gasket cells (exact global test).
        //      Words that cannot hold gasket cells keep state t: phase 2 reads them from S.
        for (int i = probe_nocompute ? np1 : threadIdx.x; i < np1; i += S::THREADS) {
            const int c = (int)p1list[i];
            const int ji = c >> 6, k = c & 63;
            if (i < ni1) {
                uint32_t sum[S::V], centre[S::V];
                vstrip<C, EIGHT, S::V, 2>(sbuf, ji, k, pv, sum, centre);
                uint32_t* dst = reinterpret_cast<uint32_t*>(ibuf + row_off<1>(ji)) + k;  // V rows of one quad
#pragma unroll
                for (int j = 0; j < S::V; ++j) {
                    const uint32_t m = member_mask<C>((uint32_t)j);
                    dst[j * (PITCH / 4)] = (sum[j] & m) | (centre[j] & ~m);
                }
            } else {
                uint32_t centre;
                const uint32_t sum = word_sum<C, EIGHT, 2>(sbuf, ji, k, pv, centre);
                const uint32_t m = word_mask<C>((int)x0 + (k - 4) * S::V, (int)y0 + ji - 1, (int)n);
                reinterpret_cast<uint32_t*>(ibuf + row_off<1>(ji))[k] = (sum & m) | (centre & ~m);
            }
        }
        __syncthreads();

        // ---- phase 2: state t+2 on the tile's gasket words, in runs of V rows (I rows t-1..t+V),
        //      blended with state t and written over state t in the staging slot (phase 1 is
        //      done with it; the store pass below reads the slot).  Item = t * 64 + k for the
        //      run's first tile row t (I row t = tile row t - 1; S row t + 2 = tile row t).
        for (int i = probe_nocompute ? np2 : threadIdx.x; i < np2; i += S::THREADS) {
            const int c = (int)p2list[i];
            const int t0 = c >> 6, k = c & 63;
            uint32_t sum[S::V], centre[S::V];
            vstrip_p2<C, EIGHT, S::V>(ibuf, sbuf, t0, k, pv, sum, centre);
            uint32_t* sp0 = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(sbuf) + row_off<2>(t0 + 2)) + k;
#pragma unroll
            for (int j = 0; j < S::V; ++j) {  // tile rows t0 .. t0+V-1: one quad, one skew
                uint32_t* sp = sp0 + j * (PITCH / 4);
                const uint32_t m = member_mask<C>((uint32_t)j);
                *sp = (sum[j] & m) | (*sp & ~m);
            }
        }
        __syncthreads();

        // ---- store: every touched sector whole (its slot row now holds state t+2)
        if (active && !probe_nostore) {
            const int k0 = 4 + 8 * g;
            const uint32_t* srow = reinterpret_cast<const uint32_t*>(sbuf + row_off<2>(t + 2));
            const uint4 a = *reinterpret_cast<const uint4*>(srow + k0);
            const uint4 b = *reinterpret_cast<const uint4*>(srow + k0 + 4);
            const uint32_t out[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            st_sector(grid + (y0 + t) * rowstride + x0 * C + g * 32, out, v8, false);
        }
    }
    cp_async_wait<0>();
    peer_epilogue_signal(grid, epi, signal_epoch);  // partitioned CA with the fused exchange only
}

// ---- host: the work lists (tile-independent supersets) ----------------------
struct TbLists {
    uint16_t* lists = nullptr;  // [staged chunks | phase-1 words | phase-2 words] (smem byte offsets)
    int ns = 0, np1 = 0, ng1 = 0, ni1 = 0, np2 = 0;
};

// Cells of the staged window: c in [-CC, TT+CC), r in [-2, TT+1]; staged word k
// (0..39) holds cells (k-4)*V .. (k-4)*V+V-1.
template <int C>
void build_lists(bool eight, std::vector<uint32_t>& out, int& ns, int& np1, int& ng1, int& ni1, int& np2) {
    using S = TB<C>;
    const int TT = S::TT, CC = S::CC, V = S::V;
    const int W = TT + 2 * CC, H = TT + 4;  // window: column c -> c + CC, row r -> r + 2
    auto mod = [&](int v) { return ((v % TT) + TT) % TT; };
    // superset membership: every neighbouring tile assumed to be a gasket tile
    auto member_sup = [&](int c, int r) { return (mod(c) & ~mod(r)) == 0; };
    auto own = [&](int c, int r) { return c >= 0 && c < TT && r >= 0 && r < TT && (c & ~r) == 0; };
    std::vector<char> D1(W * H, 0), need(W * H, 0);
    auto at = [&](std::vector<char>& v, int c, int r) -> char& { return v[(r + 2) * W + (c + CC)]; };
    auto inwin = [&](int c, int r) { return c >= -CC && c < TT + CC && r >= -2 && r < TT + 2; };
    std::vector<std::pair<int, int>> offs = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}};
    if (eight) offs.insert(offs.end(), {{1, 1}, {1, -1}, {-1, 1}, {-1, -1}});
    // D1: cells phase 2 reads (the tile's gasket cells and their neighbours)
    for (int r = 0; r < TT; ++r)
        for (int c = 0; c < TT; ++c)
            if (own(c, r)) {
                at(D1, c, r) = 1;
                for (auto [dx, dy] : offs) at(D1, c + dx, r + dy) = 1;
            }
    // state t needed: D1 itself, the neighbours of D1's (superset) gasket cells,
    // and the tile's touched sectors whole (the off-gasket blend of the store)
    for (int r = -1; r <= TT; ++r)
        for (int c = -CC; c < TT + CC; ++c)
            if (at(D1, c, r)) {
                at(need, c, r) = 1;
                if (member_sup(c, r))
                    for (auto [dx, dy] : offs)
                        if (inwin(c + dx, r + dy)) at(need, c + dx, r + dy) = 1;
            }
    for (int r = 0; r < TT; ++r)
        for (int g = 0; g < ROWB / 32; ++g)
            if (((g * S::SC) & ~r) == 0)
                for (int c = g * S::SC; c < (g + 1) * S::SC; ++c) at(need, c, r) = 1;
    out.clear();
    for (int r = -2; r < TT + 2; ++r)
        for (int q = 0; q < CHUNKS; ++q) {
            bool any = false;
            for (int c = (q - 1) * CC; c < q * CC; ++c) any = any || at(need, c, r);
            const int j = r + 2;
            if (any) out.push_back((uint32_t)(j * 16 + q));
        }
    ns = (int)out.size();
    // phase 1: words of rows -1..TT holding a D1 cell.  The tile's own gasket words come
    // in aligned runs of V rows (word w holds gasket cells of row t iff w*V subset of t,
    // which leaves t's low log2(V) bits free): one entry per run, the byte offset of
    // (I row r0 + 1, word k).  Then ring words that may hold gasket cells (neighbouring
    // tile assumed a gasket tile), then the rest (copied); single-word entries are
    // byte offset (I row ji, word k) | ji << 16 | k << 24.
    std::vector<uint32_t> inner, ring, copy;
    for (int r = -1; r <= TT; ++r)
        for (int k = 0; k < 4 * CHUNKS; ++k) {
            bool d = false, gsk = false;
            for (int c = (k - 4) * V; c < (k - 3) * V; ++c) {
                d = d || at(D1, c, r);
                gsk = gsk || member_sup(c, r);
            }
            const bool in_tile = r >= 0 && r < TT && k >= 4 && k < 4 + TT / V;
            if (in_tile && gsk) {  // exact inside the tile: part of a run
                if (r % V == 0) inner.push_back((uint32_t)((r + 1) * 64 + k));
                continue;
            }
            if (!d) continue;
            const int ji = r + 1;
            const uint32_t e = (uint32_t)(ji * 64 + k);
            (gsk ? ring : copy).push_back(e);
        }
    ni1 = (int)inner.size();
    ng1 = ni1 + (int)ring.size();
    np1 = ng1;  // (the `copy` words are read from S by phase 2, not copied into I)
    out.insert(out.end(), inner.begin(), inner.end());
    out.insert(out.end(), ring.begin(), ring.end());
    // phase 2: the tile's gasket words, one entry per aligned run of V rows: the byte
    // offset of (I row t, word k) (I rows t..t+V+1 are tile rows t-1..t+V)
    np2 = 0;
    for (int t = 0; t < TT; t += V)
        for (int w = 0; w < TT / V; ++w)
            if (((w * V) & ~t) == 0) {
                out.push_back((uint32_t)(t * 64 + w + 4));
                ++np2;
            }
}

template <int C>
const TbLists* tb_lists(bool eight) {
    static std::mutex mu;
    static std::map<std::pair<int, bool>, TbLists> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(dev, eight);
    auto it = cache.find(key);
    if (it != cache.end()) return &it->second;
    std::vector<uint32_t> v;
    TbLists L;
    build_lists<C>(eight, v, L.ns, L.np1, L.ng1, L.ni1, L.np2);
    std::vector<uint16_t> v16(v.begin(), v.end());  // every entry is a shared-memory offset < 2^16
    if (cudaMalloc(&L.lists, v16.size() * 2) != cudaSuccess ||
        cudaMemcpy(L.lists, v16.data(), v16.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return &(cache[key] = L);
}

template <int C, int KIND, int NST>
cudaError_t launch_ck(const LaunchArgs& a, int r_t) {
    using S = TB<C>;
    // tile range: the whole gasket, or (partitioned launches, gm_run_part2) the digit-order
    // sub-gasket range [sg_begin, sg_end) of level part_level; the order table groups
    // tiles by those sub-gaskets, so the range is a contiguous run of it
    uint32_t lo, hi;
    tile_range(a, r_t, lo, hi);
    if (hi == lo) return cudaSuccess;
    const uint32_t ntiles = hi - lo;
    const TbLists* L = tb_lists<C>(KIND == KIND_NSUM8);
    const uint32_t* order = rowmajor_table(r_t, order_level(a, r_t));
    if (order != nullptr) order += lo;
    if (L == nullptr || order == nullptr) return cudaErrorMemoryAllocation;
    const size_t smem = (size_t)NST * S::SBUF + S::IBUF + 2 * (size_t)(L->ns + L->np1 + L->np2);
    auto* kern = stencil_tb2<C, KIND, NST>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, smem);
    uint64_t blocks = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > ntiles) blocks = ntiles;
    kern<<<(unsigned)blocks, S::THREADS, smem, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid),
                                                          reinterpret_cast<const uint8_t*>(a.src), a.n, ntiles,
                                                          a.param, order, L->lists, L->ns, L->np1, L->ng1, L->ni1, L->np2, a.flags,
                                                          reinterpret_cast<PeerEpilogue*>(a.peer_epi), a.wait_epoch,
                                                          a.signal_epoch);
    note_launch();
    return cudaGetLastError();
}

template <int C, int KIND>
cudaError_t launch_kind(const LaunchArgs& a, int r_t) {
    // a 2-deep ring: 3 CTAs per SM for byte cells (a 3-deep ring costs a CTA per SM)
    return launch_ck<C, KIND, 2>(a, r_t);
}

template <int C>
cudaError_t launch_c(const LaunchArgs& a, int r) {
    int k = 0;
    while ((1 << k) < TB<C>::TT) ++k;
    if (r - k > 15) return cudaErrorNotSupported;  // tile-order table limit
    if (a.kind == KIND_NSUM4) return launch_kind<C, KIND_NSUM4>(a, r - k);
    if (a.kind == KIND_NSUM8) return launch_kind<C, KIND_NSUM8>(a, r - k);
    return cudaErrorNotSupported;
}

}  // namespace

// Two fused CA steps: grid <- step(step(src)); grid must equal src off the gasket.
// cudaErrorNotSupported for grids narrower than one tile or cell widths other than 1, 2, 4.
cudaError_t launch_stencil_tb2(const LaunchArgs& a) {
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    switch (a.cell_bytes) {
    case 1: if (a.n >= TB<1>::TT) return launch_c<1>(a, r); break;
    case 2: if (a.n >= TB<2>::TT) return launch_c<2>(a, r); break;
    case 4: if (a.n >= TB<4>::TT) return launch_c<4>(a, r); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
