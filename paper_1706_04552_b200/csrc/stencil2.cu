// stencil2.cu -- tuned lambda neighbour-sum kernel, v2 (strategy STRAT_TUNED,
// KIND_NSUM4 / KIND_NSUM8, cells of 1, 2 or 4 bytes).  Default stencil path;
// GM_FLAG_STENCIL_V1 selects the v1 kernel in stencil.cu for A/B runs.
//
// Same decomposition and DRAM rules as v1 (stencil.cu): one CTA per lambda
// tile of TT x TT cells whose rows are one 128-byte line, only the 16-byte
// chunks some gasket cell's neighbourhood reads are staged (cp.async with the
// .L2::64B fetch-size hint), one thread per touched 32-byte sector, every
// touched sector stored whole.  What changed, from the ncu profile of v1
// (issue-bound at 54% issue slots, barrier + scoreboard stalls, DRAM 53%):
//
//  * arithmetic in split lanes.  Byte cells are spread into two 16-bit-lane
//    words with one PRMT each (even cells, odd cells); a 9-cell sum of bytes
//    never carries out of its 16-bit lane, so plain IADD3s replace the
//    emulated __vadd4 (5+ instructions each).  Neighbours one cell left/right
//    are one funnel shift of the other parity's word.  2-byte cells use 32-bit
//    lanes the same way; 4-byte cells are plain 32-bit words.  One PRMT packs
//    the result back.  About 16 instructions per 4-byte word instead of ~40.
//  * an NST-stage cp.async ring with a single barrier per tile: tile i+NST-1
//    is issued right after the barrier that ends tile i-1's compute, so
//    NST-1 tiles per CTA are in flight (v1: one, plus a second barrier).
//  * the chunk list holds the shared-memory offset of every needed chunk;
//    interior tiles skip all bounds tests (edge tiles zero-fill as before).
//  * each touched sector leaves as one 256-bit store (st.global.v8.b32).
//
// Semantics: backends.py:127-141 (_cell_value NEIGHBOR_SUM: param + in-grid
// 4-neighbours, out-of-grid = 0, result wraps to the cell width) and our
// labelled 8-neighbour extension; only gasket cells change.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <exception>
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

constexpr int ROWB = 128;                 // tile row bytes (one line)
constexpr int PITCH = ROWB + 48;          // smem row: 16 B halo | 128 B row | 16 B halo | 16 B pad
constexpr int CHUNKS = (ROWB + 32) / 16;  // 10 staged 16-byte chunks per row

template <int C>
struct T2 {
    static constexpr int V = 4 / C;           // cells per 4-byte word
    static constexpr int TT = ROWB / C;       // tile edge (cells)
    static constexpr int SC = 32 / C;         // cells per sector
    static constexpr int NSEC = ROWB / 32;    // sectors per tile row
    static constexpr int ROWS = TT + 2;       // staged rows (-1 .. TT)
    static constexpr int BUF = ROWS * PITCH;  // bytes per staged tile
    static constexpr int NTOUCH = 9 * SC;     // touched sectors per tile (1,2,2,4 per row group)
    static constexpr int THREADS = (NTOUCH + 31) / 32 * 32;
};

__device__ __forceinline__ bool row_in(int t, int tt) { return t >= 0 && t < tt; }

template <int C>
__device__ __forceinline__ bool sec_touched(int t, int g) {
    return row_in(t, T2<C>::TT) && g >= 0 && g < T2<C>::NSEC && ((g * T2<C>::SC) & ~t) == 0;
}
template <int C>
__device__ __forceinline__ bool cell_member(int t, int c) {
    return row_in(t, T2<C>::TT) && c >= 0 && c < T2<C>::TT && (c & ~t) == 0;
}
// sector g of staged tile row t is read by some gasket cell's neighbourhood
template <int C, bool EIGHT>
__device__ __forceinline__ bool sec_needed(int t, int g) {
    constexpr int SC = T2<C>::SC;
    bool need = sec_touched<C>(t - 1, g) || sec_touched<C>(t, g) || sec_touched<C>(t + 1, g);
    need = need || sec_touched<C>(t, g + 1) || cell_member<C>(t, g * SC - 1);
    if (EIGHT) {
        need = need || sec_touched<C>(t - 1, g + 1) || sec_touched<C>(t + 1, g + 1);
        need = need || cell_member<C>(t - 1, g * SC - 1) || cell_member<C>(t + 1, g * SC - 1);
    }
    return need;
}
// chunk q of staged row j (j = tile row + 1; q = 0 left halo, 1..8 row, 9 right halo)
template <int C, bool EIGHT>
__device__ __forceinline__ bool chunk_needed(int j, int q) {
    constexpr int TT = T2<C>::TT;
    const int t = j - 1;
    if (q == 0) return EIGHT ? (row_in(t - 1, TT) || row_in(t, TT) || row_in(t + 1, TT)) : row_in(t, TT);
    if (q == CHUNKS - 1)
        return EIGHT ? (cell_member<C>(t - 1, TT - 1) || cell_member<C>(t, TT - 1) || cell_member<C>(t + 1, TT - 1))
                     : cell_member<C>(t, TT - 1);
    return sec_needed<C, EIGHT>(t, (q - 1) >> 1);
}

template <int C, int KIND, int NST>
__global__ void __launch_bounds__(T2<C>::THREADS) stencil_v2(uint8_t* __restrict__ grid, const uint8_t* __restrict__ src,
                                                             int64_t n, uint32_t tile_lo, uint32_t tile_hi, int r_t,
                                                             int part_level, uint64_t param, int flags,
                                                             const uint32_t* __restrict__ order, PeerEpilogue* epi,
                                                             uint64_t wait_epoch, uint64_t signal_epoch,
                                                             const int64_t* __restrict__ sg_off, int64_t pitch,
                                                             uint32_t per, const uint8_t* __restrict__ edge,
                                                             const uint8_t* __restrict__ border, int bb_lg) {
    using S = T2<C>;
    peer_prologue_wait(epi, wait_epoch);  // partitioned CA with the fused exchange only
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* chunks = reinterpret_cast<uint32_t*>(smem + NST * S::BUF);  // needed chunks: smem off | j << 16 | q << 24
    __shared__ uint16_t tab[243];
    __shared__ int nchunks;
    digit_table_init(tab);
    // row-major list (consecutive threads stage consecutive chunks of one row)
    if (threadIdx.x < 32) {
        int cnt = 0;
        for (int base = 0; base < S::ROWS * CHUNKS; base += 32) {
            const int i = base + threadIdx.x;
            const int j = i / CHUNKS, q = i - j * CHUNKS;
            const bool need = i < S::ROWS * CHUNKS && chunk_needed<C, EIGHT>(j, q);
            const unsigned m = __ballot_sync(0xffffffffu, need);
            // bit 28: the tile's own line needs chunks in both 64-byte halves -> fetch it
            // whole (one DRAM access instead of two; GM_FLAG_FETCH_MIXED)
            bool both = false;
            if (need && q >= 1 && q <= 8) {
                bool lo = false, hi = false;
                for (int qq = 1; qq <= 4; ++qq) lo = lo || chunk_needed<C, EIGHT>(j, qq);
                for (int qq = 5; qq <= 8; ++qq) hi = hi || chunk_needed<C, EIGHT>(j, qq);
                both = lo && hi;
            }
            if (need)
                chunks[cnt + __popc(m & ((1u << threadIdx.x) - 1u))] =
                    (uint32_t)(j * PITCH + q * 16) | ((uint32_t)j << 16) | ((uint32_t)q << 24) | ((uint32_t)both << 28);
            cnt += __popc(m);
        }
        if (threadIdx.x == 0) nchunks = cnt;
    }
    __syncthreads();
    const int nch = nchunks;
    const int64_t rowbytes = n * C;  // the global grid's row (bounds)
    const int64_t rowstride = pitch;  // the buffers' row pitch (addresses; tiled storage: its blocks')
    // with a 2-deep ring there is shared memory left for the chunks' grid offsets (one add
    // per chunk when staging interior tiles); the 3-deep ring keeps 3 CTAs per SM without
    [[maybe_unused]] int32_t* goff = reinterpret_cast<int32_t*>(chunks + S::ROWS * CHUNKS);
    if constexpr (NST == 2) {
        for (int i = threadIdx.x; i < nch; i += S::THREADS) {
            const uint32_t c = chunks[i];
            goff[i] = (int32_t)((int64_t)((c >> 16) & 0xffu) * rowstride + (int64_t)((c >> 24) & 15u) * 16);
        }
        __syncthreads();
    }
    const bool dst_from_src = (flags & GM_FLAG_DST_FROM_SRC) != 0;
    // staging fetches whole 128-byte lines (.L2::128B) by default: the pass is bound by
    // the number of DRAM accesses, not bytes (n=2^17 NSUM8: 428 us vs 441 us with the
    // .L2::64B hint, which moves 1.10 instead of ~1.44 GB); GM_FLAG_FETCH_HALF = halves
    const bool fetch_line = (flags & GM_FLAG_FETCH_HALF) == 0;
    const bool fetch256 = (flags & GM_FLAG_FETCH256) != 0;
    const bool fetch_mixed = (flags & GM_FLAG_FETCH_MIXED) != 0;
    const bool v8 = (reinterpret_cast<uintptr_t>(grid) & 31u) == 0;
#ifdef GM_AB_VARIANTS
    const bool probe_nostore = (flags & GM_FLAG_PROBE_NOSTORE) != 0;
#else
    constexpr bool probe_nostore = false;  // design probe: A/B builds only
#endif
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
    const bool store_cs = (flags & GM_FLAG_STORE_CS) != 0;
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(smem);
    uint32_t pv;
    if constexpr (C == 1) pv = 0x00010001u * (uint32_t)(param & 0xffu);
    else if constexpr (C == 2) pv = (uint32_t)(param & 0xffffu);
    else pv = (uint32_t)param;

    // this thread's touched sector (t, g): row groups of SC rows with 1,2,2,4 sectors
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
    const uint32_t tmask = member_mask<C>((uint32_t)t);
    uint32_t wmask[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) wmask[i] = (((8 * g + i) * S::V) & ~t) == 0 ? tmask : 0u;

    // tile visiting order: lambda digit order, or (GM_FLAG_ROWMAJOR) the precomputed
    // table `order` = member tiles row-major within each level-L sub-gasket, so that
    // concurrently running CTAs stage horizontally adjacent tiles (same DRAM pages)
    const bool chunked = (flags & GM_FLAG_CHUNKED) != 0;
    // bb_lg >= 0: the bounding box at tile granularity (GM_MAP_BB_VEC) -- tile index i covers
    // every tile of the 2^bb_lg x 2^bb_lg tile grid, and tiles off the gasket exit
    auto tile_xy = [&](uint32_t tile, uint32_t& bx, uint32_t& by) {
        if (bb_lg >= 0) {
            bx = tile & ((1u << bb_lg) - 1u);
            by = tile >> bb_lg;
        } else if (order == nullptr) {
            lambda_digit_order(tile, tab, bx, by);
        } else {
            const uint32_t v = __ldg(order + tile);
            bx = v & 0xffffu;
            by = v >> 16;
        }
    };
    const uint32_t span = tile_hi - tile_lo;
    const uint32_t chunk = chunked ? (span + gridDim.x - 1) / gridDim.x : 1u;
    const uint32_t step = chunked ? 1u : gridDim.x;
    const uint32_t first = tile_lo + blockIdx.x * chunk;
    const uint32_t last = chunked ? min(tile_hi, first + chunk) : tile_hi;  // exclusive
    // (a CTA without tiles still takes part in the fused exchange's completion count)
    const uint32_t count = first >= last ? 0u : (last - first + step - 1) / step;

    // byte offset of this CTA's tile #idx's sub-gasket block (tiled partition storage)
    auto tile_off = [&](uint32_t idx) -> int64_t {
        return sg_off != nullptr ? __ldg(sg_off + (first + idx * step - tile_lo) / per) : 0;
    };
    // order-table entry of this CTA's tile #idx
    auto order_v = [&](uint32_t idx) -> uint32_t {
        return (order != nullptr && idx < count) ? __ldg(order + first + idx * step) : 0u;
    };
    auto stage = [&](uint32_t idx, uint32_t v) {  // stage this CTA's tile #idx into ring slot idx % NST
        if (idx >= count || probe_noload) return;
        uint32_t bx, by;
        if (bb_lg >= 0 || order == nullptr) {
            tile_xy(first + idx * step, bx, by);
            if (bb_lg >= 0 && (bx & ~by) != 0) return;  // (bounding box: a tile off the gasket)
        } else {
            bx = v & 0xffffu;
            by = v >> 16;
        }
        const int64_t x0 = (int64_t)bx * S::TT, y0 = (int64_t)by * S::TT;
        const uint32_t sb = smem0 + (idx % NST) * S::BUF;
        const uint8_t* srct = src + tile_off(idx);
        const uint8_t* base = srct + (y0 - 1) * rowstride + x0 * C - 16;  // staged (row 0, chunk 0)
        const bool interior = y0 > 0 && y0 + S::TT < n && x0 > 0 && x0 + S::TT < n;
        // a static left edge (CA runs, edge.cu): the left halo chunks of the tile's own rows
        // come from the dense edge cache instead of one sparse grid line each
        const bool ls = edge != nullptr && order != nullptr && left_static(bx, by);  // (cache: order-table index)
        const uint8_t* ecol = edge + (ls ? (int64_t)(first + idx * step - tile_lo) * S::TT * 16 - 16 : 0);  // + j*16
        auto from_edge = [&](uint32_t c) {  // chunk 0 of staged row j = tile row j-1 in [0, TT)
            return ls && (c & 0x0f000000u) == 0 && ((c >> 16) & 0xffu) - 1u < (uint32_t)S::TT;
        };
        if (interior) {
            for (int i = threadIdx.x; i < nch; i += S::THREADS) {
                const uint32_t c = chunks[i];
                int64_t go;
                if constexpr (NST == 2) {
                    go = goff[i];
                } else {
                    go = (int64_t)((c >> 16) & 0xffu) * rowstride + (int64_t)((c >> 24) & 15u) * 16;
                }
                if (from_edge(c)) cp_async16(sb + (c & 0xffffu), ecol + ((c >> 16) & 0xffu) * 16, 16, true);
                else if (fetch256) cp_async16_256(sb + (c & 0xffffu), base + go, 16);
                else cp_async16(sb + (c & 0xffffu), base + go, 16, fetch_line || (fetch_mixed && (c >> 28)));
            }
        } else {
            for (int i = threadIdx.x; i < nch; i += S::THREADS) {
                const uint32_t c = chunks[i];
                const int j = (int)((c >> 16) & 0xffu), qq = (int)((c >> 24) & 15u);
                const int64_t y = y0 + j - 1;
                const int64_t xb = x0 * C + (qq - 1) * 16;
                const bool in = y >= 0 && y < n && xb >= 0 && xb < rowbytes;
                if (from_edge(c)) cp_async16(sb + (c & 0xffffu), ecol + j * 16, 16, true);
                else cp_async16(sb + (c & 0xffffu), in ? srct + y * rowstride + xb : src, in ? 16 : 0,
                                fetch_line || (fetch_mixed && (c >> 28)));
            }
        }
    };

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        stage((uint32_t)s, order_v((uint32_t)s));
        cp_async_commit();
    }
    for (uint32_t idx = 0; idx < count; ++idx) {
        cp_async_wait<NST - 2>();  // this thread's copies of tile idx have landed
        __syncthreads();           // everyone's have; everyone is done with tile idx-1's slot
        // refill the slot tile idx-1 used.  The order entry is loaded here, after the
        // barrier, so the staging starts an L2 round trip after the previous tile's stores:
        // n=2^17 NSUM8 427 vs 436 us, NSUM4 430 vs 451 us with the entry loaded a tile ahead
        stage(idx + NST - 1, order_v(idx + NST - 1));
        cp_async_commit();
        if (border != nullptr) {
            // in-place launch (src aliases grid; edge.cu): the neighbouring tiles' gasket cells
            // this tile reads may already hold new values -- put their pre-launch values into
            // the staged window (8 reader positions; a patch with the old value is always right)
            if (threadIdx.x < 8) {
                uint32_t bx, by;
                tile_xy(first + idx * step, bx, by);
                constexpr int TT = S::TT;
                const int p = threadIdx.x;
                int px, py, ox, oy, sl;
                switch (p) {
                case 0: px = -1; py = -1; ox = -1; oy = -1; sl = 4; break;
                case 1: px = 0; py = -1; ox = 0; oy = -1; sl = 2; break;
                case 2: px = 1; py = -1; ox = 0; oy = -1; sl = 3; break;
                case 3: px = -1; py = TT - 1; ox = -1; oy = 0; sl = 4; break;
                case 4: px = 0; py = TT; ox = 0; oy = 1; sl = 0; break;
                case 5: px = TT; py = TT - 2; ox = 1; oy = 0; sl = 1; break;
                case 6: px = TT; py = TT - 1; ox = 1; oy = 0; sl = 2; break;
                default: px = TT; py = TT; ox = 1; oy = 1; sl = 0; break;
                }
                const int64_t ntx = n / TT, tx = (int64_t)bx + ox, ty = (int64_t)by + oy;
                if (tx >= 0 && ty >= 0 && tx < ntx && ty < ntx && (tx & ~ty) == 0) {
                    uint8_t* d = smem + (idx % NST) * S::BUF + (py + 1) * PITCH + 16 + px * C;
                    const uint8_t* b = border + ((ty * ntx + tx) * 8 + sl) * C;
#pragma unroll
                    for (int k = 0; k < C; ++k) d[k] = b[k];
                }
            }
            __syncthreads();
        }
        if (active) {
            uint32_t bx, by;
            tile_xy(first + idx * step, bx, by);
            if (bb_lg >= 0 && (bx & ~by) != 0) continue;  // (bounding box: a tile off the gasket)
            const int64_t x0 = (int64_t)bx * S::TT, y0 = (int64_t)by * S::TT;
            const uint8_t* b = smem + (idx % NST) * S::BUF;
            const uint32_t* up = reinterpret_cast<const uint32_t*>(b + t * PITCH);  // staged row t = tile row t-1
            const int k0 = 4 + 8 * g;  // first word of the sector (4 halo words on the left)
            uint32_t w[3][10];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const uint32_t* row = up + r * (PITCH / 4);
                const uint4 a = *reinterpret_cast<const uint4*>(row + k0);
                const uint4 c = *reinterpret_cast<const uint4*>(row + k0 + 4);
                w[r][1] = a.x; w[r][2] = a.y; w[r][3] = a.z; w[r][4] = a.w;
                w[r][5] = c.x; w[r][6] = c.y; w[r][7] = c.z; w[r][8] = c.w;
                if (EIGHT || r == 1) {
                    w[r][0] = row[k0 - 1];
                    w[r][9] = row[k0 + 8];
                } else {
                    w[r][0] = w[r][9] = 0u;
                }
            }
            uint32_t out[8];
            if (probe_nocompute) {
#pragma unroll
                for (int i = 0; i < 8; ++i) out[i] = w[0][i + 1] ^ w[2][i + 1];
            } else {
                sector_sums<C, EIGHT>(w, pv, out);
            }
            uint8_t* gp = grid + tile_off(idx) + (y0 + t) * rowstride + x0 * C + g * 32;
            if (dst_from_src) {
#pragma unroll
                for (int i = 0; i < 8; ++i) out[i] = (out[i] & wmask[i]) | (w[1][i + 1] & ~wmask[i]);
            } else {  // off-gasket cells from the grid itself (still a whole-sector write)
                // read with the 64-byte fetch hint: only this tile touches the line, so the rest
                // of a 128-byte fetch is wasted (n=2^17 NSUM8 571 vs 586 us; byte-masked stores
                // of the gasket cells instead, with the L2's sector fill: 704 us)
                uint32_t old[8];
                ld_sector(gp, false, v8, old);
#pragma unroll
                for (int i = 0; i < 8; ++i) out[i] = (out[i] & wmask[i]) | (old[i] & ~wmask[i]);
            }
            if (!probe_nostore) st_sector(gp, out, v8, store_cs);
        }
    }
    cp_async_wait<0>();
    peer_epilogue_signal(grid, epi, signal_epoch);  // partitioned CA with the fused exchange only
}

template <int C, int KIND, int NST>
cudaError_t launch_ck(const LaunchArgs& a, int r_t) {
    using S = T2<C>;
    uint32_t lo, hi;
    tile_range(a, r_t, lo, hi);
    const int bb_lg = a.mapping == MAP_BB_VEC ? r_t : -1;  // bounding box: every tile of the grid
    if (bb_lg >= 0) {
        lo = 0;
        hi = 1u << (2 * r_t);
    }
    if (hi == lo) return cudaSuccess;
    const uint32_t ntiles = hi - lo;
    const size_t smem = (size_t)NST * S::BUF + (NST == 2 ? 8 : 4) * S::ROWS * CHUNKS;
    auto* kern = stencil_v2<C, KIND, NST>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, smem);
    uint64_t blocks = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > ntiles) blocks = ntiles;
    if (getenv("GASKET_DEBUG_OCC")) fprintf(stderr, "stencil_v2<C=%d,K=%d,NST=%d>: %d CTAs/SM, smem %zu\n", C, KIND, NST, per_sm, smem);
    const uint32_t* order = nullptr;
    if (!(a.flags & GM_FLAG_DIGIT_ORDER) && bb_lg < 0) order = rowmajor_table(r_t, order_level(a, r_t));
    kern<<<(unsigned)blocks, S::THREADS, smem, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid),
                                                          reinterpret_cast<const uint8_t*>(a.src), a.n, lo, hi, r_t,
                                                          a.part_level, a.param, a.flags, order,
                                                          reinterpret_cast<PeerEpilogue*>(a.peer_epi), a.wait_epoch,
                                                          a.signal_epoch, a.sg_off, row_pitch(a),
                                                          tiles_per_subgasket(a, r_t), bb_lg < 0 ? a.edge : nullptr,
                                                          bb_lg < 0 ? a.border : nullptr, bb_lg);
    note_launch();
    return cudaGetLastError();
}

template <int C, int KIND>
cudaError_t launch_kind(const LaunchArgs& a, int r_t) {
    // ring depth: GM_FLAG_STAGES2 / default 3 (byte cells; 2-byte and 4-byte tiles are smaller: 4).
    // With the static edge cache (CA runs) the 2-deep ring: more CTAs per SM pay off once the
    // sparse left-halo lines are gone (n=2^17 NSUM8 int8 378 vs 406 us, 4 vs 3 CTAs per SM;
    // n=2^16 NSUM4 int16 191 vs 227 us, int32 273 vs 317 us); without the cache the 2-deep
    // ring is slower (int8 499 vs 438 us).  The in-place launch (border patches, one more
    // barrier per tile) also prefers it: n=2^16 int32 NSUM4 364 vs 479 us, n=2^17 int8 NSUM8
    // 472 vs 535 us
    if ((a.flags & GM_FLAG_STAGES2) || a.edge != nullptr || a.border != nullptr) return launch_ck<C, KIND, 2>(a, r_t);
    if constexpr (C == 1) return launch_ck<C, KIND, 3>(a, r_t);
    else return launch_ck<C, KIND, 4>(a, r_t);
}

template <int C>
cudaError_t launch_c(const LaunchArgs& a, int r) {
    int k = 0;
    while ((1 << k) < T2<C>::TT) ++k;
    if (a.kind == KIND_NSUM4) return launch_kind<C, KIND_NSUM4>(a, r - k);
    if (a.kind == KIND_NSUM8) return launch_kind<C, KIND_NSUM8>(a, r - k);
    return cudaErrorNotSupported;
}

}  // namespace

// Device table of the member tiles of a level-q gasket (tile edge 1), packed
// bx | by << 16, ordered sub-gasket by sub-gasket (level-L digit order, the
// order tile ranges of partitioned launches refer to) and row-major inside each
// sub-gasket (block row Y ascending, then the columns l subset of Y).  Built on
// the host once per (device, q, L) and kept for the life of the process.
// Why: concurrently running CTAs then stage/store horizontally adjacent tiles,
// i.e. the same rows and DRAM pages at the same time (scripts/probe_gasket.cu:
// tile reads 43.7 -> 48.6 G lines/s, partial-line writes 39.7 -> 44.5 G lines/s;
// stencil n=2^17 518 -> 436 us, write pass n=2^16 118 -> 104 us).
void rowmajor_order_host(int q, int L, std::vector<uint32_t>& v) {
    uint64_t nsg = 1;
    for (int i = 0; i < L; ++i) nsg *= 3u;
    const int m = q - L;
    v.clear();
    for (uint64_t sg = 0; sg < nsg; ++sg) {
        uint32_t sx = 0, sy = 0, d = (uint32_t)sg;
        for (int i = 0; i < L; ++i, d /= 3u) {  // digit i -> level i+1: 1 = (0,1), 2 = (1,1)
            sx |= (uint32_t)(d % 3u == 2u) << i;
            sy |= (uint32_t)(d % 3u != 0u) << i;
        }
        for (uint32_t Y = 0; Y < (1u << m); ++Y) {
            for (uint32_t l = Y;; l = (l - 1) & Y) {  // subsets of Y, descending; reversed below
                v.push_back(((sx << m) + l) | (((sy << m) + Y) << 16));
                if (l == 0) break;
            }
            std::reverse(v.end() - (1u << __builtin_popcount(Y)), v.end());
        }
    }
}

const uint32_t* rowmajor_table(int q, int L) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, uint32_t*> cache;
    if (q > 15 || L > q || L < 0) return nullptr;  // caller falls back to digit order
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(dev, q, L);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<uint32_t> v;
    try {
        rowmajor_order_host(q, L, v);
    } catch (const std::exception&) {  // (host allocation) -- no exception crosses the C ABI
        return nullptr;
    }
    uint32_t* d_tab = nullptr;
    if (cudaMalloc(&d_tab, v.size() * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (cudaMemcpy(d_tab, v.data(), v.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d_tab);
        return nullptr;
    }
    cache[key] = d_tab;
    return d_tab;
}

cudaError_t launch_stencil_v2(const LaunchArgs& a) {
    if (a.flags & (GM_FLAG_OMEGA_ORDER | GM_FLAG_STENCIL_V1)) return cudaErrorNotSupported;
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    switch (a.cell_bytes) {
    case 1: if (a.n >= T2<1>::TT) return launch_c<1>(a, r); break;
    case 2: if (a.n >= T2<2>::TT) return launch_c<2>(a, r); break;
    case 4: if (a.n >= T2<4>::TT) return launch_c<4>(a, r); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
