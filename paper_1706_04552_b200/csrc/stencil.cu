// stencil.cu -- tuned lambda neighbour-sum kernel with shared-memory tile staging
// (strategy STRAT_TUNED, KIND_NSUM4 / KIND_NSUM8, cells of 1, 2 or 4 bytes).
//
// One CTA works on one lambda tile at a time (tiles of TT x TT cells whose
// rows are one 128-byte line; tile index -> tile by the digit-order closed
// form of lambda, CTAs interleaved over tiles so concurrently staged tiles are
// spatial neighbours and share halo sectors in L2):
//   1. stage rows -1..TT of the tile plus a 16-byte halo chunk on each side
//      into shared memory with cp.async (16-byte chunks, double-buffered: the
//      next tile is in flight while this one is computed).  Only chunks of
//      sectors that hold a neighbour of some gasket cell are fetched (the exact
//      sector set of roofline.stencil_read_sectors); out-of-grid rows/columns
//      are zero-filled (the reference's "out-of-grid neighbours read 0").
//   2. every thread takes touched 32-byte sectors of the tile from a constant
//      per-tile list (t, g), g subset of t >> 5 -- exactly the sectors holding
//      gasket cells -- and computes their 4-byte words in SIMD (per-byte or
//      per-halfword adds, neighbour cells by funnel shifts, the 8-neighbourhood
//      as 3x3 column sums minus the centre);
//   3. each touched sector is stored whole (two 16-byte stores).  Off-gasket
//      cells come from the snapshot when GM_FLAG_DST_FROM_SRC says grid and src
//      agree off the gasket (engine.launch, CA ping-pong), otherwise from the
//      grid's own sector, loaded first -- so DRAM never sees a partial-sector
//      write (which would cost a read-modify-write, scripts/probe_partial.cu).
// Semantics: backends.py:127-141 (_cell_value) for 4 neighbours, our 8-neighbour
// extension for KIND_NSUM8; sums wrap to the cell width.
#include "gasket.cuh"
#include "launch.h"
#include "../../include/gasket_b200.h"

namespace gm {
namespace {

constexpr int ROWB = 128;              // tile row bytes
constexpr int PITCH = ROWB + 48;       // smem row: 16 B halo + row + 16 B halo + 16 B pad (bank spread)
constexpr int CHUNKS = (ROWB + 32) / 16;  // staged 16-byte chunks per row (halo, 8 row chunks, halo)

template <int C>
struct SG {
    static constexpr int V = 4 / C;          // cells per 4-byte word
    static constexpr int TT = ROWB / C;      // tile edge in cells
    static constexpr int SC = 32 / C;        // cells per sector
    static constexpr int NSEC = ROWB / 32;   // sectors per tile row (4)
    static constexpr int ROWS = TT + 2;      // staged rows
    static constexpr int BUF = ROWS * PITCH; // bytes per staged tile
    // touched sectors per tile: rows come in 4 groups of SC rows whose row pattern
    // t >> log2(SC) is 0,1,2,3 -> 1,2,2,4 touched sectors per row = 9 * SC in all
    static constexpr int NTOUCH = 9 * SC;
    static constexpr int THREADS = (NTOUCH + 31) / 32 * 32;  // one thread per touched sector
};

template <int C>
__device__ __forceinline__ uint32_t vadd(uint32_t a, uint32_t b) {
    if constexpr (C == 1) return __vadd4(a, b);
    else if constexpr (C == 2) return __vadd2(a, b);
    else return a + b;
}
template <int C>
__device__ __forceinline__ uint32_t vsub(uint32_t a, uint32_t b) {
    if constexpr (C == 1) return __vsub4(a, b);
    else if constexpr (C == 2) return __vsub2(a, b);
    else return a - b;
}
template <int C>
__device__ __forceinline__ uint32_t lft(uint32_t prev, uint32_t cur) {  // cell j-1 for every cell j
    if constexpr (C == 4) return prev;
    else return __funnelshift_l(prev, cur, 8 * C);
}
template <int C>
__device__ __forceinline__ uint32_t rgt(uint32_t cur, uint32_t next) {  // cell j+1 for every cell j
    if constexpr (C == 4) return next;
    else return __funnelshift_r(cur, next, 8 * C);
}
template <int C>
__device__ __forceinline__ uint32_t member_mask(uint32_t t) {  // cells j of a word with j subset of t & (V-1)
    if constexpr (C == 1) {
        const uint32_t p = t & 3u;
        return p == 0 ? 0x000000ffu : p == 1 ? 0x0000ffffu : p == 2 ? 0x00ff00ffu : 0xffffffffu;
    } else if constexpr (C == 2) {
        return (t & 1u) ? 0xffffffffu : 0x0000ffffu;
    } else {
        return 0xffffffffu;
    }
}

template <int C>
__device__ __forceinline__ bool row_in(int t) { return t >= 0 && t < SG<C>::TT; }
template <int C>
__device__ __forceinline__ bool sec_touched(int t, int g) {
    return row_in<C>(t) && g >= 0 && g < SG<C>::NSEC && ((g * SG<C>::SC) & ~t) == 0;
}
template <int C>
__device__ __forceinline__ bool cell_member(int t, int c) {
    return row_in<C>(t) && c >= 0 && c < SG<C>::TT && (c & ~t) == 0;
}
template <int C, bool EIGHT>
__device__ __forceinline__ bool sec_needed(int t, int g) {
    constexpr int SC = SG<C>::SC;
    bool need = sec_touched<C>(t - 1, g) || sec_touched<C>(t, g) || sec_touched<C>(t + 1, g);
    need = need || sec_touched<C>(t, g + 1) || cell_member<C>(t, g * SC - 1);
    if (EIGHT) {
        need = need || sec_touched<C>(t - 1, g + 1) || sec_touched<C>(t + 1, g + 1);
        need = need || cell_member<C>(t - 1, g * SC - 1) || cell_member<C>(t + 1, g * SC - 1);
    }
    return need;
}

__device__ __forceinline__ uint4 ld_cg16(const void* p, bool line) {
    uint4 v;
    if (line)
        asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        asm volatile("ld.global.cg.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// An L2 miss of a plain load or cp.async fetches the whole 128-byte line from DRAM;
// with the .L2::64B fetch-size hint only the 64-byte half holding the chunk comes in
// (scripts/probe_fetch.cu: half the DRAM bytes, same per-line rate).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool zero_fill, bool line) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int src_bytes = zero_fill ? 0 : 16;
    if (line)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
    else
        asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
                     : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Chunk (j, q) of a staged tile holds a cell some gasket cell's neighbourhood reads
// (tile-local test; grid-boundary rows/columns are zero-filled at staging time).
template <int C, bool EIGHT>
__device__ __forceinline__ bool chunk_needed(int j, int q) {
    using S = SG<C>;
    const int t = j - 1;
    if (q == 0) return EIGHT ? (row_in<C>(t - 1) || row_in<C>(t) || row_in<C>(t + 1)) : row_in<C>(t);
    if (q == CHUNKS - 1)
        return EIGHT ? (cell_member<C>(t - 1, S::TT - 1) || cell_member<C>(t, S::TT - 1) ||
                        cell_member<C>(t + 1, S::TT - 1))
                     : cell_member<C>(t, S::TT - 1);
    return sec_needed<C, EIGHT>(t, (q - 1) >> 1);
}

// Issue the staging copies of one tile from the precomputed chunk list.
template <int C>
__device__ __forceinline__ void stage_tile(uint8_t* buf, const uint16_t* chunks, int nchunks,
                                           const uint8_t* __restrict__ src, int64_t n, int64_t x0, int64_t y0,
                                           bool line) {
    using S = SG<C>;
    const int64_t rowstride = n * C;
    for (int i = threadIdx.x; i < nchunks; i += S::THREADS) {
        const int j = chunks[i] >> 4, q = chunks[i] & 15;
        const int64_t y = y0 + j - 1;
        const int64_t xb = x0 * C + (q - 1) * 16;  // byte column of the chunk
        const bool in = y >= 0 && y < n && xb >= 0 && xb < rowstride;
        cp_async16(buf + j * PITCH + q * 16, in ? src + y * rowstride + xb : src, !in, line);
    }
}

template <int C, int KIND>
__global__ void __launch_bounds__(SG<C>::THREADS) stencil_tile(uint8_t* __restrict__ grid,
                                                               const uint8_t* __restrict__ src, int64_t n,
                                                               uint32_t tile_lo, uint32_t tile_hi, int r_t, int part_level,
                                                               uint64_t param, int flags) {
    using S = SG<C>;
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* bufs[2] = {smem, smem + S::BUF};
    uint16_t* chunks = reinterpret_cast<uint16_t*>(smem + 2 * S::BUF);  // needed (row, chunk) list
    __shared__ uint16_t tab[243];
    __shared__ int nchunks;
    digit_table_init(tab);
    if (threadIdx.x == 0) nchunks = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < S::ROWS * CHUNKS; i += S::THREADS) {
        const int j = i / CHUNKS, q = i - j * CHUNKS;
        if (chunk_needed<C, EIGHT>(j, q)) chunks[atomicAdd(&nchunks, 1)] = (uint16_t)((j << 4) | q);
    }
    __syncthreads();
    const int nch = nchunks;
    const int64_t rowstride = n * C;
    const bool dst_from_src = (flags & GM_FLAG_DST_FROM_SRC) != 0;
    const bool fetch_line = (flags & GM_FLAG_FETCH_LINE) != 0;
    const uint32_t pw = C == 1 ? 0x01010101u * (uint32_t)(param & 0xffu)
                               : C == 2 ? 0x00010001u * (uint32_t)(param & 0xffffu) : (uint32_t)param;

    // this thread's touched sector (t, g): rows in groups of SC with 1,2,2,4 sectors each
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

    // Tiles in [tile_lo, tile_hi) (digit order of lambda: a range of level-L
    // sub-gaskets).  Visiting order (flags): GM_FLAG_ROWMAJOR visits each
    // sub-gasket's member tiles in row-major order so consecutive tiles are
    // horizontal neighbours sharing the 128-byte halo line; GM_FLAG_CHUNKED gives
    // every CTA a contiguous run of tiles instead of interleaving CTAs.
    const bool rowmajor = (flags & GM_FLAG_ROWMAJOR) != 0;
    const bool chunked = (flags & GM_FLAG_CHUNKED) != 0;
    const int L = part_level < 0 ? 0 : part_level;
    const int q = r_t - L;
    uint32_t per_sg = 1;
    for (int i = 0; i < q; ++i) per_sg *= 3u;
    auto tile_xy = [&](uint32_t tile, uint32_t& bx, uint32_t& by) {
        if (!rowmajor) {
            lambda_digit_order(tile, tab, bx, by);
            return;
        }
        const uint32_t sg = tile / per_sg, k = tile - sg * per_sg;
        uint32_t sx = 0, sy = 0, l, Y;
        if (L > 0) lambda_digit_order(sg, tab, sx, sy);
        tile_rowmajor(k, q, l, Y);
        bx = (sx << q) + l;
        by = (sy << q) + Y;
    };
    const uint32_t span = tile_hi - tile_lo;
    const uint32_t chunk = chunked ? (span + gridDim.x - 1) / gridDim.x : 1u;
    const uint32_t step = chunked ? 1u : gridDim.x;
    uint32_t tile = tile_lo + blockIdx.x * chunk;
    const uint32_t tile_end = chunked ? min(tile_hi, tile + chunk) : tile_hi;
    if (tile >= tile_end) return;
    uint32_t bx, by;
    tile_xy(tile, bx, by);
    stage_tile<C>(bufs[0], chunks, nch, src, n, (int64_t)bx * S::TT, (int64_t)by * S::TT, fetch_line);
    cp_async_commit();
    int cur = 0;
    for (; tile < tile_end; tile += step) {
        const int64_t x0 = (int64_t)bx * S::TT, y0 = (int64_t)by * S::TT;
        const uint32_t next = tile + step;
        uint32_t nbx = 0, nby = 0;
        if (next < tile_end) {  // prefetch the next tile into the other buffer
            tile_xy(next, nbx, nby);
            stage_tile<C>(bufs[cur ^ 1], chunks, nch, src, n, (int64_t)nbx * S::TT, (int64_t)nby * S::TT, fetch_line);
        }
        cp_async_commit();
        cp_async_wait_prev();
        __syncthreads();

        if (active) {
            const uint8_t* b = bufs[cur];
            const uint32_t* up = reinterpret_cast<const uint32_t*>(b + t * PITCH);  // smem row t-1
            const uint32_t* md = up + PITCH / 4;
            const uint32_t* dn = md + PITCH / 4;
            const int k0 = 4 + 8 * g;  // first word of the sector (4 halo words on the left)
            uint32_t r[3][10];         // words k0-1 .. k0+8 of rows t-1, t, t+1
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const uint32_t* row = k == 0 ? up : k == 1 ? md : dn;
                if (!EIGHT && k != 1) {
                    const uint4 a = *reinterpret_cast<const uint4*>(row + k0);
                    const uint4 c = *reinterpret_cast<const uint4*>(row + k0 + 4);
                    r[k][1] = a.x; r[k][2] = a.y; r[k][3] = a.z; r[k][4] = a.w;
                    r[k][5] = c.x; r[k][6] = c.y; r[k][7] = c.z; r[k][8] = c.w;
                    r[k][0] = r[k][9] = 0;
                    continue;
                }
                const uint4 a = *reinterpret_cast<const uint4*>(row + k0);
                const uint4 c = *reinterpret_cast<const uint4*>(row + k0 + 4);
                r[k][0] = row[k0 - 1];
                r[k][1] = a.x; r[k][2] = a.y; r[k][3] = a.z; r[k][4] = a.w;
                r[k][5] = c.x; r[k][6] = c.y; r[k][7] = c.z; r[k][8] = c.w;
                r[k][9] = row[k0 + 8];
            }
            uint32_t out[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint32_t s;
                if (EIGHT) {
                    const uint32_t A = vadd<C>(vadd<C>(r[0][i], r[1][i]), r[2][i]);
                    const uint32_t B = vadd<C>(vadd<C>(r[0][i + 1], r[1][i + 1]), r[2][i + 1]);
                    const uint32_t D = vadd<C>(vadd<C>(r[0][i + 2], r[1][i + 2]), r[2][i + 2]);
                    s = vadd<C>(vadd<C>(lft<C>(A, B), B), rgt<C>(B, D));
                    s = vadd<C>(vsub<C>(s, r[1][i + 1]), pw);
                } else {
                    s = vadd<C>(vadd<C>(lft<C>(r[1][i], r[1][i + 1]), rgt<C>(r[1][i + 1], r[1][i + 2])),
                                vadd<C>(vadd<C>(r[0][i + 1], r[2][i + 1]), pw));
                }
                const bool touched = (((8 * g + i) * S::V) & ~t) == 0;
                const uint32_t m = touched ? tmask : 0u;
                out[i] = (s & m) | (r[1][i + 1] & ~m);
            }
            uint8_t* gp = grid + (y0 + t) * rowstride + x0 * C + g * 32;
            if (!dst_from_src) {  // off-gasket cells from the grid itself (whole-sector write)
                const uint4 o0 = ld_cg16(gp, fetch_line);
                const uint4 o1 = ld_cg16(gp + 16, fetch_line);
                const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool touched = (((8 * g + i) * S::V) & ~t) == 0;
                    const uint32_t m = touched ? tmask : 0u;
                    out[i] = (out[i] & m) | (old[i] & ~m);
                }
            }
            reinterpret_cast<uint4*>(gp)[0] = make_uint4(out[0], out[1], out[2], out[3]);
            reinterpret_cast<uint4*>(gp)[1] = make_uint4(out[4], out[5], out[6], out[7]);
        }
        __syncthreads();  // buffer `cur` is refilled by the next iteration's prefetch
        cur ^= 1;
        bx = nbx;
        by = nby;
    }
    cp_async_wait_all();
}

template <int C, int KIND>
cudaError_t launch_ck(const LaunchArgs& a, int r_t) {
    using S = SG<C>;
    uint32_t lo, hi;
    tile_range(a, r_t, lo, hi);
    if (hi == lo) return cudaSuccess;
    const uint32_t ntiles = hi - lo;
    const size_t smem = 2 * S::BUF + 2 * S::ROWS * CHUNKS + 16;
    auto* kern = stencil_tile<C, KIND>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, smem);
    uint64_t blocks = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > ntiles) blocks = ntiles;
    kern<<<(unsigned)blocks, S::THREADS, smem, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid),
                                                        reinterpret_cast<const uint8_t*>(a.src), a.n, lo, hi, r_t, a.part_level, a.param,
                                                        a.flags);
    note_launch();
    return cudaGetLastError();
}

template <int C>
cudaError_t launch_c(const LaunchArgs& a, int r) {
    int k = 0;
    while ((1 << k) < SG<C>::TT) ++k;
    if (a.kind == KIND_NSUM4) return launch_ck<C, KIND_NSUM4>(a, r - k);
    if (a.kind == KIND_NSUM8) return launch_ck<C, KIND_NSUM8>(a, r - k);
    return cudaErrorNotSupported;
}

}  // namespace

// Neighbour-sum kernels for grids at least one 128-byte tile wide with 1-, 2- or
// 4-byte cells; cudaErrorNotSupported otherwise (the caller falls back).
cudaError_t launch_stencil_tile(const LaunchArgs& a) {
    if (a.flags & GM_FLAG_OMEGA_ORDER) return cudaErrorNotSupported;
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    switch (a.cell_bytes) {
    case 1: if (a.n >= SG<1>::TT) return launch_c<1>(a, r); break;
    case 2: if (a.n >= SG<2>::TT) return launch_c<2>(a, r); break;
    case 4: if (a.n >= SG<4>::TT) return launch_c<4>(a, r); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
