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
constexpr int PITCH = ROWB + 32;       // smem row: 16 B left halo + row + 16 B right halo
constexpr int THREADS = 256;

template <int C>
struct SG {
    static constexpr int V = 4 / C;          // cells per 4-byte word
    static constexpr int TT = ROWB / C;      // tile edge in cells
    static constexpr int SC = 32 / C;        // cells per sector
    static constexpr int NSEC = ROWB / 32;   // sectors per tile row (4)
    static constexpr int ROWS = TT + 2;      // staged rows
    static constexpr int BUF = ROWS * PITCH; // bytes per staged tile
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

__device__ __forceinline__ uint4 ld_cg16(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool zero_fill) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int src_bytes = zero_fill ? 0 : 16;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Issue the staging copies of one tile (rows -1..TT, chunks 0..9 of 16 bytes).
template <int C, bool EIGHT>
__device__ __forceinline__ void stage_tile(uint8_t* buf, const uint8_t* __restrict__ src, int64_t n, int64_t x0,
                                           int64_t y0) {
    using S = SG<C>;
    const int64_t rowstride = n * C;
    constexpr int CHUNKS = PITCH / 16;  // 10
    for (int i = threadIdx.x; i < S::ROWS * CHUNKS; i += THREADS) {
        const int j = i / CHUNKS, q = i - j * CHUNKS;
        const int t = j - 1;
        const int64_t y = y0 + t;
        const bool yin = y >= 0 && y < n;
        bool need;
        const uint8_t* gp;
        if (q == 0) {  // left halo: only its last cell (x0-1) is read
            need = EIGHT ? (row_in<C>(t - 1) || row_in<C>(t) || row_in<C>(t + 1)) : row_in<C>(t);
            gp = src + y * rowstride + x0 * C - 16;
            if (need && (!yin || x0 == 0)) { cp_async16(buf + j * PITCH, src, true); continue; }
        } else if (q == CHUNKS - 1) {  // right halo: only its first cell (x0+TT) is read
            need = EIGHT ? (cell_member<C>(t - 1, S::TT - 1) || cell_member<C>(t, S::TT - 1) ||
                            cell_member<C>(t + 1, S::TT - 1))
                         : cell_member<C>(t, S::TT - 1);
            gp = src + y * rowstride + (x0 + S::TT) * C;
            if (need && (!yin || x0 + S::TT >= n)) { cp_async16(buf + j * PITCH + q * 16, src, true); continue; }
        } else {
            need = sec_needed<C, EIGHT>(t, (q - 1) >> 1);
            gp = src + y * rowstride + x0 * C + (q - 1) * 16;
            if (need && !yin) { cp_async16(buf + j * PITCH + q * 16, src, true); continue; }
        }
        if (need) cp_async16(buf + j * PITCH + q * 16, gp, false);
    }
}

template <int C, int KIND>
__global__ void __launch_bounds__(THREADS) stencil_tile(uint8_t* __restrict__ grid, const uint8_t* __restrict__ src,
                                                        int64_t n, uint32_t ntiles, uint64_t param, int flags) {
    using S = SG<C>;
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* bufs[2] = {smem, smem + S::BUF};
    uint16_t* secs = reinterpret_cast<uint16_t*>(smem + 2 * S::BUF);  // touched (t, g) list
    __shared__ uint16_t tab[243];
    __shared__ int nsecs;
    digit_table_init(tab);
    if (threadIdx.x == 0) {
        int k = 0;
        for (int t = 0; t < S::TT; ++t)
            for (int g = 0; g < S::NSEC; ++g)
                if (((g * S::SC) & ~t) == 0) secs[k++] = (uint16_t)((t << 2) | g);
        nsecs = k;
    }
    __syncthreads();
    const int64_t rowstride = n * C;
    const bool dst_from_src = (flags & GM_FLAG_DST_FROM_SRC) != 0;
    const uint32_t pw = C == 1 ? 0x01010101u * (uint32_t)(param & 0xffu)
                               : C == 2 ? 0x00010001u * (uint32_t)(param & 0xffffu) : (uint32_t)param;

    uint32_t tile = blockIdx.x;
    if (tile >= ntiles) return;
    uint32_t bx, by;
    lambda_digit_order(tile, tab, bx, by);
    stage_tile<C, EIGHT>(bufs[0], src, n, (int64_t)bx * S::TT, (int64_t)by * S::TT);
    cp_async_commit();
    int cur = 0;
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t x0 = (int64_t)bx * S::TT, y0 = (int64_t)by * S::TT;
        // prefetch the next tile into the other buffer
        const uint32_t next = tile + gridDim.x;
        uint32_t nbx = 0, nby = 0;
        if (next < ntiles) {
            lambda_digit_order(next, tab, nbx, nby);
            stage_tile<C, EIGHT>(bufs[cur ^ 1], src, n, (int64_t)nbx * S::TT, (int64_t)nby * S::TT);
        }
        cp_async_commit();
        cp_async_wait_prev();
        __syncthreads();

        const uint8_t* b = bufs[cur];
        for (int e = threadIdx.x; e < nsecs; e += THREADS) {
            const int t = secs[e] >> 2, g = secs[e] & 3;
            const uint32_t* up = reinterpret_cast<const uint32_t*>(b + t * PITCH);  // smem row t-1
            const uint32_t* md = up + PITCH / 4;
            const uint32_t* dn = md + PITCH / 4;
            const int k0 = 4 + 8 * g;  // first word of the sector (4 halo words on the left)
            uint32_t out[8];
            // words k0-1 .. k0+8 of each row
            uint32_t pu = up[k0 - 1], pm = md[k0 - 1], pd = dn[k0 - 1];
            uint32_t cu = up[k0], cm = md[k0], cd = dn[k0];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t nu = up[k0 + i + 1], nm = md[k0 + i + 1], nd = dn[k0 + i + 1];
                const int w = 8 * g + i;  // word index in the tile row
                uint32_t s;
                if (EIGHT) {
                    const uint32_t A = vadd<C>(vadd<C>(pu, pm), pd);
                    const uint32_t B = vadd<C>(vadd<C>(cu, cm), cd);
                    const uint32_t Cc = vadd<C>(vadd<C>(nu, nm), nd);
                    s = vadd<C>(vadd<C>(lft<C>(A, B), B), rgt<C>(B, Cc));
                    s = vadd<C>(vsub<C>(s, cm), pw);
                } else {
                    s = vadd<C>(vadd<C>(lft<C>(pm, cm), rgt<C>(cm, nm)), vadd<C>(vadd<C>(cu, cd), pw));
                }
                const bool touched = ((w * S::V) & ~t) == 0;
                const uint32_t m = touched ? member_mask<C>((uint32_t)t) : 0u;
                out[i] = (s & m) | (cm & ~m);
                pu = cu; pm = cm; pd = cd;
                cu = nu; cm = nm; cd = nd;
            }
            uint8_t* gp = grid + (y0 + t) * rowstride + x0 * C + g * 32;
            if (!dst_from_src) {  // off-gasket cells from the grid itself (whole-sector write)
                const uint4 o0 = ld_cg16(gp);
                const uint4 o1 = ld_cg16(gp + 16);
                const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool touched = (((8 * g + i) * S::V) & ~t) == 0;
                    const uint32_t m = touched ? member_mask<C>((uint32_t)t) : 0u;
                    out[i] = (out[i] & m) | (old[i] & ~m);
                }
            }
            reinterpret_cast<uint4*>(gp)[0] = make_uint4(out[0], out[1], out[2], out[3]);
            reinterpret_cast<uint4*>(gp)[1] = make_uint4(out[4], out[5], out[6], out[7]);
        }
        __syncthreads();  // buffer `cur` is refilled two tiles from now
        cur ^= 1;
        bx = nbx;
        by = nby;
    }
    cp_async_wait_all();
}

template <int C, int KIND>
cudaError_t launch_ck(const LaunchArgs& a, int r_t) {
    using S = SG<C>;
    uint32_t ntiles = 1;
    for (int i = 0; i < r_t; ++i) ntiles *= 3u;
    const size_t smem = 2 * S::BUF + 2 * S::TT * S::NSEC + 16;
    auto* kern = stencil_tile<C, KIND>;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
    uint64_t blocks = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > ntiles) blocks = ntiles;
    kern<<<(unsigned)blocks, THREADS, smem, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid),
                                                        reinterpret_cast<const uint8_t*>(a.src), a.n, ntiles, a.param,
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
