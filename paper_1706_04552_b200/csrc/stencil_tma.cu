// stencil_tma.cu -- tuned lambda neighbour-sum kernel with TMA tile staging
// (strategy STRAT_TUNED, KIND_NSUM4 / KIND_NSUM8, cells of 1, 2 or 4 bytes).
//
// Same decomposition and arithmetic as stencil.cu (one CTA per lambda tile of
// TT x TT cells with 128-byte rows, one thread per touched 32-byte sector,
// whole-sector stores), but the tile plus halo is staged by the Tensor Memory
// Accelerator: per tile one elected thread issues two 2-D tensor copies,
//   main  box: bytes [x0-16, x0+128) x rows [y0-1, y0+TT]   (144 B x (TT+2))
//   right box: bytes [x0+128, x0+144) x rows [y0+TT-2, y0+TT] (the only rows
//              whose gasket cells read the right neighbour)
// into an NSTAGE-deep ring in shared memory, completing on an mbarrier.  The
// tensor map's out-of-bounds fill is zero, which is exactly the reference's
// "out-of-grid neighbours read 0" (engine.py:37-38).  L2 read misses fetch
// whole 128-byte lines anyway (profiles/r1_probes.md), so staging whole rows
// costs no DRAM traffic over the needed-sector set, and the threads are free
// of copy bookkeeping.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>

#include "gasket.cuh"
#include "launch.h"
#include "../../include/gasket_b200.h"

namespace gm {
namespace {

constexpr int ROWB = 128;   // tile row bytes
constexpr int BOXW = 144;   // main box width: 16 B left halo + 128 B row
constexpr int NSTAGE = 3;   // staged tiles per CTA (tile j computed while j+1, j+2 land)

template <int C>
struct TG {
    static constexpr int V = 4 / C;
    static constexpr int TT = ROWB / C;
    static constexpr int SC = 32 / C;
    static constexpr int NSEC = ROWB / 32;
    static constexpr int ROWS = TT + 2;
    static constexpr int MAIN = ROWS * BOXW;                     // bytes of the main box
    static constexpr int RIGHT = (MAIN + 127) / 128 * 128;        // right box (3 x 16 B), TMA needs 128-B alignment
    static constexpr int STAGE = RIGHT + 128;
    static constexpr int NTOUCH = 9 * SC;
    static constexpr int THREADS = (NTOUCH + 31) / 32 * 32;
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
__device__ __forceinline__ uint32_t lft(uint32_t prev, uint32_t cur) {
    if constexpr (C == 4) return prev;
    else return __funnelshift_l(prev, cur, 8 * C);
}
template <int C>
__device__ __forceinline__ uint32_t rgt(uint32_t cur, uint32_t next) {
    if constexpr (C == 4) return next;
    else return __funnelshift_r(cur, next, 8 * C);
}
template <int C>
__device__ __forceinline__ uint32_t member_mask(uint32_t t) {
    if constexpr (C == 1) {
        const uint32_t p = t & 3u;
        return p == 0 ? 0x000000ffu : p == 1 ? 0x0000ffffu : p == 2 ? 0x00ff00ffu : 0xffffffffu;
    } else if constexpr (C == 2) {
        return (t & 1u) ? 0xffffffffu : 0x0000ffffu;
    } else {
        return 0xffffffffu;
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint4 ld_cg16(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int C, int KIND>
__global__ void __launch_bounds__(TG<C>::THREADS) stencil_tma(const __grid_constant__ CUtensorMap main_map,
                                                              const __grid_constant__ CUtensorMap right_map,
                                                              uint8_t* __restrict__ grid, int64_t n,
                                                              uint32_t tile_lo, uint32_t tile_hi, uint64_t param,
                                                              int flags) {
    using S = TG<C>;
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[NSTAGE];
    __shared__ uint16_t tab[243];
    digit_table_init(tab);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t rowstride = n * C;
    const bool dst_from_src = (flags & GM_FLAG_DST_FROM_SRC) != 0;
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
    // the right-halo word of the last sector is staged only for rows TT-2..TT (smem rows TT-1..TT+1)
    const int rrow = t - (S::TT - 1);  // right-box row of staged row t+k is rrow+k (valid for 0..2)

    auto issue = [&](uint32_t tile, int slot) {
        uint32_t bx, by;
        lambda_digit_order(tile, tab, bx, by);
        const int x0 = (int)(bx * S::TT), y0 = (int)(by * S::TT);
        uint8_t* dst = smem + slot * S::STAGE;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before async writes
        mbar_expect_tx(&bars[slot], S::MAIN + 48);
        tma_load_2d(dst, &main_map, x0 - 16 / C, y0 - 1, &bars[slot]);
        tma_load_2d(dst + S::RIGHT, &right_map, x0 + S::TT, y0 + S::TT - 2, &bars[slot]);
    };

    uint32_t tile = tile_lo + blockIdx.x;
    if (tile >= tile_hi) return;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NSTAGE - 1; ++s)
            if (tile + s * gridDim.x < tile_hi) issue(tile + s * gridDim.x, s);
    }
    int slot = 0;
    uint32_t phase = 0;
    for (; tile < tile_hi; tile += gridDim.x) {
        // keep NSTAGE-1 tiles in flight: refill the slot freed at the end of the previous iteration
        if (threadIdx.x == 0) {
            const uint32_t ahead = tile + (NSTAGE - 1) * gridDim.x;
            if (ahead < tile_hi) issue(ahead, (slot + NSTAGE - 1) % NSTAGE);
        }
        uint32_t bx, by;
        lambda_digit_order(tile, tab, bx, by);
        const int64_t x0 = (int64_t)bx * S::TT, y0 = (int64_t)by * S::TT;
        mbar_wait(&bars[slot], phase);

        if (active) {
            const uint8_t* b = smem + slot * S::STAGE;
            const uint32_t* right = reinterpret_cast<const uint32_t*>(b + S::RIGHT);
            const int k0 = 4 + 8 * g;  // first word of the sector (4 halo words on the left)
            uint32_t r[3][10];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const uint32_t* row = reinterpret_cast<const uint32_t*>(b + (t + k) * BOXW);
                const uint4 a = *reinterpret_cast<const uint4*>(row + k0);
                const uint4 c = *reinterpret_cast<const uint4*>(row + k0 + 4);
                r[k][0] = row[k0 - 1];
                r[k][1] = a.x; r[k][2] = a.y; r[k][3] = a.z; r[k][4] = a.w;
                r[k][5] = c.x; r[k][6] = c.y; r[k][7] = c.z; r[k][8] = c.w;
                const int rr = rrow + k;
                r[k][9] = g < S::NSEC - 1 ? row[k0 + 8] : (rr >= 0 && rr < 3 ? right[rr * 4] : 0u);
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
            if (!dst_from_src) {
                const uint4 o0 = ld_cg16(gp);
                const uint4 o1 = ld_cg16(gp + 16);
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
        __syncthreads();  // slot is refilled by the next iteration's issue
        if (++slot == NSTAGE) {
            slot = 0;
            phase ^= 1u;
        }
    }
}

// ---------------------------------------------------------------------------
// host side: tensor maps (cached per source buffer)
// ---------------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_map(CUtensorMap* m, const void* base, int64_t n, int c, uint32_t box_bytes, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const CUtensorMapDataType dt = c == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : c == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)(n * c)};
    const cuuint32_t box[2] = {box_bytes / (uint32_t)c, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int C, int KIND>
cudaError_t launch_ck(const LaunchArgs& a, int r_t) {
    using S = TG<C>;
    uint32_t lo, hi;
    tile_range(a, r_t, lo, hi);
    if (hi == lo) return cudaSuccess;
    CUtensorMap main_map, right_map;
    if (!make_map(&main_map, a.src, a.n, C, BOXW, S::ROWS) || !make_map(&right_map, a.src, a.n, C, 16, 3))
        return cudaErrorNotSupported;
    const size_t smem = (size_t)NSTAGE * S::STAGE;
    auto* kern = stencil_tma<C, KIND>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, smem);
    uint64_t blocks = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > hi - lo) blocks = hi - lo;
    kern<<<(unsigned)blocks, S::THREADS, smem, a.stream>>>(main_map, right_map, reinterpret_cast<uint8_t*>(a.grid),
                                                            a.n, lo, hi, a.param, a.flags);
    note_launch();
    return cudaGetLastError();
}

template <int C>
cudaError_t launch_c(const LaunchArgs& a, int r) {
    int k = 0;
    while ((1 << k) < TG<C>::TT) ++k;
    if (a.kind == KIND_NSUM4) return launch_ck<C, KIND_NSUM4>(a, r - k);
    if (a.kind == KIND_NSUM8) return launch_ck<C, KIND_NSUM8>(a, r - k);
    return cudaErrorNotSupported;
}

}  // namespace

// TMA-staged neighbour sums; cudaErrorNotSupported for shapes it does not cover
// (the caller falls back to stencil.cu).  Measured on B200 (n=2^17 int8 NSUM8):
// with GM_FLAG_DST_FROM_SRC the cp.async kernel of stencil.cu is faster
// (461 vs 517 us: it stages only the needed chunks and fits 4 CTAs/SM); without
// it this kernel is (672 us vs >2 ms), so it is the default only there.
cudaError_t launch_stencil_tma(const LaunchArgs& a) {
    if (a.flags & (GM_FLAG_OMEGA_ORDER | GM_FLAG_ROWMAJOR | GM_FLAG_CHUNKED | GM_FLAG_NO_TMA)) return cudaErrorNotSupported;
    if ((a.flags & GM_FLAG_DST_FROM_SRC) && !(a.flags & GM_FLAG_FORCE_TMA)) return cudaErrorNotSupported;
    if (a.n > (int64_t(1) << 30)) return cudaErrorNotSupported;  // TMA coordinates are int32
    if ((reinterpret_cast<uintptr_t>(a.src) & 15) != 0) return cudaErrorNotSupported;
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    switch (a.cell_bytes) {
    case 1: if (a.n >= TG<1>::TT) return launch_c<1>(a, r); break;
    case 2: if (a.n >= TG<2>::TT) return launch_c<2>(a, r); break;
    case 4: if (a.n >= TG<4>::TT) return launch_c<4>(a, r); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
