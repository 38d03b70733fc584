// tuned.cu -- B200-tuned lambda kernels (strategy STRAT_TUNED).
//
// Same index set as the paper-literal kernels (every gasket cell of every
// lambda-mapped rho x rho tile, written exactly once), reorganised for HBM:
//   * persistent grid (148 SMs x 8 CTAs x 256 threads), grid-stride over
//     work items = (tile t, tile row ty, 16-byte row segment s);
//   * lambda per item from a 243-entry digit table in shared memory (the
//     closed form of blockmap.py:91-108: per-axis "digit != 0"/"digit == 2"
//     masks, bit-interleaved), ~20 integer ops, no per-level loop;
//   * tiles visited in base-3 digit order of the compact index by default, so
//     consecutive items are spatially adjacent tiles (L2/DRAM-page locality);
//     GM_FLAG_OMEGA_ORDER visits them in the reference's b = wy*W + wx order;
//   * one 16-byte vector store per touched row segment: full segments are
//     stored directly, partial ones are blended (load + select + store) so
//     off-gasket cells keep their pre-launch values (engine.py:201,
//     backends.py:155-156) and every DRAM write is a whole 16-byte half-sector;
//   * neighbour sums (backends.py:127-141 + our 8-neighbour extension) in
//     SIMD-within-a-register (per-byte/per-halfword adds via vadd4/vadd2,
//     neighbour shifts via funnel shifts), wrap-to-width exactly like the
//     reference's int64-then-truncate numba path.
#include "gasket.cuh"
#include "launch.h"
#include "../../include/gasket_b200.h"

namespace gm {

// ---------------------------------------------------------------------------
// 16-byte segment helpers (4 x 32-bit words, little-endian cell order)
// ---------------------------------------------------------------------------

template <int C>
__device__ __forceinline__ uint32_t splat_word(uint64_t param, int w) {
    if (C == 1) return 0x01010101u * (uint32_t)(param & 0xffu);
    if (C == 2) return 0x00010001u * (uint32_t)(param & 0xffffu);
    if (C == 4) return (uint32_t)param;
    return (w & 1) ? (uint32_t)(param >> 32) : (uint32_t)param;
}

// Byte mask of word w for the member cells j (j subset of pat) of a segment.
template <int C>
__device__ __forceinline__ uint32_t member_word_mask(uint32_t pat, int w) {
    uint32_t m = 0;
    if (C == 1) {
#pragma unroll
        for (int b = 0; b < 4; ++b) m |= (((4 * w + b) & ~pat) == 0 ? 0xffu : 0u) << (8 * b);
    } else if (C == 2) {
#pragma unroll
        for (int b = 0; b < 2; ++b) m |= (((2 * w + b) & ~pat) == 0 ? 0xffffu : 0u) << (16 * b);
    } else if (C == 4) {
        m = ((w & ~pat) == 0) ? 0xffffffffu : 0u;
    } else {
        m = (((w >> 1) & ~pat) == 0) ? 0xffffffffu : 0u;
    }
    return m;
}

__device__ __forceinline__ uint4 ld16(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ uint4 ld16_cg(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st16(void* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

__device__ __forceinline__ uint32_t w_of(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Per-lane SIMD add of C-byte cells packed in a 32-bit word.
template <int C>
__device__ __forceinline__ uint32_t vadd(uint32_t a, uint32_t b) {
    if (C == 1) return __vadd4(a, b);
    if (C == 2) return __vadd2(a, b);
    return a + b;
}

// Neighbour words: cell j's left neighbour is cell j-1 (prev word's top cell
// shifts in), right neighbour is cell j+1.  C <= 4 only.
template <int C>
__device__ __forceinline__ uint32_t left_word(uint32_t prev, uint32_t cur) {
    if (C == 4) return prev;
    return __funnelshift_l(prev, cur, 8 * C);
}
template <int C>
__device__ __forceinline__ uint32_t right_word(uint32_t cur, uint32_t next) {
    if (C == 4) return next;
    return __funnelshift_r(cur, next, 8 * C);
}

// One stencil row: the 16-byte segment plus the cell left of it (in the top
// bits of `lw`) and the cell right of it (in the low bits of `rw`).
struct Row16 {
    uint32_t w[4];
    uint32_t lw, rw;
};

template <int C>
__device__ __forceinline__ void load_row16(Row16& r, const uint8_t* base, int64_t n, int64_t y, int64_t x0) {
    static_assert(C <= 4, "row helpers pack cells in 32-bit words");
    if (y < 0 || y >= n) {
        r.w[0] = r.w[1] = r.w[2] = r.w[3] = r.lw = r.rw = 0;
        return;
    }
    const uint8_t* p = base + (y * n + x0) * C;
    const uint4 v = ld16(p);
    r.w[0] = v.x; r.w[1] = v.y; r.w[2] = v.z; r.w[3] = v.w;
    constexpr int V = 16 / C;
    r.lw = x0 > 0 ? ((uint32_t)ld_cell<C>(p, -1) << (32 - 8 * C)) : 0u;
    r.rw = x0 + V < n ? (uint32_t)ld_cell<C>(p, V) : 0u;
}

template <int C, bool EIGHT>
__device__ __forceinline__ void nsum16(const Row16& up, const Row16& mid, const Row16& dn, uint32_t p, uint32_t out[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t ml = left_word<C>(i == 0 ? mid.lw : mid.w[i - 1], mid.w[i]);
        const uint32_t mr = right_word<C>(mid.w[i], i == 3 ? mid.rw : mid.w[i + 1]);
        uint32_t s = vadd<C>(p, vadd<C>(ml, mr));
        s = vadd<C>(s, vadd<C>(up.w[i], dn.w[i]));
        if (EIGHT) {
            const uint32_t ul = left_word<C>(i == 0 ? up.lw : up.w[i - 1], up.w[i]);
            const uint32_t ur = right_word<C>(up.w[i], i == 3 ? up.rw : up.w[i + 1]);
            const uint32_t dl = left_word<C>(i == 0 ? dn.lw : dn.w[i - 1], dn.w[i]);
            const uint32_t dr = right_word<C>(dn.w[i], i == 3 ? dn.rw : dn.w[i + 1]);
            s = vadd<C>(s, vadd<C>(vadd<C>(ul, ur), vadd<C>(dl, dr)));
        }
        out[i] = s;
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------

// SB = segment bytes = min(16, rho*C); V = SB / C cells per segment.
template <int C, int SB, int KIND, bool DIGIT_ORDER>
__global__ void __launch_bounds__(256) lambda_tuned(uint8_t* __restrict__ grid, const uint8_t* __restrict__ src,
                                                    int64_t n, int k, uint32_t W, uint64_t n_items, int seg_shift,
                                                    uint64_t param, int flags) {
    __shared__ uint16_t tab[243];
    digit_table_init(tab);
    __syncthreads();
    constexpr int V = SB / C;
    const uint32_t rho = 1u << k;
    const uint32_t seg_mask = (1u << seg_shift) - 1u;
    const bool dst_from_src = (flags & GM_FLAG_DST_FROM_SRC) != 0;

    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_items;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)g & seg_mask;
        const uint32_t ty = (uint32_t)(g >> seg_shift) & (rho - 1u);
        const uint32_t t = (uint32_t)(g >> (seg_shift + k));
        const uint32_t tx0 = s * V;
        if (tx0 & ~ty) continue;  // no gasket cell in this row segment
        uint32_t bx, by;
        if (DIGIT_ORDER) {
            lambda_digit_order(t, tab, bx, by);
        } else {
            const uint32_t wy = t / W;
            lambda_table(t - wy * W, wy, tab, bx, by);
        }
        const int64_t x0 = (int64_t)bx * rho + tx0;
        const int64_t y = (int64_t)by * rho + ty;
        const uint32_t pat = ty & (V - 1u);  // member cells j of the segment: j subset of pat
        uint8_t* dst = grid + (y * n + x0) * C;

        if constexpr (SB == 16 && KIND != KIND_COUNT && (KIND == KIND_CONST || C <= 4)) {
            uint32_t val[4];
            if constexpr (KIND == KIND_CONST) {
#pragma unroll
                for (int i = 0; i < 4; ++i) val[i] = splat_word<C>(param, i);
            } else {
                Row16 up, mid, dn;
                load_row16<C>(up, src, n, y - 1, x0);
                load_row16<C>(mid, src, n, y, x0);
                load_row16<C>(dn, src, n, y + 1, x0);
                nsum16<C, KIND == KIND_NSUM8>(up, mid, dn, splat_word<C>(param, 0), val);
                if (pat != V - 1u && dst_from_src) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t m = member_word_mask<C>(pat, i);
                        val[i] = (mid.w[i] & ~m) | (val[i] & m);
                    }
                    st16(dst, make_uint4(val[0], val[1], val[2], val[3]));
                    continue;
                }
            }
            if (pat != V - 1u) {  // partial segment: keep off-gasket cells
                const uint4 old = ld16_cg(dst);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t m = member_word_mask<C>(pat, i);
                    val[i] = (w_of(old, i) & ~m) | (val[i] & m);
                }
            }
            st16(dst, make_uint4(val[0], val[1], val[2], val[3]));
        } else {
            // narrow segments (rho*C < 16), 64-bit stencils and coverage counting:
            // per-cell path (cell_op = store, or atomic count for KIND_COUNT).
            (void)dst;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                if ((j & ~pat) == 0) cell_op<C, KIND>(grid, src, n, x0 + j, y, param);
            }
        }
    }
}

template <int C, int SB, int KIND>
static cudaError_t launch_t(const LaunchArgs& a) {
    int k = 0;
    while ((1 << k) < a.rho) ++k;
    int seg_shift = 0;
    while ((SB << seg_shift) < a.rho * C) ++seg_shift;
    uint64_t tiles = 1;
    for (int i = 0; i < a.r_b; ++i) tiles *= 3;
    const uint64_t n_items = (tiles << k) << seg_shift;
    int sms = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    uint64_t blocks = (n_items + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    uint8_t* g = reinterpret_cast<uint8_t*>(a.grid);
    const uint8_t* s = reinterpret_cast<const uint8_t*>(a.src);
    if (a.flags & GM_FLAG_OMEGA_ORDER)
        lambda_tuned<C, SB, KIND, false><<<(unsigned)blocks, 256, 0, a.stream>>>(
            g, s, a.n, k, (uint32_t)a.width, n_items, seg_shift, a.param, a.flags);
    else
        lambda_tuned<C, SB, KIND, true><<<(unsigned)blocks, 256, 0, a.stream>>>(
            g, s, a.n, k, (uint32_t)a.width, n_items, seg_shift, a.param, a.flags);
    note_launch();
    return cudaGetLastError();
}

template <int C, int KIND>
static cudaError_t launch_sb(const LaunchArgs& a) {
    const int64_t row_bytes = (int64_t)a.rho * C;
    if (row_bytes >= 16) return launch_t<C, (16 / C >= 1 ? 16 : C), KIND>(a);
    if (row_bytes == 8) return launch_t<C, (8 >= C ? 8 : C), KIND>(a);
    if (row_bytes == 4) return launch_t<C, (4 >= C ? 4 : C), KIND>(a);
    if (row_bytes == 2) return launch_t<C, (2 >= C ? 2 : C), KIND>(a);
    return launch_t<C, C, KIND>(a);
}

template <int C>
static cudaError_t launch_c(const LaunchArgs& a) {
    switch (a.kind) {
    case KIND_CONST: return launch_sb<C, KIND_CONST>(a);
    case KIND_NSUM4: return launch_sb<C, KIND_NSUM4>(a);
    case KIND_NSUM8: return launch_sb<C, KIND_NSUM8>(a);
    case KIND_COUNT: return launch_sb<4, KIND_COUNT>(a);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_tuned(const LaunchArgs& a) {
    // host-mapped grids: row-ordered whole-line schedule for the write pass (hostrows.cu)
    if (a.flags & GM_FLAG_HOST_ROWS) {
        const cudaError_t eh = launch_host_rows(a);
        if (eh != cudaErrorNotSupported) return eh;
        cudaGetLastError();
    }
    // neighbour sums on grids at least one 128-byte tile wide: shared-memory tiles (stencil.cu)
    if (a.kind == KIND_NSUM4 || a.kind == KIND_NSUM8) {
        if (!(a.flags & GM_FLAG_FORCE_TMA)) {  // v2 tiles (stencil2.cu) unless a variant is asked for
            const cudaError_t e2 = launch_stencil_v2(a);
            if (e2 != cudaErrorNotSupported) return e2;
            cudaGetLastError();
        }
#ifdef GM_AB_VARIANTS
        // A/B builds only: the superseded TMA-staged (stencil_tma.cu) and v1 (stencil.cu) tiles
        const cudaError_t et = launch_stencil_tma(a);
        if (et != cudaErrorNotSupported) return et;
        cudaGetLastError();
        const cudaError_t es = launch_stencil_tile(a);
        if (es != cudaErrorNotSupported) return es;
        cudaGetLastError();
#endif
    }
    // the write pass: line-tile slabs, unit -> tile computed per unit (write.cu)
    if (a.kind == KIND_CONST || a.kind == KIND_COUNT) {
        const cudaError_t ew = launch_write(a);
        if (ew != cudaErrorNotSupported) return ew;
        cudaGetLastError();
    }
    // otherwise the warp-per-tile-band kernel (stream.cu)
    const cudaError_t e = launch_stream(a);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
    switch (a.cell_bytes) {
    case 1: return launch_c<1>(a);
    case 2: return launch_c<2>(a);
    case 4: return launch_c<4>(a);
    case 8: return launch_c<8>(a);
    }
    return cudaErrorInvalidValue;
}

}  // namespace gm
