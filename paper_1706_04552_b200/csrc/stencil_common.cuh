// stencil_common.cuh -- device helpers shared by the tuned neighbour-sum kernels
// (stencil2.cu single step, stencil_tb.cu two fused steps): cp.async staging with
// the .L2::64B fetch hint, whole-sector loads/stores, and the split-lane SIMD
// arithmetic (cells spread into carry-free 16/32-bit lanes, see stencil2.cu).
#pragma once
#include <cstdint>

namespace gm {
namespace sc {

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem, int src_bytes, bool line) {
    if (line)
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem), "r"(src_bytes)
                     : "memory");
    else
        asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem), "r"(src_bytes)
                     : "memory");
}
// 256-byte prefetch-size variant (the line and its neighbour), for A/B runs
__device__ __forceinline__ void cp_async16_256(uint32_t smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ld_sector(const uint8_t* p, bool line, bool v8, uint32_t (&v)[8]) {
    if (!v8) {
        const uint4 a = __ldcg(reinterpret_cast<const uint4*>(p));
        const uint4 b = __ldcg(reinterpret_cast<const uint4*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else if (line)
        asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "l"(p));
    else
        asm volatile("ld.global.cg.L2::64B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "l"(p));
}
// one 256-bit store when the grid is 32-byte aligned (device allocations),
// else two 16-byte stores (e.g. a page-locked numpy array mapped over PCIe)
__device__ __forceinline__ void st_sector(uint8_t* p, const uint32_t (&v)[8], bool v8, bool cs) {
    if (v8 && cs) {
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                     "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else if (v8) {
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                     "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else {
        reinterpret_cast<uint4*>(p)[0] = make_uint4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<uint4*>(p)[1] = make_uint4(v[4], v[5], v[6], v[7]);
    }
}

// ---- split-lane arithmetic --------------------------------------------------
// even(w)/odd(w): the word's even/odd cells, each in its own lane wide enough
// that sums of up to 9 cells never carry into the next lane.
template <int C>
__device__ __forceinline__ uint32_t even_cells(uint32_t w) {
    if constexpr (C == 1) return __byte_perm(w, 0u, 0x4240);  // bytes 0,2 -> 16-bit lanes
    else return w & 0xffffu;                                  // C == 2: cell 0 -> 32-bit lane
}
template <int C>
__device__ __forceinline__ uint32_t odd_cells(uint32_t w) {
    if constexpr (C == 1) return __byte_perm(w, 0u, 0x4341);  // bytes 1,3 -> 16-bit lanes
    else return w >> 16;
}
// lanes shifted one cell pair: lane i <- lane i-1 (lane 0 from the previous word)
template <int C>
__device__ __forceinline__ uint32_t lane_up(uint32_t prev, uint32_t cur) {
    if constexpr (C == 1) return __funnelshift_l(prev, cur, 16);
    else return prev;
}
// lane i <- lane i+1 (last lane from the next word)
template <int C>
__device__ __forceinline__ uint32_t lane_dn(uint32_t cur, uint32_t next) {
    if constexpr (C == 1) return __funnelshift_r(cur, next, 16);
    else return next;
}
template <int C>
__device__ __forceinline__ uint32_t pack_cells(uint32_t e, uint32_t o) {
    if constexpr (C == 1) return __byte_perm(e, o, 0x6240);
    else return __byte_perm(e, o, 0x5410);
}
// gasket cells of a word of tile row t (cell j member iff j subset of t & (V-1))
template <int C>
__device__ __forceinline__ uint32_t member_mask(uint32_t t) {
    if constexpr (C == 1) {
        // byte j of the word is a gasket cell iff j subset of (t & 3): a byte-permute of
        // all-ones / zero with the selector for that pattern (0x4440, 0x4400, 0x4040, 0x0000)
        const uint32_t sel = (uint32_t)(0x0000404044004440ull >> ((t & 3u) << 4));
        return __byte_perm(0xffffffffu, 0u, sel);
    } else if constexpr (C == 2) {
        return (t & 1u) ? 0xffffffffu : 0x0000ffffu;
    } else {
        return 0xffffffffu;
    }
}

// The NW result words of a run of NW words (a sector: NW = 8) from the staged rows
// (w[r][p] = word k0-1+p of rows t-1, t, t+1).
template <int C, bool EIGHT, int NW = 8>
__device__ __forceinline__ void sector_sums(const uint32_t (&w)[3][NW + 2], uint32_t pv, uint32_t (&out)[NW]) {
    if constexpr (C == 4) {
        if constexpr (EIGHT) {
            uint32_t s[NW + 2];
#pragma unroll
            for (int p = 0; p < NW + 2; ++p) s[p] = w[0][p] + w[1][p] + w[2][p];
#pragma unroll
            for (int i = 0; i < NW; ++i) out[i] = s[i] + s[i + 1] + s[i + 2] - w[1][i + 1] + pv;
        } else {
#pragma unroll
            for (int i = 0; i < NW; ++i) out[i] = w[1][i] + w[1][i + 2] + w[0][i + 1] + w[2][i + 1] + pv;
        }
    } else {
        if constexpr (EIGHT) {
            uint32_t ce[NW + 2], co[NW + 2];
#pragma unroll
            for (int p = 0; p < NW + 2; ++p) {
                ce[p] = even_cells<C>(w[0][p]) + even_cells<C>(w[1][p]) + even_cells<C>(w[2][p]);
                co[p] = odd_cells<C>(w[0][p]) + odd_cells<C>(w[1][p]) + odd_cells<C>(w[2][p]);
            }
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                const int p = i + 1;
                const uint32_t both = ce[p] + co[p];
                // box sum minus the centre plus param; the centre is part of the box, so no borrow
                const uint32_t re = both + lane_up<C>(co[p - 1], co[p]) - even_cells<C>(w[1][p]) + pv;
                const uint32_t ro = both + lane_dn<C>(ce[p], ce[p + 1]) - odd_cells<C>(w[1][p]) + pv;
                out[i] = pack_cells<C>(re, ro);
            }
        } else {
            uint32_t em[NW + 2], om[NW + 2];
#pragma unroll
            for (int p = 0; p < NW + 2; ++p) {
                em[p] = even_cells<C>(w[1][p]);
                om[p] = odd_cells<C>(w[1][p]);
            }
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                const int p = i + 1;
                const uint32_t re = even_cells<C>(w[0][p]) + even_cells<C>(w[2][p]) + om[p] + lane_up<C>(om[p - 1], om[p]) + pv;
                const uint32_t ro = odd_cells<C>(w[0][p]) + odd_cells<C>(w[2][p]) + em[p] + lane_dn<C>(em[p], em[p + 1]) + pv;
                out[i] = pack_cells<C>(re, ro);
            }
        }
    }
}

}  // namespace sc
}  // namespace gm
