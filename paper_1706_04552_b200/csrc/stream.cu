// stream.cu -- warp-per-tile-band lambda kernel (strategy STRAT_TUNED, n*C >= 128 bytes):
// since round 2 only the paths the dedicated kernels do not take -- GM_FLAG_OMEGA_ORDER
// launches (b = wy*W + wx order, every kind) and neighbour sums on 8-byte cells.  The
// write pass and the coverage audit run in write.cu, neighbour sums in stencil2.cu.
//
// Decomposition.  lambda maps the compact tile index onto tiles of TT x TT
// cells whose rows are exactly one 128-byte line (TT = 32 * WB / C, WB = 4-byte
// words, 8 for 64-bit cells).  One warp owns one band of BAND rows of one
// tile: lane l holds word l of every row, so every warp-wide load or store is
// a single fully-coalesced L1 wavefront.  Tiles are visited in the row-major
// order of rowmajor_table (stencil2.cu) with the (tile, band) units interleaved
// over the warps, so the warps running together store the same rows of
// horizontally neighbouring tiles (shared DRAM pages: 118 -> 104 us at n=2^16
// against the lambda digit order, GM_FLAG_DIGIT_ORDER, which hands each warp a
// contiguous run of units instead).
//
// DRAM-traffic rules (measured with scripts/probe_partial.cu: a partial
// 32-byte-sector write costs a full-sector DRAM read-modify-write):
//   * stencils load, per 32-byte sector, only the sectors holding a neighbour
//     of some gasket cell (exact dilation test per lane, the same sector set
//     as roofline.stencil_read_sectors);
//   * with GM_FLAG_DST_FROM_SRC (grid == snapshot off the gasket, the
//     engine.launch / CA ping-pong case, engine.py:201) every touched sector is
//     written whole, non-gasket cells from the snapshot -> no RMW reads;
//   * otherwise, and for the constant write pass, only gasket cells are
//     stored; the per-row cell pattern is uniform across the warp, so a row is
//     at most two store instructions.
// Semantics: backends.py:127-222 (_cell_value + the numba block loops), with
// results wrapping to the cell width.
#include "gasket.cuh"
#include "launch.h"
#include "../../include/gasket_b200.h"

namespace gm {
namespace {

template <int C> struct WordT { using T = uint32_t; };
template <> struct WordT<8> { using T = uint64_t; };

template <int C>
struct Geo {
    static constexpr int WB = C <= 4 ? 4 : 8;   // bytes per lane word
    static constexpr int V = WB / C;             // cells per lane word
    static constexpr int TT = 32 * V;            // tile edge (cells) = one warp-row
    static constexpr int SC = 32 / C;            // cells per 32-byte sector
    static constexpr int NSEC = TT / SC;         // sectors per tile row
    static constexpr int LPS = 32 / WB;          // lanes per sector
};

template <int C>
__device__ __forceinline__ typename WordT<C>::T splat(uint64_t p) {
    if constexpr (C == 1) return 0x01010101u * (uint32_t)(p & 0xffu);
    else if constexpr (C == 2) return 0x00010001u * (uint32_t)(p & 0xffffu);
    else if constexpr (C == 4) return (uint32_t)p;
    else return p;
}

template <int C>
__device__ __forceinline__ typename WordT<C>::T wadd(typename WordT<C>::T a, typename WordT<C>::T b) {
    if constexpr (C == 1) return __vadd4(a, b);
    else if constexpr (C == 2) return __vadd2(a, b);
    else return a + b;
}

// Byte mask of the gasket cells of a word in tile row t: cell j member iff j subset of (t & (V-1)).
template <int C>
__device__ __forceinline__ typename WordT<C>::T cell_mask(uint32_t t) {
    if constexpr (C == 1) {
        const uint32_t p = t & 3u;
        return p == 0 ? 0x000000ffu : p == 1 ? 0x0000ffffu : p == 2 ? 0x00ff00ffu : 0xffffffffu;
    } else if constexpr (C == 2) {
        return (t & 1u) ? 0xffffffffu : 0x0000ffffu;
    } else if constexpr (C == 4) {
        return 0xffffffffu;
    } else {
        return ~0ull;
    }
}

template <class W>
__device__ __forceinline__ W shfl_up1(W v) {
    if constexpr (sizeof(W) == 8) {
        const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, 1);
        const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), 1);
        return ((uint64_t)hi << 32) | lo;
    } else {
        return __shfl_up_sync(0xffffffffu, v, 1);
    }
}
template <class W>
__device__ __forceinline__ W shfl_dn1(W v) {
    if constexpr (sizeof(W) == 8) {
        const uint32_t lo = __shfl_down_sync(0xffffffffu, (uint32_t)v, 1);
        const uint32_t hi = __shfl_down_sync(0xffffffffu, (uint32_t)(v >> 32), 1);
        return ((uint64_t)hi << 32) | lo;
    } else {
        return __shfl_down_sync(0xffffffffu, v, 1);
    }
}

// Left / right neighbour cells of every cell of the word.
template <int C>
__device__ __forceinline__ typename WordT<C>::T left_of(typename WordT<C>::T prev, typename WordT<C>::T cur) {
    if constexpr (Geo<C>::V == 1) return prev;
    else return __funnelshift_l(prev, cur, 8 * C);
}
template <int C>
__device__ __forceinline__ typename WordT<C>::T right_of(typename WordT<C>::T cur, typename WordT<C>::T next) {
    if constexpr (Geo<C>::V == 1) return next;
    else return __funnelshift_r(cur, next, 8 * C);
}

// Tile-local membership helpers (t may be -1 or TT for halo rows).
template <int C>
__device__ __forceinline__ bool row_in(int t) { return t >= 0 && t < Geo<C>::TT; }
template <int C>
__device__ __forceinline__ bool sec_touched(int t, int g) {
    return row_in<C>(t) && g >= 0 && g < Geo<C>::NSEC && ((g * Geo<C>::SC) & ~t) == 0;
}
template <int C>
__device__ __forceinline__ bool cell_member(int t, int c) {
    return row_in<C>(t) && c >= 0 && c < Geo<C>::TT && (c & ~t) == 0;
}

// Sector g of source row t is read by some gasket cell's neighbourhood.
template <int C, bool EIGHT>
__device__ __forceinline__ bool sec_needed(int t, int g) {
    constexpr int SC = Geo<C>::SC;
    bool need = sec_touched<C>(t - 1, g) || sec_touched<C>(t, g) || sec_touched<C>(t + 1, g);
    // first cell of sector g+1 (a member whenever g+1 is touched) reads the last cell of g
    need = need || sec_touched<C>(t, g + 1);
    // last cell of sector g-1 reads the first cell of g
    need = need || cell_member<C>(t, g * SC - 1);
    if (EIGHT) {
        need = need || sec_touched<C>(t - 1, g + 1) || sec_touched<C>(t + 1, g + 1);
        need = need || cell_member<C>(t - 1, g * SC - 1) || cell_member<C>(t + 1, g * SC - 1);
    }
    return need;
}

template <int C, int KIND, int BAND, bool DIGIT_ORDER>
__global__ void __launch_bounds__(256) lambda_stream(uint8_t* __restrict__ grid, const uint8_t* __restrict__ src,
                                                     int64_t n, uint32_t tile_lo, uint32_t tile_hi, int band_shift,
                                                     uint32_t W, uint64_t param, int flags,
                                                     const uint32_t* __restrict__ order) {
    using WT = typename WordT<C>::T;
    using G = Geo<C>;
    constexpr bool EIGHT = KIND == KIND_NSUM8;
    __shared__ uint16_t tab[243];
    digit_table_init(tab);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t u_lo = (uint64_t)tile_lo << band_shift;
    const uint64_t units = ((uint64_t)tile_hi << band_shift) - u_lo;
    // contiguous chunk of units per warp: lambda once per tile, bands of a tile in order;
    // with a precomputed tile order (GM_FLAG_ROWMAJOR) units are interleaved over the
    // warps instead, so concurrently running warps work on neighbouring tiles
    const bool interleave = order != nullptr;
    const uint64_t chunk = interleave ? 1 : (units + nwarps - 1) / nwarps;
    const uint64_t u_begin = u_lo + warp0 * chunk;
    const uint64_t u_end = interleave ? u_lo + units : (u_begin + chunk < u_lo + units ? u_begin + chunk : u_lo + units);
    const uint64_t u_step = interleave ? nwarps : 1;
    const int64_t rowstride = n * C;  // bytes
    const int g = lane / G::LPS;      // this lane's sector in the tile row
    const int c0 = lane * G::V;       // first cell of this lane's word
    const bool dst_from_src = (flags & GM_FLAG_DST_FROM_SRC) != 0;
    const WT pv = splat<C>(param);
    constexpr int R = BAND + 2;
    [[maybe_unused]] WT w[R];
    [[maybe_unused]] WT lh[R], rh[R];

    uint32_t cur_tile = 0xffffffffu;
    int64_t x0 = 0, y0 = 0;
    int prev_t0 = -BAND;
    for (uint64_t u = u_begin; u < u_end; u += u_step) {
        const uint32_t tile = (uint32_t)(u >> band_shift);
        const int t0 = (int)(u & ((1u << band_shift) - 1u)) * BAND;
        const bool same_tile = tile == cur_tile;
        if (!same_tile) {
            uint32_t bx, by;
            if (order != nullptr) {
                const uint32_t v = __ldg(order + tile);
                bx = v & 0xffffu;
                by = v >> 16;
            } else if (DIGIT_ORDER) {
                lambda_digit_order(tile, tab, bx, by);
            } else {
                const uint32_t wy = tile / W;
                lambda_table(tile - wy * W, wy, tab, bx, by);
            }
            cur_tile = tile;
            x0 = (int64_t)bx * G::TT;
            y0 = (int64_t)by * G::TT;
        }
        uint8_t* drow = grid + (y0 + t0) * rowstride + x0 * C + lane * G::WB;

        if constexpr (KIND == KIND_COUNT) {
#pragma unroll
            for (int i = 0; i < BAND; ++i) {
                static_assert(KIND != KIND_COUNT || C == 4, "coverage counters are uint32 cells");
                if ((c0 & ~(t0 + i)) == 0) atomicAdd(reinterpret_cast<unsigned int*>(drow + (int64_t)i * rowstride), 1u);
            }
        } else if constexpr (KIND == KIND_CONST) {
            // rows come in groups of V (t0 is a multiple of V): within a group the word's
            // touched flag is constant and slot j's cell pattern is j (cells k subset of j)
#pragma unroll
            for (int q = 0; q < BAND / G::V; ++q) {
                const int tq = t0 + q * G::V;
                if ((c0 & ~tq) == 0) {
                    uint8_t* p = drow + (int64_t)(q * G::V) * rowstride;
                    if constexpr (G::V == 1) {
                        *reinterpret_cast<WT*>(p) = pv;
                    } else if constexpr (G::V == 2) {
                        *reinterpret_cast<uint16_t*>(p) = (uint16_t)pv;
                        *reinterpret_cast<uint32_t*>(p + rowstride) = (uint32_t)pv;
                    } else {
                        p[0] = (uint8_t)pv;
                        *reinterpret_cast<uint16_t*>(p + rowstride) = (uint16_t)pv;
                        p[2 * rowstride] = (uint8_t)pv;
                        p[2 * rowstride + 2] = (uint8_t)pv;
                        *reinterpret_cast<uint32_t*>(p + 3 * rowstride) = (uint32_t)pv;
                    }
                }
            }
        } else {
            // ---- rows t0-1 .. t0+BAND (only sectors some neighbourhood needs); the two
            //      rows shared with the band above were loaded by this warp already
            const bool carry = same_tile && prev_t0 + BAND == t0;
            if (carry) {
                w[0] = w[BAND];
                w[1] = w[BAND + 1];
                lh[0] = lh[BAND];
                lh[1] = lh[BAND + 1];
                rh[0] = rh[BAND];
                rh[1] = rh[BAND + 1];
            }
            const uint8_t* srow = src + (y0 + t0 - 1) * rowstride + x0 * C + lane * G::WB;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (j < 2 && carry) continue;
                const int t = t0 - 1 + j;
                const int64_t y = y0 + t;
                const bool in = y >= 0 && y < n;
                const uint8_t* p = srow + (int64_t)j * rowstride;
                w[j] = (in && sec_needed<C, EIGHT>(t, g)) ? __ldg(reinterpret_cast<const WT*>(p)) : WT(0);
                const bool needl = EIGHT ? (row_in<C>(t - 1) || row_in<C>(t) || row_in<C>(t + 1)) : row_in<C>(t);
                const bool needr = EIGHT ? (cell_member<C>(t - 1, G::TT - 1) || cell_member<C>(t, G::TT - 1) ||
                                            cell_member<C>(t + 1, G::TT - 1))
                                         : cell_member<C>(t, G::TT - 1);
                lh[j] = (lane == 0 && in && x0 > 0 && needl) ? (WT)ld_cell<C>(p, -1) : WT(0);
                rh[j] = (lane == 31 && in && x0 + G::TT < n && needr) ? (WT)ld_cell<C>(p, G::V) : WT(0);
            }
            prev_t0 = t0;
            // ---- compute + store rows t0 .. t0+BAND-1
#pragma unroll
            for (int i = 0; i < BAND; ++i) {
                const int t = t0 + i;
                WT nb[3][2];  // [up/mid/dn][left/right] neighbour words
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    if (!EIGHT && k != 1) continue;
                    const WT cur = w[i + k];
                    WT prev = shfl_up1(cur);
                    WT next = shfl_dn1(cur);
                    if constexpr (G::V > 1) {
                        if (lane == 0) prev = lh[i + k] << (32 - 8 * C);
                    } else {
                        if (lane == 0) prev = lh[i + k];
                    }
                    if (lane == 31) next = rh[i + k];
                    nb[k][0] = left_of<C>(prev, cur);
                    nb[k][1] = right_of<C>(cur, next);
                }
                WT s = wadd<C>(pv, wadd<C>(nb[1][0], nb[1][1]));
                s = wadd<C>(s, wadd<C>(w[i], w[i + 2]));
                if (EIGHT) s = wadd<C>(s, wadd<C>(wadd<C>(nb[0][0], nb[0][1]), wadd<C>(nb[2][0], nb[2][1])));
                const bool word_touched = (c0 & ~t) == 0;
                uint8_t* p = drow + (int64_t)i * rowstride;
                if (dst_from_src) {
                    if (sec_touched<C>(t, g)) {  // whole sector written: no DRAM read-modify-write
                        const WT m = word_touched ? cell_mask<C>((uint32_t)t) : WT(0);
                        *reinterpret_cast<WT*>(p) = (s & m) | (w[i + 1] & ~m);
                    }
                } else if (word_touched) {
                    if constexpr (G::V == 1) {
                        *reinterpret_cast<WT*>(p) = s;
                    } else if constexpr (G::V == 2) {
                        if (t & 1) *reinterpret_cast<uint32_t*>(p) = s;
                        else *reinterpret_cast<uint16_t*>(p) = (uint16_t)s;
                    } else {
                        switch (t & 3) {
                        case 3: *reinterpret_cast<uint32_t*>(p) = s; break;
                        case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)s; break;
                        case 2: p[2] = (uint8_t)(s >> 16); p[0] = (uint8_t)s; break;
                        default: p[0] = (uint8_t)s; break;
                        }
                    }
                }
            }
        }
    }
}

template <int C, int KIND, int BAND>
cudaError_t launch_band(const LaunchArgs& a, int r_t) {
    using G = Geo<C>;
    uint32_t lo, hi;
    tile_range(a, r_t, lo, hi);
    if (hi == lo) return cudaSuccess;
    const uint32_t ntiles = hi - lo;
    int band_shift = 0;
    while ((BAND << band_shift) < G::TT) ++band_shift;
    uint32_t W = 1;
    for (int i = 0; i < r_t / 2; ++i) W *= 3u;
    const uint64_t units = (uint64_t)ntiles << band_shift;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool digit = !(a.flags & GM_FLAG_OMEGA_ORDER);
    auto* kern = digit ? lambda_stream<C, KIND, BAND, true> : lambda_stream<C, KIND, BAND, false>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    uint64_t blocks = (units * 32 + 255) / 256;
    const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (blocks > cap) blocks = cap;
    const uint32_t* order = nullptr;
    if (digit && !(a.flags & GM_FLAG_DIGIT_ORDER) && KIND != KIND_COUNT)
        order = rowmajor_table(r_t, order_level(a, r_t));
    kern<<<(unsigned)blocks, 256, 0, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid),
                                                 reinterpret_cast<const uint8_t*>(a.src), a.n, lo, hi, band_shift, W,
                                                 a.param, a.flags, order);
    note_launch();
    return cudaGetLastError();
}

template <int C>
cudaError_t launch_c(const LaunchArgs& a, int r_t) {
    switch (a.kind) {
    case KIND_CONST: return launch_band<C, KIND_CONST, 16>(a, r_t);
    case KIND_NSUM4: return launch_band<C, KIND_NSUM4, 16>(a, r_t);
    case KIND_NSUM8: return launch_band<C, KIND_NSUM8, 16>(a, r_t);
    case KIND_COUNT:
        if constexpr (C == 4) return launch_band<4, KIND_COUNT, 16>(a, r_t);
        break;
    }
    return cudaErrorInvalidValue;
}

}  // namespace

// Returns cudaErrorNotSupported when the grid is narrower than one tile row
// (the caller then uses the generic small-grid kernel in tuned.cu).
cudaError_t launch_stream(const LaunchArgs& a) {
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    auto level = [&](int tt) {
        int k = 0;
        while ((1 << k) < tt) ++k;
        return r - k;
    };
    switch (a.cell_bytes) {
    case 1: if (a.n >= Geo<1>::TT) return launch_c<1>(a, level(Geo<1>::TT)); break;
    case 2: if (a.n >= Geo<2>::TT) return launch_c<2>(a, level(Geo<2>::TT)); break;
    case 4: if (a.n >= Geo<4>::TT) return launch_c<4>(a, level(Geo<4>::TT)); break;
    case 8: if (a.n >= Geo<8>::TT) return launch_c<8>(a, level(Geo<8>::TT)); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
