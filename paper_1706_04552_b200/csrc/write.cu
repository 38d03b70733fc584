// write.cu -- the tuned lambda write pass (strategy STRAT_TUNED, KIND_CONST, n*C >= 128 bytes).
//
// What it replaces: _block_space_nb with KERNEL_CONST (backends.py:158-222 with
// _cell_value, backends.py:127-141): every gasket cell of the n x n grid gets
// `param`, nothing else is written (backends.py:155-156).
//
// Blocks.  The block-space map runs on line tiles of TT x TT cells whose rows are
// exactly one 128-byte line (TT = 128 / C, so rho = TT: 128 int8 cells).  Tile (X, Y)
// holds gasket cells iff X is a bit-subset of Y, and its cell (j, t) is
// a member iff j is a bit-subset of t.  A work unit is a band of BAND rows of one
// tile; units are tile-major and handed out round-robin over the warps, so the eight
// warps of a CTA store consecutive bands of one tile and the CTAs running together
// work on neighbouring tiles.
//
// lambda(omega) per unit, on the warp (the paper's scheme):
// lane i < q owns level i + 1, extracts base-3 digit i of the compact tile index c
// with a multiply-high by its own reciprocal of 3^i and one by 1/3, and two warp
// ballots assemble the block coordinates -- X from the levels whose digit is 2, Y
// from the levels whose digit is nonzero (blockmap.py:34-60: level mu adds
// (beta >> 1, beta != 0) << (mu - 1)).  O(1) integer steps per lane, no table, no
// loads.  c runs over the base-3 digit order of the packed rectangle (consecutive c
// are neighbouring tiles); the reference's b = wy*W + wx order is the same tile set
// (gm_map_rectangle / GM_FLAG_OMEGA_ORDER give that order).
//
// Alternatives (same cells, same values):
//   * GM_FLAG_ROWMAJOR: tiles in row-major order (block row Y, then X): c -> Y by a
//     q-step descent over the per-row member counts 3^i * 2^popc(prefix), X =
//     pdep(k, Y) as one ballot.
//   * GM_FLAG_GRID_ROWS: no blocks -- one warp per grid row (bottom row first), the
//     row's member lines left to right, 4 lines per 16-byte-lane instruction.
//
// Store modes (a partial 32-byte-sector store costs a DRAM
// read-modify-write of the sector; a whole sector does not):
//   * general (default): only gasket cells are stored, one warp-uniform store width
//     per row -- any background survives, exactly the reference's semantics; every
//     touched sector pays the read-modify-write;
//   * GM_FLAG_ZERO_BACKGROUND (opt-in): the caller asserts every off-gasket cell is 0
//     (the paper's zero-filled matrix; the reference bench's
//     make_grid zeros, engine.py:88-90, bench.py:145-150).  Each touched 32-byte
//     sector is stored whole (gasket cells = param, the rest 0): the same final grid,
//     no DRAM read.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "gasket.cuh"
#include "launch.h"
#include "../../include/gasket_b200.h"

namespace gm {
namespace {

__constant__ uint32_t c_pow3[20] = {1u,       3u,        9u,        27u,        81u,       243u,      729u,
                                    2187u,    6561u,     19683u,    59049u,     177147u,   531441u,   1594323u,
                                    4782969u, 14348907u, 43046721u, 129140163u, 387420489u, 1162261467u};

template <int C>
struct WGeo {
    static constexpr int TT = 128 / C;              // tile edge: one 128-byte line per row
    static constexpr int BAND = TT < 32 ? TT : 32;  // rows per unit
    static constexpr int LB = TT / BAND == 4 ? 2 : TT / BAND == 2 ? 1 : 0;  // log2 bands per tile
    static constexpr int LT = TT == 128 ? 7 : TT == 64 ? 6 : TT == 32 ? 5 : 4;
    static constexpr int P16 = 16 / C;              // cells per 16-byte piece
};

// Byte mask of the gasket cells of 32-bit word w (0..3) of 16-byte piece p of tile row t.
template <int C>
__device__ __forceinline__ uint32_t word_mask(int p, int w, uint32_t t) {
    if constexpr (C == 1) {
        const uint32_t j = (uint32_t)(16 * p + 4 * w);
        if (j & ~t) return 0u;
        const uint32_t b = t & 3u;
        return b == 3u ? 0xffffffffu : b == 1u ? 0x0000ffffu : b == 2u ? 0x00ff00ffu : 0x000000ffu;
    } else if constexpr (C == 2) {
        const uint32_t j = (uint32_t)(8 * p + 2 * w);
        if (j & ~t) return 0u;
        return (t & 1u) ? 0xffffffffu : 0x0000ffffu;
    } else if constexpr (C == 4) {
        const uint32_t j = (uint32_t)(4 * p + w);
        return (j & ~t) ? 0u : 0xffffffffu;
    } else {
        const uint32_t j = (uint32_t)(2 * p + (w >> 1));
        return (j & ~t) ? 0u : 0xffffffffu;
    }
}

// 32-bit word w of the cell value splatted over a word (8-byte cells: low/high halves).
template <int C>
__device__ __forceinline__ uint32_t splat_w(uint64_t p, int w) {
    if constexpr (C == 1) return 0x01010101u * (uint32_t)(p & 0xffu);
    else if constexpr (C == 2) return 0x00010001u * (uint32_t)(p & 0xffffu);
    else if constexpr (C == 4) return (uint32_t)p;
    else return (w & 1) ? (uint32_t)(p >> 32) : (uint32_t)p;
}

__device__ __forceinline__ void st_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// The gasket cells of one lane word of a row with in-line pattern t (general mode):
// the pattern is the same for every lane of the row, so each row is one store width.
template <int C>
__device__ __forceinline__ void st_members(uint8_t* p, uint32_t v, uint32_t t) {
    if constexpr (C == 1) {
        switch (t & 3u) {
        case 3: *reinterpret_cast<uint32_t*>(p) = v; break;
        case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; break;
        case 2: p[0] = (uint8_t)v; p[2] = (uint8_t)v; break;
        default: p[0] = (uint8_t)v; break;
        }
    } else if constexpr (C == 2) {
        if (t & 1u) *reinterpret_cast<uint32_t*>(p) = v;
        else *reinterpret_cast<uint16_t*>(p) = (uint16_t)v;
    } else {
        *reinterpret_cast<uint32_t*>(p) = v;
    }
}

__device__ __forceinline__ uint64_t lambda_lane_reciprocal(int lane) {
    if (lane == 0 || lane > 20) return 0;
    uint64_t p3 = 1;
    for (int i = 0; i < lane; ++i) p3 *= 3u;
    return ~0ull / p3 + 1ull;  // floor(c / 3^lane) = umulhi(c, this) for c < 2^32
}

// Dynamic work distribution.  Warps take units from a ticket counter instead of a
// static round-robin: the SMs do not run at the same speed (ncu, n=2^16 int8: SM active
// cycles from 57 K to 98 K within one 111 K-cycle launch of the grid-row kernel -- the
// SMs nearer the DRAM and L2 they write finish early), so a static split leaves the
// fast SMs idle for the tail.  q[0] = next ticket, q[1] = warps retired; the last warp
// to retire zeroes both for the next launch on the stream.
__device__ __forceinline__ uint32_t grab(uint32_t* q, int lane, uint32_t step) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(q, step);
    return __shfl_sync(0xffffffffu, t, 0);
}
__device__ __forceinline__ void retire(uint32_t* q, int lane, uint32_t nwarps) {
    if (q == nullptr || lane != 0) return;
    __threadfence();
    if (atomicAdd(q + 1, 1u) == nwarps - 1) {
        q[0] = 0u;
        q[1] = 0u;
        __threadfence();
    }
}

// lambda of compact tile index c at level q (q <= 20): every lane returns (X, Y).
__device__ __forceinline__ void lambda_lanes(uint32_t c, int q, int lane, uint64_t inv, uint32_t& X, uint32_t& Y) {
    const uint32_t qd = lane == 0 ? c : (uint32_t)__umul64hi((uint64_t)c, inv);
    const uint32_t d = qd - 3u * (__umulhi(qd, 0xAAAAAAABu) >> 1);  // digit = qd mod 3
    const bool live = lane < q;
    X = __ballot_sync(0xffffffffu, live && d == 2u);
    Y = __ballot_sync(0xffffffffu, live && d != 0u);
}

// Row-major tile index k -> member tile (X, Y): the member count of the block rows
// Y' < Y sharing Y's bits above i telescopes into 3^i * 2^(bits chosen so far), so Y
// comes out of a q-step descent; X = pdep(k', Y) is one ballot (lane i sets bit i when
// bit i of Y is set and k' has the bit at that bit's rank in Y).
__device__ __forceinline__ void tile_rows(uint32_t k, int q, int lane, uint32_t& X, uint32_t& Y) {
    uint32_t rem = k, y = 0;
    int pc = 0;
    for (int i = q - 1; i >= 0; --i) {
        const uint32_t c = c_pow3[i] << pc;
        if (rem >= c) {
            rem -= c;
            y |= 1u << i;
            ++pc;
        }
    }
    const bool bit = lane < q && ((y >> lane) & 1u) && ((rem >> __popc(y & ((1u << lane) - 1u))) & 1u);
    X = __ballot_sync(0xffffffffu, bit);
    Y = y;
}

// One warp per (tile, band) unit; 4-byte lanes, one 128-byte line per instruction:
// lane l holds word l of the row.
template <int C, bool ZERO, bool ROWMAJOR, bool COUNT = false>
__global__ void __launch_bounds__(256) gasket_write(uint8_t* __restrict__ grid, int64_t n, int q, uint32_t u_lo,
                                                    uint32_t u_hi, uint64_t param, uint32_t* __restrict__ wq,
                                                    int tshift) {
    using G = WGeo<C>;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int64_t rowstride = n * C;
    const uint32_t j = C == 8 ? (uint32_t)(lane >> 1) : (uint32_t)lane * 4u / C;  // first cell of word `lane`
    const uint32_t js = (uint32_t)(lane & ~7) * 4u / C;                            // first cell of its sector
    const uint32_t v = splat_w<C>(param, lane);
    const uint64_t inv = lambda_lane_reciprocal(lane);
    // units come 1 << tshift per ticket (consecutive bands of one tile) when the queue is there
    uint32_t u = u_lo + warp, u_end = u + 1;
    if (wq != nullptr) {
        u = u_lo + (grab(wq, lane, 1u) << tshift);
        u_end = u + (1u << tshift);
    }
    for (;;) {
        if (u >= u_hi) break;
        const uint32_t tile = u >> G::LB;
        uint32_t X, Y;
        if constexpr (ROWMAJOR) tile_rows(tile, q, lane, X, Y);
        else lambda_lanes(tile, q, lane, inv, X, Y);
        const uint32_t t0 = (u & ((1u << G::LB) - 1u)) * G::BAND;
        uint8_t* ptr = grid + ((int64_t)Y * G::TT + t0) * rowstride + (int64_t)X * 128 + lane * 4;
#pragma unroll 4
        for (int i = 0; i < G::BAND; ++i, ptr += rowstride) {
            const uint32_t t = t0 + i;
            if constexpr (ZERO) {
                // whole 32-byte sectors (8 lanes) of the touched sectors
                if (js & ~t) continue;
                *reinterpret_cast<uint32_t*>(ptr) = v & word_mask<C>(lane >> 2, lane & 3, t);
            } else {
                if (j & ~t) continue;
                if constexpr (COUNT) {
                    atomicAdd(reinterpret_cast<unsigned int*>(ptr), 1u);  // coverage audit: 4-byte counters
                } else {
                    st_members<C>(ptr, v, t);
                }
            }
        }
        if (wq != nullptr) {
            if (++u == u_end) {
                u = u_lo + (grab(wq, lane, 1u) << tshift);
                u_end = u + (1u << tshift);
            }
        } else {
            u += nwarps;
        }
    }
    retire(wq, lane, nwarps);
}

// GM_FLAG_GRID_ROWS: one warp per grid row y (bottom row first: the heaviest rows
// start first), the row's 2^popc(Y) member lines left to right.  Zero background:
// 16-byte lanes, 4 lines per instruction -- lane group g owns the lines whose index k
// has low bits g: X = pdep(g, the two lowest bits of Y) | S, S over the subsets of Y's
// other bits in increasing order.  General: 4-byte lanes, one line per instruction.
template <int C, bool ZERO, int GRAN, bool COUNT = false>
__global__ void __launch_bounds__(256) gasket_write_rows(uint8_t* __restrict__ grid, int64_t n, uint64_t param,
                                                         uint32_t* __restrict__ wq) {
    using G = WGeo<C>;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int64_t rowstride = n * C;
    constexpr uint32_t RPT = 4;  // rows per ticket
    uint32_t yy = warp, yy_end = yy + 1;
    if (wq != nullptr) {
        yy = grab(wq, lane, 1u) * RPT;
        yy_end = yy + RPT;
    }
    auto advance = [&] {
        if (wq == nullptr) {
            yy += nwarps;
        } else if (++yy == yy_end) {
            yy = grab(wq, lane, 1u) * RPT;
            yy_end = yy + RPT;
        }
    };
    for (; yy < (uint32_t)n; advance()) {
        const uint32_t y = (uint32_t)n - 1u - yy;
        const uint32_t Y = y >> G::LT, t = y & (G::TT - 1);
        if constexpr (!ZERO) {
            const uint32_t j = C == 8 ? (uint32_t)(lane >> 1) : (uint32_t)lane * 4u / C;
            if (j & ~t) continue;
            const uint32_t v = splat_w<C>(param, lane);
            uint8_t* row = grid + (int64_t)y * rowstride + lane * 4;
            uint32_t X = 0;
            do {
                if constexpr (COUNT) atomicAdd(reinterpret_cast<unsigned int*>(row + (int64_t)X * 128), 1u);
                else st_members<C>(row + (int64_t)X * 128, v, t);
                X = (X - Y) & Y;
            } while (X != 0);
        } else if constexpr (GRAN == 3) {
            // 32-byte lanes (one sector each, 256-bit stores): 8 lines per instruction
            const int p = lane & 3;
            const uint32_t g = (uint32_t)(lane >> 2);
            const int lb = min(__popc(Y), 3);
            if (g >= (1u << lb)) continue;
            if (((uint32_t)p * (32u / C)) & ~t) continue;  // sector without gasket cells
            uint32_t rem = Y, base = 0;
            for (int i = 0; i < lb; ++i) {
                const uint32_t b = rem & (0u - rem);
                rem ^= b;
                if ((g >> i) & 1u) base |= b;
            }
            uint32_t v[8];
#pragma unroll
            for (int w = 0; w < 8; ++w) v[w] = splat_w<C>(param, w) & word_mask<C>(2 * p + (w >> 2), w & 3, t);
            uint8_t* row = grid + (int64_t)y * rowstride + p * 32;
            uint32_t S = 0;
            do {
                st_v8(row + (int64_t)(base | S) * 128, v);
                S = (S - rem) & rem;
            } while (S != 0);
        } else {
            const int p = lane & 7;
            const uint32_t g = (uint32_t)(lane >> 3);
            const int pc = __popc(Y);
            if (g >= (1u << (pc < 2 ? pc : 2))) continue;
            // store granularity: GRAN 0 = the touched 32-byte sectors, 1 = the touched
            // 64-byte halves, 2 = whole lines (zeros included)
            if constexpr (GRAN == 0) {
                if ((((uint32_t)(p & ~1) * G::P16) & ~t) != 0) continue;
            } else if constexpr (GRAN == 1) {
                if ((((uint32_t)(p & ~3) * G::P16) & ~t) != 0) continue;
            }
            const uint32_t b0 = Y & (0u - Y), Y1 = Y ^ b0, b1 = Y1 & (0u - Y1), Yh = Y1 ^ b1;
            const uint32_t base = ((g & 1u) ? b0 : 0u) | ((g & 2u) ? b1 : 0u);
            uint32_t v[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) v[w] = splat_w<C>(param, w) & word_mask<C>(p, w, t);
            uint8_t* row = grid + (int64_t)y * rowstride + p * 16;
            uint32_t S = 0;
            do {
                st_v4(row + (int64_t)(base | S) * 128, v[0], v[1], v[2], v[3]);
                S = (S - Yh) & Yh;
            } while (S != 0);
        }
    }
    retire(wq, lane, nwarps);
}

// GM_FLAG_WRITE_SWEEP: the grid rows' member lines in ADDRESS order, cut into work units of
// up to KS consecutive member lines of one row and dealt round-robin over all warps, so
// the warps in flight together write one contiguous stretch of the grid (a sweep from
// the top row down) instead of one far-apart row each.  Unit u -> (block row Y, row t,
// chunk j) by a binary search in the per-block-row unit prefix (nY + 1 entries, built
// once per size).  Zero background: 16-byte lanes, 4 lines per instruction, the touched
// sectors; general: 4-byte lanes, one line per instruction, the gasket cells.
constexpr int KS = 32;  // member lines per unit

template <int C, bool ZERO>
__global__ void __launch_bounds__(256) gasket_write_sweep(uint8_t* __restrict__ grid, int64_t n,
                                                          const uint32_t* __restrict__ prefix, uint32_t nY,
                                                          uint64_t param) {
    using G = WGeo<C>;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const int64_t rowstride = n * C;
    const uint32_t total = __ldg(prefix + nY);
    for (uint32_t u = warp; u < total; u += nwarps) {
        uint32_t lo = 0, hi = nY;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid;
        }
        const uint32_t Y = lo;
        const int pc = __popc(Y);
        const uint32_t chunks = pc > 5 ? 1u << (pc - 5) : 1u;
        const uint32_t rem = u - __ldg(prefix + Y);
        const uint32_t t = rem / chunks, j = rem - t * chunks;
        const int64_t y = (int64_t)Y * G::TT + t;
        if constexpr (ZERO) {
            const int p = lane & 7;
            const uint32_t g = (uint32_t)(lane >> 3);
            if (g >= (1u << (pc < 2 ? pc : 2))) continue;
            if ((((uint32_t)(p & ~1) * G::P16) & ~t) != 0) continue;  // sector without gasket cells
            const uint32_t b0 = Y & (0u - Y), Y1 = Y ^ b0, b1 = Y1 & (0u - Y1), Yh = Y1 ^ b1;
            const uint32_t base = ((g & 1u) ? b0 : 0u) | ((g & 2u) ? b1 : 0u);
            uint32_t v[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) v[w] = splat_w<C>(param, w) & word_mask<C>(p, w, t);
            uint8_t* row = grid + y * rowstride + p * 16;
            // lines 32j .. 32j+31 of the row: groups of 4 = subsets S of Yh from pdep(8j, Yh)
            uint32_t S = 0, m = 8u * j, bits = Yh;
            while (m) {
                const uint32_t low = bits & (0u - bits);
                if (m & 1u) S |= low;
                m >>= 1;
                bits ^= low;
            }
#pragma unroll 8
            for (int i = 0; i < KS / 4; ++i) {
                st_v4(row + (int64_t)(base | S) * 128, v[0], v[1], v[2], v[3]);
                S = (S - Yh) & Yh;
                if (S == 0) break;
            }
        } else {
            const uint32_t jc = C == 8 ? (uint32_t)(lane >> 1) : (uint32_t)lane * 4u / C;
            if (jc & ~t) continue;
            const uint32_t v = splat_w<C>(param, lane);
            uint8_t* row = grid + y * rowstride + lane * 4;
            uint32_t X = 0, m = KS * j, bits = Y;
            while (m) {
                const uint32_t low = bits & (0u - bits);
                if (m & 1u) X |= low;
                m >>= 1;
                bits ^= low;
            }
#pragma unroll 4
            for (int i = 0; i < KS; ++i) {
                st_members<C>(row + (int64_t)X * 128, v, t);
                X = (X - Y) & Y;
                if (X == 0) break;
            }
        }
    }
}

std::mutex g_sweep_mu;
std::map<std::pair<int, int>, uint32_t*> g_sweep_prefix;  // (device, log2 nY * 256 + TT) -> prefix

// units per block row Y: TT rows x max(1, 2^popc(Y) / KS) chunks
const uint32_t* sweep_prefix(int nYbits, int tt) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_sweep_mu);
    const std::pair<int, int> key{dev, nYbits * 256 + tt};
    auto it = g_sweep_prefix.find(key);
    if (it != g_sweep_prefix.end()) return it->second;
    const uint32_t nY = 1u << nYbits;
    std::vector<uint32_t> pre(nY + 1, 0);
    for (uint32_t Y = 0; Y < nY; ++Y) {
        const int pc = __builtin_popcount(Y);
        pre[Y + 1] = pre[Y] + (uint32_t)tt * (pc > 5 ? 1u << (pc - 5) : 1u);
    }
    uint32_t* d = nullptr;
    if (cudaMalloc(&d, pre.size() * sizeof(uint32_t)) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, pre.data(), pre.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    g_sweep_prefix[key] = d;
    return d;
}

int rows_ctas_per_sm() {
    static int v = [] {
        const char* e = getenv("GASKET_WRITE_ROWS_CTAS");
        return e ? atoi(e) : 8;
    }();
    return v;
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// The bounding-box baseline written as well as the tuned lambda kernels (GM_MAP_BB_VEC,
// the write pass only): the bounding box's thread space -- every 16-byte segment of all
// n x n cells, one lane each, grid-stride -- with the same vectorised stores.  A lane
// tests its segment's cells with the paper's membership test x & (n-1-y) == 0
// (backends.py:151-156) and stores the gasket cells of each 4-byte word (one store per
// word, the row's in-word pattern), so it differs from the lambda kernels only in the
// n^2 / 16 segment tests of the bounding box.
template <int C>
__global__ void __launch_bounds__(256) bb_vec(uint8_t* __restrict__ grid, int64_t n, int seg_shift,
                                              uint64_t param) {
    constexpr uint32_t P16 = 16 / C;  // cells per segment
    const uint64_t total = (uint64_t)n << seg_shift;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t v[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) v[w] = splat_w<C>(param, w);
    for (uint64_t sidx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; sidx < total; sidx += stride) {
        const uint32_t y = (uint32_t)(sidx >> seg_shift);
        const uint32_t x0 = (uint32_t)(sidx & ((1ull << seg_shift) - 1)) * P16;
        const uint32_t m = (uint32_t)n - 1u - y;
        if ((x0 & m) != 0) continue;  // the segment's first cell decides its high bits
        uint8_t* q = grid + (int64_t)y * n * C + (int64_t)x0 * C;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const uint32_t xw = C == 8 ? x0 + (uint32_t)(w >> 1) : x0 + (uint32_t)w * (4u / C);
            if (xw & m) continue;  // no gasket cell in this word
            st_members<C>(q + 4 * w, v[w], y);
        }
    }
}

cudaError_t launch_bb_vec(const LaunchArgs& a) {
    if (a.kind != KIND_CONST) return cudaErrorNotSupported;
    if (a.n < 1 || (a.n & (a.n - 1)) != 0 || a.n * a.cell_bytes < 16) return cudaErrorNotSupported;
    int seg_shift = 0;
    while ((int64_t(1) << seg_shift) < a.n * a.cell_bytes / 16) ++seg_shift;
    const unsigned blocks = (unsigned)sm_count() * 8u;
    uint8_t* g = reinterpret_cast<uint8_t*>(a.grid);
    switch (a.cell_bytes) {
    case 1: bb_vec<1><<<blocks, 256, 0, a.stream>>>(g, a.n, seg_shift, a.param); break;
    case 2: bb_vec<2><<<blocks, 256, 0, a.stream>>>(g, a.n, seg_shift, a.param); break;
    case 4: bb_vec<4><<<blocks, 256, 0, a.stream>>>(g, a.n, seg_shift, a.param); break;
    case 8: bb_vec<8><<<blocks, 256, 0, a.stream>>>(g, a.n, seg_shift, a.param); break;
    default: return cudaErrorNotSupported;
    }
    note_launch();
    return cudaGetLastError();
}


// units per ticket of the lambda-tile write pass (log2): one band per ticket -- concurrently
// running warps then hold consecutive bands of a tile (n=2^16 int8 back to back: 107.7 us,
// 109.1 with two bands, 109.8 with a whole tile per ticket, 115.1 static; A/B knob
// GASKET_WRITE_TICKET_SHIFT)
template <class G>
int ticket_shift() {
    static const int v = [] {
        const char* e = getenv("GASKET_WRITE_TICKET_SHIFT");
        return e ? atoi(e) : 0;
    }();
    return v < 0 ? 0 : (v > G::LB ? G::LB : v);
}

std::mutex g_wq_mu;
std::map<std::pair<int, cudaStream_t>, uint32_t*> g_wq;

// The ticket counters of the dynamic schedule, one pair per (device, stream) so launches
// on different streams never share one; nullptr (the static schedule) while a stream is
// being captured before its pair exists, or if allocation fails.
uint32_t* work_queue(cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_wq_mu);
    auto it = g_wq.find({dev, s});
    if (it != g_wq.end()) return it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return nullptr;
    }
    uint32_t* q = nullptr;
    if (cudaMalloc(&q, 2 * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (cudaMemset(q, 0, 2 * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(q);
        return nullptr;
    }
    g_wq[{dev, s}] = q;
    return q;
}

template <int C, bool ZERO, bool COUNT = false>
cudaError_t launch_c(const LaunchArgs& a, int q) {
    using G = WGeo<C>;
    // zero background: the grid-row schedule unless lambda tiles (GM_FLAG_DIGIT_ORDER), row-major
    // tiles or the address sweep are asked for (n=2^16 int8: 55.7 us vs 62-64 us for lambda tiles)
    // (4- and 8-byte cells: the address sweep, 140 vs 154 us back to back at n=2^16 int32)
    const bool zero_default = ZERO && !(a.flags & (GM_FLAG_DIGIT_ORDER | GM_FLAG_ROWMAJOR | GM_FLAG_WRITE_SWEEP |
                                                   GM_FLAG_GRID_ROWS));
    const bool rows = (a.flags & GM_FLAG_GRID_ROWS) || (zero_default && (C < 4 || q > 13));
    if (rows && a.part_level < 0) {
        // 8 CTAs of 256 threads per SM (the row walk wants many rows in flight)
        const uint64_t blocks = std::min<uint64_t>((uint64_t)sm_count() * rows_ctas_per_sm(), ((uint64_t)a.n * 32 + 255) / 256);
        const int gran = (a.flags & GM_FLAG_WRITE_LINES) && (a.flags & GM_FLAG_WRITE_HALVES) ? 3
                         : (a.flags & GM_FLAG_WRITE_LINES)                                ? 2
                         : (a.flags & GM_FLAG_WRITE_HALVES)                               ? 1
                                                                                          : 0;
        auto* kr = !ZERO || gran == 0 ? gasket_write_rows<C, ZERO, 0, COUNT>
                   : gran == 1        ? gasket_write_rows<C, ZERO, 1, COUNT>
                   : gran == 2        ? gasket_write_rows<C, ZERO, 2, COUNT>
                                      : gasket_write_rows<C, ZERO, 3, COUNT>;
        // (zero background: the static schedule -- 55 vs 75 us with tickets at n=2^16 int8)
        uint32_t* wq = (ZERO || (a.flags & GM_FLAG_STATIC_SCHEDULE)) ? nullptr : work_queue(a.stream);
        kr<<<(unsigned)blocks, 256, 0, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid), a.n, a.param, wq);
        note_launch();
        return cudaGetLastError();
    }
    if (((a.flags & GM_FLAG_WRITE_SWEEP) || (zero_default && C >= 4)) && a.part_level < 0 && !COUNT && q <= 13) {
        const uint32_t* pre = sweep_prefix(q, G::TT);
        if (!pre) return cudaErrorMemoryAllocation;
        const unsigned blocks = (unsigned)sm_count() * (unsigned)rows_ctas_per_sm();
        gasket_write_sweep<C, ZERO><<<blocks, 256, 0, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid), a.n, pre,
                                                                 1u << q, a.param);
        note_launch();
        return cudaGetLastError();
    }
    uint32_t lo, hi;
    tile_range(a, q, lo, hi);  // member tiles (digit order; partitioned launches: a sub-gasket range)
    if (hi == lo) return cudaSuccess;
    const uint64_t u_lo = (uint64_t)lo << G::LB, u_hi = (uint64_t)hi << G::LB;
    if (u_hi > 0xffffffffull) return cudaErrorNotSupported;
    const bool rowmajor = (a.flags & GM_FLAG_ROWMAJOR) && a.part_level < 0;
    auto* kern = rowmajor ? gasket_write<C, ZERO, true, COUNT> : gasket_write<C, ZERO, false, COUNT>;
    // one CTA of 8 warps per SM: fewer stores in flight keep the DRAM write stream on
    // fewer pages at a time (n=2^16 int8 zero background, back to back: 59.6 us vs 71.6
    // with 2-8 CTAs per SM; general: 114.6 vs 117.3; scripts/write_ab.py)
    const uint64_t blocks = std::min<uint64_t>((uint64_t)sm_count(), ((u_hi - u_lo) * 32 + 255) / 256);
    // tickets for the general store mode (n=2^16 int8 107.7 vs 115.1 us back to back, 2^17 314 vs 334);
    // the zero-background pass keeps the static round-robin (60.5 vs 78 us with tickets)
    uint32_t* wq = (ZERO || (a.flags & GM_FLAG_STATIC_SCHEDULE)) ? nullptr : work_queue(a.stream);
    kern<<<(unsigned)blocks, 256, 0, a.stream>>>(reinterpret_cast<uint8_t*>(a.grid), a.n, q, (uint32_t)u_lo,
                                                 (uint32_t)u_hi, a.param, wq, ticket_shift<G>());
    note_launch();
    return cudaGetLastError();
}

template <int C>
cudaError_t launch_cb(const LaunchArgs& a, int q) {
    return (a.flags & GM_FLAG_ZERO_BACKGROUND) ? launch_c<C, true>(a, q) : launch_c<C, false>(a, q);
}

}  // namespace

cudaError_t launch_bb_vector(const LaunchArgs& a) { return launch_bb_vec(a); }

// The CONST pass on grids at least one 128-byte line wide (up to 3^20 tiles);
// cudaErrorNotSupported otherwise (the caller then uses the generic kernels).
// KIND_COUNT (the coverage audit, engine.py:214-258) runs the same schedule with an
// atomic increment of a 4-byte counter per gasket cell.
cudaError_t launch_write(const LaunchArgs& a) {
    if ((a.kind != KIND_CONST && a.kind != KIND_COUNT) || (a.flags & GM_FLAG_OMEGA_ORDER)) return cudaErrorNotSupported;
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    const int lt = a.cell_bytes == 1 ? 7 : a.cell_bytes == 2 ? 6 : a.cell_bytes == 4 ? 5 : 4;  // log2 TT
    if (r < lt || r - lt > 20) return cudaErrorNotSupported;
    const int q = r - lt;
    if (a.kind == KIND_COUNT) return a.cell_bytes == 4 ? launch_c<4, false, true>(a, q) : cudaErrorNotSupported;
    switch (a.cell_bytes) {
    case 1: return launch_cb<1>(a, q);
    case 2: return launch_cb<2>(a, q);
    case 4: return launch_cb<4>(a, q);
    case 8: return launch_cb<8>(a, q);
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
