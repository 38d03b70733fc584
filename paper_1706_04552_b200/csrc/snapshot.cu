// snapshot.cu -- the pre-launch snapshot of a neighbour-sum launch, masked.
//
// engine.launch takes `src = grid.copy()` before every NEIGHBOR_SUM launch
// (engine.py:201; a full n^2 copy, outside the reference's
// timer) so that the launch reads the pre-launch state while it writes gasket
// cells of `grid`.  Every stencil kernel here (literal, tuned, fused) reads `src`
// only at gasket cells, their 4/8 neighbours, and -- for whole-sector stores --
// the touched sectors of the gasket rows.  All of those lie in the window of some
// member tile: rows -1..TT of the tile (TT = 128/C cells, one 128-byte line per
// row) and one 32-byte sector either side.  So the snapshot copies exactly those
// windows, at their own positions, into a grid-sized buffer; the rest of the buffer
// is never read.  n = 2^17 int8: 59049 tiles x 130 rows x 192 B = 1.47 GB each way
// instead of 16 GiB each way.  Whole sectors only (no partial-sector RMW).
#include <cstdint>

#include "gasket.cuh"
#include "launch.h"

namespace gm {
namespace {

constexpr int WIN_BYTES = 32 + 128 + 32;  // left sector | the tile's line | right sector
constexpr int VEC_PER_ROW = WIN_BYTES / 16;

// 16 bytes, streaming; `half`: fetch only the 64-byte half of the line on an L2 miss
// (the halo sectors of a neighbouring line)
__device__ __forceinline__ uint4 ld16(const uint8_t* p, bool half) {
    uint4 v;
    if (half)
        asm volatile("ld.global.cs.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        v = __ldcs(reinterpret_cast<const uint4*>(p));
    return v;
}

// one warp per member tile (tiles row-major, grid-stride over all warps); each lane moves
// UNROLL 16-byte pieces per round with all its loads in flight before the stores
constexpr int UNROLL = 8;

// s64 != 0 (a host grid that starts s64 bytes past a 64-byte boundary, e.g. a plain numpy
// array): each window row is the three host-aligned 64-byte units covering [-16, 144)
// (PCIe reads whole units), so that the write-back can store whole host units too; pieces
// outside the array are skipped.
__global__ void __launch_bounds__(256) snapshot_tiles(uint8_t* __restrict__ snap, const uint8_t* __restrict__ grid,
                                                      int64_t n, int cell_bytes, const uint32_t* __restrict__ order,
                                                      uint32_t ntiles, uint32_t nb, int s64) {
    const int64_t rowbytes = n * cell_bytes;
    const int64_t total = rowbytes * n;
    const int tt = 128 / cell_bytes;  // tile rows (and cells per row)
    // pieces per window row and the first one relative to the tile's line: 64-byte aligned
    // grids take one 32-byte sector either side (what every stencil kernel may read); host
    // grids off a 64-byte boundary take the three host units (boundaries at grid offsets g
    // with (g + s64) % 64 == 0) covering bytes [-16, 144): the tuned stencil's halo chunks
    // and every byte the write-back of the tile's line stores (the staged path is the tuned
    // kernel's only) -- one unit per row fewer than covering the 32-byte sectors
    const int vpr = s64 ? 12 : VEC_PER_ROW;
    const int per_tile = (tt + 2) * vpr;
    const int64_t lead = s64 ? 16 + ((s64 - 16) & 63) : 32;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < ntiles; t += nwarps) {
        const uint32_t v = __ldg(order + t);
        const uint32_t bx = v & 0xffffu, by = v >> 16;
        // halo rows / sectors that a neighbouring member tile's window already covers are
        // skipped (tile (X, Y) is a member iff X & ~Y == 0, X, Y < nb)
        const bool up = by > 0 && (bx & ~(by - 1)) == 0;
        const bool down = by + 1 < nb && (bx & ~(by + 1)) == 0;
        const bool left = bx > 0 && ((bx - 1) & ~by) == 0;
        const bool right = bx + 1 < nb && ((bx + 1) & ~by) == 0;
        const int64_t line0 = (int64_t)bx * 128;    // the tile's line
        const int64_t xb0 = line0 - lead;            // window's first byte
        const int64_t y0 = (int64_t)by * tt - 1;     // window's first row
        for (int base = 0; base < per_tile; base += 32 * UNROLL) {
            uint4 val[UNROLL];
            int64_t off[UNROLL];
#pragma unroll
            for (int k = 0; k < UNROLL; ++k) {
                const int i = base + k * 32 + lane;
                const int row = i / vpr, q = i - row * vpr;
                const int64_t y = y0 + row, xb = xb0 + q * 16;
                const bool lpart = xb < line0, rpart = xb >= line0 + 128;
                // host units (s64 != 0): on the tile's own rows the unit shared with the right
                // neighbour's window (its first unit is this window's last) is read whole by
                // that neighbour when it is a member tile (it copies its own rows whole), and
                // this window's first unit whole by this tile; rows -1 and TT, copied here only
                // when the tile above / below is not a member, keep all three units
                const bool shared_right = s64 != 0 && q >= 8 && row >= 1 && row <= tt;
                // (64-byte aligned grids: the right sector is read by the gasket cells of tile
                // column TT-1 only, i.e. on window rows tt-1 .. tt+1; its host unit is the
                // right neighbour's, so on the other rows it is not fetched at all)
                bool skip = i >= per_tile || (row == 0 && up) || (row == tt + 1 && down) ||
                            (s64 == 0 ? ((lpart && left) || (rpart && (right || row < tt - 1)))
                                      : (shared_right && right)) ||
                            y < 0 || y >= n;
                if (s64 == 0) {
                    skip = skip || xb < 0 || xb >= rowbytes;
                } else {  // host units may run into the neighbouring rows: only the array's bytes
                    const int64_t f = y * rowbytes + xb;
                    skip = skip || f < 0 || f >= total;
                }
                off[k] = skip ? -1 : y * rowbytes + xb;
                if (!skip) val[k] = ld16(grid + off[k], lpart || rpart);
            }
#pragma unroll
            for (int k = 0; k < UNROLL; ++k)
                if (off[k] >= 0) *reinterpret_cast<uint4*>(snap + off[k]) = val[k];
        }
    }
}

// The write-back half of a staged launch on a host-mapped grid: every member tile's own
// rows (one 128-byte line each) go back whole -- the touched sectors from `dst` (the
// stencil's whole-sector results), the other sectors from `snap` (the pre-launch state)
// -- so the host sees whole-line writes only.
// s64 != 0 (host grid s64 bytes past a 64-byte boundary): each line goes back as the
// host-aligned 64-byte units that cover it (12 pieces; the bytes of the neighbouring
// lines they include come, by the same rule, from `dst` or `snap`, whose host-aligned
// windows hold them; two tiles may store the same unit with the same bytes).
__global__ void __launch_bounds__(256) writeback_tiles(uint8_t* __restrict__ out, const uint8_t* __restrict__ dst,
                                                       const uint8_t* __restrict__ snap, int64_t n, int cell_bytes,
                                                       const uint32_t* __restrict__ order, uint32_t ntiles, int s64) {
    const int64_t rowbytes = n * cell_bytes;
    const int64_t total = rowbytes * n;
    const int tt = 128 / cell_bytes;
    const int sc = 32 / cell_bytes;  // cells per sector
    const int vpr = s64 ? 12 : 8;    // pieces per line (host units covering it)
    const int per_tile = tt * vpr;   // 16-byte pieces of the tile's own lines
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = warp; t < ntiles; t += nwarps) {
        const uint32_t v = __ldg(order + t);
        const int64_t xb0 = (int64_t)(v & 0xffffu) * 128, y0 = (int64_t)(v >> 16) * tt;
        for (int base = 0; base < per_tile; base += 32 * UNROLL) {
            uint4 val[UNROLL];
            int64_t off[UNROLL];
#pragma unroll
            for (int k = 0; k < UNROLL; ++k) {
                const int i = base + k * 32 + lane;
                if (s64 == 0) {
                    const int row = i >> 3, q = i & 7;
                    off[k] = i < per_tile ? (y0 + row) * rowbytes + xb0 + q * 16 : -1;
                    if (off[k] >= 0) {
                        const bool touched = (((q >> 1) * sc) & ~row) == 0;  // sector holds gasket cells
                        val[k] = __ldcs(reinterpret_cast<const uint4*>((touched ? dst : snap) + off[k]));
                    }
                } else {
                    const int row = i / vpr, q = i - row * vpr;
                    const int64_t f = (y0 + row) * rowbytes + xb0 - s64 + q * 16;
                    // the last unit is also the right neighbour's first: a member neighbour
                    // stores it (whole, with this line's bytes from dst / snap by the same rule)
                    const bool shared = q >= 8 && (int64_t)((v & 0xffffu) + 1) * 128 < rowbytes &
                                                      (((v & 0xffffu) + 1) & ~(v >> 16)) == 0;
                    off[k] = (i < per_tile && f >= 0 && f < total && !shared) ? f : -1;
                    if (off[k] >= 0) {
                        // the piece's own row, line and sector decide where its bytes come from
                        const int64_t yy = f / rowbytes, col = f - yy * rowbytes;
                        const int64_t X = col >> 7, Yb = yy / tt, t = yy - Yb * tt;
                        const int g = (int)((col & 127) >> 5);
                        const bool touched = (X & ~Yb) == 0 && (((int64_t)g * sc) & ~t) == 0;
                        val[k] = __ldcs(reinterpret_cast<const uint4*>((touched ? dst : snap) + off[k]));
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < UNROLL; ++k)
                if (off[k] >= 0) *reinterpret_cast<uint4*>(out + off[k]) = val[k];
        }
    }
}

}  // namespace

cudaError_t launch_writeback_tiles(void* out, const void* dst, const void* snap, int64_t n, int cell_bytes,
                                   cudaStream_t s, uint32_t t0, uint32_t t1) {
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4 && cell_bytes != 8) return cudaErrorNotSupported;
    const int64_t tt = 128 / cell_bytes;
    if (n < tt || (n & (n - 1)) != 0) return cudaErrorNotSupported;
    int r_t = 0;
    while ((tt << r_t) < n) ++r_t;
    const uint32_t* order = rowmajor_table(r_t, 0);
    if (order == nullptr) return cudaErrorNotSupported;
    uint32_t ntiles = 1;
    for (int i = 0; i < r_t; ++i) ntiles *= 3u;
    if (t1 > 0) {  // a range of the row-major order
        if (t1 > ntiles || t0 >= t1) return t0 == t1 ? cudaSuccess : cudaErrorInvalidValue;
        order += t0;
        ntiles = t1 - t0;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t blocks = (uint32_t)sms * 8u;
    if (blocks > (ntiles + 7) / 8) blocks = (ntiles + 7) / 8;
    const int s64 = (int)(reinterpret_cast<uintptr_t>(out) & 63u);
    if (s64 % 16 != 0) return cudaErrorNotSupported;  // (numpy data is at least 16-byte aligned)
    writeback_tiles<<<blocks, 256, 0, s>>>(reinterpret_cast<uint8_t*>(out), reinterpret_cast<const uint8_t*>(dst),
                                           reinterpret_cast<const uint8_t*>(snap), n, cell_bytes, order, ntiles, s64);
    note_launch();
    return cudaGetLastError();
}

// cudaErrorNotSupported: cell widths other than 1/2/4/8, grids narrower than a tile or
// with more than 2^15 tiles per edge (the caller then copies the whole grid).
cudaError_t launch_snapshot_stencil(void* snap, const void* grid, int64_t n, int cell_bytes, cudaStream_t s,
                                    uint32_t t0, uint32_t t1) {
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4 && cell_bytes != 8) return cudaErrorNotSupported;
    const int64_t tt = 128 / cell_bytes;
    if (n < tt || (n & (n - 1)) != 0) return cudaErrorNotSupported;
    int r_t = 0;
    while ((tt << r_t) < n) ++r_t;
    const uint32_t* order = rowmajor_table(r_t, 0);  // neighbouring tiles together: shared halo lines hit L2
    if (order == nullptr) return cudaErrorNotSupported;
    uint32_t ntiles = 1;
    for (int i = 0; i < r_t; ++i) ntiles *= 3u;
    if (t1 > 0) {  // a range of the row-major order
        if (t1 > ntiles || t0 >= t1) return t0 == t1 ? cudaSuccess : cudaErrorInvalidValue;
        order += t0;
        ntiles = t1 - t0;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t blocks = (uint32_t)sms * 8u;  // 64 warps per SM, a tile each
    if (blocks > (ntiles + 7) / 8) blocks = (ntiles + 7) / 8;
    // a grid that is not 64-byte aligned (a host numpy array) is read in host-aligned units
    const int s64 = (int)(reinterpret_cast<uintptr_t>(grid) & 63u);
    if (s64 % 16 != 0) return cudaErrorNotSupported;
    snapshot_tiles<<<blocks, 256, 0, s>>>(reinterpret_cast<uint8_t*>(snap), reinterpret_cast<const uint8_t*>(grid), n,
                                          cell_bytes, order, ntiles, 1u << r_t, s64);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gm
