// edge.cu -- the static left-edge cache of a CA run (gm_ca_edge_build, gm_ca_run).
//
// Why.  The tuned stencil kernels stage, for every member tile (X, Y), the 16-byte
// chunk left of each of its rows (the cells x0-16/C .. x0-1 its column-0 cells read).
// When the left neighbour tile (X-1, Y) is not a gasket tile (X-1 not a bit-subset of
// Y: about half of the member tiles), that chunk is the only part of its 128-byte line
// anyone reads, so every such row costs a whole sparse DRAM line fetch for one cell:
// at n=2^17 int8 that is 3.7 M of the 11.3 M lines an 8-neighbour step reads.
//
// Those cells are off-gasket, and a CA run never changes off-gasket cells (only gasket
// cells are written, backends.py:155-156; both ping-pong buffers agree off the gasket,
// the DST_FROM_SRC invariant of ca.py).  So they are gathered once per run into a dense
// array -- tile by tile in the kernels' visiting order, 16 bytes per tile row -- and
// every step stages them from there: 2 KB of contiguous bytes per tile instead of 128
// sparse lines.  Results are unchanged by construction (the same bytes land in the same
// shared-memory slots); rows -1 and TT of the staged window still come from the grid,
// since the tiles above-left and below-left may be gasket tiles.  n=2^17 int8, one step:
// NSUM8 436 -> 406 us, NSUM4 431 -> 397 us with the same 3-deep staging ring; the lighter
// staging then lets a 2-deep ring with 4 CTAs per SM win: 378 / 368 us (stencil2.cu).  (The
// fused 2/4/6-step kernel, bound by its arithmetic, gained nothing and does not use it.)
#include <algorithm>

#include "launch.h"

// ---------------------------------------------------------------------------
// The in-place neighbour-sum launch (engine.launch semantics, engine.py:201, without a
// grid-sized snapshot).  Every CTA stages its tile's window before it writes the tile, so
// a tile only needs pre-launch values of the cells it reads from OTHER tiles that can
// change, i.e. gasket cells of neighbouring tiles.  Tile cell (x, y) is a gasket cell iff
// x is a bit-subset of y, so those are at most 8 reader positions, all of them one of 5
// cells of their owner tile (tile coordinates, TT = tile edge):
//   slot 0 (0,0)   slot 1 (0,TT-2)   slot 2 (0,TT-1)   slot 3 (1,TT-1)   slot 4 (TT-1,TT-1)
// read at (-1,-1) [upper-left tile, slot 4], (0,-1) / (1,-1) [tile above, slots 2 / 3],
// (-1,TT-1) [left tile, slot 4], (0,TT) [tile below, slot 0], (TT,TT-2) / (TT,TT-1) [right
// tile, slots 1 / 2], (TT,TT) [lower-right tile, slot 0] -- the K6 corner set of SURVEY
// §8e at tile scale.  border_snapshot_kernel copies those 5 cells of every member tile
// into border[(by * ntx + bx) * 8 + slot]; the stencil kernel patches its staged window
// from there (stencil2.cu).  n=2^17 int8: 0.3 M cells instead of a 1.2 GB masked copy.
// ---------------------------------------------------------------------------

namespace gm {
namespace {

__global__ void __launch_bounds__(256) border_snapshot_kernel(uint8_t* __restrict__ border,
                                                              const uint8_t* __restrict__ grid, int64_t n, int c,
                                                              int lt, const uint32_t* __restrict__ order,
                                                              uint32_t ntiles) {
    const int tt = 1 << lt;
    const int64_t ntx = n >> lt;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < (uint64_t)ntiles * 5u;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(k / 5u), slot = (uint32_t)(k - (uint64_t)i * 5u);
        const uint32_t v = __ldg(order + i);
        const int64_t bx = v & 0xffffu, by = v >> 16;
        const int cx = slot == 3 ? 1 : slot == 4 ? tt - 1 : 0;
        const int cy = slot == 0 ? 0 : slot == 1 ? tt - 2 : tt - 1;
        const uint8_t* s = grid + ((by * tt + cy) * n + bx * tt + cx) * c;
        uint8_t* d = border + ((by * ntx + bx) * 8 + slot) * c;
        for (int b = 0; b < c; ++b) d[b] = s[b];
    }
}

__global__ void __launch_bounds__(256) edge_build_kernel(uint4* __restrict__ edge, const uint8_t* __restrict__ src,
                                                         const uint32_t* __restrict__ order, uint32_t ntiles, int lt,
                                                         const int64_t* __restrict__ sg_off, int64_t pitch,
                                                         uint32_t per) {
    const uint64_t total = (uint64_t)ntiles << lt;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(k >> lt), r = (uint32_t)(k & ((1u << lt) - 1u));
        const uint32_t v = __ldg(order + i);
        const uint32_t bx = v & 0xffffu, by = v >> 16;
        if (!left_static(bx, by)) continue;
        const int64_t off = sg_off != nullptr ? __ldg(sg_off + i / per) : 0;
        const uint8_t* p = src + off + ((int64_t)(by << lt) + r) * pitch + (int64_t)bx * 128 - 16;
        edge[k] = __ldcs(reinterpret_cast<const uint4*>(p));
    }
}

bool edge_geometry(const LaunchArgs& a, int& lt, int& r_t, uint32_t& lo, uint32_t& hi) {
    if (a.cell_bytes != 1 && a.cell_bytes != 2 && a.cell_bytes != 4) return false;
    lt = a.cell_bytes == 1 ? 7 : a.cell_bytes == 2 ? 6 : 5;  // log2 of the tile edge (one 128-byte line)
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    if (r < lt || r - lt > 15) return false;  // the row-major tile table's limit
    r_t = r - lt;
    tile_range(a, r_t, lo, hi);
    return true;
}

}  // namespace

int64_t edge_cache_bytes(const LaunchArgs& a) {
    int lt, r_t;
    uint32_t lo, hi;
    if (!edge_geometry(a, lt, r_t, lo, hi)) return 0;
    return ((int64_t)(hi - lo) << lt) * 16;
}

int64_t border_bytes(int64_t n, int cell_bytes) {
    const int lt = cell_bytes == 1 ? 7 : cell_bytes == 2 ? 6 : 5;
    const int64_t ntx = n >> lt;
    return ntx * ntx * 8 * cell_bytes;
}

cudaError_t launch_border_snapshot(uint8_t* border, const void* grid, int64_t n, int cell_bytes, cudaStream_t s) {
    LaunchArgs a{};
    a.n = n;
    a.cell_bytes = cell_bytes;
    int lt, r_t;
    uint32_t lo, hi;
    if (!edge_geometry(a, lt, r_t, lo, hi)) return cudaErrorNotSupported;
    const uint32_t* order = rowmajor_table(r_t, 0);
    if (order == nullptr) return cudaErrorMemoryAllocation;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t work = (uint64_t)(hi - lo) * 5u;
    const unsigned blocks = (unsigned)std::min<uint64_t>((uint64_t)sms * 8u, (work + 255) / 256);
    border_snapshot_kernel<<<blocks, 256, 0, s>>>(border, reinterpret_cast<const uint8_t*>(grid), n, cell_bytes, lt,
                                                  order, hi - lo);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_edge_build(const LaunchArgs& a, uint8_t* edge) {
    int lt, r_t;
    uint32_t lo, hi;
    if (!edge_geometry(a, lt, r_t, lo, hi)) return cudaErrorNotSupported;
    if (hi == lo) return cudaSuccess;
    const uint32_t* order = rowmajor_table(r_t, order_level(a, r_t));
    if (order == nullptr) return cudaErrorMemoryAllocation;
    uint32_t per = 1;
    if (a.part_level >= 0)
        for (int i = 0; i < r_t - a.part_level; ++i) per *= 3u;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    edge_build_kernel<<<(unsigned)sms * 8u, 256, 0, a.stream>>>(reinterpret_cast<uint4*>(edge),
                                                                 reinterpret_cast<const uint8_t*>(a.src), order + lo,
                                                                 hi - lo, lt, a.sg_off, row_pitch(a), per);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gm
