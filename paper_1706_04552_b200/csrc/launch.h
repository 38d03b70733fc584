// launch.h -- internal launch descriptors shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace gm {

struct LaunchArgs {
    void* grid;            // device (or mapped host) pointer, n*n cells of cell_bytes
    const void* src;       // pre-launch snapshot (may equal grid only for CONST)
    int64_t n;             // grid edge
    int rho;               // block edge
    int r_b;               // block-scale level
    int64_t width, height; // packing_dims(r_b)
    int mapping;           // gm::Mapping
    int strategy;          // gm::Strategy
    int kind;              // gm::Kind
    int cell_bytes;        // 1, 2, 4, 8
    uint64_t param;        // int32 param sign-extended to 64 bits
    const int32_t* tab_x;  // TABLE strategy lookup table (device)
    const int32_t* tab_y;
    int ntab;
    int flags;             // GM_FLAG_* (see include/gasket_b200.h)
    cudaStream_t stream;
    // partitioned launches (tuned kernels only): restrict to level-part_level
    // sub-gaskets [sg_begin, sg_end) in digit order; part_level < 0 = whole gasket
    int part_level = -1;
    uint32_t sg_begin = 0, sg_end = 0;
    // fused peer halo exchange (gm_run_part_peer, peer_epilogue.cuh): device descriptor,
    // the peers' epoch to wait for before reading, the epoch to signal after writing
    void* peer_epi = nullptr;
    uint64_t wait_epoch = 0, signal_epoch = 0;
    // tiled partition storage (gm_run_part_tiled): the rank's sub-gaskets [sg_begin, sg_end)
    // each in its own ringed block; sg_off[k] = byte offset from grid / src to the virtual
    // origin of sub-gasket sg_begin + k (where global cell (0, 0) would sit), pitch = row
    // bytes of those blocks.  nullptr = the dense n x n layout (pitch n * cell_bytes).
    const int64_t* sg_off = nullptr;
    int64_t pitch = 0;
    // static left-edge cache of a CA run (gm_ca_edge_build, edge.cu): for tile #i of the
    // launch's tile range whose left neighbour tile is not a gasket tile, the 16-byte chunk
    // left of each of its TT rows at edge + (i * TT + row) * 16; nullptr = read the grid
    const uint8_t* edge = nullptr;
    // in-place neighbour-sum launch (src == grid): the pre-launch border cells of every
    // member tile (launch_border_snapshot, edge.cu); the tuned stencil patches its staged
    // window from there.  nullptr = src is a separate pre-launch state.
    const uint8_t* border = nullptr;
    // an explicit tile range [range_lo, range_hi) of the whole-grid row-major tile order
    // (contiguous block rows; the banded staged host path) -- used when range_hi > range_lo
    uint32_t range_lo = 0, range_hi = 0;
};

// The left neighbour of member tile (bx, by) holds no gasket cell (so its cells never
// change in a CA run: backends.py:155-156) and lies inside the grid.
__host__ __device__ inline bool left_static(uint32_t bx, uint32_t by) {
    return bx > 0 && ((bx - 1) & ~by) != 0;
}

// row pitch in bytes of a launch's buffers
inline int64_t row_pitch(const LaunchArgs& a) { return a.pitch > 0 ? a.pitch : a.n * a.cell_bytes; }

// tiles per sub-gasket of a partitioned launch tiled at level r_t (3^(r_t - part_level))
inline uint32_t tiles_per_subgasket(const LaunchArgs& a, int r_t) {
    uint32_t per = 1;
    if (a.part_level >= 0)
        for (int i = 0; i < r_t - a.part_level; ++i) per *= 3u;
    return per;
}

// Tile-index range [lo, hi) of a launch whose kernel tiles the gasket at level r_t.
inline void tile_range(const LaunchArgs& a, int r_t, uint32_t& lo, uint32_t& hi) {
    uint32_t all = 1;
    for (int i = 0; i < r_t; ++i) all *= 3u;
    if (a.range_hi > a.range_lo) {
        hi = a.range_hi < all ? a.range_hi : all;
        lo = a.range_lo < hi ? a.range_lo : hi;
        return;
    }
    if (a.part_level < 0 || a.part_level > r_t) { lo = 0; hi = all; return; }
    uint32_t per = 1;
    for (int i = 0; i < r_t - a.part_level; ++i) per *= 3u;
    lo = a.sg_begin * per;
    hi = a.sg_end * per;
    if (hi > all) hi = all;
    if (lo > hi) lo = hi;
}

void note_launch();

// cudaFuncAttributeMaxDynamicSharedMemorySize for `kern` on the current device, set once
// per (kernel, device) -- the attribute is per device context (capi.cu)
void ensure_dynamic_smem(const void* kern, size_t smem);

// Sub-gasket level whose groups the row-major tile order keeps together: the partition
// level for partitioned launches (their tile ranges are digit-order sub-gasket ranges),
// else 0 (one row-major sweep) -- or GASKET_TILE_ORDER_LEVEL for experiments.
int order_level(const LaunchArgs& a, int r_t);

cudaError_t launch_literal(const LaunchArgs& a);
cudaError_t launch_tuned(const LaunchArgs& a);
cudaError_t launch_stream(const LaunchArgs& a);
cudaError_t launch_write(const LaunchArgs& a);
cudaError_t launch_bb_vector(const LaunchArgs& a);  // GM_MAP_BB_VEC (write.cu)
cudaError_t launch_stencil_tile(const LaunchArgs& a);
cudaError_t launch_host_rows(const LaunchArgs& a);
cudaError_t launch_stencil_tma(const LaunchArgs& a);
cudaError_t launch_stencil_v2(const LaunchArgs& a);
cudaError_t launch_stencil_tb2(const LaunchArgs& a);
cudaError_t launch_stencil_tb(const LaunchArgs& a, int steps);  // steps = 2, 4 or 6
cudaError_t launch_edge_build(const LaunchArgs& a, uint8_t* edge);  // edge.cu
int64_t edge_cache_bytes(const LaunchArgs& a);                   // edge.cu (0: no tiled kernel)
int64_t border_bytes(int64_t n, int cell_bytes);                  // edge.cu
cudaError_t launch_border_snapshot(uint8_t* border, const void* grid, int64_t n, int cell_bytes, cudaStream_t s);
// (t0, t1): a tile range of the whole-grid row-major order; t1 == 0: every member tile
cudaError_t launch_snapshot_stencil(void* snap, const void* grid, int64_t n, int cell_bytes, cudaStream_t s,
                                    uint32_t t0 = 0, uint32_t t1 = 0);
cudaError_t launch_writeback_tiles(void* out, const void* dst, const void* snap, int64_t n, int cell_bytes, cudaStream_t s,
                                   uint32_t t0 = 0, uint32_t t1 = 0);
cudaError_t launch_host_rows_copyback(void* out, const void* dst, const void* snap, int64_t n, int cell_bytes,
                                      cudaStream_t s);
// member tiles of a level-q gasket, row-major inside each level-L sub-gasket (stencil2.cu)
const uint32_t* rowmajor_table(int q, int L);
void rowmajor_order_host(int q, int L, std::vector<uint32_t>& v);
cudaError_t launch_peer_put(const void* mine, const uint64_t* peers, const int64_t* idx, const int64_t* didx,
                            int64_t k, int cell_bytes,
                            const uint64_t* peer_flags, int rank, int world, uint64_t epoch, cudaStream_t s);
cudaError_t launch_peer_wait(const uint64_t* flags, int rank, int world, uint64_t epoch, uint64_t timeout_ns,
                             uint32_t* status, cudaStream_t s);

}  // namespace gm
