// launch.h -- internal launch descriptors shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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
};

void note_launch();

cudaError_t launch_literal(const LaunchArgs& a);
cudaError_t launch_tuned(const LaunchArgs& a);
cudaError_t launch_stream(const LaunchArgs& a);
cudaError_t launch_stencil_tile(const LaunchArgs& a);

}  // namespace gm
