// probe_stride.cu -- design probe: DRAM efficiency of tile-column (64 KB row
// stride) access vs row-contiguous access, for full-sector and byte-masked
// (RMW) stores.  Buffer = 65536 x 65536 bytes (the n=2^16 int8 grid).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int64_t N = 65536;

// unit u = (tile column c, band b) of W bytes x 16 rows; tiles visited in a scrambled order
template <int W, bool FULL>
__global__ void k_tile(uint8_t* g, int64_t units, int64_t ncol, int scramble) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = warp; u < units; u += nw) {
        int64_t uu = scramble ? (u * 40503) % units : u;
        const int64_t c = uu % ncol, b = uu / ncol;
        uint8_t* p = g + (b * 16) * N + c * W;
        for (int r = 0; r < 16; ++r) {
            uint8_t* q = p + r * N;
            if (W == 128) {
                if (FULL) reinterpret_cast<uint32_t*>(q)[lane] = 0x01010101u;
                else q[lane * 4] = 1;
            } else {
                if (FULL) reinterpret_cast<uint4*>(q)[lane] = make_uint4(1, 1, 1, 1);
                else q[lane * 16] = 1;
            }
        }
    }
}

__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}

int main() {
    uint8_t *g, *fl;
    unsigned* sink;
    CK(cudaMalloc(&g, N * N));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(g, 0, N * N));
    CK(cudaMemset(fl, 0, 1ll << 30));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 8, block = 256;
    // cover 1/4 of the grid rows (16384 rows) to keep runs short: units = cols * (16384/16)
    for (int variant = 0; variant < 8; ++variant) {
        const int W = (variant & 1) ? 512 : 128;
        const bool full = (variant & 2) != 0;
        const int scramble = (variant & 4) != 0;
        const int64_t ncol = N / W, units = ncol * (16384 / 16);
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            k_flush<<<grid, block>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
            cudaEventRecord(a);
            if (W == 128 && full) k_tile<128, true><<<grid, block>>>(g, units, ncol, scramble);
            if (W == 128 && !full) k_tile<128, false><<<grid, block>>>(g, units, ncol, scramble);
            if (W == 512 && full) k_tile<512, true><<<grid, block>>>(g, units, ncol, scramble);
            if (W == 512 && !full) k_tile<512, false><<<grid, block>>>(g, units, ncol, scramble);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double bytes = 16384.0 * N;
        printf("W=%3d %-7s %-9s %8.1f us  %6.0f GB/s (touched bytes; RMW doubles DRAM traffic)\n", W,
               full ? "full" : "bytes", scramble ? "scramble" : "ordered", best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
