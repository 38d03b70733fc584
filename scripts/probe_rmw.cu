// probe_rmw.cu -- ceiling of the CONST write pass's store pattern with perfect locality.
// The n = 2^16 int8 write pass stores, in each of 2.52 M lines, the gasket bytes of one
// grid row (row y: bytes x subset of y): 1, 2, 2 or 4 partially written sectors per
// line.  Here the same per-line patterns are stored into 2.52 M CONSECUTIVE lines of a
// buffer (line i takes the pattern of row i mod 128, i.e. y_lo = i & 127), so DRAM sees
// the same partial-sector read-modify-writes in address order.
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void st_masked(uint8_t* p, uint32_t v, uint32_t t) {
    switch (t & 3u) {
    case 3: *reinterpret_cast<uint32_t*>(p) = v; break;
    case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; break;
    case 2: p[2] = (uint8_t)(v >> 16); p[0] = (uint8_t)v; break;
    default: p[0] = (uint8_t)v; break;
    }
}

// warp per line, lanes = 4-byte words; word j holds gasket bytes iff 4j subset of t
__global__ void k_lines(uint8_t* g, int64_t nlines, int64_t stride_lines) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nlines; i += nw) {
        const uint32_t t = (uint32_t)(i & 127);
        if (((lane * 4) & ~t) == 0) st_masked(g + i * stride_lines * 128 + lane * 4, 0x01010101u, t);
    }
}

// stencil-shaped traffic in address order: A's lines [0, nread) read whole, B's lines
// [0, nwrite) get the touched sectors (pattern of row i mod 128) stored whole; each warp
// moves 8 consecutive lines per iteration with all loads in flight before any use
__global__ void k_copy(const uint8_t* __restrict__ A, uint8_t* __restrict__ B, int64_t nread, int64_t nwrite,
                       unsigned* sink) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    const int64_t nmax = (nread > nwrite ? nread : nwrite + 7) / 8;
    for (int64_t u = warp; u < nmax; u += nw) {
        const int64_t l0 = u * 8;
        uint4 v[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {  // lanes 0..31 x 16 B = 4 lines per instruction
            const int64_t line = l0 + k * 4 + (lane >> 3);
            v[k] = line < nread ? __ldcg(reinterpret_cast<const uint4*>(A + line * 128) + (lane & 7)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int64_t line = l0 + k * 4 + (lane >> 3);
            const uint32_t t = (uint32_t)(line & 127);
            const int g = (lane & 7) >> 1;  // 2 lanes (32 B) per sector
            if (line < nwrite && ((g * 32) & ~t) == 0)
                reinterpret_cast<uint4*>(B + line * 128)[lane & 7] = make_uint4(1, 1, 1, 1);
        }
        acc ^= v[0].x ^ v[1].y;
    }
    if (acc == 0x12345u) atomicAdd(sink, 1u);
}

__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}

int main() {
    const int64_t nlines = 128ll * 19683;  // 128 * 3^9 = the write pass's line count at n = 2^16 int8
    uint8_t *g, *fl;
    unsigned* sink;
    CK(cudaMalloc(&g, nlines * 128 * 4));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(g, 0, nlines * 128 * 4));
    CK(cudaMemset(fl, 0, 1ll << 30));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int64_t stride : {1, 2, 4}) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            k_flush<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
            cudaEventRecord(a);
            k_lines<<<148 * 8, 256>>>(g, nlines, stride);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
        }
        printf("consecutive lines x stride %lld: %8.1f us  %.1f G lines/s\n", (long long)stride, best * 1e3,
               nlines / (best * 1e-3) / 1e9);
    }
    {
        const int64_t nread = 11264000, nwrite = 128ll * 59049;  // n = 2^17 NSUM8: ~1.44 GB line reads, 7.56 M lines
        uint8_t *A, *B;
        CK(cudaMalloc(&A, nread * 128));
        CK(cudaMalloc(&B, nwrite * 128));
        CK(cudaMemset(A, 1, nread * 128));
        CK(cudaMemset(B, 0, nwrite * 128));
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            k_flush<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
            cudaEventRecord(a);
            k_copy<<<148 * 8, 256>>>(A, B, nread, nwrite, sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
        }
        printf("stencil-shaped traffic in address order (11.26 M line reads + 7.56 M partial-line writes): %8.1f us\n",
               best * 1e3);
    }
    return 0;
}
