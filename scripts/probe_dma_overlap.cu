// probe_dma_overlap.cu -- design probe (not product): does copy-engine traffic (cudaMemcpyAsync
// H2D + D2H of a dense slab) overlap with SM read-modify-writes of mapped host memory?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

// RMW of every `gap`-th 128-byte line (16-byte lanes, 8 lanes per line)
__global__ void rmw(uint8_t* p, int64_t nlines, int gap) {
    const int lane = threadIdx.x & 31, sub = lane >> 3, q = lane & 7;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int PER = 8;
    for (int64_t base = warp * 4 * PER; base < nlines; base += nw * 4 * PER) {
        uint4 x[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int64_t l = base + i * 4 + sub;
            if (l < nlines) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x[i].x), "=r"(x[i].y), "=r"(x[i].z), "=r"(x[i].w) : "l"(p + l * gap * 128 + q * 16));
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int64_t l = base + i * 4 + sub;
            if (l < nlines) { x[i].y ^= 1; *reinterpret_cast<uint4*>(p + l * gap * 128 + q * 16) = x[i]; }
        }
    }
}

int main() {
    const int64_t bytes = 1ll << 30, slab = 80ll << 20;
    uint8_t *h, *h2, *d;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h2, slab, cudaHostAllocDefault));
    CK(cudaMalloc(&d, slab));
    uint8_t* dm;
    CK(cudaHostGetDevicePointer((void**)&dm, h, 0));
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int gap = 3;
    const int64_t nlines = (300ll << 20) / 128 / 1;  // ~2.4 M lines, like the n=2^16 write pass
    auto timeit = [&](bool sm, bool dma) -> float {
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        cudaStreamWaitEvent(s1, a, 0);
        cudaStreamWaitEvent(s2, a, 0);
        if (sm) rmw<<<148 * 8, 256, 0, s1>>>(dm, nlines, gap);
        if (dma) {
            cudaMemcpyAsync(d, h2, slab, cudaMemcpyHostToDevice, s2);
            cudaMemcpyAsync(h2, d, slab, cudaMemcpyDeviceToHost, s2);
        }
        cudaEvent_t e1, e2;
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        cudaEventRecord(e1, s1);
        cudaEventRecord(e2, s2);
        cudaStreamWaitEvent(0, e1, 0);
        cudaStreamWaitEvent(0, e2, 0);
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    };
    for (int rep = 0; rep < 2; ++rep) {
        printf("SM RMW of %lld lines alone: %.2f ms\n", (long long)nlines, timeit(true, false));
        printf("DMA 80 MB H2D then D2H alone: %.2f ms\n", timeit(false, true));
        printf("both concurrently: %.2f ms\n", timeit(true, true));
    }
    CK(cudaGetLastError());
    return 0;
}
