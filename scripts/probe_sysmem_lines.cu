// probe_sysmem_lines.cu -- design probe (not product): SM reads / read-modify-writes of
// mapped pinned host memory in whole 128-byte lines or 64-byte halves, every `gap`-th
// line, with and without an L2 prefetch-size hint on the loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int HINT>
__device__ __forceinline__ uint4 ld(const uint8_t* p) {
    uint4 t;
    if (HINT == 0) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(p));
    else if (HINT == 1) asm volatile("ld.global.cv.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(p));
    else if (HINT == 2) asm volatile("ld.global.cv.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(p));
    else asm volatile("ld.relaxed.sys.global.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(p));
    return t;
}

// LANES = 16-byte lanes per line (8: whole line, 4: first half); RMW: write back
template <int HINT, int LANES, bool RMW>
__global__ void k(uint8_t* p, int64_t nlines, int gap, unsigned* sink) {
    const int lane = threadIdx.x & 31, sub = lane >> 3, q = lane & 7;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    constexpr int PER = 8;
    for (int64_t base = warp * 4 * PER; base < nlines; base += nw * 4 * PER) {
        uint4 x[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int64_t l = base + i * 4 + sub;
            if (l < nlines && q < LANES) x[i] = ld<HINT>(p + l * gap * 128 + q * 16);
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int64_t l = base + i * 4 + sub;
            if (l >= nlines || q >= LANES) continue;
            if (RMW) { x[i].y ^= 1; *reinterpret_cast<uint4*>(p + l * gap * 128 + q * 16) = x[i]; }
            else acc ^= x[i].x;
        }
    }
    if (acc == 0x1234567u) atomicAdd(sink, 1u);
}

template <int HINT, int LANES, bool RMW>
float run(uint8_t* d, int64_t bytes, int gap, unsigned* sink) {
    const int64_t nlines = bytes / 128 / gap;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<HINT, LANES, RMW><<<148 * 8, 256>>>(d, nlines, gap, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) k<HINT, LANES, RMW><<<148 * 8, 256>>>(d, nlines, gap, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return (float)(nlines * LANES * 16) * 3 / (ms * 1e-3f) / 1e9f;  // useful GB/s (one direction)
}

int main() {
    const int64_t bytes = 1ll << 30;
    uint8_t* h;
    unsigned* sink;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    CK(cudaMalloc(&sink, 4));
    for (int64_t i = 0; i < bytes; i += 4096) h[i] = 0;
    uint8_t* d;
    CK(cudaHostGetDevicePointer((void**)&d, h, 0));
    const char* hn[4] = {"cv", "cv.L2::128B", "cv.L2::256B", "relaxed.sys.L2::128B"};
    for (int gap : {1, 2, 8}) {
        printf("gap %d: every %d-th line\n", gap, gap);
        printf("  read  line  %-22s %7.1f GB/s\n", hn[0], run<0, 8, false>(d, bytes, gap, sink));
        printf("  read  line  %-22s %7.1f GB/s\n", hn[1], run<1, 8, false>(d, bytes, gap, sink));
        printf("  read  line  %-22s %7.1f GB/s\n", hn[2], run<2, 8, false>(d, bytes, gap, sink));
        printf("  read  line  %-22s %7.1f GB/s\n", hn[3], run<3, 8, false>(d, bytes, gap, sink));
        printf("  read  half  %-22s %7.1f GB/s\n", hn[0], run<0, 4, false>(d, bytes, gap, sink));
        printf("  read  half  %-22s %7.1f GB/s\n", hn[1], run<1, 4, false>(d, bytes, gap, sink));
        printf("  rmw   line  %-22s %7.1f GB/s (each way)\n", hn[0], run<0, 8, true>(d, bytes, gap, sink));
        printf("  rmw   line  %-22s %7.1f GB/s (each way)\n", hn[1], run<1, 8, true>(d, bytes, gap, sink));
        printf("  rmw   line  %-22s %7.1f GB/s (each way)\n", hn[3], run<3, 8, true>(d, bytes, gap, sink));
        printf("  rmw   half  %-22s %7.1f GB/s (each way)\n", hn[0], run<0, 4, true>(d, bytes, gap, sink));
        printf("  rmw   half  %-22s %7.1f GB/s (each way)\n", hn[1], run<1, 4, true>(d, bytes, gap, sink));
    }
    CK(cudaGetLastError());
    return 0;
}
