// probe_sysmem.cu -- design probe for the zero-copy host transport: bandwidth of
// SM loads/stores to mapped pinned host memory over PCIe (not part of the product).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

// stride: bytes between consecutive 16-B accesses of consecutive threads (16 = dense)
template <int MODE>
__global__ void k_sys(uint8_t* p, int64_t nvec, int64_t stride, unsigned* sink, int ilp) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (int64_t v = tid; v < nvec; v += nth * 4) {
        uint4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t w = v + i * nth;
            if (w < nvec && MODE != 1) { uint4 t; asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "l"(p + w * stride)); x[i] = t; }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t w = v + i * nth;
            if (w >= nvec) continue;
            if (MODE == 0) acc ^= x[i].x;
            else if (MODE == 1) *reinterpret_cast<uint4*>(p + w * stride) = make_uint4(1, 2, 3, 4);
            else { x[i].y ^= 1; *reinterpret_cast<uint4*>(p + w * stride) = x[i]; }
        }
    }
    if (acc == 0x1234567u) atomicAdd(sink, 1u);
}

int main(int argc, char** argv) {
    const int64_t bytes = 1ll << 30;
    uint8_t* h;
    unsigned* sink;
    const bool thp = argc > 1 && !strcmp(argv[1], "thp");
    if (thp) {  // anonymous mmap with transparent huge pages, then page-locked + mapped
        void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        madvise(m, bytes, MADV_HUGEPAGE);
        memset(m, 0, bytes);
        h = (uint8_t*)m;
        CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped));
        printf("THP-backed host buffer\n");
    } else {
        CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    }
    CK(cudaMalloc(&sink, 4));
    for (int64_t i = 0; i < bytes; i += 4096) h[i] = 0;
    uint8_t* d;
    CK(cudaHostGetDevicePointer((void**)&d, h, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"read", "write", "rmw"};
    for (int mode = 0; mode < 3; ++mode)
        for (int64_t stride : {16ll, 32ll, 128ll, 512ll, 4096ll, 65536ll})
            for (int blocks : {148 * 16}) {
                const int64_t nvec = bytes / stride;
                float best = 1e9;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    if (mode == 0) k_sys<0><<<blocks, 256>>>(d, nvec, stride, sink, 4);
                    if (mode == 1) k_sys<1><<<blocks, 256>>>(d, nvec, stride, sink, 4);
                    if (mode == 2) k_sys<2><<<blocks, 256>>>(d, nvec, stride, sink, 4);
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                const double moved = (double)nvec * 16 * (mode == 2 ? 2 : 1);
                printf("%-5s stride %4lld  blocks %5d  %8.2f ms  %6.1f GB/s useful (16 B per access)\n", names[mode],
                       (long long)stride, blocks, best, moved / (best * 1e-3) / 1e9);
            }
    // copy-engine reference
    uint8_t* dd;
    CK(cudaMalloc(&dd, bytes));
    cudaEventRecord(a);
    cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy H2D 1 GiB %.2f ms %.1f GB/s\n", ms, bytes / (ms * 1e-3) / 1e9);
    cudaEventRecord(a);
    cudaMemcpyAsync(h, dd, bytes, cudaMemcpyDeviceToHost);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy D2H 1 GiB %.2f ms %.1f GB/s\n", ms, bytes / (ms * 1e-3) / 1e9);
    return 0;
}
