// probe_dies.cu -- design probe: does it matter which die's SMs touch which addresses?
// B200 is two dies, each with half the SMs, half the L2 and half the HBM stacks.  Reads
// of a 64 MB window at various offsets, done only by the SMs of one "half" (by %smid),
// with 1 CTA per SM.  If the memory behind an address range belongs to one die, the
// local half should read it faster than the remote half.
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// CTAs on SMs of the selected half read the window (grid-stride over the active CTAs)
__global__ void k_half(const uint4* __restrict__ p, int64_t n16, int half, int nsm, unsigned* sink, unsigned* slot) {
    __shared__ int rank;
    const unsigned sm = smid();
    const bool mine = half == 2 || (half == 0 ? sm < (unsigned)nsm / 2 : sm >= (unsigned)nsm / 2);
    if (threadIdx.x == 0) rank = mine ? (int)atomicAdd(slot, 1u) : -1;
    __syncthreads();
    if (rank < 0) return;
    const int active = half == 2 ? nsm : nsm / 2;
    unsigned acc = 0;
    for (int64_t i = (int64_t)rank * blockDim.x + threadIdx.x; i < n16; i += (int64_t)active * blockDim.x)
        acc ^= __ldcg(p + i).x;
    if (acc == 0x1234567u) atomicAdd(sink, 1u);
}

__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int64_t total = 16ll << 30, win = 64ll << 20;
    uint8_t *buf, *fl;
    unsigned *sink, *slot;
    CK(cudaMalloc(&buf, total));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMalloc(&slot, 4));
    CK(cudaMemset(buf, 1, total));
    CK(cudaMemset(fl, 0, 1ll << 30));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("SMs %d; window 64 MB; GB/s when read by SMs [0,n/2) | [n/2,n) | all\n", nsm);
    for (int64_t off = 0; off + win <= total; off += (off < (1ll << 30) ? (128ll << 20) : (1ll << 30))) {
        float t[3];
        for (int half = 0; half < 3; ++half) {
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                k_flush<<<nsm * 8, 256>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
                CK(cudaMemset(slot, 0, 4));
                cudaEventRecord(a);
                k_half<<<nsm, 1024>>>(reinterpret_cast<const uint4*>(buf + off), win / 16, half, nsm, sink, slot);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                CK(cudaGetLastError());
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = std::min(best, ms);
            }
            t[half] = best;
        }
        printf("offset %6lld MB: %7.0f | %7.0f | %7.0f\n", (long long)(off >> 20), win / (t[0] * 1e-3) / 1e9,
               win / (t[1] * 1e-3) / 1e9, win / (t[2] * 1e-3) / 1e9);
    }
    return 0;
}
