// probe_sweep.cu -- design probe for the CONST write pass at n = 2^16 int8: the
// same byte-masked (read-modify-write) stores of the gasket cells, visited
//   tiles : warp per (member tile, 16-row band), tiles row-major (the product order)
//   sweep : warp per (row, member line), units in address order (row y, then the
//           lines l subset of y >> 7 ascending), interleaved over warps so the warps
//           running together store consecutive lines of the same rows
// Both write exactly the gasket cells (checked against each other).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int R = 16;
constexpr int64_t N = 1ll << R;
constexpr int Q = R - 7;

__device__ __forceinline__ uint32_t byte_mask(uint32_t t) {
    const uint32_t sel = (uint32_t)(0x0000404044004440ull >> ((t & 3u) << 4));
    return __byte_perm(0xffffffffu, 0u, sel);
}
__device__ __forceinline__ void st_masked(uint8_t* p, uint32_t v, uint32_t t) {
    // the stream.cu pattern: rows with t&3 = 0,1,2,3 store 1 byte, 2 bytes, 2 bytes, 4 bytes
    switch (t & 3u) {
    case 3: *reinterpret_cast<uint32_t*>(p) = v; break;
    case 1: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; break;
    case 2: p[2] = (uint8_t)(v >> 16); p[0] = (uint8_t)v; break;
    default: p[0] = (uint8_t)v; break;
    }
}

__global__ void k_tiles(uint8_t* g, const uint32_t* tiles, int64_t ntiles) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = warp; u < ntiles * 8; u += nw) {
        const uint32_t v = tiles[u >> 3];
        const int64_t x0 = (int64_t)(v & 0xffff) * 128, y0 = (int64_t)(v >> 16) * 128;
        const int t0 = (int)(u & 7) * 16;
        for (int i = 0; i < 16; ++i) {
            const int t = t0 + i;
            if (((lane * 4) & ~t) == 0) st_masked(g + (y0 + t) * N + x0 + lane * 4, 0x01010101u, (uint32_t)t);
        }
    }
}

// F(Y) = number of member lines in block rows < Y of one grid row band (per grid row):
// sum over set bits b of Y of 3^b * 2^popcount(Y >> (b+1))
__device__ __forceinline__ uint32_t lines_before(uint32_t Y) {
    uint32_t f = 0, p3 = 1, above = __popc(Y);
    for (int b = 0; b < 20 && (Y >> b); ++b) {
        if ((Y >> b) & 1u) { --above; f += p3 << above; }
        p3 *= 3u;
    }
    return f;
}
__device__ __forceinline__ uint32_t pdep(uint32_t i, uint32_t mask) {
    uint32_t out = 0;
    while (mask) {
        const uint32_t low = mask & (0u - mask);
        if (i & 1u) out |= low;
        i >>= 1;
        mask ^= low;
    }
    return out;
}

// units precomputed in address order: y << 16 | l
__global__ void k_sweep(uint8_t* g, const uint32_t* units, int64_t nunits) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = warp; u < nunits; u += nw) {
        const uint32_t v = __ldg(units + u);
        const uint32_t y = v >> 16, l = v & 0xffffu, t = y & 127u;
        if (((lane * 4) & ~t) == 0) st_masked(g + (int64_t)y * N + (int64_t)l * 128 + lane * 4, 0x01010101u, t);
    }
}

__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}
__global__ void k_sum(const uint8_t* g, int64_t n, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 8; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = reinterpret_cast<const uint64_t*>(g)[i];
        acc += __popcll(v) + (v % 1000003ull) * (uint64_t)(i % 7);
    }
    atomicAdd(out, acc);
}

int main() {
    uint8_t *g, *fl;
    unsigned* sink;
    unsigned long long* sum;
    CK(cudaMalloc(&g, N * N));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMalloc(&sum, 8));
    CK(cudaMemset(fl, 0, 1ll << 30));
    std::vector<uint32_t> rm;
    for (uint32_t Y = 0; Y < (1u << Q); ++Y)
        for (uint32_t l = 0; l < (1u << Q); ++l)
            if ((l & ~Y) == 0) rm.push_back(l | (Y << 16));
    const int64_t nt = (int64_t)rm.size();
    uint32_t* d_rm;
    CK(cudaMalloc(&d_rm, nt * 4));
    CK(cudaMemcpy(d_rm, rm.data(), nt * 4, cudaMemcpyHostToDevice));
    const int64_t nunits = nt * 128;
    std::vector<uint32_t> un;
    un.reserve(nunits);
    for (uint32_t y = 0; y < (uint32_t)N; ++y) {
        const uint32_t Y = y >> 7;
        for (uint32_t l = 0; l < (1u << Q); ++l)
            if ((l & ~Y) == 0) un.push_back((y << 16) | l);
    }
    uint32_t* d_un;
    CK(cudaMalloc(&d_un, nunits * 4));
    CK(cudaMemcpy(d_un, un.data(), nunits * 4, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    unsigned long long sums[2];
    for (int kind = 0; kind < 2; ++kind) {
        CK(cudaMemset(g, 0, N * N));
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            k_flush<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
            cudaEventRecord(e0);
            if (kind == 0) k_tiles<<<148 * 8, 256>>>(g, d_rm, nt);
            else k_sweep<<<148 * 8, 256>>>(g, d_un, nunits);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        CK(cudaMemset(sum, 0, 8));
        k_sum<<<148 * 8, 256>>>(g, N * N, sum);
        CK(cudaMemcpy(&sums[kind], sum, 8, cudaMemcpyDeviceToHost));
        printf("%-6s %8.1f us  %.1f G lines/s  checksum %llu\n", kind == 0 ? "tiles" : "sweep", best * 1e3,
               nunits / (best * 1e-3) / 1e9, sums[kind]);
    }
    printf("same cells: %s\n", sums[0] == sums[1] ? "yes" : "NO");
    return 0;
}
