// probe_fetch.cu -- design probe: how many bytes does DRAM deliver when a
// kernel reads only part of each 128-byte line?  (2 GiB buffer, one access
// unit per line, L2 flushed before each launch.)  Run under ncu for
// dram__bytes_read.sum and lts__t_sectors_srcunit_tex_op_read.sum; the event
// times printed here are the non-profiled numbers.
//   ./probe_fetch [l2_fetch_granularity_bytes]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int64_t BYTES = 1ll << 31;

__device__ __forceinline__ uint4 ld_plain(const void* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ uint4 ld_cg(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_na(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_64b(const void* p) {
    uint4 v;
    asm volatile("ld.global.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_ef(const void* p) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// MODE: 0 plain, 1 cg, 2 nc.no_allocate, 3 L2::64B hint, 4 evict_first, 5 cp.async.cg 16, 6 TMA bulk
// LANES lanes x 16 B per unit at byte offset OFF of line (unit * STRIDE_LINES)
template <int MODE, int LANES, int OFF, int STRIDE_LINES>
__global__ void k_sparse(const uint8_t* __restrict__ p, int64_t units, unsigned* sink) {
    __shared__ __align__(128) uint4 st[256 * 2];
    __shared__ __align__(8) unsigned long long bar;
    unsigned acc = 0;
    if (MODE == 6) {
        if (threadIdx.x == 0) {
            const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
        }
        __syncthreads();
        // one thread per unit issues a LANES*16-byte bulk copy; phase-tracked mbarrier per block iteration
        unsigned phase = 0;
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
        for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < units; base += (int64_t)gridDim.x * blockDim.x) {
            const int64_t u = base + threadIdx.x;
            const int64_t cnt = units - base < blockDim.x ? units - base : blockDim.x;
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"((unsigned)(cnt * LANES * 16)) : "memory");
            __syncthreads();
            if (u < units) {
                const uint8_t* a = p + u * STRIDE_LINES * 128 + OFF;
                const unsigned s = (unsigned)__cvta_generic_to_shared(&st[threadIdx.x * 2]);
                asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(s), "l"(a), "r"(LANES * 16), "r"(b) : "memory");
            }
            asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W; }" ::"r"(b), "r"(phase) : "memory");
            phase ^= 1;
            acc ^= st[threadIdx.x * 2].x;
            __syncthreads();
        }
        if (acc == 0x12345678u) atomicAdd(sink, 1u);
        return;
    }
    const int64_t nt = units * LANES;
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nt; h += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = h / LANES;
        const int part = (int)(h % LANES);
        const uint8_t* a = p + u * STRIDE_LINES * 128 + OFF + part * 16;
        uint4 v;
        if (MODE == 0) v = ld_plain(a);
        else if (MODE == 1) v = ld_cg(a);
        else if (MODE == 2) v = ld_na(a);
        else if (MODE == 3) v = ld_64b(a);
        else if (MODE == 4) v = ld_ef(a);
        else {
            const unsigned s = (unsigned)__cvta_generic_to_shared(&st[threadIdx.x]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(a) : "memory");
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            v = st[threadIdx.x];
        }
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1u);
}

// writes: each thread stores one whole 32-byte sector (st.global.v8) at sector
// index s of unit u; MASK = which sectors of each 128-byte line are written
template <int MASK, int STRIDE_LINES>
__global__ void k_wsparse(const uint8_t* __restrict__ pc, int64_t units, unsigned* sink) {
    uint8_t* p = const_cast<uint8_t*>(pc);
    constexpr int NS = (MASK & 1) + ((MASK >> 1) & 1) + ((MASK >> 2) & 1) + ((MASK >> 3) & 1);
    const int64_t nt = units * NS;
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nt; h += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = h / NS;
        int k = (int)(h % NS), s = 0;
        for (int b = 0; b < 4; ++b)
            if ((MASK >> b) & 1) {
                if (k == 0) { s = b; break; }
                --k;
            }
        uint8_t* a = p + u * STRIDE_LINES * 128 + s * 32;
        const unsigned v = (unsigned)h;
        asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(a), "r"(v) : "memory");
    }
    if (units < 0) atomicAdd(sink, 1u);
}

__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}

typedef void (*kfn)(const uint8_t*, int64_t, unsigned*);
struct Case {
    const char* name;
    kfn f;
    int bytes_per_unit;
    int stride_lines;
};

int main(int argc, char** argv) {
    size_t g0 = 0;
    CK(cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity));
    if (argc > 1) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1])));
    size_t g1 = 0;
    CK(cudaDeviceGetLimit(&g1, cudaLimitMaxL2FetchGranularity));
    printf("L2 fetch granularity limit: default %zu, now %zu\n", g0, g1);
    uint8_t *buf, *fl;
    unsigned* sink;
    CK(cudaMalloc(&buf, BYTES));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 1, BYTES));
    CK(cudaMemset(fl, 0, 1ll << 30));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const Case cases[] = {
        {"st 32B sector0/line", k_wsparse<1, 1>, 32, 1},
        {"st 64B sectors01/line", k_wsparse<3, 1>, 64, 1},
        {"st 64B sectors02/line", k_wsparse<5, 1>, 64, 1},
        {"st 96B sectors012/line", k_wsparse<7, 1>, 96, 1},
        {"st 128B/line (dense)", k_wsparse<15, 1>, 128, 1},
        {"st 32B sector0 / 2 lines", k_wsparse<1, 2>, 32, 2},
        {"ld 32B/line", k_sparse<0, 2, 0, 1>, 32, 1},
        {"ld 16B/line", k_sparse<0, 1, 0, 1>, 16, 1},
        {"ld.cg 32B/line", k_sparse<1, 2, 0, 1>, 32, 1},
        {"ld.nc.na 32B/line", k_sparse<2, 2, 0, 1>, 32, 1},
        {"ld.L2::64B 32B/line", k_sparse<3, 2, 0, 1>, 32, 1},
        {"ld.cs 32B/line", k_sparse<4, 2, 0, 1>, 32, 1},
        {"cp.async 32B/line", k_sparse<5, 2, 0, 1>, 32, 1},
        {"cp.async 16B/line", k_sparse<5, 1, 0, 1>, 16, 1},
        {"tma 32B/line", k_sparse<6, 2, 0, 1>, 32, 1},
        {"tma 16B/line", k_sparse<6, 1, 0, 1>, 16, 1},
        {"ld 32B sector3/line", k_sparse<0, 2, 96, 1>, 32, 1},
        {"ld 64B/line", k_sparse<0, 4, 0, 1>, 64, 1},
        {"ld 32B/2 lines", k_sparse<0, 2, 0, 2>, 32, 2},
        {"ld 32B/4 lines", k_sparse<0, 2, 0, 4>, 32, 4},
        {"cp.async 32B/2 lines", k_sparse<5, 2, 0, 2>, 32, 2},
        {"tma 32B/2 lines", k_sparse<6, 2, 0, 2>, 32, 2},
        {"ld 128B/line (dense)", k_sparse<0, 8, 0, 1>, 128, 1},
        {"ld 128B per 8 lines", k_sparse<0, 8, 0, 8>, 128, 8},
        {"ld 128B per 64 lines", k_sparse<0, 8, 0, 64>, 128, 64},
        {"ld 128B per 512 lines", k_sparse<0, 8, 0, 512>, 128, 512},
        {"ld 128B per 1024 lines", k_sparse<0, 8, 0, 1024>, 128, 1024},
        {"ld.L2::64B 64B per 8 lines", k_sparse<3, 4, 0, 8>, 64, 8},
        {"ld.L2::64B 64B per 512 lines", k_sparse<3, 4, 0, 512>, 64, 512},
    };
    for (const Case& c : cases) {
        const int64_t units = BYTES / 128 / c.stride_lines;  // sparse strides read fewer units (same buffer span)
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            k_flush<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
            cudaEventRecord(a);
            c.f<<<148 * 8, 256>>>(buf, units, sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double useful = (double)units * c.bytes_per_unit;
        printf("%-26s %8.1f us  useful %6.0f GB/s  units %.3e\n", c.name, best * 1e3, useful / (best * 1e-3) / 1e9,
               (double)units);
    }
    return 0;
}
