// probe_partial.cu -- micro-benchmark: how does B200 HBM treat partial-sector
// writes?  (Design probe for the gasket write pass; not part of the product.)
// Each kernel touches every 32-byte sector of a 2 GiB buffer once in a
// different way; run under ncu to read dram__bytes_{read,write}.sum.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_full32(uint8_t* p, int64_t nsec) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsec; s += (int64_t)gridDim.x * blockDim.x) {
        uint4* q = reinterpret_cast<uint4*>(p + s * 32);
        q[0] = make_uint4(1, 1, 1, 1);
        q[1] = make_uint4(1, 1, 1, 1);
    }
}
// lane pairs cover one sector (coalesced full sector)
__global__ void k_full32_pair(uint8_t* p, int64_t nhalf) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nhalf; h += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint4*>(p)[h] = make_uint4(2, 2, 2, 2);
}
__global__ void k_half16(uint8_t* p, int64_t nsec) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsec; s += (int64_t)gridDim.x * blockDim.x)
        *reinterpret_cast<uint4*>(p + s * 32) = make_uint4(3, 3, 3, 3);
}
__global__ void k_byte1(uint8_t* p, int64_t nsec) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsec; s += (int64_t)gridDim.x * blockDim.x)
        p[s * 32] = 4;
}
__global__ void k_u64(uint8_t* p, int64_t nsec) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsec; s += (int64_t)gridDim.x * blockDim.x)
        *reinterpret_cast<uint64_t*>(p + s * 32) = 5;
}
// 32 lanes write 8 scattered bytes of one sector each (gasket-like byte pattern), 4 sectors per warp instr
__global__ void k_warp_bytes(uint8_t* p, int64_t nsec) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s4 = warp; s4 < nsec / 4; s4 += nwarps) {
        const int sec = lane >> 3, b = lane & 7;
        p[(s4 * 4 + sec) * 32 + (b * 4 + (b & 1))] = 6;  // 8 bytes per sector, scattered
    }
}
__global__ void k_rmw16(uint8_t* p, int64_t nsec) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsec; s += (int64_t)gridDim.x * blockDim.x) {
        uint4* q = reinterpret_cast<uint4*>(p + s * 32);
        uint4 v = *q;
        v.x ^= 0x01010101u;
        *q = v;
    }
}
__global__ void k_rmw32_pair(uint8_t* p, int64_t nhalf) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nhalf; h += (int64_t)gridDim.x * blockDim.x) {
        uint4* q = reinterpret_cast<uint4*>(p) + h;
        uint4 v = *q;
        v.y ^= 0x01010101u;
        *q = v;
    }
}
// 4 independent rmw per thread (ILP)
__global__ void k_rmw32_pair_ilp4(uint8_t* p, int64_t nhalf) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nhalf; h += 4 * stride) {
        uint4* q = reinterpret_cast<uint4*>(p);
        uint4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) if (h + i * stride < nhalf) v[i] = q[h + i * stride];
#pragma unroll
        for (int i = 0; i < 4; ++i) if (h + i * stride < nhalf) { v[i].y ^= 0x01010101u; q[h + i * stride] = v[i]; }
    }
}
__global__ void k_read(const uint8_t* p, int64_t nhalf, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nhalf; h += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = reinterpret_cast<const uint4*>(p)[h];
        acc ^= v.x ^ v.w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1u);
}
// sparse: byte in every 4th sector (like a gasket row with few members)
__global__ void k_byte_sparse(uint8_t* p, int64_t nsec) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsec / 4; s += (int64_t)gridDim.x * blockDim.x)
        p[s * 128 + 5] = 7;
}
// 32-byte sector reads (lane pairs) at a stride of `step` sectors: DRAM fetch granularity probe
__global__ void k_read_sparse(const uint8_t* p, int64_t nsec, int step, unsigned* sink) {
    unsigned acc = 0;
    const int64_t nh = (nsec / step) * 2;
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nh; h += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = (h >> 1) * step;
        uint4 v = reinterpret_cast<const uint4*>(p + s * 32)[h & 1];
        acc ^= v.x ^ v.w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1u);
}
__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = p[i];
        acc ^= v.x;
    }
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}

int main() {
    const int64_t bytes = 2ll << 30;
    const int64_t nsec = bytes / 32;
    uint8_t *buf, *fl;
    unsigned* sink;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(buf, 0, bytes));
    CK(cudaMemset(fl, 0, 1ll << 30));
    const int grid = 148 * 8, block = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto flush = [&]() { k_flush<<<grid, block>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink); };
    struct T { const char* name; int id; double useful; };
    T tests[] = {{"full32", 0, 1.0}, {"full32_pair", 1, 1.0}, {"half16", 2, 0.5}, {"byte1", 3, 1.0 / 32},
                 {"u64", 4, 0.25}, {"warp_bytes8", 5, 0.25}, {"rmw16", 6, 0.5}, {"rmw32_pair", 7, 1.0},
                 {"rmw32_pair_ilp4", 8, 1.0}, {"read", 9, 1.0}, {"byte_sparse4", 10, 1.0 / 128},
                 {"read_every2nd_sector", 11, 0.5}, {"read_every4th_sector", 12, 0.25}};
    for (auto& t : tests) {
        for (int rep = 0; rep < 3; ++rep) {
            flush();
            cudaEventRecord(a);
            switch (t.id) {
            case 0: k_full32<<<grid, block>>>(buf, nsec); break;
            case 1: k_full32_pair<<<grid, block>>>(buf, nsec * 2); break;
            case 2: k_half16<<<grid, block>>>(buf, nsec); break;
            case 3: k_byte1<<<grid, block>>>(buf, nsec); break;
            case 4: k_u64<<<grid, block>>>(buf, nsec); break;
            case 5: k_warp_bytes<<<grid, block>>>(buf, nsec); break;
            case 6: k_rmw16<<<grid, block>>>(buf, nsec); break;
            case 7: k_rmw32_pair<<<grid, block>>>(buf, nsec * 2); break;
            case 8: k_rmw32_pair_ilp4<<<grid, block>>>(buf, nsec * 2); break;
            case 9: k_read<<<grid, block>>>(buf, nsec * 2, sink); break;
            case 10: k_byte_sparse<<<grid, block>>>(buf, nsec); break;
            case 11: k_read_sparse<<<grid, block>>>(buf, nsec, 2, sink); break;
            case 12: k_read_sparse<<<grid, block>>>(buf, nsec, 4, sink); break;
            }
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("%-18s %8.1f us  sectors/s %.3e  touched-sector GB/s %.0f\n", t.name, ms * 1e3,
                       (t.id == 10 ? nsec / 4 : nsec) / (ms * 1e-3), (t.id == 10 ? bytes / 4 : bytes) / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
