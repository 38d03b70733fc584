// probe_gasket.cu -- design probe: DRAM cost of the gasket's own access set in
// different visiting orders, at n = 2^17 int8 (16 GiB per buffer).
//
// Unit of access = one 128-byte line (y, l) with l subset of (y >> 7) (the lines
// holding gasket cells; 128 * 3^10 = 7.56M lines).  Kernels:
//   read  : load the line (16 B per lane, 8 lanes per line, .L2::64B hint)
//   write : store the line's touched 32-byte sectors whole (g subset of (y>>5)&3)
//   copy  : read from A, write the touched sectors to B
// Orders:
//   rows  : warp w walks row y = w (grid-stride), member lines ascending
//   tiles : warp w walks tile (l, Y) = the w-th member tile (digit order), 128 rows
//   tilesrm: as tiles, member tiles in row-major order (Y, then l)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int R = 17;
constexpr int64_t N = 1ll << R;
constexpr int Q = R - 7;  // tile level (tile = 128 x 128 cells)

__device__ __forceinline__ uint4 ld64(const uint8_t* p) {
    uint4 v;
    asm volatile("ld.global.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st16(uint8_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// one line (y, l): lanes sub = 0..7 each 16 bytes
template <int MODE>
__device__ __forceinline__ unsigned do_line(const uint8_t* a, uint8_t* b, int64_t y, int64_t l, int sub) {
    const int64_t off = y * N + l * 128 + sub * 16;
    unsigned acc = 0;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (MODE != 1) {
        v = ld64(a + off);
        acc = v.x ^ v.w;
    }
    if (MODE != 0) {
        const int g = sub >> 1;
        if (((g & ~(int)(y >> 5)) & 3) == 0) st16(b + off, make_uint4(v.x + 1, v.y, v.z, v.w));
    }
    return acc;
}

// rows order: 4 lines per warp instruction (8 lanes each)
template <int MODE>
__global__ void k_rows(const uint8_t* a, uint8_t* b, unsigned* sink) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    for (int64_t y = warp; y < N; y += nw) {
        const uint32_t Y = (uint32_t)(y >> 7);
        const int cnt = 1 << __popc(Y);
        for (int k = grp; k < cnt; k += 4) {
            // k-th subset of Y in ascending order = pdep(k, Y)
            uint32_t l = 0, m = Y, kk = (uint32_t)k;
            while (m) {
                const uint32_t low = m & (0u - m);
                if (kk & 1u) l |= low;
                kk >>= 1;
                m ^= low;
            }
            acc ^= do_line<MODE>(a, b, y, l, sub);
        }
    }
    if (acc == 0x12345u) atomicAdd(sink, 1u);
}

// tiles order: warp handles one member tile (128 rows x 1 line), 4 rows per instruction
template <int MODE>
__global__ void k_tiles(const uint8_t* a, uint8_t* b, const uint32_t* tiles, int64_t ntiles, unsigned* sink) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    for (int64_t t = warp; t < ntiles; t += nw) {
        const uint32_t v = tiles[t];
        const int64_t l = v & 0xffff, Yb = v >> 16;
        for (int r = grp; r < 128; r += 4) acc ^= do_line<MODE>(a, b, Yb * 128 + r, l, sub);
    }
    if (acc == 0x12345u) atomicAdd(sink, 1u);
}

// strips order: warp handles the member tiles of one 8-line-aligned strip of a tile
// row in lockstep: for each row, the member lines side by side (4 per instruction)
template <int MODE>
__global__ void k_strips(const uint8_t* a, uint8_t* b, const uint32_t* strips, int64_t nstrips, unsigned* sink) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned acc = 0;
    for (int64_t t = warp; t < nstrips; t += nw) {
        const uint32_t v = strips[t];
        const uint32_t X8 = v & 0xffff, Yb = v >> 16;
        const uint32_t low = Yb & 7u;
        const int cnt = 1 << __popc(low);
        for (int r = 0; r < 128; ++r) {
            for (int k = grp; k < cnt; k += 4) {
                uint32_t j = 0, m = low, kk = (uint32_t)k;
                while (m) {
                    const uint32_t lo = m & (0u - m);
                    if (kk & 1u) j |= lo;
                    kk >>= 1;
                    m ^= lo;
                }
                acc ^= do_line<MODE>(a, b, (int64_t)Yb * 128 + r, (int64_t)X8 * 8 + j, sub);
            }
        }
    }
    if (acc == 0x12345u) atomicAdd(sink, 1u);
}

__global__ void k_flush(const uint4* p, int64_t n, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) acc ^= p[i].x;
    if (acc == 0x9999u) atomicAdd(sink, 1u);
}

int main() {
    uint8_t *a, *b, *fl;
    unsigned* sink;
    CK(cudaMalloc(&a, N * N));
    CK(cudaMalloc(&b, N * N));
    CK(cudaMalloc(&fl, 1ll << 30));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(a, 1, N * N));
    CK(cudaMemset(b, 0, N * N));
    CK(cudaMemset(fl, 0, 1ll << 30));
    // member tiles: digit order and row-major
    std::vector<uint32_t> dig, rm;
    uint32_t nt = 1;
    for (int i = 0; i < Q; ++i) nt *= 3;
    for (uint32_t c = 0; c < nt; ++c) {
        uint32_t x = 0, y = 0, d = c;
        for (int i = 0; i < Q; ++i, d /= 3) { x |= (uint32_t)(d % 3 == 2) << i; y |= (uint32_t)(d % 3 != 0) << i; }
        dig.push_back(x | (y << 16));
    }
    rm = dig;
    std::sort(rm.begin(), rm.end(), [](uint32_t p, uint32_t q) {
        return (p >> 16) != (q >> 16) ? (p >> 16) < (q >> 16) : (p & 0xffff) < (q & 0xffff);
    });
    // strips: (X8, Y) with X8 subset of Y >> 3, row-major
    std::vector<uint32_t> st;
    for (uint32_t Y = 0; Y < (1u << Q); ++Y)
        for (uint32_t X8 = 0; X8 < (1u << (Q - 3)); ++X8)
            if ((X8 & ~(Y >> 3)) == 0) st.push_back(X8 | (Y << 16));
    const int64_t ns = (int64_t)st.size();
    uint32_t* d_st;
    CK(cudaMalloc(&d_st, ns * 4));
    CK(cudaMemcpy(d_st, st.data(), ns * 4, cudaMemcpyHostToDevice));
    uint32_t *d_dig, *d_rm;
    CK(cudaMalloc(&d_dig, nt * 4));
    CK(cudaMalloc(&d_rm, nt * 4));
    CK(cudaMemcpy(d_dig, dig.data(), nt * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_rm, rm.data(), nt * 4, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double lines = 128.0 * nt;
    const char* modes[] = {"read", "write", "copy"};
    for (int order = 0; order < 4; ++order) {
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                k_flush<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(fl), (1ll << 30) / 16, sink);
                cudaEventRecord(e0);
                const int grid = 148 * 8, block = 256;
                if (order == 3) {
                    if (mode == 0) k_strips<0><<<grid, block>>>(a, b, d_st, ns, sink);
                    if (mode == 1) k_strips<1><<<grid, block>>>(a, b, d_st, ns, sink);
                    if (mode == 2) k_strips<2><<<grid, block>>>(a, b, d_st, ns, sink);
                } else if (order == 0) {
                    if (mode == 0) k_rows<0><<<grid, block>>>(a, b, sink);
                    if (mode == 1) k_rows<1><<<grid, block>>>(a, b, sink);
                    if (mode == 2) k_rows<2><<<grid, block>>>(a, b, sink);
                } else {
                    const uint32_t* t = order == 1 ? d_dig : d_rm;
                    if (mode == 0) k_tiles<0><<<grid, block>>>(a, b, t, nt, sink);
                    if (mode == 1) k_tiles<1><<<grid, block>>>(a, b, t, nt, sink);
                    if (mode == 2) k_tiles<2><<<grid, block>>>(a, b, t, nt, sink);
                }
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = std::min(best, ms);
            }
            printf("%-8s %-6s %8.1f us  %6.1f G lines/s\n", order == 0 ? "rows" : order == 1 ? "tiles" : order == 2 ? "tilesrm" : "strips",
                   modes[mode], best * 1e3, lines / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
