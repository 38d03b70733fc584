// hostrows.cu -- write pass over a host-mapped grid (zero-copy transport).
//
// Same cells and values as every other write-pass kernel (backends.py:158-222
// with the CONST _cell_value): the gasket cells of the grid, each written once.
// Only the schedule differs, because over PCIe the cost model changes
// (scripts/probe_sysmem.cu): reads travel in 64-byte units, small writes are
// TLP-rate bound, and accesses that hop to a new 4 KB host page every time run
// at a fraction of the link rate.  So the grid is walked row by row: in row
// y = 128*Y + y_lo the gasket's 128-byte tile lines are the lines l that are
// bit-subsets of Y (the lambda tiles of block row Y), and every one of them has
// the same in-line cell pattern (cells c subset of y_lo).  A work unit is one
// row and a chunk of K consecutive member lines; consecutive units cover
// consecutive lines of the same row, so host pages are hit K-at-a-time, and
// every line is read once, blended and written back whole.
#include <map>
#include <mutex>
#include <vector>

#include "gasket.cuh"
#include "launch.h"
#include "../../include/gasket_b200.h"

namespace gm {
namespace {

constexpr int K = 64;  // member lines per work unit (e2e n=2^16: 7.95 ms; 8.3 at K=32, 8.7 at K=8, 9.5 at K=4)

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

template <int C>
__device__ __forceinline__ uint32_t splat4(uint64_t p) {
    if constexpr (C == 1) return 0x01010101u * (uint32_t)(p & 0xffu);
    else if constexpr (C == 2) return 0x00010001u * (uint32_t)(p & 0xffffu);
    else return (uint32_t)p;
}

// cells of lane word w (4 bytes) that are gasket cells in a row with in-line pattern yl
template <int C>
__device__ __forceinline__ uint32_t word_mask(int w, uint32_t yl) {
    constexpr int V = 4 / C;
    if (((uint32_t)(w * V) & ~yl) != 0) return 0u;
    if constexpr (C == 1) {
        const uint32_t p = yl & 3u;
        return p == 0 ? 0x000000ffu : p == 1 ? 0x0000ffffu : p == 2 ? 0x00ff00ffu : 0xffffffffu;
    } else if constexpr (C == 2) {
        return (yl & 1u) ? 0xffffffffu : 0x0000ffffu;
    } else {
        return 0xffffffffu;
    }
}

// MODE 0: whole-line read-modify-write (host-mapped grids: PCIe moves 64-byte units)
// MODE 1: whole-sector read-modify-write of the touched sectors only (DRAM: no partial-sector fills)
// MODE 2: byte-masked stores of the gasket cells only (the L2 merges / read-modify-writes)
template <int C, int MODE>
__global__ void __launch_bounds__(256) host_rows_write(uint8_t* __restrict__ grid, int64_t n, int rbits,
                                                       const uint64_t* __restrict__ prefix, uint32_t nY,
                                                       uint64_t param) {
    constexpr int TT = 128 / C;  // cells per line
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total = prefix[nY];
    const uint32_t pv = splat4<C>(param);
    const int64_t rowstride = n * C;
    for (uint64_t u = warp0; u < total; u += nwarps) {
        // block row Y: largest Y with prefix[Y] <= u
        uint32_t lo = 0, hi = nY;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid;
        }
        const uint32_t Y = lo;
        const uint32_t lines = 1u << __popc(Y);
        const uint32_t chunks = (lines + K - 1) / K;
        const uint64_t rem = u - __ldg(prefix + Y);
        const uint32_t y_lo = (uint32_t)(rem / chunks);
        const uint32_t j = (uint32_t)(rem - (uint64_t)y_lo * chunks);
        const int64_t y = (int64_t)Y * TT + y_lo;
        const uint32_t m = word_mask<C>(lane, y_lo);
        uint8_t* row = grid + y * rowstride + lane * 4;
        const uint32_t i0 = j * K;
        const int cnt = (int)min((uint32_t)K, lines - i0);
        // sector of this lane's word holds gasket cells / is entirely gasket cells
        constexpr int SC = 32 / C;  // cells per sector
        const uint32_t g = (uint32_t)(lane * 4 / 32);
        const bool sec_touched = ((g * SC) & ~y_lo) == 0;
        const bool sec_full = ((g * SC + SC - 1) & ~y_lo) == 0;
        bool do_load, do_store;
        if constexpr (MODE == 0) {
            // whole 64-byte halves (the PCIe read unit) of the line that hold gasket cells
            const uint32_t half0 = (uint32_t)((lane * 4 / 64) * (64 / C));  // first cell of this lane's half
            const bool half_touched = (half0 & ~y_lo) == 0;
            do_load = half_touched && m != 0xffffffffu;
            do_store = half_touched;
        }
        else if constexpr (MODE == 1) { do_load = sec_touched && !sec_full; do_store = sec_touched; }
        else { do_load = false; do_store = m != 0u; }
        // line k of the unit: its offset from the row start is pdep(i0 + k, Y) * 128, kept as
        // 32-bit offsets (rows are < 2^31 bytes) so that K lines in flight stay in registers
        uint32_t old[K], off[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            off[k] = pdep(i0 + k, Y) * 128u;
            old[k] = 0u;
            if (k < cnt && do_load) old[k] = *reinterpret_cast<volatile uint32_t*>(row + off[k]);
        }
        if constexpr (MODE == 2) {
            // masked stores: the row's in-word pattern is uniform across the warp
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k >= cnt || !do_store) continue;
                uint8_t* b = row + off[k];
                if (m == 0xffffffffu) *reinterpret_cast<uint32_t*>(b) = pv;
                else if (m == 0x0000ffffu) *reinterpret_cast<uint16_t*>(b) = (uint16_t)pv;
                else if (m == 0x00ff00ffu) { b[0] = (uint8_t)pv; b[2] = (uint8_t)pv; }
                else b[0] = (uint8_t)pv;
            }
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (k < cnt && do_store)
                    *reinterpret_cast<uint32_t*>(row + off[k]) = (m == 0xffffffffu) ? pv : ((pv & m) | (old[k] & ~m));
        }
    }
}

// The write-back of a staged neighbour-sum launch (gm_writeback_tiles) in the same
// row-major walk: the member lines of each row go to the host whole, sector by sector
// from `dst` (sectors holding gasket cells: the kernel's results) or `snap` (the rest).
template <int C>
__global__ void __launch_bounds__(256) host_rows_copyback(uint8_t* __restrict__ out, const uint8_t* __restrict__ dst,
                                                          const uint8_t* __restrict__ snap, int64_t n,
                                                          const uint64_t* __restrict__ prefix, uint32_t nY) {
    constexpr int TT = 128 / C;
    constexpr int SC = 32 / C;  // cells per sector
    const int lane = threadIdx.x & 31;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total = prefix[nY];
    const int64_t rowstride = n * C;
    for (uint64_t u = warp0; u < total; u += nwarps) {
        uint32_t lo = 0, hi = nY;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid;
        }
        const uint32_t Y = lo;
        const uint32_t lines = 1u << __popc(Y);
        const uint32_t chunks = (lines + K - 1) / K;
        const uint64_t rem = u - __ldg(prefix + Y);
        const uint32_t y_lo = (uint32_t)(rem / chunks);
        const uint32_t j = (uint32_t)(rem - (uint64_t)y_lo * chunks);
        const int64_t rowoff = ((int64_t)Y * TT + y_lo) * rowstride + lane * 4;
        const uint32_t g = (uint32_t)(lane * 4 / 32);
        const uint8_t* from = (((g * SC) & ~y_lo) == 0) ? dst : snap;
        const uint32_t i0 = j * K;
        const int cnt = (int)min((uint32_t)K, lines - i0);
        uint32_t v[K], off[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            off[k] = pdep(i0 + k, Y) * 128u;
            if (k < cnt) v[k] = __ldcs(reinterpret_cast<const unsigned int*>(from + rowoff + off[k]));
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (k < cnt) *reinterpret_cast<uint32_t*>(out + rowoff + off[k]) = v[k];
    }
}

// MODE 0 with 16-byte lanes: 8 lanes per line, 4 lines per warp instruction, KL lines of
// a row per unit -- twice the lines in flight per warp for the same registers
constexpr int KL = 128;
template <int C>
__global__ void __launch_bounds__(256) host_rows_write16(uint8_t* __restrict__ grid, int64_t n,
                                                         const uint64_t* __restrict__ prefix, uint32_t nY,
                                                         uint64_t param, int zero_bg) {
    constexpr int TT = 128 / C;
    constexpr int PER = KL / 4;  // lines per lane per unit
    const int lane = threadIdx.x & 31;
    const int sub = lane >> 3, q = lane & 7;  // line of the group of 4, 16-byte chunk of the line
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total = prefix[nY];
    const uint32_t pv = splat4<C>(param);
    const int64_t rowstride = n * C;
    for (uint64_t u = warp0; u < total; u += nwarps) {
        uint32_t lo = 0, hi = nY;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid;
        }
        const uint32_t Y = lo;
        const uint32_t lines = 1u << __popc(Y);
        const uint32_t chunks = (lines + KL - 1) / KL;
        const uint64_t rem = u - __ldg(prefix + Y);
        const uint32_t y_lo = (uint32_t)(rem / chunks);
        const uint32_t j = (uint32_t)(rem - (uint64_t)y_lo * chunks);
        uint8_t* row = grid + ((int64_t)Y * TT + y_lo) * rowstride + q * 16;
        const uint32_t i0 = j * KL;
        const int cnt = (int)min((uint32_t)KL, lines - i0);
        // this lane's 4 words (cells 4q*V/4 ..) and its 64-byte half (the PCIe read unit)
        uint32_t m[4];
        bool full = true;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            m[w] = word_mask<C>(4 * q + w, y_lo);
            full = full && m[w] == 0xffffffffu;
        }
        const bool half_touched = (((uint32_t)(q >> 2) * (64 / C)) & ~y_lo) == 0;
        // GM_FLAG_ZERO_BACKGROUND: the off-gasket cells are 0, nothing to read back
        const bool do_load = half_touched && !full && !zero_bg;
        uint4 old[PER];
        uint32_t off[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int k = 4 * i + sub;
            off[i] = pdep(i0 + k, Y) * 128u;
            old[i] = make_uint4(0, 0, 0, 0);
            if (k < cnt && do_load) old[i] = __ldcv(reinterpret_cast<const uint4*>(row + off[i]));
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int k = 4 * i + sub;
            if (k < cnt && half_touched)
                *reinterpret_cast<uint4*>(row + off[i]) =
                    make_uint4((pv & m[0]) | (old[i].x & ~m[0]), (pv & m[1]) | (old[i].y & ~m[1]),
                               (pv & m[2]) | (old[i].z & ~m[2]), (pv & m[3]) | (old[i].w & ~m[3]));
        }
    }
}

// host_rows_write16 for a grid whose base is not 128-byte aligned (a plain numpy array:
// malloc puts the data 16 bytes into a page).  PCIe moves host-aligned 64-byte units, so a
// grid line that straddles two host lines would cost two reads and two writes per half.
// Here every job is one HOST-aligned 128-byte line, decoded chunk by chunk (16-byte lanes,
// flat chunk index f from the array start; a host line starts where f = -s16 mod 8):
//   job A of member line X of row y: host line [128X - s, 128X - s + 128) of the row -- the
//     first 128 - s bytes of line X and the last s bytes of the line before it (previous
//     row's last line when X = 0);
//   job B: host line X + 1, only when it holds bytes of line X that no job A covers (line
//     X + 1 of the row is not a member line; the grid's very last line).
// Each host line is written by exactly one job; chunks outside the array are never read
// or written.  Per host 64-byte half: stored whole (reading the chunks that are not all
// gasket cells) when any of its chunks holds gasket cells.
constexpr int KLS = 64;  // member lines per unit (two host lines each: half of KL's registers)
template <int C>
__global__ void __launch_bounds__(256) host_rows_write16_shift(uint8_t* __restrict__ grid, int64_t n,
                                                               const uint64_t* __restrict__ prefix, uint32_t nY,
                                                               uint64_t param, int zero_bg, int s16) {
    constexpr int TT = 128 / C;
    constexpr int PER = KLS / 4;
    const int lane = threadIdx.x & 31;
    const int sub = lane >> 3, j = lane & 7;
    const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total = prefix[nY];
    const uint32_t pv = splat4<C>(param);
    const int64_t cpr = n * C / 16;          // chunks per row
    const int64_t nchunks = cpr * n;
    int cpr_shift = 0;
    while ((int64_t(1) << cpr_shift) < cpr) ++cpr_shift;
    const uint32_t nL = (uint32_t)(n / TT);  // lines per row
    // chunk f (flat) -> 4 word masks of its gasket cells; false if outside the array
    auto decode = [&](int64_t f, uint32_t (&m)[4]) -> bool {
        if (f < 0 || f >= nchunks) return false;
        const int64_t y = f >> cpr_shift;
        const uint32_t cidx = (uint32_t)(f & (cpr - 1));
        const uint32_t L = cidx >> 3, q = cidx & 7u;
        const uint32_t Yr = (uint32_t)(y >> (__ffs(TT) - 1)), yl = (uint32_t)(y & (TT - 1));
        const bool mem = (L & ~Yr) == 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) m[w] = mem ? word_mask<C>(4 * (int)q + w, yl) : 0u;
        return true;
    };
    for (uint64_t u = warp0; u < total; u += nwarps) {
        uint32_t lo = 0, hi = nY;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid;
        }
        const uint32_t Y = lo;
        const uint32_t lines = 1u << __popc(Y);
        const uint32_t chunks = (lines + KLS - 1) / KLS;
        const uint64_t rem = u - __ldg(prefix + Y);
        const uint32_t y_lo = (uint32_t)(rem / chunks);
        const uint32_t jj = (uint32_t)(rem - (uint64_t)y_lo * chunks);
        const int64_t y = (int64_t)Y * TT + y_lo;
        const uint32_t i0 = jj * KLS;
        const int cnt = (int)min((uint32_t)KLS, lines - i0);
        uint4 oldA[PER], oldB[PER];
        uint32_t mA[PER][4], mB[PER][4];
        int64_t fA[PER];
        bool stA[PER], stB[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int k = 4 * i + sub;
            const uint32_t X = pdep(i0 + (uint32_t)k, Y);
            const bool valid = k < cnt;
            fA[i] = y * cpr + 8 * (int64_t)X - s16 + j;
            const bool inA = valid && decode(fA[i], mA[i]);
            // job B: host line X + 1 holds the tail of line X that no job A covers
            const bool needB = valid && (((X + 1) & ~Y) != 0 || X + 1 == nL) && !(X + 1 == nL && y + 1 < n);
            const bool inB = needB && j < s16 && decode(fA[i] + 8, mB[i]);
            if (!inB) mB[i][0] = mB[i][1] = mB[i][2] = mB[i][3] = 0u;
            if (!inA) mA[i][0] = mA[i][1] = mA[i][2] = mA[i][3] = 0u;
            // host 64-byte half (4 lanes) holds gasket cells -> stored whole
            const bool tA = (mA[i][0] | mA[i][1] | mA[i][2] | mA[i][3]) != 0;
            const bool tB = (mB[i][0] | mB[i][1] | mB[i][2] | mB[i][3]) != 0;
            const unsigned ba = __ballot_sync(0xffffffffu, tA), bb = __ballot_sync(0xffffffffu, tB);
            const unsigned hm = 0xfu << (lane & ~3);
            stA[i] = inA && (ba & hm) != 0;
            // job B: only the chunks of line X (j < s16) of the host line's first half(s)
            stB[i] = inB && (bb & hm) != 0;
            const bool fullA = (mA[i][0] & mA[i][1] & mA[i][2] & mA[i][3]) == 0xffffffffu;
            const bool fullB = (mB[i][0] & mB[i][1] & mB[i][2] & mB[i][3]) == 0xffffffffu;
            oldA[i] = make_uint4(0, 0, 0, 0);
            oldB[i] = make_uint4(0, 0, 0, 0);
            if (stA[i] && !fullA && !zero_bg) oldA[i] = __ldcv(reinterpret_cast<const uint4*>(grid + fA[i] * 16));
            if (stB[i] && !fullB && !zero_bg) oldB[i] = __ldcv(reinterpret_cast<const uint4*>(grid + (fA[i] + 8) * 16));
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            if (stA[i])
                *reinterpret_cast<uint4*>(grid + fA[i] * 16) =
                    make_uint4((pv & mA[i][0]) | (oldA[i].x & ~mA[i][0]), (pv & mA[i][1]) | (oldA[i].y & ~mA[i][1]),
                               (pv & mA[i][2]) | (oldA[i].z & ~mA[i][2]), (pv & mA[i][3]) | (oldA[i].w & ~mA[i][3]));
            if (stB[i])
                *reinterpret_cast<uint4*>(grid + (fA[i] + 8) * 16) =
                    make_uint4((pv & mB[i][0]) | (oldB[i].x & ~mB[i][0]), (pv & mB[i][1]) | (oldB[i].y & ~mB[i][1]),
                               (pv & mB[i][2]) | (oldB[i].z & ~mB[i][2]), (pv & mB[i][3]) | (oldB[i].w & ~mB[i][3]));
        }
    }
}

std::mutex g_mu;
std::map<std::pair<int, int>, uint64_t*> g_prefix;  // (device, nYbits*1024 + rows per block row) -> table

uint64_t* prefix_table(int nYbits, int rows, uint32_t& nY, int kl = K) {
    nY = 1u << nYbits;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    const int key = (kl * 64 + nYbits) * 1024 + rows;
    auto it = g_prefix.find({dev, key});
    if (it != g_prefix.end()) return it->second;
    std::vector<uint64_t> pre(nY + 1, 0);
    for (uint32_t Y = 0; Y < nY; ++Y) {
        const uint64_t lines = 1ull << __builtin_popcount(Y);
        pre[Y + 1] = pre[Y] + (uint64_t)((lines + kl - 1) / kl) * rows;  // rows per block row = tile edge
    }
    uint64_t* d = nullptr;
    if (cudaMalloc(&d, pre.size() * sizeof(uint64_t)) != cudaSuccess) return nullptr;
    cudaMemcpy(d, pre.data(), pre.size() * sizeof(uint64_t), cudaMemcpyHostToDevice);
    g_prefix[{dev, key}] = d;
    return d;
}

template <int C>
cudaError_t launch_c(const LaunchArgs& a, int r) {
    const int mode = !(a.flags & GM_FLAG_EXPLICIT_RMW) ? 2 : (a.flags & GM_FLAG_WHOLE_LINES) ? 0 : 1;
    constexpr int TT = 128 / C;
    int k = 0;
    while ((1 << k) < TT) ++k;
    uint32_t nY;
    uint64_t* pre = prefix_table(r - k, TT, nY);
    if (!pre) return cudaErrorMemoryAllocation;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint8_t* g = reinterpret_cast<uint8_t*>(a.grid);
    const int shift = (int)(reinterpret_cast<uintptr_t>(a.grid) & 127u);
    if (mode == 0 && shift != 0 && shift % 16 == 0 && C <= 4) {
        // a grid that does not start on a 128-byte boundary: host-aligned jobs
        uint32_t nYs;
        uint64_t* pres = prefix_table(r - k, TT, nYs, KLS);
        if (!pres) return cudaErrorMemoryAllocation;
        host_rows_write16_shift<C><<<sms * 8, 256, 0, a.stream>>>(g, a.n, pres, nYs, a.param,
                                                                  (a.flags & GM_FLAG_ZERO_BACKGROUND) ? 1 : 0,
                                                                  shift / 16);
    } else if (mode == 0) {
        uint32_t nY16;
        uint64_t* pre16 = prefix_table(r - k, TT, nY16, KL);
        if (!pre16) return cudaErrorMemoryAllocation;
        host_rows_write16<C><<<sms * 8, 256, 0, a.stream>>>(g, a.n, pre16, nY16, a.param,
                                                            (a.flags & GM_FLAG_ZERO_BACKGROUND) ? 1 : 0);
    }
    else if (mode == 1) host_rows_write<C, 1><<<sms * 8, 256, 0, a.stream>>>(g, a.n, r, pre, nY, a.param);
    else host_rows_write<C, 2><<<sms * 8, 256, 0, a.stream>>>(g, a.n, r, pre, nY, a.param);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

template <int C>
cudaError_t launch_copyback_c(void* out, const void* dst, const void* snap, int64_t n, int r, cudaStream_t s) {
    constexpr int TT = 128 / C;
    int k = 0;
    while ((1 << k) < TT) ++k;
    uint32_t nY;
    uint64_t* pre = prefix_table(r - k, TT, nY);
    if (!pre) return cudaErrorMemoryAllocation;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    host_rows_copyback<C><<<sms * 8, 256, 0, s>>>(reinterpret_cast<uint8_t*>(out),
                                                  reinterpret_cast<const uint8_t*>(dst),
                                                  reinterpret_cast<const uint8_t*>(snap), n, pre, nY);
    note_launch();
    return cudaGetLastError();
}

// Row-ordered write-back of the member tiles' own lines (1/2/4-byte cells, n >= one
// 128-byte line, power of two); cudaErrorNotSupported otherwise.
cudaError_t launch_host_rows_copyback(void* out, const void* dst, const void* snap, int64_t n, int cell_bytes,
                                      cudaStream_t s) {
    if (n < 1 || (n & (n - 1)) != 0) return cudaErrorNotSupported;
    int r = 0;
    while ((int64_t(1) << r) < n) ++r;
    switch (cell_bytes) {
    case 1: if (n >= 128) return launch_copyback_c<1>(out, dst, snap, n, r, s); break;
    case 2: if (n >= 64) return launch_copyback_c<2>(out, dst, snap, n, r, s); break;
    case 4: if (n >= 32) return launch_copyback_c<4>(out, dst, snap, n, r, s); break;
    }
    return cudaErrorNotSupported;
}

// CONST write pass on a grid at least one 128-byte line wide with 1/2/4-byte cells.
cudaError_t launch_host_rows(const LaunchArgs& a) {
    if (a.kind != KIND_CONST || a.part_level >= 0) return cudaErrorNotSupported;
    int r = 0;
    while ((int64_t(1) << r) < a.n) ++r;
    switch (a.cell_bytes) {
    case 1: if (a.n >= 128) return launch_c<1>(a, r); break;
    case 2: if (a.n >= 64) return launch_c<2>(a, r); break;
    case 4: if (a.n >= 32) return launch_c<4>(a, r); break;
    }
    return cudaErrorNotSupported;
}

}  // namespace gm
