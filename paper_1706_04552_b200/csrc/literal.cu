// literal.cu -- paper-literal launch shapes, one CUDA block
// per reference block, exactly as the numba kernels walk them:
//   * bb_literal      <- backends.py:143-156 _bounding_box_nb: n_b x n_b blocks of
//                        rho x rho threads, each thread tests x & (n-1-y).
//     (EXIT variant: the block first tests bx & (n_b-1-by) -- the "fair" BB of
//      SURVEY §7 hard part 5 -- and exits as a whole.)
//   * lambda_literal  <- backends.py:158-222 _block_space_nb: 3^floor(r_b/2) x
//                        3^ceil(r_b/2) blocks; lambda(omega) computed once per
//                        block by warp 0 (lane per level + redux.sync.or, the
//                        paper's warp-shuffle reduction), broadcast through
//                        shared memory, then the intra-block strategy:
//                        SUBBOX (rho x rho threads, tx & (rho-1-ty)),
//                        TABLE (3^k threads reading the shared lookup table),
//                        UNROLL (3^k threads re-running lambda at tile scale).
// Blocks with more than 1024 natural threads (rho > 32, or 3^k > 1024) loop.
#include "gasket.cuh"
#include "launch.h"

namespace gm {

struct Pow3Magic {
    uint64_t m[21];
    constexpr Pow3Magic() : m() {
        uint64_t p = 1;
        for (int d = 0; d < 21; ++d) {
            m[d] = d == 0 ? 0ull : (~0ull / p) + 1ull;
            p *= 3ull;
        }
    }
};
__device__ const Pow3Magic g_pow3 = Pow3Magic();

template <int C, int KIND, bool EXIT>
__global__ void bb_literal(void* __restrict__ grid, const void* __restrict__ src, int64_t n, int rho,
                           int64_t nb, uint64_t param) {
    const int64_t bx = blockIdx.x;
    const int64_t by = (int64_t)blockIdx.z * gridDim.y + blockIdx.y;
    if (EXIT && (bx & (nb - 1 - by)) != 0) return;  // tile holds no gasket cell
    for (int ty = threadIdx.y; ty < rho; ty += blockDim.y) {
        const int64_t y = by * rho + ty;
        const int64_t m = n - 1 - y;
        for (int tx = threadIdx.x; tx < rho; tx += blockDim.x) {
            const int64_t x = bx * rho + tx;
            if ((x & m) == 0) cell_op<C, KIND>(grid, src, n, x, y, param);
        }
    }
}

// Block-level lambda: warp 0 cooperates, result broadcast via shared memory.
__device__ __forceinline__ void block_lambda(int r_b, uint32_t& ox, uint32_t& oy) {
    __shared__ uint32_t s_l[2];
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    const int nthreads = blockDim.x * blockDim.y;
    if (tid < 32) {
        const int lanes = nthreads < 32 ? nthreads : 32;
        uint32_t lx, ly;
        lambda_warp(blockIdx.x, blockIdx.y, r_b, tid, lanes, g_pow3.m, lx, ly);
        if (tid == 0) { s_l[0] = lx; s_l[1] = ly; }
    }
    __syncthreads();
    ox = s_l[0];
    oy = s_l[1];
}

template <int C, int KIND>
__global__ void lambda_subbox(void* __restrict__ grid, const void* __restrict__ src, int64_t n, int rho,
                              int r_b, uint64_t param) {
    uint32_t lx, ly;
    block_lambda(r_b, lx, ly);
    const int64_t ox = (int64_t)lx * rho, oy = (int64_t)ly * rho;
    for (int ty = threadIdx.y; ty < rho; ty += blockDim.y) {
        const int m = rho - 1 - ty;
        for (int tx = threadIdx.x; tx < rho; tx += blockDim.x)
            if ((tx & m) == 0) cell_op<C, KIND>(grid, src, n, ox + tx, oy + ty, param);
    }
}

template <int C, int KIND>
__global__ void lambda_table(void* __restrict__ grid, const void* __restrict__ src, int64_t n, int rho,
                             int r_b, const int32_t* __restrict__ tab_x, const int32_t* __restrict__ tab_y,
                             int ntab, uint64_t param) {
    uint32_t lx, ly;
    block_lambda(r_b, lx, ly);
    const int64_t ox = (int64_t)lx * rho, oy = (int64_t)ly * rho;
    for (int i = threadIdx.x; i < ntab; i += blockDim.x)
        cell_op<C, KIND>(grid, src, n, ox + __ldg(tab_x + i), oy + __ldg(tab_y + i), param);
}

template <int C, int KIND>
__global__ void lambda_unroll(void* __restrict__ grid, const void* __restrict__ src, int64_t n, int rho,
                              int r_b, int r_p, int t_width, int n_threads, uint64_t param) {
    uint32_t lx, ly;
    block_lambda(r_b, lx, ly);
    const int64_t ox = (int64_t)lx * rho, oy = (int64_t)ly * rho;
    for (int t = threadIdx.x; t < n_threads; t += blockDim.x) {
        // backends.py:201-219: thread t = (tx, ty) on the packing_dims(r_p) grid re-runs lambda.
        int ty = t / t_width, tx = t - (t / t_width) * t_width;
        int sx = 0, sy = 0;
        for (int mu = 1; mu <= r_p; ++mu) {
            int region;
            if (mu & 1) { region = ty % 3; ty /= 3; }
            else        { region = tx % 3; tx /= 3; }
            const int dx = region >> 1;
            sx += dx << (mu - 1);
            sy += (region - dx) << (mu - 1);
        }
        cell_op<C, KIND>(grid, src, n, ox + sx, oy + sy, param);
    }
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------

template <int C, int KIND>
static cudaError_t launch_bb_t(const LaunchArgs& a) {
    const int64_t nb = a.n / a.rho;
    const int bdim = a.rho < 32 ? a.rho : 32;
    // gridDim.y/z <= 65535: fold the block row index over y and z.
    const int64_t gy = nb < 32768 ? nb : 32768;
    const dim3 grid((unsigned)nb, (unsigned)gy, (unsigned)(nb / gy));
    const dim3 block(bdim, bdim);
    if (a.mapping == MAP_BB_EXIT)
        bb_literal<C, KIND, true><<<grid, block, 0, a.stream>>>(a.grid, a.src, a.n, a.rho, nb, a.param);
    else
        bb_literal<C, KIND, false><<<grid, block, 0, a.stream>>>(a.grid, a.src, a.n, a.rho, nb, a.param);
    note_launch();
    return cudaGetLastError();
}

template <int C, int KIND>
static cudaError_t launch_lambda_t(const LaunchArgs& a) {
    const dim3 grid((unsigned)a.width, (unsigned)a.height);
    switch (a.strategy) {
    case STRAT_SUBBOX: {
        const int bdim = a.rho < 32 ? a.rho : 32;
        lambda_subbox<C, KIND><<<grid, dim3(bdim, bdim), 0, a.stream>>>(a.grid, a.src, a.n, a.rho, a.r_b, a.param);
        break;
    }
    case STRAT_TABLE: {
        const int threads = a.ntab < 1024 ? (a.ntab > 0 ? a.ntab : 1) : 1024;
        lambda_table<C, KIND><<<grid, threads, 0, a.stream>>>(a.grid, a.src, a.n, a.rho, a.r_b, a.tab_x, a.tab_y,
                                                               a.ntab, a.param);
        break;
    }
    case STRAT_UNROLL: {
        int r_p = 0;
        while ((1 << r_p) < a.rho) ++r_p;
        int t_width = 1, n_threads = 1;
        for (int i = 0; i < r_p / 2; ++i) t_width *= 3;
        for (int i = 0; i < r_p; ++i) n_threads *= 3;
        const int threads = n_threads < 1024 ? n_threads : 1024;
        lambda_unroll<C, KIND><<<grid, threads, 0, a.stream>>>(a.grid, a.src, a.n, a.rho, a.r_b, r_p, t_width,
                                                                n_threads, a.param);
        break;
    }
    default:
        return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

#define GM_DISPATCH_KIND(FN, C, a)                                       \
    switch ((a).kind) {                                                  \
    case KIND_CONST: return FN<C, KIND_CONST>(a);                        \
    case KIND_NSUM4: return FN<C, KIND_NSUM4>(a);                        \
    case KIND_NSUM8: return FN<C, KIND_NSUM8>(a);                        \
    case KIND_COUNT: return FN<4, KIND_COUNT>(a);                        \
    }                                                                    \
    return cudaErrorInvalidValue;

template <int C>
static cudaError_t launch_bb_c(const LaunchArgs& a) { GM_DISPATCH_KIND(launch_bb_t, C, a) }
template <int C>
static cudaError_t launch_lambda_c(const LaunchArgs& a) { GM_DISPATCH_KIND(launch_lambda_t, C, a) }

cudaError_t launch_literal(const LaunchArgs& a) {
    if (a.mapping == MAP_BB_VEC) {
        // the bounding box written like the tuned kernels: the write pass over 16-byte segments
        // (write.cu), neighbour sums as the tuned tile stencil over every tile of the grid
        // (stencil2.cu); grids those do not cover take the literal bounding box
        const cudaError_t e = (a.kind == KIND_NSUM4 || a.kind == KIND_NSUM8) ? launch_stencil_v2(a) : launch_bb_vector(a);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
    }
    const bool bb = a.mapping == MAP_BB || a.mapping == MAP_BB_EXIT || a.mapping == MAP_BB_VEC;
    switch (a.cell_bytes) {
    case 1: return bb ? launch_bb_c<1>(a) : launch_lambda_c<1>(a);
    case 2: return bb ? launch_bb_c<2>(a) : launch_lambda_c<2>(a);
    case 4: return bb ? launch_bb_c<4>(a) : launch_lambda_c<4>(a);
    case 8: return bb ? launch_bb_c<8>(a) : launch_lambda_c<8>(a);
    }
    return cudaErrorInvalidValue;
}

}  // namespace gm
