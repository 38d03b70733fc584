#include <tuple>
#include <set>
#include <mutex>
#include <cstdlib>
#include <algorithm>
// capi.cu -- extern "C" drop-in boundary (include/gasket_b200.h).
//
// Validation mirrors the reference's ValueError conditions (core.py:40-41,
// 46-47, 121-124; engine.py:53-54, 198-199) so the Python layer can re-raise
// them with the reference's messages; no entry point falls back to the CPU.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/gasket_b200.h"
#include "gasket.cuh"
#include "launch.h"

namespace gm {
cudaError_t launch_map_blocks(const int64_t*, const int64_t*, int64_t, int, int64_t*, int64_t*, cudaStream_t);
cudaError_t launch_map_rectangle(int, int64_t*, int64_t*, cudaStream_t);
cudaError_t launch_bijection(const int64_t*, const int64_t*, int64_t, int64_t, int64_t*, int64_t*, cudaStream_t);
cudaError_t launch_coverage_blocks(const int64_t*, const int64_t*, int64_t, const int32_t*, const int32_t*, int, int,
                                   int64_t, uint32_t*, cudaStream_t);
cudaError_t launch_fill_hash(void*, int64_t, int, uint64_t, int, cudaStream_t);
cudaError_t launch_coverage_check(const uint32_t*, int64_t, unsigned long long*, int64_t*, int64_t*, int64_t,
                                  cudaStream_t);
cudaError_t launch_checksum(const void*, int64_t, int, uint64_t*, cudaStream_t);
cudaError_t launch_count_equal(const void*, const void*, int64_t, unsigned long long*, cudaStream_t);
cudaError_t launch_l2_flush(const void*, int64_t, uint64_t*, cudaStream_t);
cudaError_t launch_gather(const void*, int, const int64_t*, int64_t, void*, cudaStream_t);
cudaError_t launch_scatter(void*, int, const int64_t*, int64_t, const void*, cudaStream_t);
cudaError_t launch_copy_cells(void*, const void*, int, const int64_t*, const int64_t*, int64_t, cudaStream_t);
cudaError_t launch_fill_hash_window(void*, int64_t, int64_t, int, int64_t, int64_t, int64_t, int64_t, uint64_t, int,
                                    cudaStream_t);

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace gm

namespace {
thread_local std::string t_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

int cuda_rc(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return GM_OK;
    return fail(GM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }
int log2i(int64_t v) {
    int r = 0;
    while ((int64_t(1) << r) < v) ++r;
    return r;
}

int check_common(int64_t n, int32_t cell_bytes, int32_t rho, int32_t kind) {
    if (!pow2(n)) return fail(GM_EINVAL, "edge length must be a power of two >= 1, got %lld", (long long)n);
    if (log2i(n) > 40) return fail(GM_EINVAL, "scale level must be in [0, 40], got %d", log2i(n));
    if (rho < 1 || (rho & (rho - 1))) return fail(GM_EINVAL, "block edge must be a power of two >= 1, got %d", rho);
    if (rho > n) return fail(GM_EINVAL, "block edge %d exceeds grid edge %lld", rho, (long long)n);
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4 && cell_bytes != 8)
        return fail(GM_EINVAL, "cell width must be 1, 2, 4 or 8 bytes, got %d", cell_bytes);
    if (kind < GM_KIND_CONST || kind > GM_KIND_COUNT) return fail(GM_EINVAL, "unknown kernel kind %d", kind);
    return GM_OK;
}

int run(const gm::LaunchArgs& a) {
    cudaError_t e;
    if (a.mapping == GM_MAP_LAMBDA && a.strategy == GM_STRAT_TUNED)
        e = gm::launch_tuned(a);
    else
        e = gm::launch_literal(a);
    return cuda_rc(e, "kernel launch");
}

gm::LaunchArgs make_args(const gm_cfg_t* c, void* grid, const void* src, const int32_t* tx, const int32_t* ty,
                         int32_t ntab, void* stream) {
    gm::LaunchArgs a{};
    a.grid = grid;
    a.src = src;
    a.n = c->n;
    a.rho = c->rho;
    a.r_b = log2i(c->n / c->rho);
    a.width = 1;
    a.height = 1;
    for (int i = 0; i < a.r_b / 2; ++i) a.width *= 3;
    for (int i = 0; i < (a.r_b + 1) / 2; ++i) a.height *= 3;
    a.mapping = c->mapping;
    a.strategy = c->strategy;
    a.kind = c->kind;
    a.cell_bytes = c->cell_bytes;
    a.param = (uint64_t)(int64_t)c->param;
    a.tab_x = tx;
    a.tab_y = ty;
    a.ntab = ntab;
    a.flags = c->flags;
    a.stream = reinterpret_cast<cudaStream_t>(stream);
    return a;
}

int launch_cfg(const gm_cfg_t* c, void* grid, const void* src, const int32_t* tx, const int32_t* ty, int32_t ntab,
               void* stream) {
    if (!c) return fail(GM_EINVAL, "null config");
    if (int rc = check_common(c->n, c->cell_bytes, c->rho, c->kind)) return rc;
    if (!grid) return fail(GM_EINVAL, "null grid");
    if (c->kind != GM_KIND_CONST && c->kind != GM_KIND_COUNT) {
        if (!src) return fail(GM_EINVAL, "neighbour kernels need a src snapshot");
        if (src == grid)
            return fail(GM_EINVAL, "neighbour kernels read the pre-launch snapshot: src must not alias grid");
    }
    if (c->mapping != GM_MAP_BB && c->mapping != GM_MAP_LAMBDA && c->mapping != GM_MAP_BB_EXIT &&
        c->mapping != GM_MAP_BB_VEC)
        return fail(GM_EINVAL, "unknown mapping %d", c->mapping);
    const int r_b = log2i(c->n / c->rho);
    if (c->mapping == GM_MAP_LAMBDA) {
        if (c->strategy < GM_STRAT_UNROLL || c->strategy > GM_STRAT_TUNED)
            return fail(GM_EINVAL, "block-space launches need an intra-block strategy (got %d)", c->strategy);
        if (r_b > 20) return fail(GM_EINVAL, "block-space level r_b=%d exceeds the device limit 20", r_b);
        if (c->strategy == GM_STRAT_TABLE && ntab > 0 && (!tx || !ty))
            return fail(GM_EINVAL, "TABLE strategy needs the lookup table");
    } else {
        if (log2i(c->n) > 31) return fail(GM_EINVAL, "bounding-box grid edge 2^%d exceeds the device limit", log2i(c->n));
    }
    return run(make_args(c, grid, src, tx, ty, ntab, stream));
}

}  // namespace

namespace gm {
void ensure_dynamic_smem(const void* kern, size_t smem) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, size_t>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert(std::make_tuple(kern, dev, smem)).second) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        // the largest shared-memory carveout: the tiled kernels size their CTAs so that
        // several share an SM's shared memory (the driver's default choice may not)
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    }
}

int order_level(const LaunchArgs& a, int r_t) {
    if (a.part_level >= 0) return a.part_level;
    static const int env = [] {
        const char* e = getenv("GASKET_TILE_ORDER_LEVEL");
        return e ? atoi(e) : 0;
    }();
    return env < 0 ? 0 : (env > r_t ? r_t : env);
}
}  // namespace gm

extern "C" {

int gm_launch(const gm_cfg_t* cfg, void* grid, const void* src, const int32_t* tab_x, const int32_t* tab_y,
              int32_t ntab, void* stream) {
    return launch_cfg(cfg, grid, src, tab_x, tab_y, ntab, stream);
}

int gm_run_bounding_box(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t rho, int32_t kind,
                        int32_t param, int32_t early_exit, void* stream) {
    gm_cfg_t c{};
    c.n = n;
    c.rho = rho;
    if (early_exit == 2 && kind == GM_KIND_COUNT)
        return fail(GM_EINVAL, "the vectorised bounding box has no coverage-counting form");
    c.mapping = early_exit == 2 ? GM_MAP_BB_VEC : early_exit ? GM_MAP_BB_EXIT : GM_MAP_BB;
    c.strategy = GM_STRAT_SUBBOX;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    return launch_cfg(&c, grid, src, nullptr, nullptr, 0, stream);
}

int gm_run_block_space(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t rho, int32_t r_b,
                       int32_t strategy, const int32_t* tab_x, const int32_t* tab_y, int32_t ntab, int32_t kind,
                       int32_t param, int32_t flags, void* stream) {
    if (pow2(n) && pow2(rho) && rho <= n && log2i(n / rho) != r_b)
        return fail(GM_EINVAL, "r_b=%d does not match n=%lld, rho=%d", r_b, (long long)n, rho);
    gm_cfg_t c{};
    c.n = n;
    c.rho = rho;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = strategy;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    c.flags = flags;
    return launch_cfg(&c, grid, src, tab_x, tab_y, ntab, stream);
}

int gm_run_part(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* stream) {
    gm_cfg_t c{};
    c.n = n;
    c.rho = 1;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = GM_STRAT_TUNED;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    c.flags = flags & ~GM_FLAG_OMEGA_ORDER;  // partitions are digit-order ranges
    if (int rc = check_common(n, cell_bytes, 1, kind)) return rc;
    if (!grid) return fail(GM_EINVAL, "null grid");
    if (kind != GM_KIND_CONST && (!src || src == grid))
        return fail(GM_EINVAL, "neighbour kernels need a separate src snapshot");
    const int r = log2i(n);
    // the tuned kernels tile at 128-byte rows: a sub-gasket must hold whole tiles
    const int64_t tile = cell_bytes <= 4 ? 128 / cell_bytes : 32;
    if (level < 0 || (n >> level) < tile)
        return fail(GM_EINVAL, "partition level %d too deep for n=2^%d (sub-gaskets narrower than a tile)", level, r);
    uint64_t nsg = 1;
    for (int i = 0; i < level; ++i) nsg *= 3;
    if (sg_begin > sg_end || sg_end > nsg) return fail(GM_EINVAL, "sub-gasket range [%u, %u) outside [0, %llu)",
                                                       sg_begin, sg_end, (unsigned long long)nsg);
    gm::LaunchArgs a = make_args(&c, grid, src, nullptr, nullptr, 0, stream);
    a.part_level = level;
    a.sg_begin = sg_begin;
    a.sg_end = sg_end;
    return cuda_rc(gm::launch_tuned(a), "partition launch");
}

int gm_gather_cells(const void* grid, int32_t cell_bytes, const int64_t* idx, int64_t count, void* out, void* stream) {
    return cuda_rc(gm::launch_gather(grid, cell_bytes, idx, count, out, reinterpret_cast<cudaStream_t>(stream)),
                   "gather_cells");
}

int gm_scatter_cells(void* grid, int32_t cell_bytes, const int64_t* idx, int64_t count, const void* in,
                     void* stream) {
    return cuda_rc(gm::launch_scatter(grid, cell_bytes, idx, count, in, reinterpret_cast<cudaStream_t>(stream)),
                   "scatter_cells");
}

int gm_map_blocks(const int64_t* wx, const int64_t* wy, int64_t count, int32_t r_b, int64_t* lx, int64_t* ly,
                  void* stream) {
    if (count < 0) return fail(GM_EINVAL, "negative count");
    if (r_b < 0 || r_b > 62) return fail(GM_EINVAL, "scale level r_b must be in [0, 62], got %d", r_b);
    if (count && (!wx || !wy || !lx || !ly)) return fail(GM_EINVAL, "null array");
    return cuda_rc(gm::launch_map_blocks(wx, wy, count, r_b, lx, ly, reinterpret_cast<cudaStream_t>(stream)),
                   "map_blocks");
}

int gm_map_rectangle(int32_t r_b, int64_t* lx, int64_t* ly, void* stream) {
    if (r_b < 0 || r_b > 40) return fail(GM_EINVAL, "scale level must be in [0, 40], got %d", r_b);
    if (!lx || !ly) return fail(GM_EINVAL, "null array");
    return cuda_rc(gm::launch_map_rectangle(r_b, lx, ly, reinterpret_cast<cudaStream_t>(stream)), "map_rectangle");
}

int gm_coverage(const gm_cfg_t* cfg, uint32_t* counts, const int32_t* tab_x, const int32_t* tab_y, int32_t ntab,
                void* stream) {
    if (!cfg) return fail(GM_EINVAL, "null config");
    gm_cfg_t c = *cfg;
    c.kind = GM_KIND_COUNT;
    c.cell_bytes = 4;
    return launch_cfg(&c, counts, nullptr, tab_x, tab_y, ntab, stream);
}

int gm_coverage_blocks(const int64_t* bx, const int64_t* by, int64_t nblocks, const int32_t* lx, const int32_t* ly,
                       int32_t nlocal, int32_t rho, int64_t n, uint32_t* counts, void* stream) {
    if (nblocks < 0 || nlocal < 0 || rho < 1 || n < 1) return fail(GM_EINVAL, "bad coverage shape");
    return cuda_rc(gm::launch_coverage_blocks(bx, by, nblocks, lx, ly, nlocal, rho, n, counts,
                                              reinterpret_cast<cudaStream_t>(stream)),
                   "coverage_blocks");
}

int gm_coverage_check(const uint32_t* counts, int64_t n, unsigned long long* totals, int64_t* dup_idx,
                      int64_t* miss_idx, int64_t cap, void* stream) {
    if (!counts || !totals || (cap > 0 && (!dup_idx || !miss_idx)) || cap < 0)
        return fail(GM_EINVAL, "gm_coverage_check: bad buffers");
    if (!pow2(n) || n < 2) return fail(GM_EINVAL, "gm_coverage_check: edge must be a power of two >= 2");
    return cuda_rc(gm::launch_coverage_check(counts, n, totals, dup_idx, miss_idx, cap,
                                             reinterpret_cast<cudaStream_t>(stream)), "coverage check");
}

int gm_bijection_check(const int64_t* cx, const int64_t* cy, int64_t nblocks, int64_t n_b, int64_t* owner,
                       int64_t* result, void* stream) {
    if (!pow2(n_b)) return fail(GM_EINVAL, "n_b must be a power of two");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (int rc = cuda_rc(gm::launch_bijection(cx, cy, nblocks, n_b, owner, result, s), "bijection")) return rc;
    return GM_OK;
}

int gm_snapshot_stencil(void* snap, const void* grid, int64_t n, int32_t cell_bytes, void* stream) {
    if (!snap || !grid || snap == grid) return fail(GM_EINVAL, "gm_snapshot_stencil needs distinct buffers");
    if (n < 1) return fail(GM_EINVAL, "bad edge");
    const cudaError_t e = gm::launch_snapshot_stencil(snap, grid, n, cell_bytes, reinterpret_cast<cudaStream_t>(stream));
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_snapshot_stencil: needs 1/2/4/8-byte cells, a power-of-two edge >= one 128-byte "
                               "tile and <= 2^15 tiles per edge");
    }
    return cuda_rc(e, "masked snapshot");
}

int gm_snapshot_stencil_range(void* snap, const void* grid, int64_t n, int32_t cell_bytes, uint32_t t0, uint32_t t1,
                              void* stream) {
    if (!snap || !grid || snap == grid) return fail(GM_EINVAL, "gm_snapshot_stencil_range needs distinct buffers");
    if (n < 1 || t1 < t0) return fail(GM_EINVAL, "gm_snapshot_stencil_range: bad edge or range");
    if (t0 == t1) return GM_OK;
    const cudaError_t e =
        gm::launch_snapshot_stencil(snap, grid, n, cell_bytes, reinterpret_cast<cudaStream_t>(stream), t0, t1);
    if (e == cudaErrorNotSupported || e == cudaErrorInvalidValue) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_snapshot_stencil_range: unsupported grid or tile range [%u, %u)", t0, t1);
    }
    return cuda_rc(e, "masked snapshot (tile range)");
}

int gm_writeback_tiles_range(void* out, const void* dst, const void* snap, int64_t n, int32_t cell_bytes, uint32_t t0,
                             uint32_t t1, void* stream) {
    if (!out || !dst || !snap || out == dst || out == snap) return fail(GM_EINVAL, "gm_writeback_tiles_range: bad buffers");
    if (n < 1 || t1 < t0) return fail(GM_EINVAL, "gm_writeback_tiles_range: bad edge or range");
    if (t0 == t1) return GM_OK;
    const cudaError_t e =
        gm::launch_writeback_tiles(out, dst, snap, n, cell_bytes, reinterpret_cast<cudaStream_t>(stream), t0, t1);
    if (e == cudaErrorNotSupported || e == cudaErrorInvalidValue) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_writeback_tiles_range: unsupported grid or tile range [%u, %u)", t0, t1);
    }
    return cuda_rc(e, "tile write-back (tile range)");
}

int gm_writeback_tiles(void* out, const void* dst, const void* snap, int64_t n, int32_t cell_bytes, void* stream) {
    if (!out || !dst || !snap || out == dst || out == snap) return fail(GM_EINVAL, "gm_writeback_tiles: bad buffers");
    if (n < 1) return fail(GM_EINVAL, "bad edge");
    // the row-ordered walk (host pages K lines at a time) for 1/2/4-byte cells on 64-byte
    // aligned grids, else per tile (host grids off a 64-byte boundary: in host-aligned units)
    const bool aligned = (reinterpret_cast<uintptr_t>(out) & 63u) == 0;
    cudaError_t e = aligned ? gm::launch_host_rows_copyback(out, dst, snap, n, cell_bytes,
                                                            reinterpret_cast<cudaStream_t>(stream))
                            : cudaErrorNotSupported;
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        e = gm::launch_writeback_tiles(out, dst, snap, n, cell_bytes, reinterpret_cast<cudaStream_t>(stream));
    }
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_writeback_tiles: needs 1/2/4/8-byte cells, a power-of-two edge >= one 128-byte "
                               "tile and <= 2^15 tiles per edge");
    }
    return cuda_rc(e, "tile write-back");
}

int gm_fill_hash(void* buf, int64_t n, int32_t cell_bytes, uint64_t seed, int32_t mode, void* stream) {
    if (n < 1) return fail(GM_EINVAL, "bad edge");
    return cuda_rc(gm::launch_fill_hash(buf, n, cell_bytes, seed, mode, reinterpret_cast<cudaStream_t>(stream)),
                   "fill_hash");
}

int gm_checksum(const void* buf, int64_t count, int32_t cell_bytes, uint64_t* out_dev, void* stream) {
    return cuda_rc(gm::launch_checksum(buf, count, cell_bytes, out_dev, reinterpret_cast<cudaStream_t>(stream)),
                   "checksum");
}

int gm_count_equal(const void* a, const void* b, int64_t count, int32_t cell_bytes, unsigned long long* out_dev,
                   void* stream) {
    const int64_t bytes = count * cell_bytes;
    if (bytes % 16) return fail(GM_EINVAL, "count_equal needs a multiple of 16 bytes");
    return cuda_rc(gm::launch_count_equal(a, b, bytes, out_dev, reinterpret_cast<cudaStream_t>(stream)),
                   "count_equal");
}

int gm_l2_flush(const void* buf, int64_t bytes, uint64_t* sink_dev, void* stream) {
    return cuda_rc(gm::launch_l2_flush(buf, bytes, sink_dev, reinterpret_cast<cudaStream_t>(stream)), "l2_flush");
}

int gm_host_map(void* host, int64_t bytes, int32_t register_if_needed, void** dev_ptr, int32_t* registered) {
    if (!host || !dev_ptr || bytes <= 0) return fail(GM_EINVAL, "bad host buffer");
    if (registered) *registered = 0;
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, host);
    if (e == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer) {
        *dev_ptr = at.devicePointer;  // already page-locked (e.g. torch pin_memory) and mapped
        return GM_OK;
    }
    cudaGetLastError();
    if (!register_if_needed) return fail(GM_EINVAL, "host buffer is not page-locked");
    e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
    } else if (e != cudaSuccess) {
        return cuda_rc(e, "cudaHostRegister");
    } else if (registered) {
        *registered = 1;
    }
    return cuda_rc(cudaHostGetDevicePointer(dev_ptr, host, 0), "cudaHostGetDevicePointer");
}

int gm_host_unmap(void* host) {
    cudaError_t e = cudaHostUnregister(host);
    if (e == cudaErrorHostMemoryNotRegistered) {
        cudaGetLastError();
        return GM_OK;
    }
    return cuda_rc(e, "cudaHostUnregister");
}

int gm_set_l2_fetch_granularity(int32_t bytes) {
    return cuda_rc(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes), "cudaDeviceSetLimit");
}

int gm_ca_step2(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                int32_t flags, void* stream) {
    return gm_ca_steps(grid, src, n, cell_bytes, kind, param, 2, flags, stream);
}

int gm_ca_steps(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                int32_t steps, int32_t flags, void* stream) {
    if (steps != 2 && steps != 4 && steps != 6) return fail(GM_EINVAL, "gm_ca_steps: steps must be 2, 4 or 6");
    gm_cfg_t c{};
    c.n = n;
    c.rho = 1;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = GM_STRAT_TUNED;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    c.flags = flags;
    if (int rc = check_common(n, cell_bytes, 1, kind)) return rc;
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_ca_steps: kind must be NSUM4 or NSUM8");
    if (!grid || !src || src == grid) return fail(GM_EINVAL, "gm_ca_steps needs distinct grid and src buffers");
    gm::LaunchArgs a = make_args(&c, grid, src, nullptr, nullptr, 0, stream);
    const cudaError_t e = gm::launch_stencil_tb(a, steps);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_ca_steps: needs 1-, 2- or 4-byte cells (1 or 2 for 6 steps) and n >= one 128-byte "
                               "tile (<= 2^15 tiles per edge)");
    }
    return cuda_rc(e, "fused multi-step CA launch");
}

namespace {
// the launch descriptor of a CA run: n, cells, kind, the sub-gasket range (level < 0: all)
int ca_args(gm::LaunchArgs& a, const char* who, void* grid, const void* src, int64_t n, int32_t cell_bytes,
            int32_t kind, int32_t param, int32_t level, uint32_t sg_begin, uint32_t sg_end, const int64_t* sg_off,
            int64_t pitch, void* stream) {
    gm_cfg_t c{};
    c.n = n;
    c.rho = 1;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = GM_STRAT_TUNED;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    if (int rc = check_common(n, cell_bytes, 1, kind)) return rc;
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4) return fail(GM_EINVAL, "%s: 1-, 2- or 4-byte cells", who);
    if (n * cell_bytes < 128) return fail(GM_EINVAL, "%s: the grid must be at least one 128-byte tile wide", who);
    if (level >= 0) {
        uint64_t nsg = 1;
        for (int i = 0; i < level; ++i) nsg *= 3;
        if ((n >> level) * cell_bytes < 128) return fail(GM_EINVAL, "partition level %d too deep", level);
        if (sg_begin > sg_end || sg_end > nsg)
            return fail(GM_EINVAL, "sub-gasket range [%u, %u) outside [0, %llu)", sg_begin, sg_end, (unsigned long long)nsg);
    }
    if (sg_off != nullptr && (pitch % 32 != 0 || level < 0)) return fail(GM_EINVAL, "%s: bad tiled layout", who);
    a = make_args(&c, grid, src, nullptr, nullptr, 0, stream);
    a.part_level = level;
    a.sg_begin = sg_begin;
    a.sg_end = sg_end;
    a.sg_off = sg_off;
    a.pitch = sg_off != nullptr ? pitch : 0;
    return GM_OK;
}
}  // namespace

int gm_ca_edge_bytes(int64_t n, int32_t cell_bytes, int32_t level, uint32_t sg_begin, uint32_t sg_end, int64_t* bytes) {
    if (!bytes) return fail(GM_EINVAL, "gm_ca_edge_bytes: null output");
    gm::LaunchArgs a{};
    if (int rc = ca_args(a, "gm_ca_edge_bytes", nullptr, nullptr, n, cell_bytes, GM_KIND_NSUM8, 1, level, sg_begin,
                         sg_end, nullptr, 0, nullptr))
        return rc;
    *bytes = gm::edge_cache_bytes(a);
    if (*bytes == 0 && n * cell_bytes >= 128)
        return fail(GM_EINVAL, "gm_ca_edge_bytes: more than 2^15 tiles per edge");
    return GM_OK;
}

int gm_ca_edge_build(void* edge, const void* src, int64_t n, int32_t cell_bytes, int32_t level, uint32_t sg_begin,
                     uint32_t sg_end, const int64_t* sg_off, int64_t pitch, void* stream) {
    if (!edge || !src) return fail(GM_EINVAL, "gm_ca_edge_build: null buffer");
    gm::LaunchArgs a{};
    if (int rc = ca_args(a, "gm_ca_edge_build", nullptr, src, n, cell_bytes, GM_KIND_NSUM8, 1, level, sg_begin, sg_end,
                         sg_off, pitch, stream))
        return rc;
    const cudaError_t e = gm::launch_edge_build(a, reinterpret_cast<uint8_t*>(edge));
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_ca_edge_build: more than 2^15 tiles per edge");
    }
    return cuda_rc(e, "edge cache build");
}

int gm_ca_run(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param, int32_t steps,
              const void* edge, int32_t flags, void* stream) {
    if (steps != 1 && steps != 2 && steps != 4 && steps != 6) return fail(GM_EINVAL, "gm_ca_run: steps must be 1, 2, 4 or 6");
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_ca_run: kind must be NSUM4 or NSUM8");
    if (!grid || !src || src == grid) return fail(GM_EINVAL, "gm_ca_run needs distinct grid and src buffers");
    gm::LaunchArgs a{};
    if (int rc = ca_args(a, "gm_ca_run", grid, src, n, cell_bytes, kind, param, -1, 0, 0, nullptr, 0, stream)) return rc;
    a.flags = (flags & ~GM_FLAG_DST_FROM_SRC) | (steps == 1 ? GM_FLAG_DST_FROM_SRC : 0);
    // the single-step kernel stages from the cache; the fused kernels are bound by their
    // arithmetic, not staging (n=2^17 NSUM8 with the cache: 1 step 436 -> 406 us, 2/4/6
    // steps 1-2% slower), so they read the grid
    a.edge = steps == 1 ? reinterpret_cast<const uint8_t*>(edge) : nullptr;
    const cudaError_t e = steps == 1 ? gm::launch_stencil_v2(a) : gm::launch_stencil_tb(a, steps);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_ca_run: no tiled kernel for these cells (6 steps: 1- or 2-byte cells; <= 2^15 tiles "
                               "per edge)");
    }
    return cuda_rc(e, "CA launch");
}

int gm_border_bytes(int64_t n, int32_t cell_bytes, int64_t* bytes) {
    if (!bytes) return fail(GM_EINVAL, "gm_border_bytes: null output");
    gm::LaunchArgs a{};
    if (int rc = ca_args(a, "gm_border_bytes", nullptr, nullptr, n, cell_bytes, GM_KIND_NSUM8, 1, -1, 0, 0, nullptr, 0,
                         nullptr))
        return rc;
    *bytes = gm::border_bytes(n, cell_bytes);
    return GM_OK;
}

int gm_run_inplace(void* grid, void* border, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                   void* stream) {
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_run_inplace: kind must be NSUM4 or NSUM8");
    if (!grid || !border || border == grid) return fail(GM_EINVAL, "gm_run_inplace: needs the grid and a border buffer");
    gm::LaunchArgs a{};
    if (int rc = ca_args(a, "gm_run_inplace", grid, grid, n, cell_bytes, kind, param, -1, 0, 0, nullptr, 0, stream))
        return rc;
    a.flags = GM_FLAG_DST_FROM_SRC;  // off-gasket cells come from the staged window (the grid itself)
    a.border = reinterpret_cast<const uint8_t*>(border);
    cudaError_t e = gm::launch_border_snapshot(reinterpret_cast<uint8_t*>(border), grid, n, cell_bytes, a.stream);
    if (e == cudaSuccess) e = gm::launch_stencil_v2(a);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_run_inplace: no tiled kernel for these cells (<= 2^15 tiles per edge)");
    }
    return cuda_rc(e, "in-place neighbour-sum launch");
}

int gm_run_tiles(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param, int32_t flags,
                 uint32_t t0, uint32_t t1, void* stream) {
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_run_tiles: kind must be NSUM4 or NSUM8");
    if (!grid || !src || src == grid) return fail(GM_EINVAL, "gm_run_tiles needs distinct grid and src buffers");
    if (t1 < t0) return fail(GM_EINVAL, "gm_run_tiles: bad tile range");
    if (t0 == t1) return GM_OK;
    gm::LaunchArgs a{};
    if (int rc = ca_args(a, "gm_run_tiles", grid, src, n, cell_bytes, kind, param, -1, 0, 0, nullptr, 0, stream)) return rc;
    a.flags = flags & ~GM_FLAG_DIGIT_ORDER;  // (tile ranges refer to the row-major order)
    a.range_lo = t0;
    a.range_hi = t1;
    const cudaError_t e = gm::launch_stencil_v2(a);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_run_tiles: no tiled kernel for these cells");
    }
    return cuda_rc(e, "tuned step (tile range)");
}

int gm_dev_alloc(int64_t bytes, void** out) {
    if (bytes <= 0 || !out) return fail(GM_EINVAL, "gm_dev_alloc: bad size/out");
    return cuda_rc(cudaMalloc(out, (size_t)bytes), "cudaMalloc");
}

int gm_dev_free(void* p) { return cuda_rc(cudaFree(p), "cudaFree"); }

int gm_ipc_get_handle(void* base, void* handle_out) {
    if (!base || !handle_out) return fail(GM_EINVAL, "gm_ipc_get_handle: null argument");
    cudaIpcMemHandle_t h;
    if (int rc = cuda_rc(cudaIpcGetMemHandle(&h, base), "cudaIpcGetMemHandle")) return rc;
    memcpy(handle_out, &h, sizeof(h));
    return GM_OK;
}

int gm_ipc_open_handle(const void* handle, void** out) {
    if (!handle || !out) return fail(GM_EINVAL, "gm_ipc_open_handle: null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    return cuda_rc(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int gm_ipc_close(void* p) { return cuda_rc(cudaIpcCloseMemHandle(p), "cudaIpcCloseMemHandle"); }

int gm_peer_halo_put(const void* mine, const uint64_t* peers, const int64_t* idx, int64_t count, int32_t cell_bytes,
                     const uint64_t* peer_flags, int32_t rank, int32_t world, uint64_t epoch, void* stream) {
    if (!mine || !peers || !peer_flags || (count && !idx) || count < 0) return fail(GM_EINVAL, "gm_peer_halo_put: bad arguments");
    if (world < 1 || rank < 0 || rank >= world) return fail(GM_EINVAL, "gm_peer_halo_put: rank %d outside world %d", rank, world);
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4 && cell_bytes != 8)
        return fail(GM_EINVAL, "gm_peer_halo_put: cell_bytes must be 1, 2, 4 or 8");
    return cuda_rc(gm::launch_peer_put(mine, peers, idx, nullptr, count, cell_bytes, peer_flags, rank, world, epoch,
                                       reinterpret_cast<cudaStream_t>(stream)), "peer_halo_put");
}

int gm_peer_halo_put_to(const void* mine, const uint64_t* peers, const int64_t* idx, const int64_t* didx,
                        int64_t count, int32_t cell_bytes, const uint64_t* peer_flags, int32_t rank, int32_t world,
                        uint64_t epoch, void* stream) {
    if (!mine || !peers || !peer_flags || (count && (!idx || !didx)) || count < 0)
        return fail(GM_EINVAL, "gm_peer_halo_put_to: bad arguments");
    if (world < 1 || world > 255 || rank < 0 || rank >= world)
        return fail(GM_EINVAL, "gm_peer_halo_put_to: rank %d outside world %d", rank, world);
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4 && cell_bytes != 8)
        return fail(GM_EINVAL, "gm_peer_halo_put_to: cell_bytes must be 1, 2, 4 or 8");
    return cuda_rc(gm::launch_peer_put(mine, peers, idx, didx, count, cell_bytes, peer_flags, rank, world, epoch,
                                       reinterpret_cast<cudaStream_t>(stream)), "peer_halo_put_to");
}

int gm_copy_cells(void* dst, const void* src, int32_t cell_bytes, const int64_t* dst_idx, const int64_t* src_idx,
                  int64_t count, void* stream) {
    if (count < 0 || (count && (!dst || !src || !dst_idx || !src_idx))) return fail(GM_EINVAL, "gm_copy_cells: bad arguments");
    return cuda_rc(gm::launch_copy_cells(dst, src, cell_bytes, dst_idx, src_idx, count,
                                         reinterpret_cast<cudaStream_t>(stream)), "copy_cells");
}

int gm_fill_hash_window(void* out, int64_t pitch, int64_t n, int32_t cell_bytes, int64_t x0, int64_t y0, int64_t w,
                        int64_t h, uint64_t seed, int32_t mode, void* stream) {
    if (!out || n < 1 || pitch < w * cell_bytes) return fail(GM_EINVAL, "gm_fill_hash_window: bad arguments");
    return cuda_rc(gm::launch_fill_hash_window(out, pitch, n, cell_bytes, x0, y0, w, h, seed, mode,
                                               reinterpret_cast<cudaStream_t>(stream)), "fill_hash_window");
}

int gm_run_part_tiled(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                      int32_t steps, int32_t level, uint32_t sg_begin, uint32_t sg_end, const int64_t* sg_off,
                      int64_t pitch, void* epilogue, uint64_t wait_epoch, uint64_t signal_epoch, const void* edge,
                      void* stream) {
    if (steps != 1 && steps != 2 && steps != 4 && steps != 6)
        return fail(GM_EINVAL, "gm_run_part_tiled: steps must be 1, 2, 4 or 6");
    gm_cfg_t c{};
    c.n = n;
    c.rho = 1;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = GM_STRAT_TUNED;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    c.flags = steps == 1 ? GM_FLAG_DST_FROM_SRC : 0;
    if (int rc = check_common(n, cell_bytes, 1, kind)) return rc;
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_run_part_tiled: kind must be NSUM4 or NSUM8");
    if (!grid || !src || src == grid || !sg_off) return fail(GM_EINVAL, "gm_run_part_tiled: bad buffers");
    if (cell_bytes != 1 && cell_bytes != 2 && cell_bytes != 4) return fail(GM_EINVAL, "gm_run_part_tiled: 1-, 2- or 4-byte cells");
    const int64_t tile = 128 / cell_bytes;
    if (level < 0 || (n >> level) < tile) return fail(GM_EINVAL, "partition level %d too deep", level);
    if (pitch < (n >> level) * cell_bytes + 32 || pitch % 32 != 0)
        return fail(GM_EINVAL, "gm_run_part_tiled: pitch %lld must cover a sub-gasket row plus its ring, a multiple of 32",
                    (long long)pitch);
    uint64_t nsg = 1;
    for (int i = 0; i < level; ++i) nsg *= 3;
    if (sg_begin > sg_end || sg_end > nsg) return fail(GM_EINVAL, "sub-gasket range [%u, %u) outside [0, %llu)",
                                                       sg_begin, sg_end, (unsigned long long)nsg);
    gm::LaunchArgs a = make_args(&c, grid, src, nullptr, nullptr, 0, stream);
    a.part_level = level;
    a.sg_begin = sg_begin;
    a.sg_end = sg_end;
    a.sg_off = sg_off;
    a.pitch = pitch;
    a.peer_epi = epilogue;
    a.wait_epoch = epilogue ? wait_epoch : 0;
    a.signal_epoch = epilogue ? signal_epoch : 0;
    a.edge = steps == 1 ? reinterpret_cast<const uint8_t*>(edge) : nullptr;  // (see gm_ca_run)
    const cudaError_t e = steps == 1 ? gm::launch_stencil_v2(a) : gm::launch_stencil_tb(a, steps);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_run_part_tiled: no tiled kernel for these cells (6 steps: 1- or 2-byte cells)");
    }
    return cuda_rc(e, "tiled partition launch");
}

int gm_peer_halo_wait(const uint64_t* flags, int32_t rank, int32_t world, uint64_t epoch, uint64_t timeout_ns,
                      uint32_t* status, void* stream) {
    if (!flags || !status) return fail(GM_EINVAL, "gm_peer_halo_wait: null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(GM_EINVAL, "gm_peer_halo_wait: rank %d outside world %d", rank, world);
    return cuda_rc(gm::launch_peer_wait(flags, rank, world, epoch, timeout_ns, status,
                                        reinterpret_cast<cudaStream_t>(stream)), "peer_halo_wait");
}

int gm_run_part2(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                 int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* stream) {
    return gm_run_part_steps(grid, src, n, cell_bytes, kind, param, 2, flags, level, sg_begin, sg_end, stream);
}

int gm_run_part_steps(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                      int32_t steps, int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* stream) {
    if (steps != 2 && steps != 4 && steps != 6) return fail(GM_EINVAL, "gm_run_part_steps: steps must be 2, 4 or 6");
    gm_cfg_t c{};
    c.n = n;
    c.rho = 1;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = GM_STRAT_TUNED;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    c.flags = flags;
    if (int rc = check_common(n, cell_bytes, 1, kind)) return rc;
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_run_part_steps: kind must be NSUM4 or NSUM8");
    if (!grid || !src || src == grid) return fail(GM_EINVAL, "gm_run_part_steps needs distinct grid and src buffers");
    const int r = log2i(n);
    const int64_t tile = cell_bytes <= 4 ? 128 / cell_bytes : 32;
    if (level < 0 || (n >> level) < tile)
        return fail(GM_EINVAL, "partition level %d too deep for n=2^%d (sub-gaskets narrower than a tile)", level, r);
    uint64_t nsg = 1;
    for (int i = 0; i < level; ++i) nsg *= 3;
    if (sg_begin > sg_end || sg_end > nsg) return fail(GM_EINVAL, "sub-gasket range [%u, %u) outside [0, %llu)",
                                                       sg_begin, sg_end, (unsigned long long)nsg);
    gm::LaunchArgs a = make_args(&c, grid, src, nullptr, nullptr, 0, stream);
    a.part_level = level;
    a.sg_begin = sg_begin;
    a.sg_end = sg_end;
    const cudaError_t e = gm::launch_stencil_tb(a, steps);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_run_part_steps: needs 1-, 2- or 4-byte cells (1 or 2 for 6 steps)");
    }
    return cuda_rc(e, "partitioned fused multi-step CA launch");
}

int gm_run_part_peer(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                     int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* epilogue,
                     uint64_t wait_epoch, uint64_t signal_epoch, void* stream) {
    gm_cfg_t c{};
    c.n = n;
    c.rho = 1;
    c.mapping = GM_MAP_LAMBDA;
    c.strategy = GM_STRAT_TUNED;
    c.kind = kind;
    c.cell_bytes = cell_bytes;
    c.param = param;
    c.flags = flags & ~(GM_FLAG_OMEGA_ORDER | GM_FLAG_STENCIL_V1 | GM_FLAG_FORCE_TMA);
    if (int rc = check_common(n, cell_bytes, 1, kind)) return rc;
    if (kind != GM_KIND_NSUM4 && kind != GM_KIND_NSUM8) return fail(GM_EINVAL, "gm_run_part_peer: kind must be NSUM4 or NSUM8");
    if (!grid || !src || src == grid || !epilogue) return fail(GM_EINVAL, "gm_run_part_peer: bad buffers or descriptor");
    const int64_t tile = cell_bytes <= 4 ? 128 / cell_bytes : 32;
    if (level < 0 || (n >> level) < tile) return fail(GM_EINVAL, "partition level %d too deep", level);
    uint64_t nsg = 1;
    for (int i = 0; i < level; ++i) nsg *= 3;
    if (sg_begin > sg_end || sg_end > nsg) return fail(GM_EINVAL, "sub-gasket range [%u, %u) outside [0, %llu)",
                                                       sg_begin, sg_end, (unsigned long long)nsg);
    gm::LaunchArgs a = make_args(&c, grid, src, nullptr, nullptr, 0, stream);
    a.part_level = level;
    a.sg_begin = sg_begin;
    a.sg_end = sg_end;
    a.peer_epi = epilogue;
    a.wait_epoch = wait_epoch;
    a.signal_epoch = signal_epoch;
    // only the v2 tile kernel (one step) and the fused multi-step kernel (GM_FLAG_TWO_STEPS,
    // GM_FLAG_FOUR_STEPS, GM_FLAG_SIX_STEPS) carry the fused exchange: no silent fallback to a kernel without it
    const cudaError_t e = (flags & GM_FLAG_SIX_STEPS)    ? gm::launch_stencil_tb(a, 6)
                          : (flags & GM_FLAG_FOUR_STEPS) ? gm::launch_stencil_tb(a, 4)
                          : (flags & GM_FLAG_TWO_STEPS)  ? gm::launch_stencil_tb(a, 2)
                                                         : gm::launch_stencil_v2(a);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        return fail(GM_EINVAL, "gm_run_part_peer: needs 1-, 2- or 4-byte cells");
    }
    return cuda_rc(e, "partitioned CA step with fused peer exchange");
}

int gm_tile_order(int32_t q, int32_t level, uint32_t* out, int64_t capacity) {
    if (q < 0 || q > 15 || level < 0 || level > q || out == nullptr) return fail(GM_EINVAL, "gm_tile_order: bad q/level");
    std::vector<uint32_t> v;
    gm::rowmajor_order_host(q, level, v);
    if ((int64_t)v.size() > capacity) return fail(GM_EINVAL, "gm_tile_order: capacity < 3^q");
    std::copy(v.begin(), v.end(), out);
    return GM_OK;
}

uint64_t gm_launch_count(void) { return gm::g_launches.load(); }
const char* gm_last_error(void) { return t_err.c_str(); }
const char* gm_version(void) { return "gasket_b200 0.1.0 sm_100a"; }

}  // extern "C"
