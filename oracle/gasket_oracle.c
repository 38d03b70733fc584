/*
 * gasket_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file.  It is loaded (via oracle/oracle.py) only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs,
 * and there only as the checker or the timed CPU baseline.
 *
 * Every function restates one reference function, cited as file:line relative
 * to /root/reference/pkg/src/gasketmap/.  Parity of this restatement is pinned
 * by tests/test_oracle_golden.py against fixtures generated from the live
 * reference (tests/golden/make_golden.py) and, when /root/reference is present,
 * against the reference itself (tests/test_oracle_vs_reference.py).
 *
 * The 8-neighbour kernel (KIND_NSUM8) has no reference implementation.  It is
 * our labelled extension of _cell_value (backends.py:127-141) from the four
 * von-Neumann offsets to the eight Moore offsets with identical conventions
 * (param + in-grid neighbours, out-of-grid = 0, wrap to the cell width, read
 * the pre-launch snapshot).  Its parity is pinned only by construction: the
 * NSUM4 path that shares the code is pinned to the reference.
 *
 * Integer semantics follow the numba backend (the reference's default,
 * backends.py:39-50): the sum is formed in 64-bit from an int32 param and the
 * neighbour cells, then truncated to the cell width on store.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KIND_CONST 0
#define KIND_NSUM4 1
#define KIND_NSUM8 2
/* backends.py:32-34 */
#define STRAT_UNROLL 0
#define STRAT_TABLE 1
#define STRAT_SUBBOX 2

static int nthr(int t) {
#ifdef _OPENMP
    return t > 0 ? t : omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

int go_max_threads(void) { return nthr(0); }

/* Python floor division / modulo on int64 (numpy semantics). */
static inline int64_t py_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}
static inline int64_t py_mod(int64_t a, int64_t b) {
    int64_t m = a % b;
    if (m != 0 && ((m < 0) != (b < 0))) m += b;
    return m;
}

/* blockmap.py:91-108  map_blocks_array -- the vectorised lambda(omega). */
void go_map_blocks(const int64_t* wx, const int64_t* wy, int64_t count, int r_b,
                   int64_t* lx, int64_t* ly, int threads) {
#pragma omp parallel for num_threads(nthr(threads)) schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        int64_t ax = 0, ay = 0, div_x = 1, div_y = 1, step = 1;
        for (int mu = 1; mu <= r_b; ++mu) {
            int64_t region;
            if (mu & 1) {
                region = py_mod(py_div(wy[i], div_y), 3);
                div_y *= 3;
            } else {
                region = py_mod(py_div(wx[i], div_x), 3);
                div_x *= 3;
            }
            int64_t dx = region >> 1;
            ax += dx * step;
            ay += (region - dx) * step;
            step <<= 1;
        }
        lx[i] = ax;
        ly[i] = ay;
    }
}

/* The full packed rectangle in the reference's b = wy*W + wx order
 * (blockmap.py:140-141, engine.py:233-235, backends.py:103-105). */
void go_map_rectangle(int r_b, int64_t* lx, int64_t* ly, int threads) {
    int64_t W = 1, H = 1;
    for (int i = 0; i < r_b / 2; ++i) W *= 3;           /* core.py:64-72 */
    for (int i = 0; i < (r_b + 1) / 2; ++i) H *= 3;
    int64_t total = W * H;
#pragma omp parallel for num_threads(nthr(threads)) schedule(static)
    for (int64_t b = 0; b < total; ++b) {
        int64_t wy = b / W, wx = b - wy * W;
        int64_t ax = 0, ay = 0, div_x = 1, div_y = 1, step = 1;
        for (int mu = 1; mu <= r_b; ++mu) {
            int64_t region;
            if (mu & 1) { region = (wy / div_y) % 3; div_y *= 3; }
            else        { region = (wx / div_x) % 3; div_x *= 3; }
            int64_t dx = region >> 1;
            ax += dx * step;
            ay += (region - dx) * step;
            step <<= 1;
        }
        lx[b] = ax;
        ly[b] = ay;
    }
}

/* ------------------------------------------------------------------------ */
/* Per-cell kernels: backends.py:127-141 (_cell_value), generated per width. */
/* ------------------------------------------------------------------------ */

#define DEFINE_CELL_KERNELS(T, SUF)                                                        \
static inline T cell_value_##SUF(const T* src, int64_t n, int64_t x, int64_t y, int kind,  \
                                 int32_t param) {                                          \
    if (kind == KIND_CONST) return (T)(int64_t)param;                                      \
    uint64_t t = (uint64_t)(int64_t)param;                                                 \
    const T* row = src + y * n;                                                            \
    if (x > 0) t += (uint64_t)(int64_t)row[x - 1];                                         \
    if (x < n - 1) t += (uint64_t)(int64_t)row[x + 1];                                     \
    if (y > 0) t += (uint64_t)(int64_t)row[x - n];                                         \
    if (y < n - 1) t += (uint64_t)(int64_t)row[x + n];                                     \
    if (kind == KIND_NSUM8) { /* our extension: Moore diagonals, same conventions */       \
        if (y > 0 && x > 0) t += (uint64_t)(int64_t)row[x - n - 1];                        \
        if (y > 0 && x < n - 1) t += (uint64_t)(int64_t)row[x - n + 1];                    \
        if (y < n - 1 && x > 0) t += (uint64_t)(int64_t)row[x + n - 1];                    \
        if (y < n - 1 && x < n - 1) t += (uint64_t)(int64_t)row[x + n + 1];                \
    }                                                                                      \
    return (T)t;                                                                           \
}                                                                                          \
                                                                                           \
/* backends.py:143-156  _bounding_box_nb */                                                \
static void bb_##SUF(T* grid, const T* src, int64_t n, int64_t rho, int kind,              \
                     int32_t param, int threads) {                                         \
    int64_t nb = n / rho;                                                                  \
    _Pragma("omp parallel for num_threads(nthr(threads)) schedule(static)")                \
    for (int64_t b = 0; b < nb * nb; ++b) {                                                \
        int64_t by = b / nb, bx = b - by * nb;                                             \
        for (int64_t ty = 0; ty < rho; ++ty) {                                             \
            int64_t y = by * rho + ty, m = n - 1 - y;                                      \
            for (int64_t tx = 0; tx < rho; ++tx) {                                         \
                int64_t x = bx * rho + tx;                                                 \
                if ((x & m) == 0) grid[y * n + x] = cell_value_##SUF(src, n, x, y, kind, param); \
            }                                                                              \
        }                                                                                  \
    }                                                                                      \
}                                                                                          \
                                                                                           \
/* backends.py:158-222  _block_space_nb */                                                 \
static void bs_##SUF(T* grid, const T* src, int64_t n, int64_t rho, int r_b, int64_t width, \
                     int64_t nblocks, int strategy, const int64_t* tab_x,                  \
                     const int64_t* tab_y, int64_t ntab, int r_p, int64_t t_width,         \
                     int kind, int32_t param, int threads) {                               \
    _Pragma("omp parallel for num_threads(nthr(threads)) schedule(static)")                \
    for (int64_t b = 0; b < nblocks; ++b) {                                                \
        int64_t wy = b / width, wx = b - wy * width;                                       \
        int64_t lx = 0, ly = 0, div_x = 1, div_y = 1, step = 1;                            \
        for (int mu = 1; mu <= r_b; ++mu) {                   /* :171-181 */               \
            int64_t region;                                                                \
            if (mu & 1) { region = (wy / div_y) % 3; div_y *= 3; }                         \
            else        { region = (wx / div_x) % 3; div_x *= 3; }                         \
            int64_t dx = region >> 1;                                                      \
            lx += dx * step;                                                               \
            ly += (region - dx) * step;                                                    \
            step <<= 1;                                                                    \
        }                                                                                  \
        int64_t ox = lx * rho, oy = ly * rho;                  /* :182-183 */              \
        if (strategy == STRAT_SUBBOX) {                        /* :184-191 */              \
            for (int64_t ty = 0; ty < rho; ++ty) {                                         \
                int64_t m = rho - 1 - ty, y = oy + ty;                                     \
                for (int64_t tx = 0; tx < rho; ++tx)                                       \
                    if ((tx & m) == 0) {                                                   \
                        int64_t x = ox + tx;                                               \
                        grid[y * n + x] = cell_value_##SUF(src, n, x, y, kind, param);     \
                    }                                                                      \
            }                                                                              \
        } else if (strategy == STRAT_TABLE) {                  /* :192-196 */              \
            for (int64_t i = 0; i < ntab; ++i) {                                           \
                int64_t x = ox + tab_x[i], y = oy + tab_y[i];                              \
                grid[y * n + x] = cell_value_##SUF(src, n, x, y, kind, param);             \
            }                                                                              \
        } else {                                               /* :197-222 */              \
            int64_t n_threads = 1;                                                         \
            for (int i = 0; i < r_p; ++i) n_threads *= 3;                                  \
            for (int64_t t = 0; t < n_threads; ++t) {                                      \
                int64_t ty = t / t_width, tx = t - ty * t_width;                           \
                int64_t sx = 0, sy = 0, tdx = 1, tdy = 1, ts = 1;                          \
                for (int mu = 1; mu <= r_p; ++mu) {                                        \
                    int64_t region;                                                        \
                    if (mu & 1) { region = (ty / tdy) % 3; tdy *= 3; }                     \
                    else        { region = (tx / tdx) % 3; tdx *= 3; }                     \
                    int64_t dx = region >> 1;                                              \
                    sx += dx * ts;                                                         \
                    sy += (region - dx) * ts;                                              \
                    ts <<= 1;                                                              \
                }                                                                          \
                int64_t x = ox + sx, y = oy + sy;                                          \
                grid[y * n + x] = cell_value_##SUF(src, n, x, y, kind, param);             \
            }                                                                              \
        }                                                                                  \
    }                                                                                      \
}

DEFINE_CELL_KERNELS(int8_t, i8)
DEFINE_CELL_KERNELS(int16_t, i16)
DEFINE_CELL_KERNELS(int32_t, i32)
DEFINE_CELL_KERNELS(int64_t, i64)

/* backends.py:225-231  run_bounding_box (numba leg). Returns 0 or -1 on bad width. */
int go_run_bounding_box(void* grid, const void* src, int64_t n, int cell_bytes, int64_t rho,
                        int kind, int32_t param, int threads) {
    switch (cell_bytes) {
    case 1: bb_i8((int8_t*)grid, (const int8_t*)src, n, rho, kind, param, threads); return 0;
    case 2: bb_i16((int16_t*)grid, (const int16_t*)src, n, rho, kind, param, threads); return 0;
    case 4: bb_i32((int32_t*)grid, (const int32_t*)src, n, rho, kind, param, threads); return 0;
    case 8: bb_i64((int64_t*)grid, (const int64_t*)src, n, rho, kind, param, threads); return 0;
    }
    return -1;
}

/* backends.py:234-272  run_block_space (numba leg: width, r_p, t_width at :247-255). */
int go_run_block_space(void* grid, const void* src, int64_t n, int cell_bytes, int64_t rho,
                       int r_b, int strategy, const int64_t* tab_x, const int64_t* tab_y,
                       int64_t ntab, int kind, int32_t param, int threads) {
    int64_t width = 1, nblocks = 1, t_width = 1;
    int r_p = 0;
    for (int i = 0; i < r_b / 2; ++i) width *= 3;
    for (int i = 0; i < r_b; ++i) nblocks *= 3;
    while ((1LL << r_p) < rho) ++r_p;
    for (int i = 0; i < r_p / 2; ++i) t_width *= 3;
    if (strategy != STRAT_TABLE) ntab = 0;
    switch (cell_bytes) {
    case 1: bs_i8((int8_t*)grid, (const int8_t*)src, n, rho, r_b, width, nblocks, strategy, tab_x, tab_y, ntab, r_p, t_width, kind, param, threads); return 0;
    case 2: bs_i16((int16_t*)grid, (const int16_t*)src, n, rho, r_b, width, nblocks, strategy, tab_x, tab_y, ntab, r_p, t_width, kind, param, threads); return 0;
    case 4: bs_i32((int32_t*)grid, (const int32_t*)src, n, rho, r_b, width, nblocks, strategy, tab_x, tab_y, ntab, r_p, t_width, kind, param, threads); return 0;
    case 8: bs_i64((int64_t*)grid, (const int64_t*)src, n, rho, r_b, width, nblocks, strategy, tab_x, tab_y, ntab, r_p, t_width, kind, param, threads); return 0;
    }
    return -1;
}

/* ------------------------------------------------------------------------ */
/* Synthetic inputs and checksums (shared definition with the CUDA library;  */
/* no reference counterpart -- test/bench plumbing).                         */
/* ------------------------------------------------------------------------ */

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* mode 0 "strict": every cell random; mode 1 "CA": gasket cells random, 0 elsewhere. */
void go_fill_hash(void* buf, int64_t n, int cell_bytes, uint64_t seed, int mode, int threads) {
#pragma omp parallel for num_threads(nthr(threads)) schedule(static)
    for (int64_t y = 0; y < n; ++y) {
        int64_t m = n - 1 - y;
        for (int64_t x = 0; x < n; ++x) {
            uint64_t v = splitmix64(seed ^ (((uint64_t)y << 32) | (uint64_t)x));
            if (mode == 1 && (x & m) != 0) v = 0;
            int64_t i = y * n + x;
            switch (cell_bytes) {
            case 1: ((uint8_t*)buf)[i] = (uint8_t)v; break;
            case 2: ((uint16_t*)buf)[i] = (uint16_t)v; break;
            case 4: ((uint32_t*)buf)[i] = (uint32_t)v; break;
            default: ((uint64_t*)buf)[i] = v; break;
            }
        }
    }
}

/* H = sum_i ((2i+1) * K) * v_i  (mod 2^64), v_i the cell as an unsigned word. */
uint64_t go_checksum(const void* buf, int64_t count, int cell_bytes, int threads) {
    const uint64_t K = 0x9E3779B97F4A7C15ULL;
    uint64_t h = 0;
#pragma omp parallel for num_threads(nthr(threads)) schedule(static) reduction(+ : h)
    for (int64_t i = 0; i < count; ++i) {
        uint64_t v;
        switch (cell_bytes) {
        case 1: v = ((const uint8_t*)buf)[i]; break;
        case 2: v = ((const uint16_t*)buf)[i]; break;
        case 4: v = ((const uint32_t*)buf)[i]; break;
        default: v = ((const uint64_t*)buf)[i]; break;
        }
        h += ((2 * (uint64_t)i + 1) * K) * v;
    }
    return h;
}

/* engine.py:214-258 verify_coverage, counting leg: counts[y][x] += 1 for every
 * (block, local cell) the launch shape writes; writes outside the grid dropped. */
void go_coverage_blocks(const int64_t* bx, const int64_t* by, int64_t nblocks, const int64_t* lx,
                        const int64_t* ly, int64_t nlocal, int64_t rho, int64_t n, int64_t* counts) {
    for (int64_t b = 0; b < nblocks; ++b)
        for (int64_t i = 0; i < nlocal; ++i) {
            int64_t x = bx[b] * rho + lx[i], y = by[b] * rho + ly[i];
            if (x >= 0 && x < n && y >= 0 && y < n) counts[y * n + x] += 1;
        }
}

/* ------------------------------------------------------------------------ */
/* Row bands of a multi-step CA run at sizes the full-grid oracle cannot     */
/* hold (n = 2^17 int8 is 16 GiB per grid, 2^18 is 64 GiB).                  */
/*                                                                          */
/* Same arithmetic as bb_* / bs_* above: every step is one NEIGHBOR_SUM      */
/* launch with engine.launch's snapshot semantics (engine.py:201, src = the  */
/* pre-launch grid): each gasket cell x & (n-1-y) == 0 (backends.py:155-156) */
/* gets _cell_value (backends.py:127-141) of the previous state, off-gasket  */
/* cells never change.  Only the cell order differs (rows, the x that are    */
/* bit-subsets of y ascending)   ; writes are disjoint, so order is moot.   */
/*                                                                          */
/* The input is the synthetic grid go_fill_hash(seed, mode) builds.  Rows     */
/* [y0, y1) after s steps depend on rows [y0-s, y1+s) of the input, so the    */
/* window is filled with `smax` extra rows on each side (clipped to the      */
/* grid, where out-of-grid = 0 is exact); cells next to a window edge that    */
/* is not a grid edge go stale one row per step and never reach the band.    */
/* outs[i] receives rows [y0, y1) after steps[i] steps (0 = the input).      */
/* ------------------------------------------------------------------------ */

static void fill_rows(void* buf, int64_t n, int cell_bytes, uint64_t seed, int mode, int64_t w0, int64_t w1,
                      int threads) {
#pragma omp parallel for num_threads(nthr(threads)) schedule(static)
    for (int64_t y = w0; y < w1; ++y) {
        int64_t m = n - 1 - y;
        for (int64_t x = 0; x < n; ++x) {
            uint64_t v = splitmix64(seed ^ (((uint64_t)y << 32) | (uint64_t)x));
            if (mode == 1 && (x & m) != 0) v = 0;
            int64_t i = (y - w0) * n + x;
            switch (cell_bytes) {
            case 1: ((uint8_t*)buf)[i] = (uint8_t)v; break;
            case 2: ((uint16_t*)buf)[i] = (uint16_t)v; break;
            case 4: ((uint32_t*)buf)[i] = (uint32_t)v; break;
            default: ((uint64_t*)buf)[i] = v; break;
            }
        }
    }
}

#define DEFINE_BAND_STEP(T, SUF)                                                            \
static void band_step_##SUF(T* dst, const T* src, int64_t n, int64_t w0, int64_t w1,       \
                            int kind, int32_t param, int threads) {                        \
    _Pragma("omp parallel for num_threads(nthr(threads)) schedule(dynamic, 16)")           \
    for (int64_t y = w0; y < w1; ++y) {                                                    \
        const T* r0 = src + (y - w0) * n;                                                  \
        const T* rp = (y > w0) ? r0 - n : 0;          /* row y-1 (absent: grid or window edge) */ \
        const T* rn = (y + 1 < w1) ? r0 + n : 0;      /* row y+1 */                        \
        T* out = dst + (y - w0) * n;                                                       \
        const int64_t m = y;   /* x & (n-1-y) == 0  <=>  x is a bit-subset of y */         \
        int64_t x = 0;                                                                     \
        if (kind == KIND_CONST) {                       /* the write pass: param */        \
            do { out[x] = (T)(int64_t)param; x = (x - m) & m; } while (x != 0);            \
            continue;                                                                      \
        }                                                                                  \
        do {                                                                               \
            uint64_t t = (uint64_t)(int64_t)param;                                         \
            if (x > 0) t += (uint64_t)(int64_t)r0[x - 1];                                  \
            if (x < n - 1) t += (uint64_t)(int64_t)r0[x + 1];                              \
            if (rp) t += (uint64_t)(int64_t)rp[x];                                         \
            if (rn) t += (uint64_t)(int64_t)rn[x];                                         \
            if (kind == KIND_NSUM8) {                                                      \
                if (rp && x > 0) t += (uint64_t)(int64_t)rp[x - 1];                        \
                if (rp && x < n - 1) t += (uint64_t)(int64_t)rp[x + 1];                    \
                if (rn && x > 0) t += (uint64_t)(int64_t)rn[x - 1];                        \
                if (rn && x < n - 1) t += (uint64_t)(int64_t)rn[x + 1];                    \
            }                                                                              \
            out[x] = (T)t;                                                                 \
            x = (x - m) & m;                                                               \
        } while (x != 0);                                                                  \
    }                                                                                      \
}

DEFINE_BAND_STEP(int8_t, i8)
DEFINE_BAND_STEP(int16_t, i16)
DEFINE_BAND_STEP(int32_t, i32)
DEFINE_BAND_STEP(int64_t, i64)

int go_steps_band(void* const* outs, const int32_t* steps, int nouts, int64_t n, int cell_bytes, uint64_t seed,
                  int mode, int kind, int32_t param, int64_t y0, int64_t y1, int threads) {
    if (kind != KIND_CONST && kind != KIND_NSUM4 && kind != KIND_NSUM8) return -1;
    if (y0 < 0 || y1 > n || y0 >= y1 || nouts < 1) return -1;
    int smax = 0;
    for (int i = 0; i < nouts; ++i) {
        if (steps[i] < 0) return -1;
        if (steps[i] > smax) smax = steps[i];
    }
    const int64_t w0 = y0 - smax < 0 ? 0 : y0 - smax, w1 = y1 + smax > n ? n : y1 + smax;
    const size_t bytes = (size_t)(w1 - w0) * (size_t)n * (size_t)cell_bytes;
    char* a = (char*)malloc(bytes);
    char* b = (char*)malloc(bytes);
    if (!a || !b) { free(a); free(b); return -2; }
    fill_rows(a, n, cell_bytes, seed, mode, w0, w1, threads);
    memcpy(b, a, bytes);  /* off-gasket cells: identical in both ping-pong buffers for ever */
    const size_t off = (size_t)(y0 - w0) * (size_t)n * (size_t)cell_bytes;
    const size_t len = (size_t)(y1 - y0) * (size_t)n * (size_t)cell_bytes;
    for (int s = 0; s <= smax; ++s) {
        if (s > 0) {
            switch (cell_bytes) {
            case 1: band_step_i8((int8_t*)b, (const int8_t*)a, n, w0, w1, kind, param, threads); break;
            case 2: band_step_i16((int16_t*)b, (const int16_t*)a, n, w0, w1, kind, param, threads); break;
            case 4: band_step_i32((int32_t*)b, (const int32_t*)a, n, w0, w1, kind, param, threads); break;
            case 8: band_step_i64((int64_t*)b, (const int64_t*)a, n, w0, w1, kind, param, threads); break;
            default: free(a); free(b); return -1;
            }
            char* t = a; a = b; b = t;
        }
        for (int i = 0; i < nouts; ++i)
            if (steps[i] == s) memcpy(outs[i], a + off, len);
    }
    free(a);
    free(b);
    return 0;
}
