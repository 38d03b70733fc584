/*
 * gasket_b200.h -- C ABI of libgasket_b200.so, the sm_100a implementation of
 * the block-space map lambda(omega) and the embedded-gasket kernels it drives.
 *
 * Drop-in boundary.  Each entry point replaces one reference interface
 * (paths relative to /root/reference/pkg/src/gasketmap/):
 *
 *   gm_run_bounding_box  <- backends.run_bounding_box   backends.py:225-231
 *                           (numba kernel _bounding_box_nb, backends.py:143-156)
 *   gm_run_block_space   <- backends.run_block_space    backends.py:234-272
 *                           (numba kernel _block_space_nb, backends.py:158-222)
 *   gm_map_blocks        <- blockmap.map_blocks_array   blockmap.py:91-108
 *   gm_map_rectangle     <- the idx%W, idx//W call sites of map_blocks_array
 *                           (blockmap.py:140-141, engine.py:233-235, backends.py:103-105)
 *   gm_coverage          <- engine.verify_coverage      engine.py:214-258 (counting leg)
 *   gm_coverage_blocks   <- engine.verify_coverage with a map_fn  engine.py:236-251
 *   gm_bijection_check   <- blockmap.verify_bijection   blockmap.py:123-166
 *
 * Conventions (mirroring backends.py): grids are dense row-major n x n arrays
 * of 1/2/4/8-byte integer cells; `grid` is mutated in place and only gasket
 * cells are written; `src` is the read-only pre-launch snapshot and may alias
 * `grid` only for GM_KIND_CONST.  Pointers are device pointers or mapped
 * pinned-host pointers (cudaHostRegisterMapped / cudaHostAlloc(Mapped)).
 * Every launch is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default stream).  Results: 0 on success, otherwise a GM_E* code, with a
 * message in gm_last_error() (thread-local).  No entry point falls back to
 * the CPU.
 */
#ifndef GASKET_B200_H
#define GASKET_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* backends.py:30-34 integer tags, extended. */
#define GM_KIND_CONST 0   /* KERNEL_CONST */
#define GM_KIND_NSUM4 1   /* KERNEL_NEIGHBOR_SUM (4-neighbour) */
#define GM_KIND_NSUM8 2   /* 8-neighbour extension (no reference implementation) */
#define GM_KIND_COUNT 3   /* coverage audit: atomic per-cell uint32 counters */

#define GM_STRAT_UNROLL 0 /* STRAT_UNROLL */
#define GM_STRAT_TABLE 1  /* STRAT_TABLE */
#define GM_STRAT_SUBBOX 2 /* STRAT_SUBBOX */
#define GM_STRAT_TUNED 3  /* B200 row-segment kernel (same index set) */

#define GM_MAP_BB 0       /* engine.Mapping.BOUNDING_BOX (paper-literal) */
#define GM_MAP_LAMBDA 1   /* engine.Mapping.BLOCK_SPACE */
#define GM_MAP_BB_EXIT 2  /* bounding box with block-level early exit */
#define GM_MAP_BB_VEC 3   /* bounding box, vectorised: one lane per 16-byte segment of all n*n cells (write pass) */

/* Launch flags.  All but GM_FLAG_DST_FROM_SRC and GM_FLAG_HOST_ROWS select kernel
 * variants kept for A/B measurement (scripts/variants.py; results in
 * profiles/r1_probes.md); every variant computes the same cells except the
 * GM_FLAG_PROBE_* design probes.  The defaults are the measured-best variants. */
#define GM_FLAG_OMEGA_ORDER 1  /* tuned: visit tiles in b = wy*W + wx order */
#define GM_FLAG_DST_FROM_SRC 2 /* stencil: grid == copy of src off-gasket (engine.py:201) */
#define GM_FLAG_EXPLICIT_RMW 4 /* tuned write: load partial sectors, store whole sectors */
#define GM_FLAG_WHOLE_LINES 8  /* with EXPLICIT_RMW: read-modify-write whole 128-byte tile rows */
#define GM_FLAG_HOST_ROWS 16   /* write pass on a host-mapped grid: row-ordered whole-line schedule */
#define GM_FLAG_ROWMAJOR 32    /* tuned: visit tiles row-major per sub-gasket (the default since v2; kept for ABI) */
#define GM_FLAG_CHUNKED 64     /* tuned stencil: contiguous tile run per CTA instead of interleaved */
#define GM_FLAG_NO_TMA 128     /* A/B builds only (GASKET_AB_BUILD=1): never the TMA-staged stencil */
#define GM_FLAG_FORCE_TMA 256  /* A/B builds only: the superseded TMA-staged stencil (stencil_tma.cu) */
#define GM_FLAG_FETCH_LINE 512 /* tuned kernels: whole-line (.L2::128B) loads (stencil v2: the default since round 1d) */
#define GM_FLAG_FETCH64 1024   /* tuned write: touch each written 64-byte half with an .L2::64B load first
                                  (with GM_FLAG_FETCH_LINE: touch the whole line) */
#define GM_FLAG_STENCIL_V1 2048 /* A/B builds only: the superseded v1 stencil (stencil.cu) instead of v2 */
#define GM_FLAG_STAGES2 4096   /* tuned stencil v2: 2-deep staging ring instead of 3/4 */
#define GM_FLAG_PROBE_NOSTORE 8192  /* A/B builds only: design probe, no stores (result undefined) */
#define GM_FLAG_PROBE_NOLOAD 16384  /* A/B builds only: design probe, no staging (result undefined) */
#define GM_FLAG_PROBE_NOCOMPUTE 32768 /* A/B builds only: design probe, no arithmetic (result undefined) */
#define GM_FLAG_DIGIT_ORDER 65536 /* tuned: visit tiles in lambda digit order instead of row-major per sub-gasket */
#define GM_FLAG_STORE_CS 131072   /* tuned write pass / stencil v2: streaming (evict-first) stores */
#define GM_FLAG_BAND_MAJOR 262144 /* tuned write pass: hand out (band, tile) units band-major */
#define GM_FLAG_PREFETCH_AHEAD 524288 /* tuned write pass: L2-prefetch the lines of the unit two ahead */
#define GM_FLAG_FETCH_MIXED 1048576   /* stencil v2 with FETCH_HALF: whole-line fetch for lines needed in both halves */
#define GM_FLAG_FETCH_HALF 2097152    /* stencil v2: stage with the .L2::64B hint (64-byte halves) instead of whole lines */
#define GM_FLAG_FETCH256 4194304      /* stencil v2: stage interior tiles with the .L2::256B prefetch-size hint */
#define GM_FLAG_TWO_STEPS 8388608     /* gm_run_part_peer: two fused CA steps per launch (depth-2 halo) */
#define GM_FLAG_FOUR_STEPS 16777216   /* gm_run_part_peer: four fused CA steps per launch (depth-4 halo) */
#define GM_FLAG_SIX_STEPS 33554432    /* gm_run_part_peer: six fused CA steps per launch (depth-6 halo) */
#define GM_FLAG_ZERO_BACKGROUND 67108864 /* tuned write pass, opt-in: the caller asserts every off-gasket cell is 0
                                            (PAPER.md:442-443's zero-filled matrix); touched 32-byte sectors are
                                            stored whole (gasket cells = param, the rest 0), no DRAM read-modify-write */
#define GM_FLAG_WRITE_HALVES 134217728 /* zero-background write pass: store the touched 64-byte halves whole */
#define GM_FLAG_WRITE_LINES 268435456  /* zero-background write pass: store the touched 128-byte lines whole */
#define GM_FLAG_STATIC_SCHEDULE 4096 /* tuned write pass: static round-robin units instead of the ticket queue
                                       (A/B; shares its value with the stencil-only GM_FLAG_STAGES2) */
#define GM_FLAG_WRITE_SWEEP 1073741824 /* tuned write pass: the grid's member lines in address order, chunks of
                                          32 lines dealt round-robin over all warps (write.cu) */
#define GM_FLAG_GRID_ROWS 536870912   /* tuned write pass: no blocks -- one warp per grid row, its member lines
                                         left to right (the row enumeration; write.cu) */

#define GM_OK 0
#define GM_EINVAL 1  /* bad shape / size / tag (the reference's ValueError) */
#define GM_ECUDA 2   /* CUDA runtime error */
#define GM_ENOMEM 3

typedef struct gm_cfg {
    int64_t n;          /* grid edge, power of two */
    int32_t rho;        /* block edge, power of two, rho <= n */
    int32_t mapping;    /* GM_MAP_* */
    int32_t strategy;   /* GM_STRAT_* (ignored for bounding-box maps) */
    int32_t kind;       /* GM_KIND_* */
    int32_t cell_bytes; /* 1, 2, 4 or 8 */
    int32_t param;      /* CellKernel.param (engine.py:35-41); int32 like np.int32(param) */
    int32_t flags;      /* GM_FLAG_* */
    int32_t reserved;
} gm_cfg_t;

/* backends.py:225-231.  grid/src: n*n cells.  early_exit: 0 = the paper-literal kernel,
 * 1 = off-gasket blocks exit first (GM_MAP_BB_EXIT), 2 = vectorised (GM_MAP_BB_VEC, write
 * pass only: GM_EINVAL for neighbour sums). */
int gm_run_bounding_box(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t rho,
                        int32_t kind, int32_t param, int32_t early_exit, void* stream);

/* backends.py:234-272.  tab_x/tab_y: device int32[ntab] local offsets (TABLE only;
 * intra.build_lookup_table order), ignored by the other strategies. */
int gm_run_block_space(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t rho,
                       int32_t r_b, int32_t strategy, const int32_t* tab_x, const int32_t* tab_y,
                       int32_t ntab, int32_t kind, int32_t param, int32_t flags, void* stream);

/* Generic launch through a config struct (engine.LaunchPlan.run, engine.py:159-178). */
int gm_launch(const gm_cfg_t* cfg, void* grid, const void* src, const int32_t* tab_x,
              const int32_t* tab_y, int32_t ntab, void* stream);

/* Multi-GPU partition (no reference counterpart): the tuned kernel
 * restricted to the level-`level` sub-gaskets [sg_begin, sg_end) in base-3 digit
 * order (a contiguous tile range of the lambda digit order). */
int gm_run_part(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* stream);
/* Halo plumbing: out[i] = grid[idx[i]] / grid[idx[i]] = in[i] (linear cell indices). */
int gm_gather_cells(const void* grid, int32_t cell_bytes, const int64_t* idx, int64_t count, void* out,
                    void* stream);
int gm_scatter_cells(void* grid, int32_t cell_bytes, const int64_t* idx, int64_t count, const void* in,
                     void* stream);

/* blockmap.py:91-108: (lx, ly) = lambda(wx, wy) element-wise, int64, floor semantics. */
int gm_map_blocks(const int64_t* wx, const int64_t* wy, int64_t count, int32_t r_b, int64_t* lx,
                  int64_t* ly, void* stream);

/* lambda over the whole packed rectangle in b = wy*W + wx order (3^r_b entries). */
int gm_map_rectangle(int32_t r_b, int64_t* lx, int64_t* ly, void* stream);

/* engine.py:214-258 counting leg: counts (uint32, n*n, zeroed by the caller)
 * += 1 per cell the launch shape of `cfg` writes, using the real kernels. */
int gm_coverage(const gm_cfg_t* cfg, uint32_t* counts, const int32_t* tab_x, const int32_t* tab_y,
                int32_t ntab, void* stream);

/* engine.py:245-251 with explicit block coordinates (map_fn given): counts +=1 at
 * (bx*rho+lx, by*rho+ly) for every block and local cell; off-grid writes dropped. */
int gm_coverage_blocks(const int64_t* bx, const int64_t* by, int64_t nblocks, const int32_t* lx,
                       const int32_t* ly, int32_t nlocal, int32_t rho, int64_t n, uint32_t* counts,
                       void* stream);

/* engine.py:252-258, the comparison leg of the coverage audit, on the device: over the
 * n*n uint32 counters of gm_coverage, totals[0] = duplicates (count above membership),
 * totals[1] = misses (gasket cells with count 0); the first `cap` linear indices y*n + x of
 * each go to dup_idx / miss_idx in no particular order.  totals: device, 2 entries. */
int gm_coverage_check(const uint32_t* counts, int64_t n, unsigned long long* totals, int64_t* dup_idx,
                      int64_t* miss_idx, int64_t cap, void* stream);

/* blockmap.py:123-166 on the device.  Maps coordinates (cx, cy) (e.g. from
 * gm_map_rectangle, row-major omega order) of nblocks blocks onto the edge-n_b
 * gasket; owner must be n_b*n_b int64 scratch.  Writes result[0] = first bad
 * omega index (or -1), result[1] = number of distinct gasket cells hit. */
int gm_bijection_check(const int64_t* cx, const int64_t* cy, int64_t nblocks, int64_t n_b,
                       int64_t* owner, int64_t* result, void* stream);

/* The pre-launch snapshot of a neighbour-sum launch (engine.py:201's grid.copy()),
 * masked: copies into `snap` (n*n cells, distinct from grid) only what a one-step
 * stencil over the gasket reads -- each member 128-byte tile's rows -1..TT, the 32-byte
 * sector left of them, and the sector right of rows TT-2..TT (only tile column TT-1's
 * gasket cell, at row TT-1, reads further right) -- at the same positions; other cells
 * of snap are left as they are.  A grid off a 64-byte boundary (a host numpy array, read over PCIe in
 * host-aligned 64-byte units) gets, per window row, the units covering bytes [-16, 144)
 * of the tile's line instead: what the tuned stencil and gm_writeback_tiles read (the
 * staged host path's kernels).  Async on `stream`.  GM_EINVAL for other cell widths, edges that are
 * not a power of two >= 128/cell_bytes, or more than 2^15 tiles per edge. */
int gm_snapshot_stencil(void* snap, const void* grid, int64_t n, int32_t cell_bytes, void* stream);
/* The write-back of a staged neighbour-sum launch (host-mapped grids): writes every
 * member tile's own rows (128-byte lines) of `out` whole -- sectors holding gasket
 * cells from `dst`, the others from `snap`.  out, dst, snap: n*n cells, distinct. */
int gm_writeback_tiles(void* out, const void* dst, const void* snap, int64_t n, int32_t cell_bytes, void* stream);

/* The staged host path in bands (backends.py: a neighbour-sum launch on a host grid
 * whose src is the grid): gm_snapshot_stencil / gm_writeback_tiles and the tuned step
 * (stencil v2) restricted to the tiles [t0, t1) of the whole-grid row-major tile order
 * (gm_tile_order(q, 0); whole block rows), so that one band's write-back (device -> host)
 * overlaps the next bands' snapshots (host -> device) on another stream.  The snapshot
 * of band b+1 must be complete before band b is written back or stepped. */
int gm_snapshot_stencil_range(void* snap, const void* grid, int64_t n, int32_t cell_bytes, uint32_t t0, uint32_t t1,
                              void* stream);
int gm_writeback_tiles_range(void* out, const void* dst, const void* snap, int64_t n, int32_t cell_bytes, uint32_t t0,
                             uint32_t t1, void* stream);
int gm_run_tiles(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param, int32_t flags,
                 uint32_t t0, uint32_t t1, void* stream);

/* Synthetic inputs / checks shared with the CPU oracle (oracle/gasket_oracle.c). */
int gm_fill_hash(void* buf, int64_t n, int32_t cell_bytes, uint64_t seed, int32_t mode, void* stream);
int gm_checksum(const void* buf, int64_t count, int32_t cell_bytes, uint64_t* out_dev, void* stream);
int gm_count_equal(const void* a, const void* b, int64_t count, int32_t cell_bytes,
                   unsigned long long* out_dev, void* stream);
/* Reads `bytes` of `buf` (bigger than L2) so the next kernel starts cold. */
int gm_l2_flush(const void* buf, int64_t bytes, uint64_t* sink_dev, void* stream);

/* Host buffers for the zero-copy transport: returns the device-visible address
 * of a page-locked host range, page-locking and mapping it first when
 * register_if_needed != 0 (cudaHostRegisterMapped); *registered = 1 when this
 * call did the registration (the caller then owns a gm_host_unmap). */
int gm_host_map(void* host, int64_t bytes, int32_t register_if_needed, void** dev_ptr,
                int32_t* registered);
int gm_host_unmap(void* host);

/* Device-wide L2 fetch granularity hint (cudaLimitMaxL2FetchGranularity, 0..128 bytes). */
int gm_set_l2_fetch_granularity(int32_t bytes);

/* Number of kernels this library has launched (all entry points). */
/* Two CA steps in one pass (temporal blocking, stencil_tb.cu): grid <- kind(kind(src)),
 * each step the neighbour-sum launch with engine.launch's snapshot semantics.
 * Precondition (the CA ping-pong invariant): grid == src on every off-gasket cell.
 * kind = GM_KIND_NSUM4 or GM_KIND_NSUM8; 1-, 2- or 4-byte cells; async on `stream`. */
int gm_ca_step2(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                int32_t flags, void* stream);
/* gm_ca_step2 with `steps` = 2, 4 or 6 fused CA steps per launch (temporal blocking over
 * a `steps`-cell-deep dependency cone; 6 needs 1- or 2-byte cells):
 * grid <- step^steps(src), same preconditions. */
int gm_ca_steps(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                int32_t steps, int32_t flags, void* stream);
/* CA runs with a static left-edge cache (edge.cu, no reference
 * counterpart).  Off-gasket cells never change in a CA run (backends.py:155-156), so
 * the 16-byte chunks left of the rows of every member tile whose left neighbour tile
 * holds no gasket cell -- one sparse DRAM line per row otherwise -- are gathered once
 * into a dense cache and staged from there by every step.
 * gm_ca_edge_bytes: the cache size for the tiles of the level-`level` sub-gaskets
 * [sg_begin, sg_end) (level < 0: the whole gasket).  gm_ca_edge_build: fill it from
 * `src` (dense n x n, or the tiled blocks of gm_run_part_tiled when sg_off != NULL).
 * gm_ca_run: `steps` (1, 2, 4 or 6) CA steps src -> grid with the CA ping-pong
 * preconditions of gm_ca_steps (grid == src off the gasket) and the cache built from a
 * buffer that agrees with src off the gasket (edge = NULL: no cache; the fused 2/4/6-step
 * kernels, bound by arithmetic rather than staging, read the grid either way); flags:
 * GM_FLAG_* kernel variants (0: the defaults). */
int gm_ca_edge_bytes(int64_t n, int32_t cell_bytes, int32_t level, uint32_t sg_begin, uint32_t sg_end,
                     int64_t* bytes);
int gm_ca_edge_build(void* edge, const void* src, int64_t n, int32_t cell_bytes, int32_t level, uint32_t sg_begin,
                     uint32_t sg_end, const int64_t* sg_off, int64_t pitch, void* stream);
int gm_ca_run(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param, int32_t steps,
              const void* edge, int32_t flags, void* stream);
/* In-place neighbour-sum launch with engine.launch's snapshot semantics (engine.py:201:
 * every cell reads the pre-launch state) without a grid-sized snapshot (edge.cu): each
 * tile stages its window before it writes, so only the <= 5 border cells per member tile
 * that neighbouring tiles read can change under them; those are copied into `border`
 * (gm_border_bytes bytes, device memory, one per stream) and patched into the staged
 * windows.  kind NSUM4 / NSUM8; 1-, 2- or 4-byte cells, n >= one 128-byte tile. */
int gm_border_bytes(int64_t n, int32_t cell_bytes, int64_t* bytes);
int gm_run_inplace(void* grid, void* border, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                   void* stream);
/* Peer-memory halo exchange of the partitioned CA (peer.cu).
 * gm_dev_alloc/free: plain cudaMalloc'd buffers (allocation bases, so they can be
 * exported); gm_ipc_get_handle writes a 64-byte cudaIpcMemHandle_t; gm_ipc_open_handle
 * maps a peer's buffer.  gm_peer_halo_put copies the `count` cells at linear indices
 * `idx` from `mine` into each peer grid (peers = device array of `world` grid
 * pointers, own entry unused), then release-stores `epoch` into slot `rank` of each
 * peer's flag array (peer_flags = device array of `world` flag-array pointers).
 * gm_peer_halo_wait acquires slots != rank of the own flag array until they reach
 * `epoch`; after timeout_ns it sets bit p of *status instead of hanging. */
int gm_dev_alloc(int64_t bytes, void** out);
int gm_dev_free(void* p);
int gm_ipc_get_handle(void* base, void* handle_out);
int gm_ipc_open_handle(const void* handle, void** out);
int gm_ipc_close(void* p);
int gm_peer_halo_put(const void* mine, const uint64_t* peers, const int64_t* idx, int64_t count, int32_t cell_bytes,
                     const uint64_t* peer_flags, int32_t rank, int32_t world, uint64_t epoch, void* stream);
int gm_peer_halo_wait(const uint64_t* flags, int32_t rank, int32_t world, uint64_t epoch, uint64_t timeout_ns,
                      uint32_t* status, void* stream);
/* gm_peer_halo_put with a destination per entry (tiled partition storage): entry i copies
 * cell idx[i] of `mine` to cell (didx[i] & (2^56-1)) of rank (didx[i] >> 56)'s buffer --
 * the own rank's entries are ring copies inside `mine` -- then releases `epoch` as above. */
int gm_peer_halo_put_to(const void* mine, const uint64_t* peers, const int64_t* idx, const int64_t* didx,
                        int64_t count, int32_t cell_bytes, const uint64_t* peer_flags, int32_t rank, int32_t world,
                        uint64_t epoch, void* stream);
/* Tiled partition storage (per-rank storage = the owned level-`level`
 * sub-gaskets plus a ring, not two n x n grids).  Each owned sub-gasket is one block of
 * (m + 2R) rows x `pitch` bytes (m = n >> level; R ring rows; `pitch` >= m*cell_bytes plus
 * the ring columns, a multiple of 32); the global cell (x, y) of sub-gasket sg_begin + k
 * lives at byte sg_off[k] + y*pitch + x*cell_bytes of the buffer (sg_off: device int64[],
 * the block's virtual origin).  Rings hold the neighbours' cells (static off-gasket
 * values once, changing halo cells per exchange).
 * gm_run_part_tiled: `steps` (1, 2, 4 or 6) CA steps src -> grid over the rank's blocks
 * (one step: whole-sector blend from src; the blocks of src and grid agree off the gasket);
 * epilogue/wait/signal: the fused peer exchange of gm_run_part_peer (NULL: none; the
 * descriptor's didx then lists per-entry destinations, gm_peer_halo_put_to's format);
 * edge: the rank's static left-edge cache (gm_ca_edge_build over the same blocks; used by
 * one-step launches; NULL: none).
 * gm_copy_cells: dst[dst_idx[i]] = src[src_idx[i]] (cell indices).  gm_fill_hash_window:
 * the synthetic grid's cells [x0, x0+w) x [y0, y0+h) (0 outside n x n) into a pitched
 * block. */
int gm_run_part_tiled(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                      int32_t steps, int32_t level, uint32_t sg_begin, uint32_t sg_end, const int64_t* sg_off,
                      int64_t pitch, void* epilogue, uint64_t wait_epoch, uint64_t signal_epoch, const void* edge,
                      void* stream);
int gm_copy_cells(void* dst, const void* src, int32_t cell_bytes, const int64_t* dst_idx, const int64_t* src_idx,
                  int64_t count, void* stream);
int gm_fill_hash_window(void* out, int64_t pitch, int64_t n, int32_t cell_bytes, int64_t x0, int64_t y0, int64_t w,
                        int64_t h, uint64_t seed, int32_t mode, void* stream);
/* gm_run_part with the halo exchange fused into the step kernel (peer_epilogue.cuh):
 * `epilogue` = device descriptor (PartitionedCA(halo="peer", fused=True) builds it);
 * every CTA first acquires the peers' flags >= wait_epoch (0: no wait), the last CTA
 * to finish stores the rank's halo cells into the peers' buffers and releases
 * signal_epoch.  With GM_FLAG_TWO_STEPS / _FOUR_STEPS / _SIX_STEPS the launch is
 * gm_run_part_steps' 2 / 4 / 6 fused steps (the halo must then be of that depth).
 * Stream-ordered like every launch. */
int gm_run_part_peer(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                     int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* epilogue,
                     uint64_t wait_epoch, uint64_t signal_epoch, void* stream);
/* gm_ca_step2 restricted to the level-`level` sub-gaskets [sg_begin, sg_end) (digit
 * order), like gm_run_part: one rank's share of a partitioned CA, two steps per call.
 * The caller keeps the halo within two steps current (PartitionPlan(depth=2)). */
int gm_run_part2(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                 int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* stream);
/* gm_run_part2 with `steps` = 2, 4 or 6 fused steps per call (PartitionPlan(depth=steps)). */
int gm_run_part_steps(void* grid, const void* src, int64_t n, int32_t cell_bytes, int32_t kind, int32_t param,
                      int32_t steps, int32_t flags, int32_t level, uint32_t sg_begin, uint32_t sg_end, void* stream);
/* The tuned kernels' tile visiting order (host-side, no GPU needed): the 3^q
 * member tiles of a level-q gasket as bx | by << 16, level-`level` sub-gaskets in
 * lambda digit order, row-major inside each.  out must hold 3^q entries. */
int gm_tile_order(int32_t q, int32_t level, uint32_t* out, int64_t capacity);
uint64_t gm_launch_count(void);
const char* gm_last_error(void);
const char* gm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GASKET_B200_H */
