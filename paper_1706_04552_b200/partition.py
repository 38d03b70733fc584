"""Multi-GPU partition of the gasket by self-similar sub-gaskets.

No reference counterpart: the reference is single-process (numba ``prange``,
backends.py:147, 162).  The level-L sub-gaskets of an edge-n gasket are the
3**L member blocks of edge m = n >> L; in the base-3 digit order of the
lambda map (digit i <-> level i+1) sub-gasket s is exactly the contiguous tile
range [s * 3**(r_t-L), (s+1) * 3**(r_t-L)) of the tuned kernels, so a rank
owning the sub-gaskets [s0, s1) launches one kernel over one tile range
(``gm_run_part``).

Write passes need no communication (lambda is a bijection: ranks write
disjoint cells).  A neighbour-sum CA step reads a one-cell halo; because the
reference never writes off-gasket cells (backends.py:155-156), the only halo
cells that change are gasket cells next to another sub-gasket -- a handful of
cells at the sub-gasket corners (at most 5 per sub-gasket for 8 neighbours,
3 for 4).  ``PartitionPlan`` finds them exhaustively; ``HaloExchange`` moves
them after every step with one fixed-size ``all_gather`` (NCCL on the GPU,
gloo on CPU, or an in-process loopback for several virtual ranks on one GPU).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from .geometry import scale_level


def subgasket_block(s: int, level: int) -> tuple[int, int]:
    """Block coordinates of level-`level` sub-gasket s (digit i -> bit i: 0 top, 1 below, 2 below-right)."""
    bx = by = 0
    for i in range(level):
        s, d = divmod(s, 3)
        if d:
            by |= 1 << i
            if d == 2:
                bx |= 1 << i
    return bx, by


def subgasket_index(bx: int, by: int, level: int) -> Optional[int]:
    """Inverse of subgasket_block; None for blocks off the gasket."""
    if bx & ~by:
        return None
    s = 0
    for i in reversed(range(level)):
        yb, xb = (by >> i) & 1, (bx >> i) & 1
        s = s * 3 + (0 if not yb else (2 if xb else 1))
    return s


def rank_ranges(nsg: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced sub-gasket ranges per rank."""
    return [(r * nsg // world, (r + 1) * nsg // world) for r in range(world)]


def _is_member(x: np.ndarray, y: np.ndarray, n: int) -> np.ndarray:
    return (x & (n - 1 - y)) == 0


@dataclass
class PartitionPlan:
    n: int
    level: int
    world: int
    eight: bool = True
    depth: int = 1  # CA steps per exchange (2, 4 or 6: fused steps per launch, gm_run_part_steps)
    ranges: list[tuple[int, int]] = field(init=False)
    halo: dict[int, np.ndarray] = field(init=False)  # sub-gasket -> linear indices of changing halo cells

    def __post_init__(self) -> None:
        r = scale_level(self.n)
        if not 0 <= self.level <= r:
            raise ValueError(f"partition level {self.level} outside [0, {r}]")
        self.nsg = 3 ** self.level
        self.m = self.n >> self.level
        if self.world > self.nsg:
            # a rank without sub-gaskets would never launch, so on the fused peer path it
            # would never release its step flag and its peers would wait for it
            raise ValueError(f"{self.world} ranks exceed the {self.nsg} level-{self.level} sub-gaskets")
        self.ranges = rank_ranges(self.nsg, self.world)
        if self.depth not in (1, 2, 4, 6):
            raise ValueError("depth must be 1, 2, 4 or 6 (CA steps per halo exchange)")
        self.halo = {s: self._halo_cells_depth(s) for s in range(self.nsg)}

    # -- ownership --------------------------------------------------------
    def owner_of_subgasket(self, s: int) -> int:
        for rank, (lo, hi) in enumerate(self.ranges):
            if lo <= s < hi:
                return rank
        raise ValueError(s)

    def owner_of_cells(self, lin: np.ndarray) -> np.ndarray:
        y, x = np.divmod(lin, self.n)
        bx, by = x // self.m, y // self.m
        owners = np.empty(lin.shape, dtype=np.int64)
        for i, (a, b) in enumerate(zip(bx.tolist(), by.tolist())):
            s = subgasket_index(a, b, self.level)
            owners[i] = -1 if s is None else self.owner_of_subgasket(s)
        return owners

    # -- halo -------------------------------------------------------------
    def _halo_cells(self, s: int) -> np.ndarray:
        """Gasket cells outside sub-gasket s that a gasket cell inside s reads."""
        n, m = self.n, self.m
        bx, by = subgasket_block(s, self.level)
        ox, oy = bx * m, by * m
        ring = np.arange(-1, m + 1, dtype=np.int64)
        xs = np.concatenate([ring, ring, np.full(m, -1), np.full(m, m)])
        ys = np.concatenate([np.full(m + 2, -1), np.full(m + 2, m), np.arange(m), np.arange(m)])
        gx, gy = ox + xs, oy + ys
        ok = (gx >= 0) & (gx < n) & (gy >= 0) & (gy < n)
        xs, ys, gx, gy = xs[ok], ys[ok], gx[ok], gy[ok]
        ok = _is_member(gx, gy, n)
        xs, ys, gx, gy = xs[ok], ys[ok], gx[ok], gy[ok]
        offs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
        if self.eight:
            offs += [(1, 1), (1, -1), (-1, 1), (-1, -1)]
        read = np.zeros(xs.shape, dtype=bool)
        for dx, dy in offs:
            ix, iy = xs + dx, ys + dy
            inside = (ix >= 0) & (ix < m) & (iy >= 0) & (iy < m)
            read |= inside & _is_member(ox + np.clip(ix, 0, m - 1), oy + np.clip(iy, 0, m - 1), n)
        return np.unique(gy[read] * n + gx[read])

    def _offsets(self) -> list[tuple[int, int]]:
        offs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
        if self.eight:
            offs += [(1, 1), (1, -1), (-1, 1), (-1, -1)]
        return offs

    def _halo_cells_depth(self, s: int) -> np.ndarray:
        """Changing cells outside sub-gasket s that its next `depth` steps read: H_1 is the
        one-step halo; H_{k+1} adds every gasket cell outside s next to an H_k cell (H_k's
        later values, recomputed locally, read those one step earlier).  Off-gasket cells
        never change, and a rank holds them from the start."""
        h = self._halo_cells(s)
        if self.depth == 1 or h.size == 0:
            return h
        n, m = self.n, self.m
        bx, by = subgasket_block(s, self.level)
        ox, oy = bx * m, by * m
        cells, frontier = set(h.tolist()), set(h.tolist())
        for _ in range(self.depth - 1):
            grown = set()
            for c in frontier:
                y, x = divmod(c, n)
                for dx, dy in self._offsets():
                    gx, gy = x + dx, y + dy
                    if not (0 <= gx < n and 0 <= gy < n) or (gx & (n - 1 - gy)) != 0:
                        continue
                    if ox <= gx < ox + m and oy <= gy < oy + m:
                        continue  # own cell
                    if gy * n + gx not in cells:
                        grown.add(gy * n + gx)
            cells |= grown
            frontier = grown
        return np.array(sorted(cells), dtype=np.int64)

    def exchange_slots(self) -> tuple[list[np.ndarray], int]:
        """Per owner rank, the sorted linear indices of its cells some other rank reads."""
        need: list[set[int]] = [set() for _ in range(self.world)]
        for s in range(self.nsg):
            reader = self.owner_of_subgasket(s)
            cells = self.halo[s]
            if cells.size == 0:
                continue
            for c, o in zip(cells.tolist(), self.owner_of_cells(cells).tolist()):
                if o >= 0 and o != reader:
                    need[o].add(c)
        slots = [np.array(sorted(v), dtype=np.int64) for v in need]
        width = max([1] + [len(v) for v in slots])
        return slots, width


class LoopbackGroup:
    """In-process stand-in for a process group: `world` virtual ranks on one device.

    all_gather is called once per virtual rank; the last call completes the
    gather for everyone (ranks are stepped in order by the driver)."""

    def __init__(self, world: int) -> None:
        self.world = world
        self._parts: dict[int, torch.Tensor] = {}

    def contribute(self, rank: int, t: torch.Tensor) -> None:
        self._parts[rank] = t.clone()

    def gathered(self) -> torch.Tensor:
        return torch.cat([self._parts[r] for r in range(self.world)])


class HaloExchange:
    """Moves the changing halo cells after each step: gather own slots, one
    fixed-size all_gather, scatter the other ranks' slots."""

    def __init__(self, plan: PartitionPlan, rank: int, device: torch.device, dtype: torch.dtype,
                 group=None, loopback: Optional[LoopbackGroup] = None) -> None:
        self.plan, self.rank, self.device, self.dtype = plan, rank, device, dtype
        self.group, self.loopback = group, loopback
        slots, self.width = plan.exchange_slots()
        self.send_idx = torch.from_numpy(slots[rank]).to(device)
        recv = [slots[r] for r in range(plan.world)]
        # positions in the gathered buffer and the cells they belong to (other ranks only)
        pos, cells = [], []
        for r, v in enumerate(recv):
            if r == rank or v.size == 0:
                continue
            pos.append(r * self.width + np.arange(v.size))
            cells.append(v)
        self.recv_pos = torch.from_numpy(np.concatenate(pos) if pos else np.zeros(0, np.int64)).to(device)
        self.recv_idx = torch.from_numpy(np.concatenate(cells) if cells else np.zeros(0, np.int64)).to(device)
        self.sendbuf = torch.zeros(self.width, dtype=dtype, device=device)
        self.gathered = torch.zeros(self.width * plan.world, dtype=dtype, device=device)
        self.bytes_per_step = int(self.width * plan.world * self.sendbuf.element_size())

    # device-side gather/scatter through the C ABI; torch indexing on CPU (gloo tests)
    def _gather(self, grid: torch.Tensor) -> None:
        k = self.send_idx.numel()
        if k == 0:
            return
        if grid.is_cuda:
            from . import device as dev
            from . import native

            native.call("gm_gather_cells", grid.data_ptr(), grid.element_size(), self.send_idx.data_ptr(), k,
                        self.sendbuf.data_ptr(), dev.stream_handle())
        else:
            self.sendbuf[:k] = grid.view(-1)[self.send_idx]

    def _scatter(self, grid: torch.Tensor) -> None:
        k = self.recv_idx.numel()
        if k == 0:
            return
        vals = self.gathered[self.recv_pos]
        if grid.is_cuda:
            from . import device as dev
            from . import native

            vals = vals.contiguous()
            native.call("gm_scatter_cells", grid.data_ptr(), grid.element_size(), self.recv_idx.data_ptr(), k,
                        vals.data_ptr(), dev.stream_handle())
        else:
            grid.view(-1)[self.recv_idx] = vals

    def post(self, grid: torch.Tensor) -> None:
        """Contribute this rank's halo values (loopback: before anyone completes)."""
        self._gather(grid)
        if self.loopback is not None:
            self.loopback.contribute(self.rank, self.sendbuf)
        else:
            import torch.distributed as dist

            if self.sendbuf.is_cuda:
                dist.all_gather_into_tensor(self.gathered, self.sendbuf, group=self.group)
            else:  # gloo: list form
                dist.all_gather(list(self.gathered.chunk(self.plan.world)), self.sendbuf, group=self.group)

    def complete(self, grid: torch.Tensor) -> None:
        if self.loopback is not None:
            self.gathered.copy_(self.loopback.gathered())
        self._scatter(grid)

    def exchange(self, grid: torch.Tensor) -> None:
        self.post(grid)
        self.complete(grid)


class DeviceBuffer:
    """A plain cudaMalloc'd buffer (an allocation base, so CUDA IPC can export it),
    viewed as a torch tensor through __cuda_array_interface__."""

    _TYPESTR = {torch.int8: "|i1", torch.uint8: "|u1", torch.int16: "<i2", torch.uint16: "<u2",
                torch.int32: "<i4", torch.int64: "<i8", torch.uint64: "<u8"}

    def __init__(self, shape: tuple[int, ...], dtype: torch.dtype) -> None:
        import ctypes

        from . import native

        self.shape, self.dtype = tuple(shape), dtype
        self.nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        native.call("gm_dev_alloc", self.nbytes, ctypes.byref(p))
        self.ptr = int(p.value)
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": self._TYPESTR[dtype],
                                         "data": (self.ptr, False), "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device="cuda")

    def ipc_handle(self) -> bytes:
        from . import native

        h = (np.zeros(64, dtype=np.uint8))
        native.call("gm_ipc_get_handle", self.ptr, h.ctypes.data)
        return h.tobytes()

    def free(self) -> None:
        from . import native

        if self.ptr:
            self.tensor = None
            native.call("gm_dev_free", self.ptr)
            self.ptr = 0


class PeerHaloExchange:
    """Halo exchange over peer memory (peer.cu): each rank maps its peers' ping-pong
    buffers and flag words once (CUDA IPC, bootstrapped with all_gather_object on the
    process group), then per step writes its changing halo cells straight into every
    peer's new state and release-stores a step counter into each peer's flags; the
    next step waits (acquire) for every peer's counter.  No collective per step."""

    TIMEOUT_NS = 10_000_000_000

    def __init__(self, plan: PartitionPlan, rank: int, bufs: Sequence[DeviceBuffer], group=None,
                 entries: Optional[tuple[np.ndarray, np.ndarray]] = None) -> None:
        """entries (tiled storage): (source cells, destination rank << 56 | cell) per copy,
        own-rank destinations being ring copies; default: the dense layout's slots, each
        cell stored at the same index in every peer."""
        import torch.distributed as dist

        from . import native

        self.plan, self.rank, self.world = plan, rank, plan.world
        self.cell_bytes = bufs[0].tensor.element_size()
        if entries is None:
            slots, _ = plan.exchange_slots()
            self.send_idx = torch.from_numpy(slots[rank]).cuda()
            self.didx = None
            self.bytes_per_step = int(self.send_idx.numel() * self.cell_bytes * (self.world - 1))
        else:
            self.send_idx = torch.from_numpy(entries[0]).cuda()
            self.didx = torch.from_numpy(entries[1]).cuda()
            remote = int(((entries[1] >> 56) != rank).sum())
            self.bytes_per_step = remote * self.cell_bytes
        self.flags = DeviceBuffer((self.world,), torch.uint64)
        self.flags.tensor.zero_()
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        mine = [b.ipc_handle() for b in bufs] + [self.flags.ipc_handle()]
        everyone: list = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        import ctypes

        self._opened: list[int] = []
        ptrs = [[0] * self.world for _ in range(3)]  # buffer 0, buffer 1, flags
        for q in range(self.world):
            for j in range(3):
                if q == rank:
                    ptrs[j][q] = bufs[j].ptr if j < 2 else self.flags.ptr
                    continue
                p = ctypes.c_void_p()
                h = np.frombuffer(everyone[q][j], dtype=np.uint8).copy()
                native.call("gm_ipc_open_handle", h.ctypes.data, ctypes.byref(p))
                ptrs[j][q] = int(p.value)
                self._opened.append(int(p.value))
        self.peer_bufs = [torch.tensor(ptrs[j], dtype=torch.int64).cuda() for j in range(2)]
        self.peer_flags = torch.tensor(ptrs[2], dtype=torch.int64).cuda()
        self.bufs = bufs
        self.epoch = 0
        self._group = group
        dist.barrier(group=group)

    # ---- the exchange fused into the step kernel (peer_epilogue.cuh, gm_run_part_peer) ----
    MAX_PEERS = 16

    def epilogue(self, which: int) -> torch.Tensor:
        """Device descriptor (struct PeerEpilogue) for steps that write buffer `which`."""
        if not hasattr(self, "_epi"):
            import ctypes

            class Epi(ctypes.Structure):
                _fields_ = [("peers", ctypes.c_uint64 * self.MAX_PEERS), ("peer_flags", ctypes.c_uint64 * self.MAX_PEERS),
                            ("own_flags", ctypes.c_uint64), ("idx", ctypes.c_uint64), ("count", ctypes.c_int64),
                            ("cell_bytes", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                            ("done", ctypes.c_uint32), ("status", ctypes.c_uint32), ("didx", ctypes.c_uint64)]

            if self.world > self.MAX_PEERS:
                raise ValueError(f"the fused exchange supports up to {self.MAX_PEERS} ranks")
            pb = [t.cpu().tolist() for t in self.peer_bufs]
            pf = self.peer_flags.cpu().tolist()
            self._epi = []
            for w in range(2):
                e = Epi()
                for q in range(self.world):
                    e.peers[q] = pb[w][q]
                    e.peer_flags[q] = pf[q]
                e.own_flags = self.flags.ptr
                e.idx = self.send_idx.data_ptr()
                e.count = self.send_idx.numel()
                e.cell_bytes, e.rank, e.world = self.cell_bytes, self.rank, self.world
                e.didx = self.didx.data_ptr() if self.didx is not None else 0
                raw = np.frombuffer(bytes(e), dtype=np.uint8).copy()
                self._epi.append(torch.from_numpy(raw).cuda())
            self._epi_status_off = Epi.status.offset
        return self._epi[which]

    def check_fused(self) -> None:
        for t in getattr(self, "_epi", []):
            st = int(t[self._epi_status_off:self._epi_status_off + 4].cpu().numpy().view(np.uint32)[0])
            if st:
                from .native import GasketError

                raise GasketError(f"fused peer halo wait timed out (peer bitmask {st:#x})")

    def exchange(self, which: int) -> None:
        """After this rank wrote its new state into buffer `which`: put + wait (stream-ordered)."""
        from . import device as dev
        from . import native

        self.epoch += 1
        s = dev.stream_handle()
        if self.didx is not None:
            native.call("gm_peer_halo_put_to", self.bufs[which].ptr, self.peer_bufs[which].data_ptr(),
                        self.send_idx.data_ptr(), self.didx.data_ptr(), self.send_idx.numel(), self.cell_bytes,
                        self.peer_flags.data_ptr(), self.rank, self.world, self.epoch, s)
        else:
            native.call("gm_peer_halo_put", self.bufs[which].ptr, self.peer_bufs[which].data_ptr(),
                        self.send_idx.data_ptr(), self.send_idx.numel(), self.cell_bytes, self.peer_flags.data_ptr(),
                        self.rank, self.world, self.epoch, s)
        native.call("gm_peer_halo_wait", self.flags.ptr, self.rank, self.world, self.epoch, self.TIMEOUT_NS,
                    self.status.data_ptr(), s)

    def check(self) -> None:
        bad = int(self.status.item())
        if bad:
            from .native import GasketError

            raise GasketError(f"peer halo wait timed out (peer bitmask {bad:#x})")

    def close(self) -> None:
        import torch.distributed as dist

        from . import native

        torch.cuda.synchronize()
        dist.barrier(group=self._group)  # every peer is done storing into this rank's buffers
        for p in self._opened:
            native.call("gm_ipc_close", p)
        self._opened = []
        self.flags.free()


StepFn = Callable[[torch.Tensor, torch.Tensor, int, int], None]


class PartitionedCA:
    """One rank of the partitioned CA: full-size ping-pong buffers, own sub-gaskets
    computed by `step_fn(dst, src, sg_lo, sg_hi)` (the GPU kernel by default)."""

    def __init__(self, plan: PartitionPlan, rank: int, init: torch.Tensor, kind: int, param: int = 1,
                 group=None, loopback: Optional[LoopbackGroup] = None, step_fn: Optional[StepFn] = None,
                 adopt_init: bool = False, halo: str = "collective",
                 init_fill: Optional[Callable[[torch.Tensor], None]] = None, fused: bool = False) -> None:
        """plan.depth = 2, 4 or 6 makes every step() advance that many CA steps with one
        fused launch (gm_run_part_steps) and one halo exchange."""
        """`init_fill(t)` (peer halo only) writes the initial state into the first buffer in
        place; `init` then only gives shape and dtype (a meta tensor is enough), so a
        2^18 grid needs two full-size buffers, not three."""
        self.plan, self.rank, self.kind, self.param = plan, rank, kind, param
        self.peer = None
        if halo == "peer":
            # buffers the peers can map (CUDA IPC needs allocation bases)
            self._dbufs = [DeviceBuffer(tuple(init.shape), init.dtype) for _ in range(2)]
            if init_fill is not None:
                init_fill(self._dbufs[0].tensor)
            else:
                self._dbufs[0].tensor.copy_(init)
            self._dbufs[1].tensor.copy_(self._dbufs[0].tensor)
            self.a, self.b = self._dbufs[0].tensor, self._dbufs[1].tensor
            self.peer = PeerHaloExchange(plan, rank, self._dbufs, group=group)
            self._dst = 1  # index of the buffer the next step writes
            self.halo = None
        elif halo == "collective":
            self.a = init if adopt_init else init.clone()  # adopt: no third full-size buffer (n=2^18 int8 is 64 GiB)
            self.b = init.clone()  # both buffers agree off the gasket -> whole-sector writes from src
            self.halo = HaloExchange(plan, rank, init.device, init.dtype, group=group, loopback=loopback)
        else:
            raise ValueError("halo must be 'collective' (all_gather) or 'peer' (peer memory)")
        self.step_fn = step_fn or self._gpu_step
        self.lo, self.hi = plan.ranges[rank]
        # fused=True (peer halo): the exchange runs inside the step kernel (gm_run_part_peer)
        # -- one launch per step (per plan.depth steps), no put/wait kernels
        self.fused = bool(fused)
        if self.fused and (self.peer is None or step_fn is not None):
            raise ValueError("fused exchange needs halo='peer' and the GPU step")
        self._epoch = 0

    def _gpu_step(self, dst: torch.Tensor, src: torch.Tensor, lo: int, hi: int) -> None:
        from . import device as dev
        from . import native

        if self.plan.depth > 1:  # depth fused steps over this rank's sub-gaskets
            native.call("gm_run_part_steps", dst.data_ptr(), src.data_ptr(), self.plan.n, dst.element_size(),
                        self.kind, int(np.int32(self.param)), self.plan.depth, 0, self.plan.level, lo, hi,
                        dev.stream_handle())
            return
        native.call("gm_run_part", dst.data_ptr(), src.data_ptr(), self.plan.n, dst.element_size(), self.kind,
                    int(np.int32(self.param)), native.FLAG_DST_FROM_SRC, self.plan.level, lo, hi,
                    dev.stream_handle())

    def compute(self) -> None:
        self.step_fn(self.b, self.a, self.lo, self.hi)

    def finish(self) -> None:
        self.a, self.b = self.b, self.a
        if self.peer is not None:
            self._dst ^= 1

    def step(self) -> None:
        """compute -> exchange halo of the new state -> swap (real process group)."""
        if self.fused:
            from . import device as dev
            from . import native

            self._epoch += 1
            fl = {1: native.FLAG_DST_FROM_SRC, 2: native.FLAG_TWO_STEPS, 4: native.FLAG_FOUR_STEPS,
                  6: native.FLAG_SIX_STEPS}[self.plan.depth]
            native.call("gm_run_part_peer", self.b.data_ptr(), self.a.data_ptr(), self.plan.n, self.b.element_size(),
                        self.kind, int(np.int32(self.param)), fl, self.plan.level, self.lo,
                        self.hi, self.peer.epilogue(self._dst).data_ptr(), self._epoch - 1, self._epoch,
                        dev.stream_handle())
            self.finish()
            return
        self.compute()
        if self.peer is not None:
            self.peer.exchange(self._dst)
        else:
            self.halo.exchange(self.b)
        self.finish()

    @property
    def halo_bytes_per_step(self) -> int:
        return self.peer.bytes_per_step if self.peer is not None else self.halo.bytes_per_step

    def close(self) -> None:
        if self.peer is not None:
            self.peer.check()
            self.peer.check_fused()
            self.peer.close()
            self.a = self.b = None
            for d in self._dbufs:
                d.free()
            self.peer = None

    def owned_mask(self) -> torch.Tensor:
        """Cells of this rank's sub-gaskets (for assembling results in tests)."""
        n, m = self.plan.n, self.plan.m
        mask = torch.zeros((n, n), dtype=torch.bool, device=self.a.device)
        for s in range(self.lo, self.hi):
            bx, by = subgasket_block(s, self.plan.level)
            mask[by * m:(by + 1) * m, bx * m:(bx + 1) * m] = True
        return mask


# ---------------------------------------------------------------------------
# tiled storage: each rank holds only its sub-gaskets, each in a ringed block
# ---------------------------------------------------------------------------

RING_ROWS = 8     # >= the deepest fused kernel's reach (6 rows) -- the staged window of a tile
RING_BYTES = 128  # one line either side: the blocks' tile lines stay 128-byte aligned


class TiledLayout:
    """Per-rank storage of SURVEY §8e: the rank's level-L sub-gaskets, each one block of
    (m + 2R) rows x pitch bytes (m = n >> L, R = RING_ROWS, pitch = m*C + 2*RING_BYTES)
    holding the sub-gasket and a ring of its neighbours' cells -- not two n x n grids.
    A sub-gasket of level L is itself an edge-m gasket (its cell (x, y) is a gasket cell
    iff x is a bit-subset of y), so the tuned kernels run on a block unchanged, addressing
    it through the block's virtual origin sg_off[k] (where global cell (0, 0) would sit):
    global cell (x, y) of block k is at byte sg_off[k] + y*pitch + x*C.

    n = 2^18 int8 at L = 5: 243 blocks of 69.3 MB = 16.8 GB for the whole gasket per
    ping-pong buffer (the dense grid is 64 GiB), 2.2 GB per rank at 8 ranks."""

    def __init__(self, plan: "PartitionPlan", rank: int, cell_bytes: int) -> None:
        self.plan, self.rank, self.c = plan, rank, int(cell_bytes)
        if self.c not in (1, 2, 4):
            raise ValueError("tiled storage runs the tuned tile kernels: 1-, 2- or 4-byte cells")
        self.m = plan.m
        if self.m * self.c < 128:
            raise ValueError(f"sub-gaskets of edge {self.m} are narrower than one 128-byte tile")
        self.lo, self.hi = plan.ranges[rank]
        self.count = self.hi - self.lo
        self.R, self.P = RING_ROWS, RING_BYTES
        self.pc = self.P // self.c  # ring cells either side
        self.pitch = self.m * self.c + 2 * self.P
        self.rows = self.m + 2 * self.R
        self.block = self.rows * self.pitch
        self.nbytes = self.count * self.block
        self.origins = [tuple(v * self.m for v in subgasket_block(s, plan.level)) for s in range(self.lo, self.hi)]
        self.sg_off = np.array([k * self.block + self.R * self.pitch + self.P - oy * self.pitch - ox * self.c
                                for k, (ox, oy) in enumerate(self.origins)], dtype=np.int64)

    def cell_index(self, k: int, x, y):
        """Cell index (byte offset / C) of global cell (x, y) in block k (x, y may be arrays)."""
        return (self.sg_off[k] + np.asarray(y, dtype=np.int64) * self.pitch
                + np.asarray(x, dtype=np.int64) * self.c) // self.c

    def block_of(self, s: int) -> int:
        return s - self.lo

    def window(self, k: int) -> tuple[int, int, int, int]:
        """Global cells [x0, x1) x [y0, y1) block k holds (sub-gasket plus ring)."""
        ox, oy = self.origins[k]
        return ox - self.pc, ox + self.m + self.pc, oy - self.R, oy + self.m + self.R

    def block_view(self, buf: torch.Tensor, k: int) -> torch.Tensor:
        """Block k of a flat buffer as a (rows, pitch / C) tensor."""
        w = self.pitch // self.c
        return buf[k * (self.block // self.c):(k + 1) * (self.block // self.c)].view(self.rows, w)

    # -- filling and reading -------------------------------------------------
    def load_dense(self, buf: torch.Tensor, dense: torch.Tensor) -> None:
        """Every block's window from a dense n x n grid (0 outside the grid)."""
        n = self.plan.n
        buf.zero_()
        for k in range(self.count):
            x0, x1, y0, y1 = self.window(k)
            cx0, cx1, cy0, cy1 = max(x0, 0), min(x1, n), max(y0, 0), min(y1, n)
            v = self.block_view(buf, k)
            v[cy0 - y0:cy1 - y0, cx0 - x0:cx1 - x0].copy_(dense[cy0:cy1, cx0:cx1])

    def fill_hash(self, buf: torch.Tensor, seed: int, mode: int = 0) -> None:
        """Every block's window from the synthetic grid fill_hash(seed, mode) (no dense copy)."""
        from . import device as dev
        from . import native

        for k in range(self.count):
            x0, x1, y0, y1 = self.window(k)
            v = self.block_view(buf, k)
            native.call("gm_fill_hash_window", v.data_ptr(), self.pitch, self.plan.n, self.c, x0, y0, x1 - x0,
                        y1 - y0, seed & (2**64 - 1), mode, dev.stream_handle())

    def store_dense(self, buf: torch.Tensor, dense: torch.Tensor) -> None:
        """The rank's sub-gaskets (block interiors) into a dense n x n grid."""
        m = self.m
        for k in range(self.count):
            ox, oy = self.origins[k]
            v = self.block_view(buf, k)
            dense[oy:oy + m, ox:ox + m].copy_(v[self.R:self.R + m, self.pc:self.pc + m])


def tiled_exchange(plan: "PartitionPlan", cell_bytes: int) -> list[tuple[np.ndarray, np.ndarray]]:
    """Per SOURCE rank: (source cells in its layout, destination rank << 56 | destination
    cell) for every copy a step needs -- each changing halo cell of a sub-gasket
    (plan.halo, depth-aware) from its owner's block into the ring of the reading block;
    a destination rank equal to the source is a ring copy inside the same buffer."""
    layouts = [TiledLayout(plan, r, cell_bytes) for r in range(plan.world)]
    src: list[list[int]] = [[] for _ in range(plan.world)]
    dst: list[list[int]] = [[] for _ in range(plan.world)]
    n = plan.n
    for reader_rank, lay in enumerate(layouts):
        for k in range(lay.count):
            s = lay.lo + k
            cells = plan.halo[s]
            if cells.size == 0:
                continue
            y, x = np.divmod(cells, n)
            owners_sg = [subgasket_index(int(a) // plan.m, int(b) // plan.m, plan.level) for a, b in zip(x, y)]
            d_idx = lay.cell_index(k, x, y)
            for i, s2 in enumerate(owners_sg):
                if s2 is None:  # (never: halo cells are gasket cells)
                    continue
                o = plan.owner_of_subgasket(s2)
                src_lay = layouts[o]
                src[o].append(int(src_lay.cell_index(src_lay.block_of(s2), x[i], y[i])))
                dst[o].append(int(d_idx[i]) | (reader_rank << 56))
    return [(np.array(a, dtype=np.int64), np.array(b, dtype=np.int64)) for a, b in zip(src, dst)]


class TiledCA:
    """One rank of the partitioned CA on tiled storage (TiledLayout): two flat buffers of
    the rank's blocks, `plan.depth` steps per launch (gm_run_part_tiled), then the halo
    copies of tiled_exchange: over NCCL / gloo all_gather ("collective", the received
    values scattered into the rings plus the rank's own ring copies), over peer memory
    ("peer": gm_peer_halo_put_to), or inside the step kernel ("peer" + fused)."""

    def __init__(self, plan: "PartitionPlan", rank: int, kind: int, param: int = 1, dtype=torch.int8,
                 init: Optional[torch.Tensor] = None, seed: Optional[int] = None, group=None,
                 loopback: Optional["LoopbackGroup"] = None, halo: str = "collective", fused: bool = False,
                 edge_cache: bool = True) -> None:
        from . import device as dev
        from . import native

        dev.require_cuda()
        self.plan, self.rank, self.kind, self.param = plan, rank, kind, param
        c = torch.empty((), dtype=dtype).element_size()
        self.layout = L = TiledLayout(plan, rank, c)
        self.sg_off = torch.from_numpy(L.sg_off).cuda()
        entries = tiled_exchange(plan, c)
        self.peer = None
        numel = max(1, L.nbytes // c)
        if halo == "peer":
            self._dbufs = [DeviceBuffer((numel,), dtype) for _ in range(2)]
            self.a, self.b = self._dbufs[0].tensor, self._dbufs[1].tensor
        elif halo == "collective":
            self.a = torch.empty(numel, dtype=dtype, device="cuda")
            self.b = torch.empty(numel, dtype=dtype, device="cuda")
        else:
            raise ValueError("halo must be 'collective' or 'peer'")
        if init is not None:
            L.load_dense(self.a, init)
        elif seed is not None:
            self.a.zero_()
            L.fill_hash(self.a, seed)
        else:
            raise ValueError("pass the initial state: a dense grid (init) or a synthetic seed")
        self.b.copy_(self.a)  # both buffers agree off the gasket (rings included)
        self.lo, self.hi = L.lo, L.hi
        # the static left-edge cache of the rank's tiles (edge.cu; one-step launches use it)
        self.edge = None
        if edge_cache and plan.depth == 1 and self.hi > self.lo:
            self.edge = torch.empty(native.ca_edge_bytes(plan.n, c, plan.level, self.lo, self.hi), dtype=torch.uint8,
                                    device="cuda")
            native.call("gm_ca_edge_build", self.edge.data_ptr(), self.a.data_ptr(), plan.n, c, plan.level, self.lo,
                        self.hi, self.sg_off.data_ptr(), L.pitch, dev.stream_handle())
        self.fused = bool(fused)
        if halo == "peer":
            self.peer = PeerHaloExchange(plan, rank, self._dbufs, group=group, entries=entries[rank])
            self._dst = 1
        else:
            if self.fused:
                raise ValueError("the fused exchange needs halo='peer'")
            self._coll = _TiledCollective(plan, rank, entries, dtype, group=group, loopback=loopback)
        self._epoch = 0

    # -- one exchange round ---------------------------------------------------
    def _launch(self, epi: int = 0, wait: int = 0, signal: int = 0) -> None:
        from . import device as dev
        from . import native

        native.call("gm_run_part_tiled", self.b.data_ptr(), self.a.data_ptr(), self.plan.n, self.a.element_size(),
                    self.kind, int(np.int32(self.param)), self.plan.depth, self.plan.level, self.lo, self.hi,
                    self.sg_off.data_ptr(), self.layout.pitch, epi, wait, signal,
                    self.edge.data_ptr() if self.edge is not None else None, dev.stream_handle())

    def compute(self) -> None:
        if self.hi > self.lo:
            self._launch()

    def finish(self) -> None:
        self.a, self.b = self.b, self.a
        if self.peer is not None:
            self._dst ^= 1

    def step(self) -> None:
        """depth CA steps on the rank's blocks, then the halo copies of the new state."""
        if self.fused:
            self._epoch += 1
            self._launch(self.peer.epilogue(self._dst).data_ptr(), self._epoch - 1, self._epoch)
            self.finish()
            return
        self.compute()
        if self.peer is not None:
            self.peer.exchange(self._dst)
        else:
            self._coll.exchange(self.b)
        self.finish()

    @property
    def halo_bytes_per_step(self) -> int:
        return self.peer.bytes_per_step if self.peer is not None else self._coll.bytes_per_step

    @property
    def storage_bytes(self) -> int:
        return 2 * self.layout.nbytes + (self.edge.numel() if self.edge is not None else 0)

    def store_dense(self, dense: torch.Tensor) -> None:
        torch.cuda.synchronize()
        self.layout.store_dense(self.a, dense)

    def close(self) -> None:
        if self.peer is not None:
            self.peer.check()
            self.peer.check_fused()
            self.peer.close()
            self.a = self.b = None
            for d in self._dbufs:
                d.free()
            self.peer = None


class _TiledCollective:
    """The tiled halo copies over a process group (all_gather) or a loopback group: the
    rank's cells other ranks read go out in one fixed-size all_gather, the received
    values are scattered into this rank's rings, and the rank's own ring copies run as
    one gm_copy_cells."""

    def __init__(self, plan, rank, entries, dtype, group=None, loopback=None, device: str = "cuda") -> None:
        self.plan, self.rank, self.group, self.loopback = plan, rank, group, loopback
        W = plan.world
        # per source rank o: its unique cells read by other ranks, in a fixed order
        sends = []
        for o in range(W):
            srcs, dsts = entries[o]
            remote = (dsts >> 56) != o
            sends.append(np.unique(srcs[remote]))
        self.width = max([1] + [len(v) for v in sends])
        srcs, dsts = entries[rank]
        local = (dsts >> 56) == rank
        dev = torch.device(device)
        self.send_idx = torch.from_numpy(sends[rank]).to(dev)
        self.local_src = torch.from_numpy(srcs[local]).to(dev)
        self.local_dst = torch.from_numpy(dsts[local] & ((1 << 56) - 1)).to(dev)
        pos, cells = [], []
        for o in range(W):
            if o == rank:
                continue
            so, do = entries[o]
            mine = (do >> 56) == rank
            if not mine.any():
                continue
            slot = np.searchsorted(sends[o], so[mine])
            pos.append(o * self.width + slot)
            cells.append(do[mine] & ((1 << 56) - 1))
        self.recv_pos = torch.from_numpy(np.concatenate(pos) if pos else np.zeros(0, np.int64)).to(dev)
        self.recv_idx = torch.from_numpy(np.concatenate(cells) if cells else np.zeros(0, np.int64)).to(dev)
        self.sendbuf = torch.zeros(self.width, dtype=dtype, device=dev)
        self.gathered = torch.zeros(self.width * W, dtype=dtype, device=dev)
        self.bytes_per_step = int(self.width * W * self.sendbuf.element_size()) if W > 1 else 0

    def post(self, buf: torch.Tensor) -> None:
        from . import device as dev
        from . import native

        if self.plan.world == 1:
            return  # one rank: only its own ring copies (complete)
        k = self.send_idx.numel()
        if k:
            native.call("gm_gather_cells", buf.data_ptr(), buf.element_size(), self.send_idx.data_ptr(), k,
                        self.sendbuf.data_ptr(), dev.stream_handle())
        if self.loopback is not None:
            self.loopback.contribute(self.rank, self.sendbuf)
        else:
            import torch.distributed as dist

            dist.all_gather_into_tensor(self.gathered, self.sendbuf, group=self.group)

    def complete(self, buf: torch.Tensor) -> None:
        from . import device as dev
        from . import native

        if self.loopback is not None and self.plan.world > 1 and len(self.loopback._parts) == self.plan.world:
            self.gathered.copy_(self.loopback.gathered())
        k = self.recv_idx.numel()
        if k:
            vals = self.gathered[self.recv_pos].contiguous()
            native.call("gm_scatter_cells", buf.data_ptr(), buf.element_size(), self.recv_idx.data_ptr(), k,
                        vals.data_ptr(), dev.stream_handle())
        k = self.local_src.numel()
        if k:
            native.call("gm_copy_cells", buf.data_ptr(), buf.data_ptr(), buf.element_size(), self.local_dst.data_ptr(),
                        self.local_src.data_ptr(), k, dev.stream_handle())

    def exchange(self, buf: torch.Tensor) -> None:
        self.post(buf)
        self.complete(buf)


def run_loopback_tiled(plan: "PartitionPlan", kind: int, rounds: int, param: int = 1, dtype=torch.int8,
                       init: Optional[torch.Tensor] = None, seed: Optional[int] = None,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """All virtual ranks' tiled storage on one device; after `rounds` exchange rounds
    (each plan.depth CA steps) the sub-gaskets are written into `out` (a dense grid:
    a copy of init, or fill_hash(seed) -- off-gasket cells never change)."""
    lb = LoopbackGroup(plan.world)
    ranks = [TiledCA(plan, r, kind, param, dtype=dtype, init=init, seed=seed, loopback=lb) for r in range(plan.world)]
    for _ in range(rounds):
        for ca in ranks:
            ca.compute()
        for ca in ranks:
            ca._coll.post(ca.b)
        for ca in ranks:
            ca._coll.complete(ca.b)
        for ca in ranks:
            ca.finish()
    if out is None:
        out = init.clone()
    for ca in ranks:
        ca.store_dense(out)
    return out


def run_loopback(plan: PartitionPlan, init: torch.Tensor, kind: int, steps: int, param: int = 1,
                 step_fn: Optional[StepFn] = None) -> torch.Tensor:
    """All virtual ranks on one device; returns the assembled grid after `steps` exchange
    rounds (each plan.depth CA steps)."""
    lb = LoopbackGroup(plan.world)
    ranks = [PartitionedCA(plan, r, init, kind, param, loopback=lb, step_fn=step_fn) for r in range(plan.world)]
    for _ in range(steps):
        for ca in ranks:
            ca.compute()
        for ca in ranks:
            ca.halo.post(ca.b)
        for ca in ranks:
            ca.halo.complete(ca.b)
        for ca in ranks:
            ca.finish()
    out = init.clone()
    for ca in ranks:
        mask = ca.owned_mask()
        out[mask] = ca.a[mask]
    return out


__all__: Sequence[str] = ("subgasket_block", "subgasket_index", "rank_ranges", "PartitionPlan", "LoopbackGroup",
                          "HaloExchange", "DeviceBuffer", "PeerHaloExchange", "PartitionedCA", "run_loopback",
                          "TiledLayout", "tiled_exchange", "TiledCA", "run_loopback_tiled")
