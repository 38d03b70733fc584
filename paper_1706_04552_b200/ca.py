"""Multi-step cellular-automaton driver on the device (ping-pong +
CUDA Graphs).

A CA step is the reference's neighbour-sum launch with the pre-launch
snapshot semantics of engine.launch (engine.py:201): every step reads the
previous state and writes only gasket cells.  Two device buffers ping-pong;
both hold the same off-gasket cells for ever (the kernels never write them),
so every step may write whole sectors blended from its source
(``FLAG_DST_FROM_SRC``) -- no DRAM read-modify-write.  A pair of steps
(A->B, B->A) is captured once into a CUDA graph and replayed, which removes
the per-step Python/ctypes launch cost for long runs.

``temporal=T`` (temporal blocking) advances T = 2, 4 or 6 steps
with one fused launch (``gm_ca_steps``, stencil_tb.cu): state t is read once, the
intermediate states live only in shared memory, state t+T is written once -- 1/T
of the DRAM traffic per step.  Results are bit-identical to single steps.

``edge_cache=True`` (default): the off-gasket cells left of every member tile whose
left neighbour tile holds no gasket cell are gathered once into a dense cache
(``gm_ca_edge_build``, edge.cu) and every step stages them from there instead of
fetching one sparse DRAM line per tile row (a third of an 8-neighbour step's line
reads at n=2^17).  The cache is taken from the initial state: like the ping-pong
itself it relies on nobody changing off-gasket cells of the buffers between steps.
"""

from __future__ import annotations

import numpy as np
import torch

from . import backends, device, native
from .geometry import FractalSpec, IntraStrategy


class CARunner:
    def __init__(self, grid: torch.Tensor, kind: int = backends.KERNEL_NEIGHBOR_SUM8, param: int = 1,
                 rho: int = 64, use_graph: bool = True, temporal: int = 6, edge_cache: bool = True) -> None:
        device.require_cuda()
        if not device.is_device(grid):
            raise TypeError("CARunner works on a CUDA grid tensor")
        if kind not in (backends.KERNEL_NEIGHBOR_SUM, backends.KERNEL_NEIGHBOR_SUM8):
            raise ValueError("CA steps are neighbour-sum launches (kind 1 or 2)")
        n = device.check_square(grid)
        rho = min(rho, n)
        self.spec = FractalSpec(n=n, rho=rho)
        self.kind, self.param = kind, param
        self.bufs = (grid, grid.clone())  # fixed physical buffers (the graph captures their addresses)
        self.cur = 0                      # which buffer holds the current state
        self.use_graph = use_graph
        if temporal not in (1, 2, 4, 6):
            raise ValueError("temporal must be 1 (one step per launch), 2, 4 or 6 (fused steps per launch)")
        # the fused kernel needs whole 128-byte tiles of 1-, 2- or 4-byte cells
        self.temporal = temporal if (grid.element_size() in (1, 2, 4) and n * grid.element_size() >= 128) else 1
        if self.temporal == 6 and grid.element_size() == 4:
            self.temporal = 4  # a 6-cell cone outgrows the 4-cell halo chunk of 4-byte cells
        self._graph = None
        self.steps_done = 0
        # tiled kernels (1-, 2-, 4-byte cells, at least one 128-byte tile, <= 2^15 tiles per edge)
        c = grid.element_size()
        self._tiled = c in (1, 2, 4) and n * c >= 128 and n // (128 // c) <= (1 << 15)
        self.edge = None
        if edge_cache and self._tiled:
            self.edge = torch.empty(native.ca_edge_bytes(n, c), dtype=torch.uint8, device=grid.device)
            native.call("gm_ca_edge_build", self.edge.data_ptr(), grid.data_ptr(), n, c, -1, 0, 0, None, 0,
                        device.stream_handle())

    def _edge_ptr(self):
        return self.edge.data_ptr() if self.edge is not None else None

    def _step(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        if self._tiled:
            native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), self.spec.n, dst.element_size(), self.kind,
                        int(np.int32(self.param)), 1, self._edge_ptr(), 0, device.stream_handle())
        else:
            backends.run_block_space(dst, src, self.spec.rho, self.spec.r_b, IntraStrategy.TUNED, kind=self.kind,
                                     param=self.param, flags=native.FLAG_DST_FROM_SRC)

    def _fused(self, dst: torch.Tensor, src: torch.Tensor, steps: int) -> None:
        """`steps` (2, 4 or 6) steps src -> dst (the intermediate states never leave the SM)."""
        native.call("gm_ca_run", dst.data_ptr(), src.data_ptr(), self.spec.n, dst.element_size(), self.kind,
                    int(np.int32(self.param)), steps, self._edge_ptr(), 0, device.stream_handle())

    def _single(self) -> None:
        src, dst = self.bufs[self.cur], self.bufs[1 - self.cur]
        self._step(dst, src)
        self.cur ^= 1
        self.steps_done += 1

    def _advance(self, steps: int) -> None:
        """Advance `steps` (2, 4 or 6) fused steps from the current buffer (graph-free path)."""
        src, dst = self.bufs[self.cur], self.bufs[1 - self.cur]
        self._fused(dst, src, steps)
        self.cur ^= 1
        self.steps_done += steps

    def _capture(self) -> None:
        if self.temporal > 1:
            return self._capture_fused()
        a, b = self.bufs
        # warm up outside the capture (module load, tensor-map caches); advances two steps
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._step(b, a)
            self._step(a, b)
        torch.cuda.current_stream().wait_stream(s)
        self.steps_done += 2
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step(b, a)
            self._step(a, b)
        self._graph = g

    def _capture_fused(self) -> None:
        # fused launches alternate A->B, B->A: one graph = 2T steps (two launches)
        a, b, T = self.bufs[0], self.bufs[1], self.temporal
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._fused(b, a, T)
            self._fused(a, b, T)
        torch.cuda.current_stream().wait_stream(s)
        self.steps_done += 2 * T
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._fused(b, a, T)
            self._fused(a, b, T)
        self._graph = g

    @property
    def state(self) -> torch.Tensor:
        return self.bufs[self.cur]

    def run(self, steps: int) -> torch.Tensor:
        """Advance `steps` CA steps; returns the buffer holding the current state."""
        if steps < 0:
            raise ValueError("steps must be >= 0")
        left = steps
        per_graph = 2 * self.temporal  # steps one graph replay advances (two launches)
        if self.use_graph and left >= per_graph:
            if self.cur == 1:  # graphs start from buffer 0
                self._single()
                left -= 1
            if self._graph is None and left >= per_graph:
                self._capture()
                left -= per_graph
            while left >= per_graph:
                self._graph.replay()
                self.steps_done += per_graph
                left -= per_graph
        for k in (6, 4, 2):  # the remainder: fused launches no longer than `temporal`, then singles
            while self.temporal >= k and left >= k:
                self._advance(k)
                left -= k
        while left > 0:
            self._single()
            left -= 1
        return self.state


def run_ca(grid: torch.Tensor, steps: int, kind: int = backends.KERNEL_NEIGHBOR_SUM8, param: int = 1,
           use_graph: bool = True, temporal: int = 6, edge_cache: bool = True) -> torch.Tensor:
    """`steps` CA steps starting from `grid`; the final state is copied back into `grid`."""
    runner = CARunner(grid, kind, param, use_graph=use_graph, temporal=temporal, edge_cache=edge_cache)
    out = runner.run(steps)
    if out.data_ptr() != grid.data_ptr():
        grid.copy_(out)
    return grid
