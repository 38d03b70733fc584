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
"""

from __future__ import annotations

import torch

from . import backends, device, native
from .geometry import FractalSpec, IntraStrategy


class CARunner:
    def __init__(self, grid: torch.Tensor, kind: int = backends.KERNEL_NEIGHBOR_SUM8, param: int = 1,
                 rho: int = 64, use_graph: bool = True) -> None:
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
        self._graph = None
        self.steps_done = 0

    def _step(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        backends.run_block_space(dst, src, self.spec.rho, self.spec.r_b, IntraStrategy.TUNED, kind=self.kind,
                                 param=self.param, flags=native.FLAG_DST_FROM_SRC)

    def _single(self) -> None:
        src, dst = self.bufs[self.cur], self.bufs[1 - self.cur]
        self._step(dst, src)
        self.cur ^= 1
        self.steps_done += 1

    def _capture(self) -> None:
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

    @property
    def state(self) -> torch.Tensor:
        return self.bufs[self.cur]

    def run(self, steps: int) -> torch.Tensor:
        """Advance `steps` CA steps; returns the buffer holding the current state."""
        if steps < 0:
            raise ValueError("steps must be >= 0")
        left = steps
        if self.use_graph and left >= 2:
            if self.cur == 1:  # graph pairs start from buffer 0
                self._single()
                left -= 1
            if self._graph is None and left >= 2:
                self._capture()
                left -= 2
            while left >= 2:
                self._graph.replay()
                self.steps_done += 2
                left -= 2
        while left > 0:
            self._single()
            left -= 1
        return self.state


def run_ca(grid: torch.Tensor, steps: int, kind: int = backends.KERNEL_NEIGHBOR_SUM8, param: int = 1,
           use_graph: bool = True) -> torch.Tensor:
    """`steps` CA steps starting from `grid`; the final state is copied back into `grid`."""
    runner = CARunner(grid, kind, param, use_graph=use_graph)
    out = runner.run(steps)
    if out.data_ptr() != grid.data_ptr():
        grid.copy_(out)
    return grid
