"""Sub-gasket partition (multi-GPU path): planner, halo sets, and the
exchange protocol over a real process group (gloo, world_size 2, CPU) with the
CPU oracle as the per-rank step; the CUDA kernels through the same protocol on
one GPU with an in-process loopback group."""

import os
import socket

import numpy as np
import pytest
import torch

from paper_1706_04552_b200 import partition as P


def test_subgasket_block_index_roundtrip():
    for level in range(0, 6):
        blocks = {P.subgasket_block(s, level) for s in range(3**level)}
        assert len(blocks) == 3**level
        for s in range(3**level):
            bx, by = P.subgasket_block(s, level)
            assert bx & ~by == 0
            assert P.subgasket_index(bx, by, level) == s
    assert P.subgasket_index(1, 0, 3) is None


def test_rank_ranges_balanced():
    for nsg in (27, 243):
        for world in (1, 2, 4, 8):
            rr = P.rank_ranges(nsg, world)
            assert rr[0][0] == 0 and rr[-1][1] == nsg
            sizes = [b - a for a, b in rr]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("eight", [False, True])
def test_halo_cells_are_corner_cells(eight):
    """At most 5 (8-nbr) / 3 (4-nbr) changing halo cells per sub-gasket, all among the
    tile-relative candidates of SURVEY §8e."""
    for n, level in ((1 << 8, 3), (1 << 10, 5), (1 << 9, 2)):
        plan = P.PartitionPlan(n, level, world=4, eight=eight)
        m = plan.m
        cand8 = {(-1, -1), (0, -1), (1, -1), (-1, m - 1), (0, m), (m, m - 2), (m, m - 1), (m, m)}
        cand4 = {(0, -1), (-1, m - 1), (m, m - 1), (0, m)}
        for s in range(plan.nsg):
            bx, by = P.subgasket_block(s, level)
            rel = {(int(c % n) - bx * m, int(c // n) - by * m) for c in plan.halo[s]}
            assert rel <= (cand8 if eight else cand4), (n, level, s, rel)
            assert len(rel) <= (5 if eight else 3)


@pytest.mark.parametrize("kind", [1, 2])
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("depth", [2, 4, 6])
def test_deep_partition_matches_full_steps_cpu(kind, world, depth):
    """`depth` CA steps per exchange: with the depth-d halo (H1 grown by the gasket cells
    next to it, d-1 times) every rank's own cells after k rounds equal d*k full-grid
    oracle steps."""
    n, level = 1 << 8, 3
    plan = P.PartitionPlan(n, level, world, eight=kind == 2, depth=depth)
    import oracle

    init = oracle.fill_hash(n, np.int8, 21, 0)
    got = P.run_loopback(plan, torch.from_numpy(init), kind, 3, step_fn=_oracle_step_fn(plan, kind, 1))
    assert np.array_equal(got.numpy(), _reference_steps(init, kind, 1, 3 * depth))


def test_deeper_halo_contains_shallower():
    for eight in (False, True):
        p1 = P.PartitionPlan(1 << 10, 4, 4, eight=eight)
        p2 = P.PartitionPlan(1 << 10, 4, 4, eight=eight, depth=2)
        p4 = P.PartitionPlan(1 << 10, 4, 4, eight=eight, depth=4)
        p6 = P.PartitionPlan(1 << 10, 4, 4, eight=eight, depth=6)
        for s in range(p1.nsg):
            assert (set(p1.halo[s].tolist()) <= set(p2.halo[s].tolist()) <= set(p4.halo[s].tolist())
                    <= set(p6.halo[s].tolist()))
            assert len(p2.halo[s]) <= (13 if eight else 8)
            assert len(p4.halo[s]) <= (45 if eight else 24)


def _oracle_step_fn(plan, kind, param):
    import oracle

    def step(dst, src, lo, hi):
        tmp = dst.numpy().copy()
        oracle.run_bounding_box(tmp, src.numpy(), 1, kind, param)
        for _ in range(plan.depth - 1):  # further steps on this rank's (halo-current) local copy
            tmp2 = tmp.copy()
            oracle.run_bounding_box(tmp2, tmp, 1, kind, param)
            tmp = tmp2
        mask = np.zeros(tmp.shape, dtype=bool)
        m = plan.m
        for s in range(lo, hi):
            bx, by = P.subgasket_block(s, plan.level)
            mask[by * m:(by + 1) * m, bx * m:(bx + 1) * m] = True
        d = dst.numpy()
        d[mask] = tmp[mask]

    return step


def _reference_steps(init, kind, param, steps):
    import oracle

    a = init.copy()
    for _ in range(steps):
        b = a.copy()
        oracle.run_bounding_box(b, a, 1, kind, param)
        a = b
    return a


def test_loopback_protocol_cpu_oracle():
    import oracle

    n, level, steps = 1 << 7, 3, 5
    init = oracle.fill_hash(n, np.int8, 3, 0)
    want = _reference_steps(init, 2, 1, steps)
    for world in (1, 2, 5):
        plan = P.PartitionPlan(n, level, world, eight=True)
        got = P.run_loopback(plan, torch.from_numpy(init), 2, steps, step_fn=_oracle_step_fn(plan, 2, 1))
        assert np.array_equal(got.numpy(), want), world


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, n, level, kind, steps, out):
    import torch.distributed as dist

    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = P.PartitionPlan(n, level, world, eight=kind == 2)
        init = oracle.fill_hash(n, np.int8, 9, 0)
        ca = P.PartitionedCA(plan, rank, torch.from_numpy(init), kind, 1, step_fn=_oracle_step_fn(plan, kind, 1))
        for _ in range(steps):
            ca.step()
        want = _reference_steps(init, kind, 1, steps)
        mask = ca.owned_mask().numpy()
        out[rank] = bool(np.array_equal(ca.a.numpy()[mask], want[mask]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", [1, 2])
def test_gloo_world2_matches_single_process(kind):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, 1 << 7, 3, kind, 4, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert dict(out) == {0: True, 1: True}


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [1, 2])
def test_partition_loopback_gpu_matches_full_grid(gpu, kind):
    """The gm_run_part kernels + halo exchange (loopback, several virtual ranks on
    one GPU) == the unpartitioned tuned stencil, bit for bit."""
    be = gpu.backends
    S = gpu.geometry.IntraStrategy
    for n, level, worlds in ((1 << 12, 3, (2, 3, 8)), (1 << 14, 5, (8,)), (1 << 10, 2, (4,))):
        init = gpu.device.fill_hash(n, torch.int8, 5, 0)
        a = init.clone()
        for _ in range(4):
            b = a.clone()
            be.run_block_space(b, a, 64, (n // 64).bit_length() - 1, S.TUNED, kind=kind, param=1)
            a = b
        a6 = a.clone()
        for _ in range(2):
            b = a6.clone()
            be.run_block_space(b, a6, 64, (n // 64).bit_length() - 1, S.TUNED, kind=kind, param=1)
            a6 = b
        for world in worlds:
            plan = P.PartitionPlan(n, level, world, eight=kind == 2)
            got = P.run_loopback(plan, init, kind, 4)
            assert gpu.device.count_mismatch(got, a) == 0, (n, level, world)
            # fused steps per launch (gm_run_part_steps) with the depth-d halo: 4 steps
            for depth in (2, 4):
                plan_d = P.PartitionPlan(n, level, world, eight=kind == 2, depth=depth)
                got_d = P.run_loopback(plan_d, init, kind, 4 // depth)
                assert gpu.device.count_mismatch(got_d, a) == 0, (n, level, world, depth)
            plan6 = P.PartitionPlan(n, level, world, eight=kind == 2, depth=6)
            got6 = P.run_loopback(plan6, init, kind, 1)
            assert gpu.device.count_mismatch(got6, a6) == 0, (n, level, world, 6)


def _peer_worker(rank, world, port, n, level, kind, steps, out, depth=1, fused=False):
    """One rank of the partitioned CA with the peer-memory halo (peer.cu): both ranks
    share the one GPU of the test box and map each other's buffers with CUDA IPC."""
    import torch.distributed as dist

    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan = P.PartitionPlan(n, level, world, eight=kind == 2, depth=depth)
        init = oracle.fill_hash(n, np.int8, 9, 0)
        ca = P.PartitionedCA(plan, rank, torch.from_numpy(init).cuda(), kind, 1, group=dist.group.WORLD, halo="peer",
                             fused=fused)
        for _ in range(steps):
            ca.step()
        torch.cuda.synchronize()
        ca.peer.check()
        mask = ca.owned_mask().cpu().numpy()
        got = ca.a.cpu().numpy()[mask]
        want = _reference_steps(init, kind, 1, steps * depth)[mask]
        out[rank] = bool(np.array_equal(got, want))
        out[f"bytes{rank}"] = ca.halo_bytes_per_step
        ca.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,depth,kind,fused", [(2, 1, 1, False), (2, 1, 2, False), (2, 2, 1, False),
                                                    (2, 2, 2, False), (4, 1, 2, False), (4, 2, 2, False),
                                                    (2, 1, 1, True), (2, 1, 2, True), (4, 1, 2, True),
                                                    (2, 2, 2, True), (4, 2, 1, True), (2, 4, 2, False),
                                                    (4, 4, 2, True), (2, 4, 1, True), (2, 6, 2, True),
                                                    (4, 6, 1, False)])
def test_peer_memory_halo_processes(gpu, world, depth, kind, fused):
    """PartitionedCA(halo="peer"): no collective per step, halo cells written into the
    peers' buffers over CUDA IPC + release/acquire step flags == the oracle's steps
    (all ranks share the test box's GPU; 4 ranks exercise every-peer puts and waits)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, 1 << 10, 3, kind, 5, out, depth, fused))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert all(out[r] is True for r in range(world))
    assert all(out[f"bytes{r}"] > 0 for r in range(world))


# ---------------------------------------------------------------------------
# tiled storage (per-rank blocks with a ring)
# ---------------------------------------------------------------------------

def _window_steps(win: np.ndarray, x0: int, y0: int, n: int, kind: int, param: int, steps: int) -> np.ndarray:
    """`steps` CA steps on a window of the global grid, what a tiled block's kernel sees:
    gasket cells (global test, in-grid) get param + neighbours, neighbours outside the
    window read 0 (the window reaches past the block's sub-gasket by its ring)."""
    h, w = win.shape
    ys = np.arange(y0, y0 + h).reshape(h, 1)
    xs = np.arange(x0, x0 + w).reshape(1, w)
    member = (xs >= 0) & (xs < n) & (ys >= 0) & (ys < n) & ((xs & ~ys) == 0)
    offs = [(1, 0), (-1, 0), (0, 1), (0, -1)] + ([(1, 1), (1, -1), (-1, 1), (-1, -1)] if kind == 2 else [])
    a = win.astype(np.int64)
    for _ in range(steps):
        pad = np.zeros((h + 2, w + 2), dtype=np.int64)
        pad[1:-1, 1:-1] = a
        tot = np.full((h, w), param, dtype=np.int64)
        for dx, dy in offs:
            tot += pad[1 + dy:1 + dy + h, 1 + dx:1 + dx + w]
        a = np.where(member, tot, a)
    return a.astype(win.dtype)


@pytest.mark.parametrize("kind", [1, 2])
@pytest.mark.parametrize("world,level,depth", [(1, 2, 1), (2, 2, 1), (3, 3, 2), (4, 3, 6), (4, 2, 4), (8, 3, 1)])
def test_tiled_protocol_matches_full_steps_cpu(oracle, kind, world, level, depth):
    """The tiled storage end to end on CPU: every rank's blocks (sub-gasket + ring) loaded
    from the initial grid, each block advanced `depth` steps from its window alone (the
    numpy stand-in for gm_run_part_tiled), then the copies of tiled_exchange applied
    (remote entries into the other ranks' rings, own entries into own rings); after 3
    rounds every sub-gasket equals 3*depth full-grid oracle steps.  This pins the ring
    depth, the halo lists and the block addressing the GPU kernels use."""
    n = 1024
    plan = P.PartitionPlan(n, level, world, eight=kind == 2, depth=depth)
    init = oracle.fill_hash(n, np.int8, 17, 0)
    lays = [P.TiledLayout(plan, r, 1) for r in range(world)]
    bufs = []
    for L in lays:
        b = torch.zeros(L.nbytes, dtype=torch.int8)
        L.load_dense(b, torch.from_numpy(init))
        bufs.append(b)
    ent = P.tiled_exchange(plan, 1)
    for _ in range(3):
        new = []
        for L, b in zip(lays, bufs):
            nb = b.clone()
            for k in range(L.count):
                x0, x1, y0, y1 = L.window(k)
                v = L.block_view(b, k).numpy()
                out = _window_steps(v[:, :x1 - x0], x0, y0, n, kind, 1, depth)
                L.block_view(nb, k).numpy()[L.R:L.R + L.m, L.pc:L.pc + L.m] = out[L.R:L.R + L.m, L.pc:L.pc + L.m]
            new.append(nb)
        for o, (src, dst) in enumerate(ent):
            vals = new[o].numpy()[src]
            for q in range(world):
                sel = (dst >> 56) == q
                new[q].numpy()[dst[sel] & ((1 << 56) - 1)] = vals[sel]
        bufs = new
    want = init.copy()
    for _ in range(3 * depth):
        nxt = want.copy()
        oracle.run_bounding_box(nxt, want, 1, kind, 1)
        want = nxt
    got = torch.from_numpy(init.copy())
    for L, b in zip(lays, bufs):
        L.store_dense(b, got)
    assert np.array_equal(got.numpy(), want)


def test_tiled_storage_shrinks_with_ranks():
    """Per-rank storage = its sub-gasket blocks + rings: ~1/N of the whole gasket's blocks,
    which is itself ~1/4 of the dense grid at level 5 (243 of 1024 blocks)."""
    n, level = 1 << 18, 5
    whole = P.TiledLayout(P.PartitionPlan(n, level, 1, eight=True), 0, 1).nbytes
    assert whole < 0.27 * n * n
    for world in (2, 4, 8):
        plan = P.PartitionPlan(n, level, world, eight=True)
        per = [P.TiledLayout(plan, r, 1).nbytes for r in range(world)]
        assert max(per) <= (whole / world) * 1.04  # 243 blocks split as evenly as they go


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [1, 2])
def test_tiled_loopback_gpu_matches_full_grid(gpu, kind):
    """gm_run_part_tiled + the tiled halo copies (loopback virtual ranks on one GPU) ==
    the unpartitioned tuned kernel, bit for bit: depth 1 (single-step kernel on the
    blocks) and 2 / 4 / 6 (fused kernel), several worlds, 1/2/4-byte cells."""
    be = gpu.backends
    S = gpu.geometry.IntraStrategy
    for n, level, worlds, dt in ((1 << 12, 3, (1, 2, 3, 8), torch.int8), (1 << 14, 5, (8,), torch.int8),
                                 (1 << 12, 2, (2,), torch.int16), (1 << 12, 2, (3,), torch.int32)):
        init = gpu.device.fill_hash(n, dt, 5, 0)
        ref = {0: init}
        a = init
        for s in range(1, 13):
            b = a.clone()
            be.run_block_space(b, a, 64, (n // 64).bit_length() - 1, S.TUNED, kind=kind, param=1)
            a = b
            ref[s] = a
        for world in worlds:
            for depth, rounds in ((1, 3), (2, 2), (4, 2), (6, 2)):
                if depth == 6 and dt == torch.int32:
                    continue
                plan = P.PartitionPlan(n, level, world, eight=kind == 2, depth=depth)
                got = P.run_loopback_tiled(plan, kind, rounds, dtype=dt, init=init)
                assert gpu.device.count_mismatch(got, ref[depth * rounds]) == 0, (n, level, world, depth, str(dt))
                got = P.run_loopback_tiled(plan, kind, rounds, dtype=dt, seed=5, out=init.clone())
                assert gpu.device.count_mismatch(got, ref[depth * rounds]) == 0, ("seed", n, level, world, depth)


@pytest.mark.gpu
def test_tiled_n18_eight_ranks_vs_oracle(gpu, oracle):
    """BASELINE config 5 at its size: n = 2^18 int8, NSUM8, the level-5 partition over 8
    virtual ranks on tiled storage (the blocks of all 8 ranks: 2 x 16.8 GB instead of
    8 x 2 x 64 GiB), depth 1 (3 exchange rounds) and depth 6 (one round), against the
    oracle on sampled row bands that straddle sub-gasket boundaries."""
    from tests.gpu_compare import band_mismatches, sampled_bands

    n, seed = 1 << 18, 7
    bands = sampled_bands(n, 512, 16)
    for depth, rounds in ((1, 3), (6, 1)):
        plan = P.PartitionPlan(n, 5, 8, eight=True, depth=depth)
        out = gpu.device.fill_hash(n, torch.int8, seed, 0)
        got = P.run_loopback_tiled(plan, 2, rounds, seed=seed, out=out)
        torch.cuda.synchronize()
        bad = band_mismatches(gpu, oracle, {depth * rounds: got}, n, np.int8, seed, 0, 2, 1, bands=bands)
        assert bad == {depth * rounds: 0}, (depth, bad)
        del got, out
        torch.cuda.empty_cache()


def _tiled_peer_worker(rank, world, port, n, level, kind, rounds, out, depth=1, fused=False):
    import torch.distributed as dist

    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        plan = P.PartitionPlan(n, level, world, eight=kind == 2, depth=depth)
        init = oracle.fill_hash(n, np.int8, 9, 0)
        ca = P.TiledCA(plan, rank, kind, 1, init=torch.from_numpy(init).cuda(), group=dist.group.WORLD, halo="peer",
                       fused=fused)
        for _ in range(rounds):
            ca.step()
        got = torch.from_numpy(init.copy()).cuda()
        ca.store_dense(got)
        ca.peer.check()
        lo, hi = plan.ranges[rank]
        want = _reference_steps(init, kind, 1, rounds * depth)
        ok = True
        for s in range(lo, hi):
            bx, by = P.subgasket_block(s, level)
            m = plan.m
            ok &= bool(np.array_equal(got[by * m:(by + 1) * m, bx * m:(bx + 1) * m].cpu().numpy(),
                                      want[by * m:(by + 1) * m, bx * m:(bx + 1) * m]))
        out[rank] = ok
        out[f"bytes{rank}"] = ca.storage_bytes
        ca.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,depth,kind,fused", [(2, 1, 2, False), (2, 1, 1, True), (4, 2, 2, True),
                                                    (4, 6, 2, False), (2, 6, 1, True), (3, 4, 2, True)])
def test_tiled_peer_memory_processes(gpu, world, depth, kind, fused):
    """TiledCA(halo="peer"): per-entry destinations (gm_peer_halo_put_to / the fused
    epilogue's didx) into the peers' rings and the rank's own rings, processes sharing
    the test GPU; every rank's sub-gaskets equal the oracle's steps."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    ps = [ctx.Process(target=_tiled_peer_worker, args=(r, world, port, 1 << 10, 3, kind, 3, out, depth, fused))
          for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert all(out[r] for r in range(world)), dict(out)


@pytest.mark.parametrize("world,depth", [(2, 1), (4, 2), (8, 6), (3, 4)])
def test_tiled_collective_and_peer_move_the_same_cells(world, depth):
    """The all_gather layout of the tiled collective path (unique sends per owner, the
    receivers' gathered positions, own ring copies) delivers exactly the copies the peer
    path's per-entry destinations make: the same (destination rank, cell) <- (owner, cell)
    pairs, nothing more, nothing less."""
    plan = P.PartitionPlan(1 << 12, 4, world, eight=True, depth=depth)
    ent = P.tiled_exchange(plan, 1)
    peer = set()
    for o, (src, dst) in enumerate(ent):
        for a, b in zip(src.tolist(), dst.tolist()):
            peer.add((b >> 56, b & ((1 << 56) - 1), o, a))
    coll = set()
    colls = [P._TiledCollective(plan, r, ent, torch.int8, device="cpu") for r in range(world)]
    sends = [c.send_idx.numpy() for c in colls]
    for r, c in enumerate(colls):
        for pos, cell in zip(c.recv_pos.tolist(), c.recv_idx.tolist()):
            o, slot = divmod(pos, c.width)
            coll.add((r, cell, o, int(sends[o][slot])))
        for a, b in zip(c.local_src.tolist(), c.local_dst.tolist()):
            coll.add((r, b, r, a))
        assert c.width == colls[0].width  # one fixed-size all_gather
    assert coll == peer and len(peer) > 0
