#!/usr/bin/env python
"""Small launches of every product kernel family, for compute-sanitizer (memcheck,
racecheck, synccheck):  compute-sanitizer --tool T python scripts/sanitize_cases.py [part]

  (default)  write pass (every schedule, both store modes), paper-literal lambda / BB
             (incl. the vectorised BB), stencil v2 (NSUM4/8, 1/2/4-byte cells, whole-sector
             blend), the in-place launch, the CA step with the static edge cache, the fused CA
             kernel (T = 2, 4, 6), the banded masked snapshot + staged
             host write-back, lambda maps, coverage
  part       the partitioned CA with the peer-memory halo fused into the step kernel, two
             processes on the one GPU (CUDA IPC)
Each case is checked against the CPU oracle so a run also shows the results are right.
"""

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (checker only)
from paper_1706_04552_b200 import backends, device, native  # noqa: E402
from paper_1706_04552_b200.geometry import IntraStrategy as S  # noqa: E402


def steps(init, kind, param, k):
    a = init.copy()
    for _ in range(k):
        b = a.copy()
        oracle.run_bounding_box(b, a, 1, kind, param)
        a = b
    return a


def main_cases():
    bad = 0
    n = 512
    for dt in (np.int8, np.int16, np.int32, np.int64):
        g0 = oracle.fill_hash(n, dt, 3, 0)
        want = g0.copy()
        oracle.run_bounding_box(want, want, 1, 0, 5)
        for fl in (0, native.FLAG_ROWMAJOR, native.FLAG_GRID_ROWS, native.FLAG_WRITE_SWEEP):
            g = torch.from_numpy(g0.copy()).cuda()
            backends.run_block_space(g, g, 32, 4, S.TUNED, kind=0, param=5, flags=fl)
            bad += not np.array_equal(g.cpu().numpy(), want)
        z = torch.zeros((n, n), dtype=g.dtype, device="cuda")
        backends.run_block_space(z, z, 32, 4, S.TUNED, kind=0, param=5, assume_zero_background=True)
        wz = np.zeros((n, n), dtype=dt)
        oracle.run_bounding_box(wz, wz, 1, 0, 5)
        bad += not np.array_equal(z.cpu().numpy(), wz)
        for rho, strat in ((8, S.SUBBOX), (16, S.TABLE), (16, S.UNROLL)):
            g = torch.from_numpy(g0.copy()).cuda()
            lx, ly = backends.local_cell_arrays(strat, rho)
            backends.run_block_space(g, g, rho, (n // rho).bit_length() - 1, strat, lx, ly, kind=0, param=5)
            bad += not np.array_equal(g.cpu().numpy(), want)
        for variant in ({}, {"early_exit": True}, {"vectorized": True}):
            g = torch.from_numpy(g0.copy()).cuda()
            backends.run_bounding_box(g, g, 8, 0, 5, **variant)
            bad += not np.array_equal(g.cpu().numpy(), want)
    for dt in (np.int8, np.int16, np.int32):
        for kind in (1, 2):
            src = oracle.fill_hash(n, dt, 7, 0)
            want = src.copy()
            oracle.run_bounding_box(want, src, 1, kind, 3)
            for fl in (0, native.FLAG_DST_FROM_SRC):
                g = torch.from_numpy(src.copy()).cuda()
                backends.run_block_space(g, torch.from_numpy(src).cuda(), 64, 3, S.TUNED, kind=kind, param=3, flags=fl)
                bad += not np.array_equal(g.cpu().numpy(), want)
            # the in-place launch (src is the grid: border snapshot + patched staging windows)
            g_ip = torch.from_numpy(src.copy()).cuda()
            backends.run_block_space(g_ip, g_ip, 64, 3, S.TUNED, kind=kind, param=3)
            bad += not np.array_equal(g_ip.cpu().numpy(), want)
            # the CA step with the static left-edge cache (edge.cu: build + 2-deep staging ring)
            s_d = torch.from_numpy(src.copy()).cuda()
            c = s_d.element_size()
            edge = torch.empty(native.ca_edge_bytes(n, c), dtype=torch.uint8, device="cuda")
            native.call("gm_ca_edge_build", edge.data_ptr(), s_d.data_ptr(), n, c, -1, 0, 0, None, 0,
                        device.stream_handle())
            d_d = s_d.clone()
            native.call("gm_ca_run", d_d.data_ptr(), s_d.data_ptr(), n, c, kind, 3, 1, edge.data_ptr(), 0,
                        device.stream_handle())
            bad += not np.array_equal(d_d.cpu().numpy(), want)
            for T in (2, 4, 6):
                if T == 6 and dt == np.int32:
                    continue
                s_d = torch.from_numpy(src.copy()).cuda()
                d_d = s_d.clone()
                native.call("gm_ca_steps", d_d.data_ptr(), s_d.data_ptr(), n, s_d.element_size(), kind, 3, T, 0,
                            device.stream_handle())
                bad += not np.array_equal(d_d.cpu().numpy(), steps(src, kind, 3, T))
            # staged host path: masked snapshot -> kernel -> whole-line write-back
            os.environ[device.HOST_TRANSPORT_ENV] = "mapped"
            h = src.copy()
            backends.run_block_space(h, h, 64, 3, S.TUNED, kind=kind, param=3)
            bad += not np.array_equal(h, want)
            os.environ.pop(device.HOST_TRANSPORT_ENV)
    lx, ly = device.map_rectangle(8)
    olx, oly = oracle.map_rectangle(8)
    bad += not (np.array_equal(lx.cpu().numpy(), olx) and np.array_equal(ly.cpu().numpy(), oly))
    torch.cuda.synchronize()
    print(f"sanitize cases: {'ok' if bad == 0 else f'{bad} MISMATCHES'}", flush=True)
    return bad


def _peer_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1706_04552_b200 import partition as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    n, level = 1024, 3
    ok = True
    try:
        init = oracle.fill_hash(n, np.int8, 9, 0)
        for depth in (1, 2, 6):
            want = steps(init, 2, 1, 2 * depth)
            plan = P.PartitionPlan(n, level, world, eight=True, depth=depth)
            # dense layout, exchange fused into the step kernel
            ca = P.PartitionedCA(plan, rank, torch.from_numpy(init).cuda(), 2, 1, group=dist.group.WORLD,
                                 halo="peer", fused=True)
            for _ in range(2):
                ca.step()
            torch.cuda.synchronize()
            mask = ca.owned_mask().cpu().numpy()
            ok &= bool(np.array_equal(ca.a.cpu().numpy()[mask], want[mask]))
            ca.close()
            # tiled storage, per-entry destinations in the fused epilogue
            tc = P.TiledCA(plan, rank, 2, 1, init=torch.from_numpy(init).cuda(), group=dist.group.WORLD,
                           halo="peer", fused=True)
            for _ in range(2):
                tc.step()
            got = torch.from_numpy(init.copy()).cuda()
            tc.store_dense(got)
            ok &= bool(np.array_equal(got.cpu().numpy()[mask], want[mask]))
            tc.close()
    except Exception as e:  # report instead of leaving the parent waiting
        print(f"rank {rank}: {e!r}", flush=True)
        ok = False
    dist.destroy_process_group()
    q.put((rank, ok))


def main_part():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_peer_worker, args=(r, 2, 29611, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join()
    print(f"sanitize part (2 processes, fused peer epilogue): {'ok' if all(res.values()) else res}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "part":
        main_part()
    else:
        sys.exit(1 if main_cases() else 0)
