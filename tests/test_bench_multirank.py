"""The multi-rank bench path (torchrun, one process per rank) on the test box's one GPU:
every rank on cuda:0 with gloo plumbing (GASKET_BENCH_SHARED_GPU=1), the partitioned CA
on tiled storage with each halo transport.  Functional only (the ranks time-slice one
GPU); the 8-GPU command is scripts/part18_8gpu.sh."""

import json
import os
import signal
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("halo,temporal,storage", [("collective", 1, "tiled"), ("peer", 6, "tiled"),
                                                   ("peer-fused", 1, "tiled"), ("peer-fused", 6, "tiled"),
                                                   ("collective", 2, "dense")])
def test_bench_two_ranks_part15(gpu, halo, temporal, storage):
    env = dict(os.environ, GASKET_BENCH_SHARED_GPU="1", OMP_NUM_THREADS="1", PYTHONFAULTHANDLER="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--workload", "part15", "--halo", halo, "--temporal", str(temporal),
           "--storage", storage]
    # on a hang every rank gets SIGABRT (faulthandler prints where it waits) instead of the
    # test blocking the suite
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env, cwd=ROOT)
    try:
        stdout, stderr = p.communicate(timeout=240)
    except subprocess.TimeoutExpired:
        # torchrun starts its workers in sessions of their own: signal every descendant
        import psutil

        procs = psutil.Process(p.pid).children(recursive=True) + [psutil.Process(p.pid)]
        for q in procs:
            try:
                q.send_signal(signal.SIGABRT)
            except psutil.NoSuchProcess:
                pass
        try:
            stdout, stderr = p.communicate(timeout=30)
        except subprocess.TimeoutExpired:
            for q in procs:
                try:
                    q.kill()
                except psutil.NoSuchProcess:
                    pass
            stdout, stderr = p.communicate()
        pytest.fail(f"multi-rank bench hung (240 s); tracebacks:\n{stderr[-8000:]}")
    assert p.returncode == 0, stderr[-3000:]
    line = json.loads([x for x in stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["storage"] == storage and line["config"]["halo"] == halo
    if storage == "tiled":
        assert line["config"]["storage_bytes_per_rank"] < 2 * (1 << 30) // 4
