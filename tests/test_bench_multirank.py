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


def _run_two_ranks(args: list[str]) -> dict:
    env = dict(os.environ, GASKET_BENCH_SHARED_GPU="1", OMP_NUM_THREADS="1", PYTHONFAULTHANDLER="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2", *args]
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env, cwd=ROOT)
    try:
        stdout, stderr = p.communicate(timeout=240)
    except subprocess.TimeoutExpired:
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
    return json.loads([x for x in stdout.splitlines() if x.startswith("{")][-1])


def test_bench_two_ranks_write16(gpu):
    """The default workload at N=2 (the driver's scaling run): one independent n=2^16 grid per
    rank, weak scaling, the job's e2e from every rank's own host grid."""
    line = _run_two_ranks(["--steps", "5", "--warmup", "3"])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.parametrize("halo,temporal,storage", [("collective", 1, "tiled"), ("peer", 6, "tiled"),
                                                   ("peer-fused", 1, "tiled"), ("peer-fused", 6, "tiled"),
                                                   ("collective", 2, "dense")])
def test_bench_two_ranks_part15(gpu, halo, temporal, storage):
    line = _run_two_ranks(["--steps", "4", "--warmup", "3", "--workload", "part15", "--halo", halo, "--temporal",
                           str(temporal), "--storage", storage])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["storage"] == storage and line["config"]["halo"] == halo
    if storage == "tiled":
        assert line["config"]["storage_bytes_per_rank"] < 2 * (1 << 30) // 4
