"""bench.py's reference arm (CPU, runs here): one JSON line with the contract's
keys, the same metric/config/unit as our arm, and e2e with zero copies."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("workload", ["write16", "stencil17"])
def test_reference_arm_line(workload):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--workload", workload], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    sys.path.insert(0, str(ROOT))
    import bench

    assert line["impl"] == "reference"
    assert line["metric"] == bench._metric(workload)
    r, _, _, rho, _ = bench.WORKLOADS[workload]
    assert line["config"] == bench._config(workload, rho, 1, False)
    assert line["unit"] == "cells/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "cells/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
