"""The sweep harness on the device (the reference's bench.run_sweep,
bench.py:166-232, CSV schema :25-29): rows, counters, statuses and the crossover n0."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_run_sweep_on_device_reference_schema(gpu, golden, tmp_path):
    from paper_1706_04552_b200 import bench as B
    from paper_1706_04552_b200.engine import Mapping

    meta, _ = golden
    cfg = B.SweepConfig(r_min=6, r_max=13, rho_set=(8, 16, 32), reps=(3, 2), dtype=torch.int32,
                        mem_limit_bytes=1 << 30, time_budget_s=0.2)
    recs = B.run_sweep(cfg)
    combos = [(Mapping.BOUNDING_BOX.value, "none")] + [(Mapping.BLOCK_SPACE.value, s.value) for s in cfg.strategies]
    # one row per (r, rho, mapping/strategy), BB first within each (r, rho)
    assert [(r.r, r.rho, r.mapping, r.strategy) for r in recs] == [
        (r, rho, m, s) for r in range(6, 14) for rho in (8, 16, 32) for m, s in combos]
    golden_wc = {(w["n"], w["rho"], w["mapping"], w["strategy"] or "none"): w["counts"] for w in meta["work_counts"]}
    checked = 0
    for rec in recs:
        assert rec.status == "ok" or rec.status.startswith("ok-reps="), rec
        assert rec.wall_ns_mean is not None and rec.wall_ns_mean > 0
        key = (rec.n, rec.rho, rec.mapping, rec.strategy)
        if key in golden_wc:  # engine.work_counts of the live reference (n = 64, 256, 8192)
            assert [rec.blocks_launched, rec.threads_launched, rec.threads_useful, rec.map_ops,
                    rec.reduction_depth, rec.simulated_cost] == golden_wc[key], key
            checked += 1
        if rec.mapping == Mapping.BOUNDING_BOX.value:
            assert rec.cost_ratio is None and rec.speedup is None
        else:
            assert rec.cost_ratio is not None and rec.cost_ratio > 0
            assert rec.speedup is not None and rec.speedup > 0
    assert checked >= 24
    p = tmp_path / "sweep.csv"
    B.write_csv(recs, p)
    assert p.read_text().splitlines()[0] == meta["csv_header"]
    assert [B.record_to_row(r) for r in B.read_csv(p)] == [B.record_to_row(r) for r in recs]
    cross = B.crossover(recs)
    assert set(cross["per_rho"]) == {"8", "16", "32"}
    assert sorted(cross["best_vs_best_paper_literal_by_r"]) == list(range(6, 14))
    # at n = 2^13 the paper-literal lambda kernels beat the bounding box, whose threads land on gasket
    # cells 3^13 / 4^13 = 1.3 % of the time
    assert cross["best_vs_best_paper_literal_by_r"][13] > 1
    n0 = cross["n0_best_vs_best"]
    assert n0 is not None and 64 <= n0 <= 8192


def test_skipped_rows_keep_the_schema(gpu):
    from paper_1706_04552_b200 import bench as B

    cfg = B.SweepConfig(r_min=2, r_max=3, rho_set=(8,), reps=(2, 1), dtype=torch.int32, time_budget_s=0.1)
    recs = B.run_sweep(cfg)
    assert {r.status for r in recs if r.n < 8} == {"skipped-shape"}
    big = B.SweepConfig(r_min=15, r_max=15, rho_set=(32,), reps=(2, 1), dtype=torch.int32,
                        mem_limit_bytes=1 << 20)
    assert {r.status for r in B.run_sweep(big)} == {"skipped-mem"}
