"""Host-side sweep pieces (no GPU): problem_digest pinned to the reference, normalized_metrics
semantics (instrument.py:155-190), plan validation and the bench CSV layout (cli.py:274-292)."""

import json
import os

import numpy as np
import pytest

import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import instrument as ins
from paper_1412_4080_b200 import sweep as sw

HERE = os.path.dirname(__file__)


def _digest_case(c):
    rng = np.random.default_rng(100 + c["seed"])
    D = rng.standard_normal((c["n"], c["k"]))
    D /= np.linalg.norm(D, axis=0)
    y = rng.standard_normal(c["n"])
    y /= np.linalg.norm(y)
    dic = ds.Dictionary(D)
    part = None
    if c["grouped"]:
        groups = [np.arange(g, g + 5) for g in range(0, c["k"], 5)]
        part = ds.GroupPartition.build(dic, groups, spectral_norms=np.ones(len(groups)))
    return ds.Problem(dic, y, c["lam"], part)


def test_problem_digest_matches_reference():
    with open(os.path.join(HERE, "golden", "digest_cases.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        assert ins.problem_digest(_digest_case(c)) == c["digest"]


def _trace(strategy, flops, seconds, lam=0.3, digest="d"):
    t = ins.SolveTrace(kind="lasso", strategy=strategy, n_rows=10, n_cols=20, group_count=0, lam=lam, digest=digest)
    t.append(1, 20, 1, 1.0, flops, seconds)
    return t


def test_normalized_metrics():
    m = ins.normalized_metrics(_trace("none", 100, 2.0), _trace("static", 50, 1.0), _trace("dynamic", 25, 0.5))
    assert (m.flops_static_ratio, m.flops_dynamic_ratio, m.time_static_ratio, m.time_dynamic_ratio) == (0.5, 0.25, 0.5, 0.25)
    with pytest.raises(ValueError):   # wrong order
        ins.normalized_metrics(_trace("static", 1, 1.0), _trace("none", 1, 1.0), _trace("dynamic", 1, 1.0))
    with pytest.raises(ValueError):   # different instances
        ins.normalized_metrics(_trace("none", 1, 1.0), _trace("static", 1, 1.0, digest="x"), _trace("dynamic", 1, 1.0))
    with pytest.raises(ValueError):   # degenerate baseline
        ins.normalized_metrics(_trace("none", 0, 1.0), _trace("static", 1, 1.0), _trace("dynamic", 1, 1.0))


def test_sweep_plan_validation_and_csv(tmp_path):
    sw.SweepPlan([0.5, 0.9], algorithms=["ista", "fista"], tests=["safe", "dst3", "dome"]).validate("lasso")
    sw.SweepPlan([0.5], tests=["gst3"]).validate("group")
    for bad in (sw.SweepPlan([0.9, 0.5]), sw.SweepPlan([0.0, 0.5]), sw.SweepPlan([0.5, 1.5]),
                sw.SweepPlan([0.5], tests=["gst3"]), sw.SweepPlan([0.5], algorithms=["newton"])):
        with pytest.raises(ValueError):
            bad.validate("lasso")
    rows = [(0, "ista", "none", "-", 0.5, 10, 1000, 0.01, 0.2, 0.0),
            (0, "ista", "dynamic", "dst3", 0.5, 10, 600, 0.005, 0.2, 0.4)]
    path = tmp_path / "bench.csv"
    assert sw.write_bench_csv(rows, path, sw.SweepPlan([0.5])) == 2
    lines = path.read_text().splitlines()
    assert lines[0].startswith("# ") and lines[1] == sw.BENCH_HEADER
    assert lines[2] == "0,ista,dynamic,dst3,0.5,10,600,0.005,0.2,0.4"     # sorted like run_bench
