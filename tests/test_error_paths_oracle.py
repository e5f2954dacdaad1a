"""The oracle reproduces the reference's error paths (tests/golden/error_cases.json, recorded
from screenlab itself): FloatingPointError for non-finite iterates and failed backtracking,
RuntimeError for the radius guard and a degenerate GST3 normal, and the one overflow run the
reference completes with +inf objectives."""

import json
import os
import warnings

import numpy as np
import pytest

from oracle import screen_oracle as so
from tests.error_cases import CASES

with open(os.path.join(os.path.dirname(__file__), "golden", "error_cases.json")) as fh:
    GOLD = json.load(fh)


def oracle_outcome(c):
    prob = so.make_problem(c["D"], c["y"], c["lam"], c["groups"], c["weights"])
    cfg = so.Config(**c["cfg"])
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            return "ok", so.solve(prob, cfg)
    except (FloatingPointError, RuntimeError) as e:
        return type(e).__name__, e


@pytest.mark.parametrize("name,build", CASES, ids=[c[0] for c in CASES])
def test_oracle_error_paths_match_reference(name, build):
    ref = GOLD[name]
    kind, res = oracle_outcome(build())
    assert kind == ref["outcome"], (kind, ref)
    if kind == "ok":
        assert res.iterations == ref["iterations"]
        assert res.trace["objective"] == ref["objective"]
        assert bool(np.all(np.isfinite(res.x_star))) == ref["x_finite"]
        assert float(np.max(np.abs(res.x_star))) == pytest.approx(ref["x_absmax"], rel=1e-12)
    else:
        assert str(res).split(";")[0].split(" fell to")[0] in ref["message"]
