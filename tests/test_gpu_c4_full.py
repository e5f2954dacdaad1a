"""BASELINE config 4 at its full, benchmarked size (8192 x 262144 fp32) against the REFERENCE.

The golden trace ``tests/golden/c4_reference.npz`` was produced in the build container by
running the reference's own ``screenlab.run`` (fp64, on the fp32-rounded dictionary upcast,
``check_unit_norms=False`` -- SURVEY §8(c)) to the first iteration with duality gap <= 1e-5:
``scripts/c4_reference_run.py`` (command and timing in ``tests/golden/c4_reference.json`` and
``profiles/r02_c4_reference_thit.json``).  The GPU consumes the committed L and the same seeded
inputs, and must reproduce, per north_star: the iteration count to the gap (exactly), the
per-iteration objective, gap, kept, nnz and support traces, the final objective and x (rel 1e-4
for fp32 storage; the measured agreement is far tighter and is printed), and the screened set
(margin rule; safety is trivial when nothing is screened, which the golden records).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "c4_reference.npz")


@pytest.fixture(scope="module")
def c4():
    if not os.path.exists(GOLD):
        pytest.fail("missing tests/golden/c4_reference.npz (scripts/c4_reference_run.py)")
    g = dict(np.load(GOLD))
    w = wl.config4(seed=int(g["seed"]), ratio=float(g["ratio"]), n=int(g["n"]), k=int(g["k"]),
                   gap_tol=float(g["gap_tol"]))
    assert w.lam == float(g["lam"]), "c4 inputs drifted from the golden run"
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="f32")
    yield g, w, dic
    dic.drop_device()
    torch.cuda.empty_cache()


def test_c4_full_matches_reference(c4):
    g, w, dic = c4
    L = float(g["L"])
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=10000, rel_tol=1e-300,
                          L0=L, gap_tol=float(g["gap_tol"]))
    res = ds.run(ds.Problem(dic, w.y, w.lam), cfg)
    t_hit = int(g["t_hit"])
    tr = res.trace
    obj_rel = np.max(np.abs(np.array(tr.objective) - g["objective"][: len(tr.objective)]) / g["objective"][0])
    print(f"c4 full: GPU {res.iterations} iterations vs reference {t_hit}; "
          f"max objective rel. diff {obj_rel:.2e}")
    assert res.stop_reason == "gap"
    assert res.iterations == t_hit
    np.testing.assert_allclose(tr.objective, g["objective"], rtol=1e-4)
    np.testing.assert_allclose(tr.gap, g["gap"], rtol=1e-4, atol=1e-10)
    assert tr.kept == g["kept"].tolist()
    assert tr.sparsity == g["nnz"].tolist()
    assert tr.support == g["support"].tolist()
    assert res.lambda_max == pytest.approx(float(g["lmax"]), rel=1e-12)
    x_ref = np.zeros(int(g["k"]))
    x_ref[g["x_idx"]] = g["x_val"]
    xr = np.linalg.norm(res.x_star - x_ref) / np.linalg.norm(x_ref)
    print(f"c4 full: x rel. diff {xr:.2e}, final objective {res.final_objective!r} vs {float(g['objective'][-1])!r}")
    assert xr <= 1e-4
    assert res.final_objective == pytest.approx(float(g["objective"][-1]), rel=1e-4)
    # screened set: the reference's (recorded) -- equality; nothing screened means safety is trivial
    assert np.array_equal(res.screen_state.eliminated, g["eliminated"])


def test_c4_full_operator_norm_matches_committed_L(c4):
    """The committed L is ||D||^2 (1 + 1e-9) from an fp64 Gram eigvalsh; the device power iteration
    (Gram path) must agree, so a bench run computing its own L solves the same problem."""
    g, w, dic = c4
    nrm = ds.operator_norm(dic, tol=1e-12, max_iters=20000)
    assert nrm * nrm == pytest.approx(float(g["L"]) / (1 + 1e-9), rel=1e-9)
