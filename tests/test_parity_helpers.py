"""CPU checks of oracle/parity.py (the north_star parity rules used by the -m gpu tests)."""

import numpy as np

from oracle import parity
from oracle import screen_oracle as so
from paper_1412_4080_b200 import workloads as wl


def _run(test="dst3", ratio=0.6):
    D = wl.correlated_dictionary(40, 200, 2)
    y, _ = wl.planted_observation(D, 2, nnz=4)
    op = so.make_problem(D, y, ratio * wl.lambda_star(D, y))
    rec = parity.RadiusRecorder()
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
    ref = so.solve(op, so.Config(algorithm="fista", strategy="dynamic", test=test, max_iters=2000,
                                 rel_tol=1e-300, L0=L, gap_tol=1e-9), hook=rec)
    return op, ref, rec


def test_margin_rule_accepts_equal_sets_and_near_threshold_units_only():
    op, ref, rec = _run()
    assert ref.eliminated.size > 0 and len(rec.radius) == ref.iterations
    ok, diff, _ = parity.screened_sets_agree(op, "dst3", ref.eliminated, ref.eliminated, rec.radius)
    assert ok and diff.size == 0
    kept = np.setdiff1d(np.arange(op.k), ref.eliminated)
    values, _ = parity.unit_test_values(op, "dst3")
    far = kept[np.argmax(np.abs(values[kept][:, None] - np.array(rec.radius)[None, :]).min(axis=1))]
    ok, diff, m = parity.screened_sets_agree(op, "dst3", np.union1d(ref.eliminated, [far]), ref.eliminated,
                                             rec.radius)
    assert not ok and diff.tolist() == [far] and m[0] > 1e-9
    # a unit whose test value sits 1e-10 from a recorded threshold is a legitimate difference
    radii = list(rec.radius) + [float(values[far] - so.SCREEN_MARGIN - 1e-10)]
    ok, _, m = parity.screened_sets_agree(op, "dst3", np.union1d(ref.eliminated, [far]), ref.eliminated, radii)
    assert ok and m[0] <= 1e-9


def test_certified_safety_and_group_values():
    op, ref, _ = _run("safe", 0.8)
    safe, gap = parity.certified_safe(op, ref.eliminated)
    assert safe and gap <= 1e-10
    assert parity.certified_safe(op, np.empty(0, np.int64)) == (True, 0.0)
    D = wl.gaussian_dictionary(30, 60, 3)
    groups = [np.arange(g, g + 3) for g in range(0, 60, 3)]
    y = wl.gaussian_observation(30, 3)
    gp = so.make_problem(D, y, 0.5 * wl.lambda_star(D, y, groups), groups)
    v, gof = parity.unit_test_values(gp, "gst3")
    assert v.shape == (20,) and gof.shape == (60,) and gof[59] == 19


def test_bf16_rounding_is_nearest_even_from_fp64():
    from fractions import Fraction

    from oracle import batched_oracle as bo
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-20, 20, 2000),
                        [1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -(1.0 + 2.0 ** -8), 1.0 + 2.0 ** -8 + 2.0 ** -40]])
    got = bo.bf16_rn(v)
    for a, g in zip(v, got):
        m, e = np.frexp(abs(a))                  # a = m 2^e, m in [0.5, 1): keep 8 significant bits
        q = Fraction(float(m)) * 256
        lo = int(q)
        r = lo + (1 if (q - lo > Fraction(1, 2) or (q - lo == Fraction(1, 2) and lo % 2)) else 0)
        assert g == np.copysign(np.ldexp(r / 256.0, int(e)), a)


def test_bf16_oracle_with_two_terms_tracks_the_fp64_oracle():
    from oracle import batched_oracle as bo
    from paper_1412_4080_b200 import workloads as wl
    w = wl.config5(seed=2, n=64, k=256, batch=4, nnz=4, ratio=0.5)
    D = wl.bf16_to_f64(w.D).reshape(w.D.shape)
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-6))
    for j in range(4):
        e2 = bo.solve_bf16(D, w.y[:, j], w.lam[j], L, 60, splits=2)
        e1 = bo.solve_bf16(D, w.y[:, j], w.lam[j], L, 60, splits=1)
        ref = so.solve(so.make_problem(D, w.y[:, j], w.lam[j]),
                       so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=60, rel_tol=1e-300,
                                 L0=L, norm_aware=True))
        assert abs(e2.objective - ref.final_objective) <= 1e-9 * ref.final_objective
        assert abs(e1.objective - ref.final_objective) <= 1e-5 * ref.final_objective
        # the inflated correlation bound only ever screens less
        assert np.all(np.isin(e1.eliminated, ref.eliminated)) and np.all(np.isin(e2.eliminated, ref.eliminated))
