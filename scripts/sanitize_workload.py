"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python scripts/sanitize_workload.py [fused|sharded|batched|ops|all]

* fused   -- c1-shaped solve (1000 x 5000 fp64, ISTA + DST3) through run(): setup graph, the
             conditional-WHILE loop graph (K1/K2/K3a/K3b with last-CTA tickets); plus a group
             FISTA/GST3 solve, a FISTA/SAFE solve with backtracking REDO trips (L0 = 1) and an
             fp32 tiled-K1 solve;
* sharded -- the split phases at one rank: one collective (K2S/K3S/K1R1/K2C, FIXUP trips), two
             collectives, the peer-memory exchange (st.release.sys / ld.acquire.sys flags), the
             trip graph and the per-phase host loop;
* batched -- config-5-shaped batch (256 x 2048 bf16, 512 observations): tcgen05 CTA-pair GEMM with
             the fused screening epilogue, warp / CTA updates, screening order, sparse residual;
* ops     -- per-op entry points (correlate, apply, prox, tests, operator norm, group norms).
Exits non-zero if any result disagrees with the CPU oracle (so a sanitizer run also checks parity).
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np


def fused():
    import paper_1412_4080_b200 as ds
    from paper_1412_4080_b200 import workloads as wl
    from oracle import screen_oracle as so
    w = wl.config1()
    L = float(np.linalg.norm(w.D, 2) ** 2 * (1 + 1e-6))
    cfg = ds.SolverConfig(algorithm="ista", strategy="dynamic", test="dst3", max_iters=300, rel_tol=1e-300, L0=L,
                          gap_tol=1e-6)
    res = ds.run(ds.Problem(ds.Dictionary(w.D), w.y, w.lam), cfg)
    ref = so.solve(so.make_problem(w.D, w.y, w.lam), so.Config(algorithm="ista", strategy="dynamic", test="dst3",
                                                               max_iters=300, rel_tol=1e-300, L0=L, gap_tol=1e-6))
    assert res.iterations == ref.iterations and np.array_equal(res.screen_state.eliminated, ref.eliminated)
    # backtracking REDO trips
    D = wl.correlated_dictionary(200, 1000, 2)
    y, _ = wl.planted_observation(D, 2, nnz=10)
    lam = 0.6 * wl.lambda_star(D, y)
    c2 = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="safe", max_iters=200, rel_tol=1e-300, L0=1.0)
    r2 = ds.run(ds.Problem(ds.Dictionary(D), y, lam), c2)
    f2 = so.solve(so.make_problem(D, y, lam), so.Config(algorithm="fista", strategy="dynamic", test="safe",
                                                         max_iters=200, rel_tol=1e-300, L0=1.0))
    assert r2.iterations == f2.iterations and abs(r2.final_objective - f2.final_objective) <= 1e-9 * f2.final_objective
    # group FISTA + GST3
    w3 = wl.config3(seed=1, ratio=0.7, n=300, k=1500, group_size=10, n_active=3)
    dic3 = ds.Dictionary(w3.D)
    part = ds.GroupPartition.build(dic3, w3.groups)
    L3 = float(np.linalg.norm(w3.D, 2) ** 2 * (1 + 1e-6))
    c3 = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="gst3", max_iters=300, rel_tol=1e-300, L0=L3,
                         gap_tol=1e-7)
    r3 = ds.run(ds.Problem(dic3, w3.y, w3.lam, part), c3)
    f3 = so.solve(so.make_problem(w3.D, w3.y, w3.lam, w3.groups, part.weights, part.spectral_norms),
                  so.Config(algorithm="fista", strategy="dynamic", test="gst3", max_iters=300, rel_tol=1e-300, L0=L3,
                            gap_tol=1e-7))
    assert r3.iterations == f3.iterations and np.array_equal(r3.screen_state.eliminated, f3.eliminated)
    # fp32 tiled K1 (short columns)
    D4 = wl.gaussian_dictionary_f32(1536, 4096, 3)
    y4 = wl.gaussian_observation(1536, 3)
    lam4 = 0.3 * float(np.max(np.abs(D4.astype(np.float64).T @ y4)))
    L4 = float(np.linalg.norm(D4.astype(np.float64), 2) ** 2 * (1 + 1e-6))
    c4 = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=200, rel_tol=1e-300, L0=L4,
                         gap_tol=1e-6)
    r4 = ds.run(ds.Problem(ds.Dictionary(D4, check_unit_norms=False, dtype="f32"), y4, lam4), c4)
    f4 = so.solve(so.make_problem(D4.astype(np.float64), y4, lam4),
                  so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=200, rel_tol=1e-300,
                            L0=L4, gap_tol=1e-6, norm_aware=True))
    assert abs(r4.iterations - f4.iterations) <= 1
    print(f"fused ok: c1 {res.iterations} it, backtracking {r2.iterations} it, group {r3.iterations} it, "
          f"fp32 {r4.iterations} it")


def sharded():
    import paper_1412_4080_b200 as ds
    from paper_1412_4080_b200 import dist as pdist
    from paper_1412_4080_b200 import workloads as wl
    D = wl.correlated_dictionary(200, 2000, 5)
    y, _ = wl.planted_observation(D, 5, nnz=10)
    p = ds.Problem(ds.Dictionary(D), y, 0.6 * wl.lambda_star(D, y))
    nrm = float(np.linalg.norm(D, 2))
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=2000, rel_tol=1e-300,
                          L0=nrm * nrm * (1 + 1e-9), gap_tol=1e-9)
    a = ds.run(p, cfg)
    for coll in (1, 2, "peer"):
        for graph in (True, False):
            b = pdist.run_sharded(p, cfg, pg=None, collectives=coll, graph=graph)
            assert a.iterations == b.iterations, (coll, graph)
            assert np.array_equal(a.screen_state.eliminated, b.screen_state.eliminated)
    print(f"sharded ok: {a.iterations} it in all exchange modes")


def batched():
    import paper_1412_4080_b200 as ds
    from paper_1412_4080_b200 import workloads as wl
    from paper_1412_4080_b200.batched import solve_batched
    from oracle import batched_oracle as bo
    w = wl.config5(seed=3, n=256, k=2048, batch=512, nnz=8, ratio=0.85)
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
    D64 = dic.as_float64()
    L = float(np.linalg.norm(D64, 2) ** 2 * (1 + 1e-6))
    res = solve_batched(dic, w.y, w.lam, L, iterations=40, test="dst3", splits=1, masks=True)
    for j in (0, 111, 511):
        emu = bo.solve_bf16(D64, w.y[:, j], w.lam[j], L, 40, splits=1)
        assert abs(res.objective[j] - emu.objective) <= 1e-7 * emu.objective
        assert np.array_equal(res.eliminated(j), emu.eliminated)
    print(f"batched ok: kept min {res.kept.min()}")


def ops():
    import paper_1412_4080_b200 as ds
    from paper_1412_4080_b200 import workloads as wl
    D = wl.gaussian_dictionary(300, 1200, 4)
    dic = ds.Dictionary(D)
    v = wl.gaussian_observation(300, 4)
    assert np.allclose(dic.correlate(v), D.T @ v, rtol=1e-12, atol=1e-14)
    x = np.zeros(1200)
    x[::7] = 1.0
    assert np.allclose(dic.apply(x), D @ x, rtol=1e-12, atol=1e-13)
    nrm = ds.operator_norm(dic, tol=1e-12, max_iters=20000)
    assert abs(nrm - np.linalg.norm(D, 2)) <= 1e-8 * nrm
    part = ds.GroupPartition.build(dic, [np.arange(g, g + 6) for g in range(0, 1200, 6)])
    sn = np.array([np.linalg.norm(D[:, g], 2) for g in part.groups])
    assert np.allclose(part.spectral_norms, sn, rtol=1e-8)
    print("ops ok")


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in (("fused", fused), ("sharded", sharded), ("batched", batched), ("ops", ops)):
        if which in (name, "all"):
            fn()
