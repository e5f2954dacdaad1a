"""Generate golden vectors by running the REFERENCE implementation (screenlab).

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes ``tests/golden/solver_cases.npz`` (inputs + reference outputs of
``screenlab.run`` with a per-iteration duality-gap hook) and
``tests/golden/kernel_cases.npz`` (outputs of the reference's per-op functions
on seeded inputs).  The committed fixtures pin the CPU oracle
(``oracle/screen_oracle.py``) and, through it, the GPU engine.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import screenlab as sl  # noqa: E402  (reference, from PYTHONPATH)
from screenlab import screening  # noqa: E402

from paper_1412_4080_b200 import workloads as wl  # noqa: E402


def gap_hook(problem, sink):
    """Record r_SAFE^2 at theta_t with the pre-screening correlations."""

    def hook(info):
        if problem.kind == sl.LASSO:
            ci = float(np.max(np.abs(info.corr), initial=0.0))
            _, v = sl.dual_scale_lasso(problem, info.theta, corr_inf=ci)
        else:
            lay = problem.partition.layout(info.kept)
            _, v = sl.dual_scale_group(problem, info.theta, group_corr_norms=lay.norms(info.corr),
                                       group_weights=lay.weights)
        diff = problem.y / problem.lam - v
        sink.append(float(diff @ diff))
        if info.mask is not None:
            sink_masks.append((info.t, info.kept[info.mask].copy()))

    sink_masks = []
    hook.masks = sink_masks
    return hook


def problems():
    """(name, D, y, lam, groups) small instances covering the reference's fixtures."""
    out = []
    # identity instance (tests/conftest.py:30-39)
    out.append(("identity", np.eye(2), np.array([1.0, 0.0]), 0.8, None))
    out.append(("identity_group", np.eye(2), np.array([1.0, 0.0]), 0.8, [np.array([0]), np.array([1])]))
    for seed, n, k, ratio in ((3, 12, 30, 0.7), (11, 16, 40, 0.6), (14, 12, 30, 0.8),
                              (19, 12, 30, 0.999), (2, 30, 80, 0.5), (1, 30, 80, 0.9)):
        D = wl.gaussian_dictionary(n, k, seed)
        y = wl.gaussian_observation(n, seed)
        lam = ratio * wl.lambda_star(D, y)
        out.append((f"lasso_s{seed}_{n}x{k}_r{ratio}", D, y, lam, None))
    for seed, n, k, ratio, gs in ((12, 12, 30, 0.5, 3), (15, 12, 30, 0.7, 3), (2, 30, 80, 0.7, 4),
                                  (1, 30, 80, 0.3, 4), (19, 12, 30, 0.999, 3)):
        D = wl.gaussian_dictionary(n, k, seed)
        groups = wl.random_groups(k, gs, seed)
        y = wl.bernoulli_gaussian_observation(D, groups, seed, p=0.2)
        lam = ratio * wl.lambda_star(D, y, groups)
        out.append((f"group_s{seed}_{n}x{k}_r{ratio}", D, y, lam, groups))
    # scaled-down BASELINE shapes (c1 Gaussian / c2 correlated / c3 contiguous groups)
    D = wl.gaussian_dictionary(100, 500, 0)
    y = wl.gaussian_observation(100, 0)
    out.append(("c1mini", D, y, 0.5 * wl.lambda_star(D, y), None))
    D = wl.correlated_dictionary(100, 600, 0)
    y, _ = wl.planted_observation(D, 0, nnz=8)
    for r in (0.1, 0.5, 0.9):
        out.append((f"c2mini_r{r}", D, y, r * wl.lambda_star(D, y), None))
    w3 = wl.config3(seed=0, ratio=0.5, n=100, k=600, group_size=10, n_active=4)
    out.append(("c3mini", w3.D, w3.y, w3.lam, w3.groups))
    return out


def configs_for(name, kind):
    algos = sl.ALGORITHMS
    tests = screening.LASSO_TESTS if kind == "lasso" else screening.GROUP_TESTS
    cfgs = []
    big = name.startswith("c")
    if big:
        # BASELINE-style: L0 = ||D||^2 (1 + 1e-9), rel_tol off, gap recorded per iteration
        for algo in ("ista", "fista", "sparsa", "cp"):
            for test in tests[:2] if kind == "lasso" else tests:
                cfgs.append(dict(algorithm=algo, strategy="dynamic", test=test, max_iters=400,
                                 rel_tol=1e-300, L0="spec"))
        cfgs.append(dict(algorithm="fista", strategy="static", test=tests[0], max_iters=300,
                         rel_tol=1e-300, L0="spec"))
        return cfgs
    for algo in algos:
        cfgs.append(dict(algorithm=algo, strategy="none", test=None, max_iters=300, rel_tol=1e-10))
        for test in tests:
            cfgs.append(dict(algorithm=algo, strategy="dynamic", test=test, max_iters=300,
                             rel_tol=1e-10))
            cfgs.append(dict(algorithm=algo, strategy="static", test=test, max_iters=300,
                             rel_tol=1e-10))
    return cfgs


def main():
    arrays = {}
    manifest = []
    for pi, (name, D, y, lam, groups) in enumerate(problems()):
        dic = sl.Dictionary(D)
        part = sl.GroupPartition.build(dic, groups, weights=np.ones(2) if name == "identity_group" else None) if groups is not None else None
        p = sl.Problem(dic, y, lam, part)
        pre = f"p{pi}__"
        arrays[pre + "D"] = np.asarray(D)
        arrays[pre + "y"] = y
        if groups is not None:
            arrays[pre + "group_of"] = part.group_of
            arrays[pre + "weights"] = part.weights
            arrays[pre + "snorms"] = part.spectral_norms
        lm = sl.lambda_max(p)
        spec_L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
        op_norm = sl.operator_norm(dic)
        entry = {"name": name, "kind": p.kind, "lam": lam, "lmax": lm.value,
                 "lmax_index": lm.atom_index, "lmax_group": lm.group, "spec_L": spec_L,
                 "op_norm": op_norm, "configs": []}
        for ci, cfgd in enumerate(configs_for(name, p.kind)):
            cfgd = dict(cfgd)
            if cfgd.get("L0") == "spec":
                cfgd["L0"] = spec_L
            cfg = sl.SolverConfig(**cfgd)
            rs = []
            hook = gap_hook(p, rs)
            res = sl.run(p, cfg, iteration_hook=hook)
            obj = np.array(res.trace.objective)
            gaps = obj - 0.5 * float(y @ y) + 0.5 * lam * lam * np.array(rs) if obj.size else obj
            key = f"{pre}c{ci}__"
            arrays[key + "x_star"] = res.x_star
            arrays[key + "eliminated"] = res.screen_state.eliminated
            arrays[key + "objective"] = obj
            arrays[key + "kept"] = np.array(res.trace.kept, dtype=np.int64)
            arrays[key + "nnz"] = np.array(res.trace.sparsity, dtype=np.int64)
            arrays[key + "flops"] = np.array(res.trace.flops_cum, dtype=np.int64)
            arrays[key + "gap"] = gaps
            entry["configs"].append({"cfg": cfgd, "iterations": res.iterations,
                                     "final_objective": res.final_objective})
        manifest.append(entry)
        print(name, len(entry["configs"]), "configs", flush=True)

    # per-op golden cases (reference functions on seeded inputs)
    rng = np.random.default_rng(1234)
    kern = {}
    for i in range(20):
        v = rng.standard_normal(37) * 2
        t = float(rng.random())
        kern[f"prox_l1_{i}__v"] = v
        kern[f"prox_l1_{i}__t"] = np.array(t)
        kern[f"prox_l1_{i}__out"] = sl.prox_l1(v, t)
    D = wl.gaussian_dictionary(10, 12, 7)
    part = sl.GroupPartition.build(sl.Dictionary(D), [np.arange(0, 4), np.arange(4, 7), np.arange(7, 12)])
    for i in range(10):
        v = rng.standard_normal(12) * 3
        t = float(rng.random() * 2)
        kern[f"prox_group_{i}__v"] = v
        kern[f"prox_group_{i}__t"] = np.array(t)
        kern[f"prox_group_{i}__out"] = sl.prox_group(v, t, part)
    kern["prox_group__snorms"] = part.spectral_norms
    for i in range(10):
        n, k = int(rng.integers(2, 14)), int(rng.integers(1, 10))
        M = rng.standard_normal((n, k))
        M /= np.linalg.norm(M, axis=0)
        kern[f"opnorm_{i}__D"] = M
        kern[f"opnorm_{i}__out"] = np.array(sl.operator_norm(sl.Dictionary(M)))
    np.savez_compressed(os.path.join(HERE, "solver_cases.npz"), **arrays)
    np.savez_compressed(os.path.join(HERE, "kernel_cases.npz"), **kern)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("wrote", len(arrays), "solver arrays,", len(kern), "kernel arrays")


if __name__ == "__main__":
    main()
