"""Loader for the reference-generated golden fixtures (tests/golden/)."""

import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(HERE, "manifest.json")) as fh:
        manifest = json.load(fh)
    arr = np.load(os.path.join(HERE, "solver_cases.npz"))
    cases = []
    for pi, entry in enumerate(manifest):
        pre = f"p{pi}__"
        D = arr[pre + "D"]
        y = arr[pre + "y"]
        groups = weights = snorms = None
        if entry["kind"] == "group":
            gof = arr[pre + "group_of"]
            groups = [np.flatnonzero(gof == g) for g in range(int(gof.max()) + 1)]
            weights = arr[pre + "weights"]
            snorms = arr[pre + "snorms"]
        for ci, c in enumerate(entry["configs"]):
            key = f"{pre}c{ci}__"
            out = {f: arr[key + f] for f in ("x_star", "eliminated", "objective", "kept", "nnz",
                                              "flops", "gap")}
            out["iterations"] = c["iterations"]
            out["final_objective"] = c["final_objective"]
            cases.append(dict(pid=pi, name=entry["name"], kind=entry["kind"], D=D, y=y,
                              lam=entry["lam"], groups=groups, weights=weights, snorms=snorms,
                              cfg=c["cfg"], ref=out, lmax=entry["lmax"],
                              lmax_index=entry["lmax_index"], lmax_group=entry["lmax_group"],
                              spec_L=entry["spec_L"], op_norm=entry["op_norm"]))
    return cases


def kernel_cases():
    return np.load(os.path.join(HERE, "kernel_cases.npz"))
