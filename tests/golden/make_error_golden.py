"""Record the REFERENCE's outcome on the error-path inputs of tests/error_cases.py.

Build container only:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_error_golden.py
"""
import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import screenlab as sl  # noqa: E402

from tests.error_cases import CASES  # noqa: E402

out = {}
for name, build in CASES:
    c = build()
    dic = sl.Dictionary(c["D"], check_unit_norms=c["check_unit_norms"])
    part = sl.GroupPartition.build(dic, c["groups"], weights=c["weights"]) if c["groups"] is not None else None
    rec = {}
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = sl.run(sl.Problem(dic, c["y"], c["lam"], part), sl.SolverConfig(**c["cfg"]))
        rec = {"outcome": "ok", "iterations": r.iterations,
               "objective": [float(v) for v in r.trace.objective],
               "x_finite": bool(np.all(np.isfinite(r.x_star))),
               "x_absmax": float(np.max(np.abs(r.x_star)))}
    except Exception as e:  # noqa: BLE001  (recording which exception the reference raises)
        rec = {"outcome": type(e).__name__, "message": str(e)}
    out[name] = rec
    print(name, rec.get("outcome"), rec.get("message", rec.get("iterations")))
with open(os.path.join(HERE, "error_cases.json"), "w") as fh:
    json.dump(out, fh, indent=1)
