"""Digest fixtures from the reference's problem_digest (instrument.py:60-71).

Run in the build container (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_digest_golden.py
"""
import json
import os

import numpy as np

from screenlab.dictionary import Dictionary, GroupPartition
from screenlab.instrument import problem_digest
from screenlab.problems import Problem

out = []
for seed, (n, k, lam, grouped) in enumerate([(20, 50, 0.3, False), (30, 60, 0.1, True), (7, 9, 0.5, False)]):
    rng = np.random.default_rng(100 + seed)
    D = rng.standard_normal((n, k))
    D /= np.linalg.norm(D, axis=0)
    y = rng.standard_normal(n)
    y /= np.linalg.norm(y)
    part = None
    if grouped:
        part = GroupPartition.build(Dictionary(D), [np.arange(g, g + 5) for g in range(0, k, 5)])
    out.append({"seed": seed, "n": n, "k": k, "lam": lam, "grouped": grouped,
                "digest": problem_digest(Problem(Dictionary(D), y, lam, part))})
with open(os.path.join(os.path.dirname(__file__), "digest_cases.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(out)
