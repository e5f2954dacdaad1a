import sys, numpy as np
sys.path.insert(0, '.')
import paper_1412_4080_b200 as ds
from tests.golden_cases import load
from tests.test_gpu_parity import _cached_problem, _cfg
CASES = load()
for idx in map(int, sys.argv[1:]):
    c = CASES[idx]; ref = c["ref"]
    res = ds.run(_cached_problem(c), _cfg(c))
    print(idx, c["name"], c["cfg"], "iters", res.iterations, ref["iterations"], res.stop_reason)
    g1, g2 = np.array(res.trace.gap), ref["gap"]
    o1, o2 = np.array(res.trace.objective), ref["objective"]
    m = min(len(g1), len(g2))
    for t in list(range(0, m, max(1, m // 12))) + [m - 1]:
        print(f"  t={t+1:4d} gap {g1[t]: .6e} {g2[t]: .6e}  obj {o1[t]:.15e} {o2[t]:.15e}  L {res.trace.L[t]}")
    print("  min gaps", g1.min(), g2.min())
