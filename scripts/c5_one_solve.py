"""One c5 batched solve (setup + the 100-iteration graph), for an ncu launch list:
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file out.csv python scripts/c5_one_solve.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.batched import BatchedEngine  # noqa: E402

w = wl.config5()
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
L = ds.operator_norm(dic, tol=1e-11, max_iters=20000) ** 2 * (1 + 1e-6)
e = BatchedEngine(dic, w.y, w.lam, L, iterations=100, test="dst3")
torch.cuda.synchronize()
print("MARK setup")
e.setup()
torch.cuda.synchronize()
e.run()
torch.cuda.synchronize()
res = e.result()
print("kept min", int(res.kept.min()), "objective sum", float(res.objective.sum()))
