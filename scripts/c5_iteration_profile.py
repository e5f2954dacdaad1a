"""Per-iteration kernel times of one c5 batched solve (direct launches, events): python scripts/c5_iteration_profile.py"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import _native as nat  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.batched import BatchedEngine  # noqa: E402

w = wl.config5()
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
L = ds.operator_norm(dic, tol=1e-11, max_iters=20000) ** 2 * (1 + 1e-6)
e = BatchedEngine(dic, w.y, w.lam, L, iterations=100, test="dst3")
e.setup()
rows = []
for t in range(100):
    ms = (C.c_float * 3)()
    nat.check(e.L.dscr_batched_profile(e.h, t, e.sptr, ms))
    rows.append(list(ms) + [float(e._view(e.bufs.kept, e.b, torch.int32).sum().item())])
    if "--scan" in sys.argv:
        cbuf = e._view(e.bufs.C, 3, torch.float32)
        if t < 40:
            print("t", t, "scan range/passes/scans", cbuf.cpu().numpy().tolist())
        cbuf.zero_()
rows = np.array(rows)
kept = e._view(e.bufs.kept, e.b, torch.int32).cpu().numpy()
print("total ms", rows[:, :3].sum(0), "sum", rows[:, :3].sum())
for t in list(range(0, 10)) + list(range(10, 100, 10)):
    print(t, np.round(rows[t, :3] * 1e3, 1))
print("kept min/mean", kept.min(), kept.mean())
print("update us t=0..40:", np.round(rows[:41, 1] * 1e3, 0).astype(int).tolist())
print("screened per iteration t=1..40:", (-np.diff(rows[:41, 3])).astype(np.int64).tolist())
