"""Distribution of the per-observation support-list lengths of a c5 solve after t iterations
(direct launches): python scripts/c5_support_hist.py [t]"""
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
for t in range(100):
    ms = (C.c_float * 3)()
    nat.check(e.L.dscr_batched_profile(e.h, t, e.sptr, ms))
    if t in (1, 5, 20, 50, 99):
        for par in (0, 1):
            cnt = e._view(e.bufs.s_cnt[par], e.b, torch.int32).cpu().numpy()
            q = np.percentile(cnt, [0, 50, 90, 99, 100])
            print(f"t={t} list[{par}] support len: mean {cnt.mean():.1f} pct(0,50,90,99,100) {q}")
