"""Fused GEMM time of the first iterations of a c5 solve (dscr_batched_profile), for experiments."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import _native as nat  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.batched import BatchedEngine  # noqa: E402

w = wl.config5()
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
L = ds.operator_norm(dic, tol=1e-10) ** 2 * (1 + 1e-6)
e = BatchedEngine(dic, w.y, w.lam, L, iterations=100, test="dst3")
e.setup()
out = []
for t in range(6):
    ms = (C.c_float * 3)()
    e.L.dscr_batched_profile(e.h, t, e.sptr, ms)
    out.append(round(ms[0] * 1e3, 1))
print("GEMM us per iteration:", out)
