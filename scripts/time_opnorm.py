"""Time operator_norm (||D||_2 by block power iteration) on a BASELINE workload: python scripts/time_opnorm.py c3|c4"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = {"c1": wl.config1, "c3": wl.config3, "c4": wl.config4, "c5": wl.config5}[name]()
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype=w.dtype)
dic.device_data(torch.device("cuda", 0))
for tol, its in ((1e-10, 5000), (1e-11, 20000)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nrm = ds.operator_norm(dic, tol=tol, max_iters=its)
    torch.cuda.synchronize()
    print(f"{name} operator_norm tol {tol:g}: {1e3 * (time.perf_counter() - t0):.1f} ms -> {nrm:.15f}", flush=True)
