"""Time GroupPartition.build (group spectral norms) and operator_norm on c3."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402

w = wl.config3()
dic = ds.Dictionary(w.D, check_unit_norms=False)
ds.operator_norm(dic)
torch.cuda.synchronize()
t0 = time.perf_counter()
nrm = ds.operator_norm(dic)
torch.cuda.synchronize()
t1 = time.perf_counter()
part = ds.GroupPartition.build(dic, w.groups)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"operator_norm {1e3 * (t1 - t0):.1f} ms ({nrm:.12f}); GroupPartition.build {1e3 * (t2 - t1):.1f} ms "
      f"for {len(w.groups)} groups; norms[:3] {part.spectral_norms[:3]}")
