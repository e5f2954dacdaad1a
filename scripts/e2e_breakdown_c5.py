"""Where the end-to-end time of one c5 solve_batched call goes (host timers, synchronised)."""
import time
import numpy as np
import torch
import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import workloads as wl
from paper_1412_4080_b200.batched import BatchedEngine

w = wl.config5()
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
nrm = ds.operator_norm(dic, tol=1e-11, max_iters=20000)
L = nrm * nrm * (1.0 + 1e-6)


def tick(t, name, out):
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out.append((name, (t2 - t) * 1e3))
    return t2


for rep in range(3):
    out = []
    t = time.perf_counter()
    dic.drop_device()
    dic.device_data(torch.device("cuda", 0))
    t = tick(t, "D upload", out)
    e = BatchedEngine(dic, w.y, w.lam, L, iterations=100, test="dst3")
    t = tick(t, "engine (Y transpose+upload, workspace, create)", out)
    e.setup()
    t = tick(t, "setup kernels", out)
    e.run()
    t = tick(t, "run (capture+instantiate+100 iterations)", out)
    r = e.result()
    t = tick(t, "result D2H + lists", out)
    e.close()
    t = tick(t, "close", out)
    print(rep, " | ".join(f"{n}: {v:.1f} ms" for n, v in out))
