"""Where the end-to-end time of c5 solve_batched calls goes (pinned inputs, host timers, synchronised)."""
import time

import torch

import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import workloads as wl
from paper_1412_4080_b200.batched import BatchedEngine

w = wl.config5()
host_d = torch.empty((w.D.shape[1], w.D.shape[0]), dtype=torch.uint16, pin_memory=True)
host_d.numpy()[:] = w.D.T
host_y = torch.empty((w.y.shape[1], w.y.shape[0]), dtype=torch.float64, pin_memory=True)
host_y.numpy()[:] = w.y.T
dic = ds.Dictionary(host_d.numpy().T, check_unit_norms=False, dtype="bf16")
dic._host_tensor = host_d
L = ds.operator_norm(dic, tol=1e-11, max_iters=20000) ** 2 * (1 + 1e-6)


def tick(t, name, out):
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out.append((name, (t2 - t) * 1e3))
    return t2


for rep in range(10):
    out = []
    t = time.perf_counter()
    dic.drop_device()
    dic.device_data(torch.device("cuda", 0))
    t = tick(t, "D", out)
    e = BatchedEngine(dic, host_y.T, w.lam, L, iterations=100, test="dst3")
    t = tick(t, "engine", out)
    e.setup()
    t = tick(t, "setup", out)
    e.run()
    t = tick(t, "run", out)
    r = e.result()
    t = tick(t, "result", out)
    e.close()
    t = tick(t, "close", out)
    print(rep, f"total {sum(v for _, v in out):.1f} ms |", " | ".join(f"{n} {v:.1f}" for n, v in out), flush=True)
