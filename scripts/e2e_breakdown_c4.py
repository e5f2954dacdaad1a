"""Where the end-to-end time of one c4 ds.run call goes (host timers, synchronised)."""
import sys
import time
import types

import torch

import bench
import paper_1412_4080_b200 as ds
from paper_1412_4080_b200.solver import Engine, _solve

args = types.SimpleNamespace(workload="c4", seed=0)
works = bench.build_workload("c4", 0, pinned=True)
problems = bench.make_problems(ds, works)
dev = torch.device("cuda", 0)


def tick(t, name, out):
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out.append((name, (t2 - t) * 1e3))
    return t2


for rep in range(3):
    for p, c in problems:
        out = []
        t = time.perf_counter()
        p.dictionary.drop_device()
        p.dictionary.__dict__.pop("_problem_cache", None)
        t = tick(t, "drop", out)
        eng = Engine(p, c, device=dev)
        t = tick(t, "Engine() incl. D upload", out)
        r = _solve(eng, p, c, None)
        t = tick(t, "solve+result", out)
        eng.close()
        t = tick(t, "close", out)
        print(rep, r.iterations, f"device {r.device_seconds * 1e3:.1f} ms |",
              " | ".join(f"{n}: {v:.1f} ms" for n, v in out), flush=True)
