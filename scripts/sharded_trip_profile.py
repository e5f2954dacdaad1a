"""Per-phase device time of a column-sharded trip at one rank (events around each phase, host
loop), c4 or a smaller c4-shaped problem: python scripts/sharded_trip_profile.py [k] [trips]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import _native as nat
from paper_1412_4080_b200 import dist as pdist
from paper_1412_4080_b200 import workloads as wl

k = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
trips = int(sys.argv[2]) if len(sys.argv) > 2 else 30
w = wl.config4(k=k)
dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="f32")
L = ds.operator_norm(dic, tol=1e-10) ** 2 * (1 + 1e-6)
cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=10000, rel_tol=1e-300, L0=L,
                      gap_tol=1e-5)
prob = ds.Problem(dic, w.y, w.lam)
for mode in (1, 2):
    shard = pdist.GpuShard(prob, cfg, 0, k)
    shard.set_collectives(0, 1, mode == 1)
    for ph in (nat.PH_SETUP_LOCAL,):
        shard.phase(ph)
    # lambda_* adoption exactly as orchestrate does at one rank
    comm = shard.comm
    cand = comm[nat.CM_SETUP: nat.CM_SETUP + 3].cpu().numpy()
    lmax, gidx, sign = float(cand[0]), int(cand[1]), float(cand[2])
    comm[nat.CM_SETUP: nat.CM_SETUP + 7] = torch.tensor([lmax, gidx, sign, 0.0, 1.0, 0.0, gidx], dtype=comm.dtype,
                                                        device=comm.device)
    shard.phase(nat.PH_SETUP_ADOPT)
    shard.phase(nat.PH_SETUP_VEC)
    shard.phase(nat.PH_SETUP_FINISH)
    seq = ([nat.PH_K1, nat.PH_K2S, nat.PH_K3A, nat.PH_K3S, nat.PH_K1R1, nat.PH_K2C, nat.PH_K3B] if mode == 1 else
           [nat.PH_K1, nat.PH_K1R, nat.PH_K2, nat.PH_K3A, nat.PH_K3S, nat.PH_K3B])
    names = {v: n for n, v in vars(nat).items() if n.startswith("PH_") and isinstance(v, int)}
    acc = {ph: [] for ph in seq}
    s = torch.cuda.current_stream()
    for t in range(trips):
        for ph in seq:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            shard.phase(ph)
            e1.record(s)
            e1.synchronize()
            acc[ph].append(e0.elapsed_time(e1) * 1e3)
    print(f"collectives={mode}: median us per phase over trips 5..{trips}:",
          {names[ph]: round(float(np.median(v[5:])), 1) for ph, v in acc.items()},
          "sum", round(sum(float(np.median(v[5:])) for v in acc.values()), 1))
    shard.close()
