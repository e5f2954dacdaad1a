"""Per-GPU trip time at the shard sizes of a G-rank column-sharded c4 job, measured on ONE GPU.

A rank of a G-rank job holds K/G = 262144/G columns of the 8192-row fp32 dictionary and runs the
same trip graph (phase kernels + one all-reduce per trip) on them.  This script runs, for
G = 1, 2, 4, 8, a c4-shaped problem with K/G columns through the sharded path with a one-rank
NCCL group (trip graph, one SUM all-reduce per trip -- at one rank the all-reduce is a copy, so
its NVLink time is NOT in these numbers) for a fixed number of iterations and prints the device
time per trip next to the K1 stream time at the measured copy bandwidth.  It is a model of the
per-rank work, not a multi-GPU measurement: the solve trajectory of a K/G-column problem differs
from a shard of the K-column one, only the shapes (columns per rank, support fraction) match.

    python scripts/shard_projection.py [iters]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import dist as pdist
from paper_1412_4080_b200 import workloads as wl

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29517")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
peak = 6549.0
pp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
if os.path.exists(pp):
    peak = float(json.load(open(pp)).get("hbm_gbs", peak))
rows = []
for G in (8, 4, 2, 1):
    k = 262144 // G
    w = wl.config4(k=k)
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="f32")
    L = ds.operator_norm(dic, tol=1e-8) ** 2 * (1 + 1e-6)
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3", max_iters=iters, rel_tol=1e-300,
                          L0=L, gap_tol=1e-300)
    prob = ds.Problem(dic, w.y, w.lam)
    shard = pdist.GpuShard(prob, cfg, 0, k)
    for _ in range(2):
        pdist.orchestrate(shard, cfg, w.lam, dist.group.WORLD, collectives=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sc = pdist.orchestrate(shard, cfg, w.lam, dist.group.WORLD, collectives=1)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / max(sc.trips, 1)
    k1_us = 8192 * k * 4 / (peak * 1e9) * 1e6
    rows.append((G, k, sc.t, sc.trips, us, k1_us))
    shard.close()
    dic.drop_device()
    del shard, prob, dic, w
    torch.cuda.empty_cache()
t1 = [r for r in rows if r[0] == 1][0][4]
print(f"# c4-shaped shards on one B200, sharded path (trip graph, 1 SUM all-reduce per trip, 1-rank NCCL group), {iters} iterations")
print(f"# {'G':>2s} {'cols/rank':>9s} {'trips':>6s} {'us/trip':>9s} {'K1 stream @%.0f GB/s' % peak:>22s} {'overhead us':>12s} {'compute-only speed-up':>22s} {'efficiency':>10s}")
for G, k, t, trips, us, k1 in sorted(rows):
    print(f"  {G:2d} {k:9d} {trips:6d} {us:9.1f} {k1:22.1f} {us - k1:12.1f} {t1 / us:22.2f} {t1 / us / G:10.2f}")
print("# 'compute-only speed-up' = us/trip at G = 1 over us/trip at K/G columns; a real G-rank trip adds the NVLink all-reduce of")
print("# 2 x 8192 fp64 + scalars (128 KB) per trip, which one GPU cannot time")
dist.destroy_process_group()
