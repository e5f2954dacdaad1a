"""In-graph per-kernel timing of one solve from the engine's %globaltimer stamps.

    python scripts/timing_breakdown.py c1|c2|c3|c4|c4proxy
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.solver import Engine  # noqa: E402


def workload(name):
    if name == "c1":
        return wl.config1()
    if name == "c2":
        return wl.config2(ratio=0.1)
    if name == "c2r5":
        return wl.config2(ratio=0.5)
    if name == "c3":
        return wl.config3()
    if name == "c4":
        return wl.config4()
    D = wl.gaussian_dictionary_f32(1024, 32768, 0)
    y = wl.gaussian_observation(1024, 0)
    lam = 0.2 * float(np.max(np.abs(D.astype(np.float64).T @ y)))
    return wl.Workload("c4proxy", D, y, lam, algorithm="fista", test="dst3", gap_tol=1e-5, dtype="f32")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    w = workload(name)
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype=w.dtype)
    part = ds.GroupPartition.build(dic, w.groups) if w.groups else None
    L = ds.operator_norm(dic, tol=1e-11) ** 2 * (1 + 1e-6)
    cfg = ds.SolverConfig(algorithm=w.algorithm, strategy="dynamic", test=w.test, max_iters=w.max_iters,
                          rel_tol=1e-300, L0=L, gap_tol=w.gap_tol)
    prob = ds.Problem(dic, w.y, w.lam, part)
    for rep in range(3):
        eng = Engine(prob, cfg)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        eng.setup()
        ev1.record()
        eng.launch(0)
        ev2 = torch.cuda.Event(enable_timing=True)
        ev2.record()
        sc = eng.scalars()
        b = eng.bufs
        trips = min(sc.trips, b.max_kts)
        ts = eng.view(b.kts, trips * 8, torch.int64).cpu().numpy().reshape(trips, 8).astype(np.float64)
        rows = eng.trace_rows(sc.t)
        eng.close()
    t = sc.t
    setup_ms = ev0.elapsed_time(ev1)
    loop_ms = ev1.elapsed_time(ev2)
    d = ts[1:]           # skip the first trip
    nxt = ts[2:, 0]
    cols = {
        "K1": d[:, 1] - d[:, 0], "K1->K2 gap": d[:, 2] - d[:, 1], "K2": d[:, 3] - d[:, 2],
        "K2->K3a gap": d[:, 4] - d[:, 3], "K3a(+gap)": d[:, 6] - d[:, 4], "K3b": d[:, 7] - d[:, 6],
        "K3b->next K1": np.concatenate([nxt - d[:-1, 7], [np.nan]]),
    }
    print(f"{name}: {t} iterations, {sc.trips} trips, setup {setup_ms:.3f} ms, loop {loop_ms:.3f} ms "
          f"= {1e3 * loop_ms / max(t, 1):.2f} us/iteration")
    for k, v in cols.items():
        print(f"  {k:14s} median {np.nanmedian(v) / 1e3:8.2f} us   mean {np.nanmean(v) / 1e3:8.2f} us")
    from paper_1412_4080_b200 import _native as nat  # noqa: E402
    sup = rows[:, nat.TR_SUPPORT].astype(np.float64)
    elem = {"f64": 8, "f32": 4, "bf16": 2}[w.dtype]
    k3a = (d[:, 6] - d[:, 4]) / 1e9
    print(f"  support (x or u nonzero) median {np.median(sup):.0f}, final nnz {int(rows[-1, nat.TR_NNZ])}, "
          f"kept {int(rows[-1, nat.TR_KEPT])}; K3a reads {np.median(sup) * w.D.shape[0] * elem / 1e6:.1f} MB "
          f"-> {np.median(sup[1:len(k3a) + 1] * w.D.shape[0] * elem / k3a) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
