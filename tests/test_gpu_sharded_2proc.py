"""Column sharding with two real processes (gloo, both on cuda:0) and the CUDA phase kernels.

The kernels of the two ranks never wait on one another: every exchange is a host-side
torch.distributed collective between phases, so two processes sharing one GPU are a valid
test of the multi-rank orchestration (lambda_* argmax across ranks, owner broadcast, the MAX
and SUM exchanges, REDO/FIXUP control) with the production kernels.  NCCL itself needs one
GPU per rank and is covered at world size 1 in test_gpu_sharded.py."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [("fista", "dst3", 0.5, "lasso", 2), ("ista-bt", "dst3", 0.7, "lasso", 2),
         ("fista", "static-dst3", 0.8, "lasso", 2), ("fista", "gst3", 0.7, "group", 2),
         # one collective per trip (rank-slot gather in the SUM, FIXUP on a screened nonzero)
         ("fista", "dst3", 0.5, "lasso", 1), ("ista-bt", "dst3", 0.7, "lasso", 1), ("fista", "gst3", 0.7, "group", 1),
         ("sparsa", "dst3", 0.6, "lasso", 1)]


def _build(case):
    import paper_1412_4080_b200 as ds
    from paper_1412_4080_b200 import workloads as wl
    algo, test, ratio, kind = case[:4]
    if kind == "group":
        w = wl.config3(ratio=ratio, n=300, k=1200)
        dic = ds.Dictionary(w.D)
        part = ds.GroupPartition.build(dic, w.groups)
        p = ds.Problem(dic, w.y, w.lam, part)
    else:
        D = wl.correlated_dictionary(200, 2000, 5)
        y, _ = wl.planted_observation(D, 5, nnz=10)
        p = ds.Problem(ds.Dictionary(D), y, ratio * wl.lambda_star(D, y))
    strategy = "static" if test.startswith("static") else "dynamic"
    L0 = 1.0 if algo == "ista-bt" else None
    kw = {} if L0 is None else {"L0": L0}
    if L0 is None:
        kw["L0"] = float(np.linalg.norm(p.dictionary.as_float64(), 2) ** 2 * (1 + 1e-6))
    cfg = ds.SolverConfig(algorithm="ista" if algo == "ista-bt" else algo, strategy=strategy,
                          test=test.replace("static-", ""), max_iters=400, rel_tol=1e-9, **kw)
    return p, cfg


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    from paper_1412_4080_b200 import dist as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        p, cfg = _build(case)
        res = pdist.run_sharded(p, cfg, pg=dist.group.WORLD, device=torch.device("cuda", 0),
                                collectives=case[4])
        if rank == 0:
            q.put(("ok", res.iterations, res.x_star, np.asarray(res.screen_state.eliminated), res.final_objective,
                   list(res.trace.kept)))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put(("error", rank, repr(e)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", CASES, ids=["-".join(map(str, c[:3])) + f"-{c[4]}coll" for c in CASES])
def test_two_ranks_match_unsharded(case, monkeypatch):
    import paper_1412_4080_b200 as ds
    monkeypatch.setenv("DSCR_F23", "0")   # unsharded reference: K2 builds the support list (same order)
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    try:
        msg = q.get(timeout=240)
    finally:
        for pr in procs:
            pr.join(timeout=60)
            if pr.is_alive():
                pr.kill()
    assert msg[0] == "ok", msg
    _, iters, x, elim, obj, kept = msg
    p, cfg = _build(case)
    ref = ds.run(p, cfg)
    assert iters == ref.iterations
    assert np.array_equal(elim, np.asarray(ref.screen_state.eliminated))
    np.testing.assert_allclose(x, ref.x_star, rtol=1e-9, atol=1e-12)
    assert obj == pytest.approx(ref.final_objective, rel=1e-12)
    assert kept == list(ref.trace.kept)
