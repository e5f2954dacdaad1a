"""Column-sharded orchestration (paper_1412_4080_b200.dist) on CPU with gloo, world_size 2.

Each rank runs the numpy phase backend on its column block; the collective
sequence, the cross-rank lambda_* argmax, the owner broadcast and the
stop / backtracking-redo / fixup control are the production code paths.  The
sharded result must match the unsharded CPU oracle (iterations, screened set,
x, objective).
"""

import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_4080_b200 import dist as pdist
from paper_1412_4080_b200 import workloads as wl
from oracle import screen_oracle as so

CASES = [
    # (algorithm, test, ratio, L0 mode, gap_tol)
    ("fista", "dst3", 0.5, "spec", 1e-9),
    ("fista", "safe", 0.9, "spec", 1e-9),
    ("ista", "dst3", 0.7, "spec", 1e-8),
    ("ista", "dst3", 0.6, "one", 1e-8),      # backtracking REDO trips from L0 = 1
    ("fista", "dst3", 0.8, "one", 1e-9),
    ("sparsa", "dst3", 0.7, "spec", 1e-9),
    ("cp", "safe", 0.7, "spec", 1e-9),
    ("fista", "dst3", 1.5, "spec", 1e-9),    # trivial regime: lam > lambda_*
]


def _data(ratio):
    D = wl.correlated_dictionary(60, 301, 3)
    y, _ = wl.planted_observation(D, 3, nnz=6)
    return D, y, ratio * wl.lambda_star(D, y)


def _cfg(algo, test, L0mode, gap_tol, D):
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9)) if L0mode == "spec" else 1.0
    return so.Config(algorithm=algo, strategy="dynamic", test=test, max_iters=3000, rel_tol=1e-300, L0=L,
                     gap_tol=gap_tol, op_norm=float(np.linalg.norm(D, 2)))


def _worker(rank, world, port, out_path, case, collectives=2):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.sharded_numpy_backend import NumpyShard
        algo, test, ratio, L0mode, gap_tol = case
        D, y, lam = _data(ratio)
        cfg = _cfg(algo, test, L0mode, gap_tol, D)
        c0, c1 = pdist.shard_ranges(D.shape[1], world)[rank]
        shard = NumpyShard(D[:, c0:c1], y, lam, cfg, c0, op_norm=cfg.op_norm)
        sc = pdist.orchestrate(shard, cfg, lam, pg=dist.group.WORLD, chunk=3, collectives=collectives)
        if sc.trivial:
            local = (np.empty(0, np.int64), np.empty(0))
        else:
            local = (shard.active + c0, shard.x[shard.active])
        got = [None] * world
        dist.all_gather_object(got, (local, shard.trace, int(sc.t), bool(sc.trivial)))
        if rank == 0:
            with open(out_path, "wb") as fh:
                pickle.dump(got, fh)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("collectives", [2, 1], ids=["two-collectives", "one-collective"])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-{c[2]}-{c[3]}" for c in CASES])
def test_sharded_world2_matches_oracle(case, collectives):
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "res.pkl")
        mp.spawn(_worker, args=(2, _free_port(), out, case, collectives), nprocs=2, join=True)
        with open(out, "rb") as fh:
            got = pickle.load(fh)
    algo, test, ratio, L0mode, gap_tol = case
    D, y, lam = _data(ratio)
    ref = so.solve(so.make_problem(D, y, lam), _cfg(algo, test, L0mode, gap_tol, D))
    traces = [g[1] for g in got]
    if collectives in (1, "peer"):   # kept counts are per rank in one-collective trips (summed by the host)
        assert [t[:1] + t[2:] for t in traces[0]] == [t[:1] + t[2:] for t in traces[1]], "ranks disagree"
        traces = [[(a[0], a[1] + b[1]) + a[2:] for a, b in zip(traces[0], traces[1])]] * 2
    assert traces[0] == traces[1], "ranks disagree on the trace"
    its = got[0][2]
    assert its == ref.iterations
    if got[0][3]:
        assert ref.iterations == 0
        return
    kept = np.concatenate([g[0][0] for g in got])
    xs = np.concatenate([g[0][1] for g in got])
    x = np.zeros(D.shape[1])
    x[kept] = xs
    elim = np.setdiff1d(np.arange(D.shape[1]), kept)
    assert np.array_equal(elim, ref.eliminated)
    assert np.linalg.norm(x - ref.x_star) <= 1e-9 * max(1.0, np.linalg.norm(ref.x_star))
    np.testing.assert_allclose([t[3] for t in traces[0]], ref.trace["objective"], rtol=1e-10)
    assert [t[1] for t in traces[0]] == ref.trace["kept"]


@pytest.mark.parametrize("case", [CASES[0], CASES[3], CASES[5]], ids=["fista-dst3", "ista-backtracking", "sparsa"])
def test_sharded_world2_peer_exchange_phases(case):
    """The peer-memory exchange phase order (K3S; K3X_PUSH; K3X_REDUCE; K1R1) with the host
    mirror of the device exchange: same result as the oracle."""
    test_sharded_world2_matches_oracle(case, "peer")


def test_shard_ranges_cover_and_keep_groups_whole():
    assert pdist.shard_ranges(10, 3) == [(0, 3), (3, 7), (7, 10)]
    sizes = np.array([3, 3, 4, 2, 5, 3])
    cols, grps = pdist.shard_ranges(int(sizes.sum()), 3, sizes)
    assert cols[0][0] == 0 and cols[-1][1] == sizes.sum()
    ptr = np.concatenate(([0], np.cumsum(sizes)))
    for (c0, c1), (g0, g1) in zip(cols, grps):
        assert c0 == ptr[g0] and c1 == ptr[g1]
    for a, b in zip(cols, cols[1:]):
        assert a[1] == b[0]


def test_shard_ranges_one_group_per_rank_and_limits():
    sizes = np.array([70, 10, 10, 10])          # searchsorted by atom count would give rank 1 nothing
    cols, grps = pdist.shard_ranges(100, 4, sizes)
    assert grps == [(0, 1), (1, 2), (2, 3), (3, 4)]
    assert all(c1 > c0 for c0, c1 in cols)
    cols, grps = pdist.shard_ranges(100, 2, sizes)
    assert grps[0][1] > grps[0][0] and grps[1][1] > grps[1][0] and grps[1][1] == 4
    for world in (3, 5, 7, 8):
        sizes = np.array([1] * 3 + [50] + [1] * 5)
        cols, grps = pdist.shard_ranges(int(sizes.sum()), world, sizes)
        assert [g[1] - g[0] >= 1 for g in grps] == [True] * world
        assert grps[0][0] == 0 and grps[-1][1] == sizes.size
        assert all(a[1] == b[0] for a, b in zip(grps, grps[1:]))
    with pytest.raises(ValueError, match="groups over"):
        pdist.shard_ranges(100, 5, np.array([70, 10, 10, 10]))
    with pytest.raises(ValueError, match="columns over"):
        pdist.shard_ranges(3, 4)


def _one_rank_data(ratio=0.4):
    """A correlated dictionary with its columns reordered so that every atom the oracle screens
    sits in the last block: with the uneven ranges below, only rank 3 ever screens."""
    D0 = wl.correlated_dictionary(60, 120, 5)
    y, _ = wl.planted_observation(D0, 5, nnz=5)
    lam = ratio * wl.lambda_star(D0, y)
    L = float(np.linalg.norm(D0, 2) ** 2 * (1 + 1e-9))
    r = so.solve(so.make_problem(D0, y, lam), so.Config(algorithm="fista", strategy="dynamic", test="dst3",
                                                         max_iters=3000, rel_tol=1e-300, L0=L, gap_tol=1e-9))
    elim = np.asarray(r.eliminated)
    perm = np.concatenate([np.setdiff1d(np.arange(120), elim), elim])
    return np.asfortranarray(D0[:, perm]), y, lam, 120 - elim.size


def _uneven(n_kept):
    """Blocks of 7 / n_kept-17 / 10 kept atoms, then every screened atom on rank 3."""
    return [(0, 7), (7, n_kept - 10), (n_kept - 10, n_kept), (n_kept, 120)]


def _worker_uneven(rank, world, port, out_path, algo, collectives):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.sharded_numpy_backend import NumpyShard
        D, y, lam, n_kept = _one_rank_data()
        cfg = _cfg(algo, "dst3", "spec", 1e-9, D)
        c0, c1 = _uneven(n_kept)[rank]
        shard = NumpyShard(D[:, c0:c1], y, lam, cfg, c0, op_norm=cfg.op_norm)
        sc = pdist.orchestrate(shard, cfg, lam, pg=dist.group.WORLD, chunk=4, collectives=collectives)
        local = (shard.active + c0, shard.x[shard.active], c1 - c0 - shard.active.size)
        got = [None] * world
        dist.all_gather_object(got, (local, shard.trace, int(sc.t)))
        if rank == 0:
            with open(out_path, "wb") as fh:
                pickle.dump(got, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("collectives", [2, 1], ids=["two-collectives", "one-collective"])
@pytest.mark.parametrize("algo", ["fista", "ista"])
def test_sharded_world4_uneven_screening_on_one_rank(algo, collectives):
    """World 4 (gloo) with uneven column blocks; screening fires on
    rank 3 only, so the ranks' active lists shrink at different rates while the control path
    (radius, stop, redo/fixup) stays identical on every rank."""
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "res.pkl")
        mp.spawn(_worker_uneven, args=(4, _free_port(), out, algo, collectives), nprocs=4, join=True)
        with open(out, "rb") as fh:
            got = pickle.load(fh)
    D, y, lam, n_kept = _one_rank_data()
    assert [c1 - c0 for c0, c1 in _uneven(n_kept)] != [D.shape[1] // 4] * 4
    ref = so.solve(so.make_problem(D, y, lam), _cfg(algo, "dst3", "spec", 1e-9, D))
    screened = [g[0][2] for g in got]
    assert screened[:3] == [0, 0, 0] and screened[3] > 0, screened
    assert len({g[2] for g in got}) == 1 and got[0][2] == ref.iterations
    kept = np.concatenate([g[0][0] for g in got])
    x = np.zeros(D.shape[1])
    x[kept] = np.concatenate([g[0][1] for g in got])
    assert np.array_equal(np.setdiff1d(np.arange(D.shape[1]), kept), ref.eliminated)
    assert np.linalg.norm(x - ref.x_star) <= 1e-9 * max(1.0, np.linalg.norm(ref.x_star))
    objs = [[t[3] for t in g[1]] for g in got]
    assert all(o == objs[0] for o in objs), "ranks disagree on the objective trace"
    np.testing.assert_allclose(objs[0], ref.trace["objective"], rtol=1e-10)
