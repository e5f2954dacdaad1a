"""Two and four ranks of the native peer-memory exchange on ONE GPU, in lock step in one process.

The production kernels of every rank (K1 .. K3S, k3x_push, k3x_reduce, K1R1, K2C, K3B) run on the
same stream, phase by phase: rank 0's phase, then rank 1's, ...  All pushes precede all reduces, so
no kernel ever waits for another rank's flag (nothing spins; see the profiling guide on ranks
sharing a GPU) -- but the pushes store into the *other* ranks' receive areas, the flags carry the
device-side sequence numbers, the areas alternate by parity and the reduces sum the sections in
rank order, exactly as with one process per GPU over NVLink.  Reference: the unsharded engine."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import _native as nat  # noqa: E402
from paper_1412_4080_b200 import dist as pdist  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402


def _connect(shards):
    """dscr_peer_alloc per rank, every rank's base handed to every solver (same process: the
    pointers are used directly, no IPC handle exchange)."""
    L = shards[0].eng.L
    world = len(shards)
    bases = []
    for sh in shards:
        nbytes = int(L.dscr_peer_buffer_bytes(world, sh.ldd))
        own, hd = C.c_void_p(), (C.c_char * 64)()
        nat.check(L.dscr_peer_alloc(nbytes, C.byref(own), hd))
        bases.append(own)
    for r, sh in enumerate(shards):
        recv = (C.c_void_p * world)(*[b.value + 512 for b in bases])
        flags = (C.c_void_p * world)(*[b.value for b in bases])
        nat.check(L.dscr_solver_set_peers(sh.eng.h, r, world, recv, flags))
    return bases


def _lockstep(shards, cfg, lam, vec_tests=("dst3", "gst3"), group_weights=None):
    world = len(shards)
    for r, sh in enumerate(shards):
        sh.set_collectives(r, world, True)
    bases = _connect(shards)
    for sh in shards:
        sh.phase(nat.PH_SETUP_LOCAL)
    allc = np.stack([sh.comm[nat.CM_SETUP: nat.CM_SETUP + 3].cpu().numpy() for sh in shards])
    best = 0
    for r in range(1, world):         # max value, lowest global index on ties (problems.py:79)
        if allc[r, 0] > allc[best, 0] or (allc[r, 0] == allc[best, 0] and allc[r, 1] < allc[best, 1]):
            best = r
    lmax, gidx, sign = float(allc[best, 0]), int(allc[best, 1]), float(allc[best, 2])
    assert lam <= lmax
    w_star = float(group_weights[gidx]) if group_weights is not None else 0.0
    for r, sh in enumerate(shards):
        local_unit = gidx - sh.unit_offset if r == best else -1
        sh.comm[nat.CM_SETUP: nat.CM_SETUP + 7] = torch.tensor(
            [lmax, gidx, sign, 0.0, 1.0 if r == best else 0.0, w_star, local_unit], dtype=sh.comm.dtype).to(sh.comm.device)
        sh.phase(nat.PH_SETUP_ADOPT)
    if cfg.test in vec_tests:
        shards[best].phase(nat.PH_SETUP_VEC)
        for r, sh in enumerate(shards):
            if r != best:
                sh.vec.copy_(shards[best].vec)
    for sh in shards:
        sh.phase(nat.PH_SETUP_FINISH)
    seq = [nat.PH_K1, nat.PH_K2S, nat.PH_K3A, nat.PH_K3S, nat.PH_K3X_PUSH, nat.PH_K3X_REDUCE, nat.PH_K1R1, nat.PH_K2C,
           nat.PH_K3B]
    trips = 0
    while True:
        sc = [sh.scalars() for sh in shards]
        assert len({(s.stop, s.t, s.mode) for s in sc}) == 1, "ranks diverged"
        if sc[0].stop != nat.STOP_RUNNING or sc[0].t >= cfg.max_iters:
            break
        for _ in range(8):
            for ph in seq:
                for sh in shards:          # lock step: every rank's push before any rank's reduce
                    sh.phase(ph)
            trips += 1
    return bases, trips


@pytest.mark.parametrize("algo,ratio,cuts", [
    ("fista", 0.7, [(0, 384), (384, 1024)]),
    ("ista", 0.8, [(0, 384), (384, 1024)]),
    ("sparsa", 0.7, [(0, 384), (384, 1024)]),
    ("fista", 0.7, [(0, 100), (100, 384), (384, 900), (900, 1024)]),
], ids=["fista-2", "ista-2", "sparsa-2", "fista-4"])
def test_peer_exchange_lockstep_matches_unsharded(algo, ratio, cuts):
    n, k = 200, 1024
    D = wl.correlated_dictionary(n, k, 0)
    y, _ = wl.planted_observation(D, 0, nnz=10)
    lam = ratio * wl.lambda_star(D, y)
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm=algo, strategy="dynamic", test="dst3", max_iters=400, rel_tol=1e-300, L0=L,
                          gap_tol=1e-7)
    ref = ds.run(ds.Problem(ds.Dictionary(D), y, lam), cfg)
    assert ref.screen_state.eliminated.size > 0
    shards = [pdist.GpuShard(ds.Problem(ds.Dictionary(np.asfortranarray(D[:, c0:c1])), y, lam), cfg, c0, k)
              for c0, c1 in cuts]
    bases = []
    try:
        bases, trips = _lockstep(shards, cfg, lam)
        sols = [sh.local_solution() for sh in shards]
        sc = sols[0][3]
        assert sc.t == ref.iterations and trips >= ref.iterations
        kept = np.concatenate([s[0] + c0 for s, (c0, _) in zip(sols, cuts)])
        xs = np.concatenate([s[1] for s in sols])
        x = np.zeros(k)
        x[kept] = xs
        elim = np.setdiff1d(np.arange(k), kept)
        assert np.array_equal(elim, ref.screen_state.eliminated)
        assert np.linalg.norm(x - ref.x_star) <= 1e-9 * max(np.linalg.norm(ref.x_star), 1e-12)
        assert abs(float(sc.F) - ref.final_objective) <= 1e-12 * abs(ref.final_objective)
        # every rank reduced the same bits
        assert len({(float(s[3].F), float(s[3].gap)) for s in sols}) == 1
    finally:
        for sh in shards:
            sh.close()
        for b in bases:
            shards[0].eng.L.dscr_peer_free(b)


def test_group_peer_exchange_lockstep_matches_unsharded():
    """Group-Lasso, FISTA + dynamic GST3, two ranks holding whole groups (48 + 80 groups of 8)."""
    n, k, gs = 200, 1024, 8
    D = wl.correlated_dictionary(n, k, 1)
    groups = [np.arange(g, g + gs) for g in range(0, k, gs)]
    dic = ds.Dictionary(D)
    part = ds.GroupPartition.build(dic, groups)
    rng = np.random.default_rng(5)
    x0 = np.zeros(k)
    for g in rng.choice(len(groups), 4, replace=False):
        x0[groups[g]] = rng.standard_normal(gs)
    y = D @ x0 + 0.01 * rng.standard_normal(n)
    y /= np.linalg.norm(y)
    lmax = max(np.linalg.norm(D[:, g].T @ y) / part.weights[i] for i, g in enumerate(groups))
    lam = 0.7 * lmax
    L = float(np.linalg.norm(D, 2) ** 2 * (1 + 1e-9))
    cfg = ds.SolverConfig(algorithm="fista", strategy="dynamic", test="gst3", max_iters=400, rel_tol=1e-300, L0=L,
                          gap_tol=1e-7)
    ref = ds.run(ds.Problem(dic, y, lam, part), cfg)
    assert ref.screen_state.eliminated.size > 0
    gcuts = [(0, 48), (48, len(groups))]
    shards = []
    for g0, g1 in gcuts:
        c0, c1 = g0 * gs, g1 * gs
        sub = ds.Dictionary(np.asfortranarray(D[:, c0:c1]))
        lp = ds.GroupPartition.build(sub, [g - c0 for g in groups[g0:g1]], weights=part.weights[g0:g1],
                                     spectral_norms=part.spectral_norms[g0:g1])
        shards.append(pdist.GpuShard(ds.Problem(sub, y, lam, lp), cfg, c0, k, g0, len(groups)))
    bases = []
    try:
        bases, trips = _lockstep(shards, cfg, lam, group_weights=np.asarray(part.weights))
        sols = [sh.local_solution() for sh in shards]
        sc = sols[0][3]
        assert sc.t == ref.iterations
        kept = np.concatenate([s[0] + g0 * gs for s, (g0, _) in zip(sols, gcuts)])
        xs = np.concatenate([s[1] for s in sols])
        x = np.zeros(k)
        x[kept] = xs
        assert np.array_equal(np.setdiff1d(np.arange(k), kept), ref.screen_state.eliminated)
        assert np.linalg.norm(x - ref.x_star) <= 1e-9 * max(np.linalg.norm(ref.x_star), 1e-12)
        assert abs(float(sc.F) - ref.final_objective) <= 1e-12 * abs(ref.final_objective)
        assert len({(float(s[3].F), float(s[3].gap)) for s in sols}) == 1
    finally:
        for sh in shards:
            sh.close()
        for b in bases:
            shards[0].eng.L.dscr_peer_free(b)
