"""Column-sharded solves across GPUs (one process per GPU, torch.distributed).

SURVEY §8(e): each rank owns a contiguous block of dictionary columns (groups
kept whole) and runs the per-iteration kernels on it; per trip two collectives
join the ranks — a MAX of the correlation bound after K1 (the dual scaling needs
max |c| over *all* active atoms before any test) and a SUM of the length-N
partial residuals ``D_S a``, ``D_S b`` plus the per-rank scalars after K3a.
Every rank then computes the radius, the objective, the gap, the stop flags and
the REDO/FIXUP trip modes from identical reduced values, so all ranks take the
same control path.  lambda_* is a cross-rank argmax with the reference's
lowest-index tie break (problems.py:79); the extremal atom (or the GST3 normal)
is broadcast from its owner.

The collectives are ``torch.distributed`` all-reduces on zero-copy views of the
engine's ``comm`` region: NCCL over NVLink on GPUs, gloo in the CPU tests (which
drive the same ``orchestrate`` with a numpy phase backend).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .problem import GROUP, Dictionary, GroupPartition, Problem
from .solver import _STOP_NAMES, ScreenState, SolveResult, SolverConfig
from .instrument import SolveTrace, flops_iteration, flops_static_init, problem_digest

NEEDS_VEC = ("dst3", "dome", "gst3")


def shard_ranges(k, world, group_sizes=None):
    """[start, end) column block per rank; with groups, whole groups per rank (balanced by atom
    count).  Every rank gets at least one column (one group): a world larger than the column
    (group) count is rejected, as the engine has no zero-column shard."""
    if world < 1:
        raise ValueError("world size must be at least 1")
    if group_sizes is None:
        if world > k:
            raise ValueError(f"cannot shard {k} columns over {world} ranks (need at least one column per rank)")
        bounds = [round(r * k / world) for r in range(world + 1)]
        return [(bounds[r], bounds[r + 1]) for r in range(world)]
    sizes = np.asarray(group_sizes, dtype=np.int64)
    ng = int(sizes.size)
    if world > ng:
        raise ValueError(f"cannot shard {ng} groups over {world} ranks (need at least one group per rank)")
    ptr = np.concatenate(([0], np.cumsum(sizes)))
    g_bounds = [int(np.searchsorted(ptr, r * k / world, side="left")) for r in range(world)] + [ng]
    g_bounds[0] = 0
    for r in range(1, world):             # at least one group per rank, and room for the ranks after r
        g_bounds[r] = min(max(g_bounds[r], g_bounds[r - 1] + 1), ng - (world - r))
    return [(int(ptr[g_bounds[r]]), int(ptr[g_bounds[r + 1]])) for r in range(world)], \
           [(g_bounds[r], g_bounds[r + 1]) for r in range(world)]


def _allreduce(tensor, op, pg):
    import torch.distributed as dist
    if pg is None:
        return
    dist.all_reduce(tensor, op=op, group=pg)


def orchestrate(backend, cfg, lam, pg=None, group_weights=None, chunk=8, collectives=2, graph=None):
    """Run a sharded solve: setup exchange, then trips with two collectives (MAX after K1, SUM
    after K3A), with ``collectives="peer"`` one exchange per trip through peer memory (device
    stores into every peer's buffer + arrival flags, no host collective), or, with
    ``collectives=1``, one SUM per trip (rank-slot gather of the MAX
    quantities and test extremes, residuals on the unreduced iterate, FIXUP trip when a rank
    screens a unit carrying a nonzero coefficient; SURVEY §7 hard part 2).  The dome test
    always uses two.

    ``graph`` (default: whenever the backend can, i.e. a GPU shard with NCCL or no process
    group): the per-trip phase launches and collectives are captured once into a CUDA graph of
    ``chunk`` trips and replayed, two replays in flight, until the device stop flag is set --
    no per-phase host launches.  Every rank computes the same stop, so all ranks replay the
    same number of times and their captured collectives match."""
    import torch
    import torch.distributed as dist
    MAX, SUM = dist.ReduceOp.MAX, dist.ReduceOp.SUM
    comm = backend.comm
    world = dist.get_world_size(pg) if pg is not None else 1
    rank = dist.get_rank(pg) if pg is not None else 0
    peer = collectives == "peer" and not (cfg.strategy == "dynamic" and cfg.test == "dome")
    one = (collectives == 1 or peer) and not (cfg.strategy == "dynamic" and cfg.test == "dome")
    backend.set_collectives(rank, world, one)
    if peer:
        backend.setup_peers(pg, rank, world)

    backend.phase(nat.PH_SETUP_LOCAL)
    cand = comm[nat.CM_SETUP: nat.CM_SETUP + 3].clone()
    if pg is not None:
        parts = [torch.empty_like(cand) for _ in range(world)]
        dist.all_gather(parts, cand, group=pg)
        allc = torch.stack(parts).cpu().numpy()
    else:
        allc = cand.cpu().numpy()[None, :]
    best = 0
    for r in range(1, world):         # max value, lowest global index on ties (problems.py:79)
        if allc[r, 0] > allc[best, 0] or (allc[r, 0] == allc[best, 0] and allc[r, 1] < allc[best, 1]):
            best = r
    lmax, gidx, sign = float(allc[best, 0]), int(allc[best, 1]), float(allc[best, 2])
    trivial = lam > lmax
    w_star = float(group_weights[gidx]) if group_weights is not None else 0.0
    local_unit = gidx - backend.unit_offset if rank == best else -1
    comm[nat.CM_SETUP: nat.CM_SETUP + 7] = torch.tensor(
        [lmax, gidx, sign, 1.0 if trivial else 0.0, 1.0 if rank == best else 0.0, w_star, local_unit],
        dtype=comm.dtype).to(comm.device)
    backend.phase(nat.PH_SETUP_ADOPT)
    if not trivial and cfg.strategy != "none" and cfg.test in NEEDS_VEC:
        if rank == best:
            backend.phase(nat.PH_SETUP_VEC)
        if pg is not None:
            dist.broadcast(backend.vec, src=best, group=pg)
    backend.phase(nat.PH_SETUP_FINISH)
    if cfg.strategy == "static" and not trivial:
        backend.phase(nat.PH_STATIC_LOCAL)
        _allreduce(comm[nat.CM_MAX: nat.CM_MAX + 8], MAX, pg)
        backend.phase(nat.PH_STATIC_FINISH)
    max_sec = comm[nat.CM_MAX: nat.CM_MAX + 8]
    vec_end = nat.CM_VEC + 2 * backend.ldd
    # two collectives: scalars + vector; one collective: also the rank slots (gather by SUM)
    sum_sec = comm[nat.CM_SUM: vec_end + (nat.OC_SLOT * world if one else 0)]
    def trip():
        backend.phase(nat.PH_K1)
        if one:
            backend.phase(nat.PH_K2S)
            backend.phase(nat.PH_K3A)
            backend.phase(nat.PH_K3S)
            if peer:   # the exchange runs on the devices: stores into peer memory, flags
                backend.phase(nat.PH_K3X_PUSH)
                backend.phase(nat.PH_K3X_REDUCE)
            else:
                _allreduce(sum_sec, SUM, pg)
            backend.phase(nat.PH_K1R1)
            backend.phase(nat.PH_K2C)
        else:
            _allreduce(max_sec, MAX, pg)
            backend.phase(nat.PH_K1R)
            backend.phase(nat.PH_K2)
            backend.phase(nat.PH_K3A)
            backend.phase(nat.PH_K3S)
            _allreduce(sum_sec, SUM, pg)
        backend.phase(nat.PH_K3B)

    if graph is None:
        graph = getattr(backend, "can_capture", lambda _pg: False)(pg)
    if graph:
        # `chunk` trips (phase kernels + the collectives) captured once as a CUDA graph and
        # replayed until the device stop flag is set; trips after the stop return at entry.
        # A capture that fails (before anything was replayed) falls back to the host loop.
        try:
            backend.run_captured(trip, chunk)
        except _CaptureFailed as exc:
            import sys
            sys.stderr.write(f"dist: trip-graph capture failed ({exc.__cause__!r}); per-phase host loop\n")
            graph = False
    if not graph:
        while True:
            sc = backend.scalars()
            if sc.stop != nat.STOP_RUNNING or sc.t >= cfg.max_iters:
                break
            for _ in range(chunk):
                trip()
    backend.one_collective = one
    return backend.scalars()


class _CaptureFailed(RuntimeError):
    """The trip graph could not be captured (e.g. a collective backend without capture support)."""


class GpuShard:
    """GPU phase backend: a solver handle on this rank's column block."""

    def __init__(self, problem_local, cfg, col_offset, n_cols_total, group_offset=0, n_groups_total=0,
                 device=None):
        import torch
        from .solver import Engine
        self.eng = Engine(problem_local, cfg, device=device, desc_patch=dict(
            col_offset=col_offset, n_cols_total=n_cols_total, group_offset=group_offset,
            n_groups_total=n_groups_total))
        self.torch = torch
        b = self.eng.bufs
        self.comm = self.eng.view(b.comm, b.comm_len, torch.float64)
        self.vec = self.eng.view(b.vec, problem_local.dictionary.ldd, torch.float64)
        self.unit_offset = group_offset if problem_local.kind == GROUP else col_offset
        self.ldd = problem_local.dictionary.ldd
        self.phase_calls = 0          # dscr_solver_phase launches (each enqueues >= 1 kernel)
        self.one_collective = False
        self.launch_sptr = self.eng.sptr   # stream the phases launch on (the capture stream while capturing)
        self.graph_trips = 0
        self.graph_replays = 0

    def set_collectives(self, rank, world, one):
        nat.check(self.eng.L.dscr_solver_set_collectives(self.eng.h, int(rank), int(world), 1 if one else 0))

    def setup_peers(self, pg, rank, world):
        """Native exchange: allocate this rank's peer buffer, all-gather the CUDA IPC handles,
        open the peers' buffers and hand every rank's base to the solver."""
        import torch.distributed as dist
        if getattr(self, "peer_own", None) is not None and self.peer_key == (rank, world):
            return                      # already connected (repeated solves on this shard)
        L = self.eng.L
        nbytes = int(L.dscr_peer_buffer_bytes(world, self.ldd))
        if nbytes == 0:
            nat.check(nat.DSCR_EINVAL, "peer buffer size")
        own = C.c_void_p()
        hd = (C.c_char * 64)()
        nat.check(L.dscr_peer_alloc(nbytes, C.byref(own), hd))
        self.peer_own = own
        handles = [bytes(hd)]
        if pg is not None and world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, bytes(hd), group=pg)
        bases, self.peer_opened = [], []
        for r in range(world):
            if r == rank:
                bases.append(own.value)
                continue
            p = C.c_void_p()
            nat.check(L.dscr_peer_open(C.create_string_buffer(handles[r], 64), C.byref(p)))
            self.peer_opened.append(p)
            bases.append(p.value)
        recv = (C.c_void_p * world)(*[b + 512 for b in bases])
        flags = (C.c_void_p * world)(*bases)
        nat.check(L.dscr_solver_set_peers(self.eng.h, int(rank), int(world), recv, flags))
        self.peer_pg = pg
        self.peer_key = (rank, world)

    def phase(self, ph):
        nat.check(self.eng.L.dscr_solver_phase(self.eng.h, int(ph), self.launch_sptr))
        self.phase_calls += 1

    def can_capture(self, pg):
        """Trips can be graph-captured with no process group or an NCCL one (gloo runs on the
        host); DSCR_SHARDED_GRAPH=0 keeps the per-phase host loop."""
        import os
        import torch.distributed as dist
        if os.environ.get("DSCR_SHARDED_GRAPH", "1") == "0":
            return False
        return pg is None or dist.get_backend(pg) == "nccl"

    def run_captured(self, trip, chunk):
        """Capture `chunk` trips once (on a side stream: kernels are recorded, not run), then
        replay the graph on the engine's stream until the stop flag is set.  The stop flag and
        iteration counter of each replay are copied to pinned memory behind it; the host waits
        for replay i-1 while replay i runs, so the device never idles on the host."""
        torch = self.torch
        eng = self.eng
        cs = torch.cuda.Stream(device=eng.device)
        cs.wait_stream(eng.stream)
        g = torch.cuda.CUDAGraph()
        self.launch_sptr = C.c_void_p(cs.cuda_stream)
        calls0 = self.phase_calls
        try:
            with torch.cuda.graph(g, stream=cs):
                for _ in range(chunk):
                    trip()
        except Exception as exc:            # nothing was enqueued for execution: host loop instead
            self.phase_calls = calls0
            raise _CaptureFailed() from exc
        finally:
            self.launch_sptr = eng.sptr
        self.graph_trips = chunk
        sc_dev = eng.view(eng.bufs.scalars, 8, torch.int32)        # t, run_limit, max_iters, mode, stop, ...
        pinned = torch.zeros((2, 8), dtype=torch.int32, pin_memory=True)
        events = [torch.cuda.Event(), torch.cuda.Event()]
        replays = 0
        with torch.cuda.stream(eng.stream):
            pending = []
            while True:
                slot = replays & 1
                g.replay()
                pinned[slot].copy_(sc_dev, non_blocking=True)
                events[slot].record(eng.stream)
                pending.append(slot)
                replays += 1
                if len(pending) == 2:
                    old = pending.pop(0)
                    events[old].synchronize()
                    if int(pinned[old, 4]) != nat.STOP_RUNNING:
                        break
            eng.stream.synchronize()
        self.graph_replays = replays
        per_graph = self.phase_calls - calls0      # phase launches recorded into the graph
        self.phase_calls = calls0 + replays * per_graph
        del g

    def scalars(self):
        return self.eng.scalars()

    def local_solution(self):
        eng = self.eng
        sc = eng.scalars()
        units = eng.active_units(sc.parity)
        atoms = eng.units_to_atoms(units)
        xs = eng.vec(eng.bufs.x[sc.xi], eng.dp.k)[atoms]
        return eng.to_original(atoms), xs, eng.trace_rows(sc.t), sc

    def close(self):
        import torch.distributed as dist
        if getattr(self, "peer_own", None) is not None:
            self.torch.cuda.synchronize()
            if self.peer_pg is not None and dist.get_world_size(self.peer_pg) > 1:
                dist.barrier(group=self.peer_pg)   # no peer still stores into this buffer
            for p in self.peer_opened:
                self.eng.L.dscr_peer_close(p)
            self.eng.L.dscr_peer_free(self.peer_own)
            self.peer_own = None
        self.eng.close()


def sharded_operator_norm(dictionary_local, pg=None, tol=1e-11, max_iters=20000, device=None):
    """||D||_2 of a column-sharded dictionary: power iteration on D D^T = sum_r D_r D_r^T,
    with the length-N product summed across ranks (SUM all-reduce per step)."""
    import torch
    import torch.distributed as dist
    L = nat.lib()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    dic = dictionary_local
    Dd = dic.device_data(dev)
    n, k, ldd = dic.n_rows, dic.n_cols, dic.ldd
    q = torch.zeros(ldd, dtype=torch.float64, device=dev)
    q[:n] = 1.0 / np.sqrt(n)
    w = torch.empty(k, dtype=torch.float64, device=dev)
    z = torch.empty(ldd, dtype=torch.float64, device=dev)
    nb = int(L.dscr_apply_work_size(dic.dtype_code, ldd, k))
    work = torch.empty(nb, dtype=torch.uint8, device=dev)
    s = nat.stream_ptr()
    val = None
    for _ in range(max_iters):
        nat.check(L.dscr_correlate(dic.dtype_code, Dd.data_ptr(), ldd, n, k, q.data_ptr(), w.data_ptr(), s))
        nat.check(L.dscr_apply(dic.dtype_code, Dd.data_ptr(), ldd, n, k, w.data_ptr(), z.data_ptr(),
                               work.data_ptr(), nb, s))
        if pg is not None:
            dist.all_reduce(z, op=dist.ReduceOp.SUM, group=pg)
        new = float(torch.dot(q, z).item())
        nz = float(torch.linalg.vector_norm(z).item())
        if val is not None and abs(new - val) <= tol * max(1.0, abs(new)):
            return float(np.sqrt(max(new, 0.0)))
        val = new
        q = z / nz
    return float(np.sqrt(max(val, 0.0)))


def global_kept(rows, pg):
    """One-collective trips leave each rank's kept-atom count in its trace rows: sum them."""
    import torch
    import torch.distributed as dist
    kept = torch.tensor(np.ascontiguousarray(rows[:, nat.TR_KEPT]), dtype=torch.float64)
    if pg is not None:
        if dist.get_backend(pg) == "nccl":
            kept = kept.cuda()
        dist.all_reduce(kept, op=dist.ReduceOp.SUM, group=pg)
    rows = rows.copy()
    rows[:, nat.TR_KEPT] = kept.cpu().numpy()
    return rows


def run_sharded(problem, cfg, pg=None, device=None, chunk=8, collectives=2, graph=None):
    """Solve `problem` with its columns sharded over the ranks of `pg` (None: single rank,
    split phases without collectives).  Every rank gets the full SolveResult.  ``graph``: see
    ``orchestrate`` (None: capture the trips whenever the process group allows it)."""
    import torch.distributed as dist
    cfg.validate(problem.kind)
    world = dist.get_world_size(pg) if pg is not None else 1
    rank = dist.get_rank(pg) if pg is not None else 0
    k = problem.n_cols
    dic = problem.dictionary
    if problem.kind == GROUP:
        part = problem.partition
        order = np.concatenate(part.groups)
        if not np.array_equal(order, np.arange(k)):
            raise ValueError("sharded group problems need contiguous groups (permute columns first)")
        (c0, c1), (g0, g1) = [x[rank] for x in shard_ranges(k, world, part.group_sizes())]
        sub = Dictionary(dic.data[:, c0:c1], check_unit_norms=False, dtype=dic.dtype)
        sub.col_norm_checked = dic.col_norm_checked
        lp = GroupPartition.build(sub, [g - c0 for g in part.groups[g0:g1]], weights=part.weights[g0:g1],
                                  spectral_norms=part.spectral_norms[g0:g1])
        local = Problem(sub, problem.y, problem.lam, lp)
        shard = GpuShard(local, cfg, c0, k, g0, part.n_groups, device)
        gw = np.asarray(part.weights)
    else:
        c0, c1 = shard_ranges(k, world)[rank]
        sub = Dictionary(dic.data[:, c0:c1], check_unit_norms=False, dtype=dic.dtype)
        sub.col_norm_checked = dic.col_norm_checked
        local = Problem(sub, problem.y, problem.lam)
        shard = GpuShard(local, cfg, c0, k, 0, 0, device)
        gw = None
    import torch
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    try:
        start.record(shard.eng.stream)
        sc = orchestrate(shard, cfg, problem.lam, pg, gw, chunk, collectives, graph)
        replays = shard.graph_replays
        stop.record(shard.eng.stream)
        stop.synchronize()
        device_s = start.elapsed_time(stop) / 1e3
        if sc.status != 0:
            from .solver import _raise_status
            _raise_status(None, sc)
        kept_l, x_l, rows, sc = shard.local_solution()
        if shard.one_collective:
            rows = global_kept(rows, pg)
    finally:
        shard.close()
    if pg is not None:
        got = [None] * world
        dist.all_gather_object(got, (kept_l + c0, x_l), group=pg)
    else:
        got = [(kept_l + c0, x_l)]
    kept = np.concatenate([g[0] for g in got]).astype(np.int64)
    xs = np.concatenate([g[1] for g in got])
    order = np.argsort(kept, kind="stable")
    kept, xs = kept[order], xs[order]
    x_star = np.zeros(k)
    x_star[kept] = xs
    mask = np.ones(k, dtype=bool)
    mask[kept] = False
    trace = SolveTrace(kind=problem.kind, strategy=cfg.strategy, n_rows=problem.n_rows, n_cols=k,
                       group_count=problem.partition.n_groups if problem.kind == GROUP else 0, lam=problem.lam,
                       digest=problem_digest(problem))
    cum = 0
    if cfg.strategy == "static":                      # as run() and the reference (solvers.py:425-426)
        trace.init_flops = flops_static_init(k, problem.n_rows)
        cum = trace.init_flops
    for r in rows:
        cum += flops_iteration(problem.kind, cfg.strategy, k, problem.n_rows, int(r[nat.TR_KEPT]),
                               int(r[nat.TR_NNZ]), trace.group_count)
        trace.append(int(r[nat.TR_T]), int(r[nat.TR_KEPT]), int(r[nat.TR_NNZ]), float(r[nat.TR_OBJ]), cum,
                     float(r[nat.TR_NS]) * 1e-9)
        trace.gap.append(float(r[nat.TR_GAP]))
        trace.radius.append(float(r[nat.TR_RADIUS]))
        trace.support.append(int(r[nat.TR_SUPPORT]))
        trace.L.append(float(r[nat.TR_L]))
    if sc.trivial:
        res = SolveResult(np.zeros(k), 0, trace, 0.5 * float(problem.y @ problem.y),
                          ScreenState(np.arange(k, dtype=np.int64), np.empty(0, np.int64), cfg.test),
                          lambda_max=float(sc.lmax), stop_reason="trivial", device_seconds=device_s)
    else:
        final = trace.objective[-1] if trace.objective else 0.5 * float(problem.y @ problem.y)
        res = SolveResult(x_star, int(sc.t), trace, final,
                          ScreenState(np.flatnonzero(mask).astype(np.int64), kept, cfg.test),
                          lambda_max=float(sc.lmax), gap=float(sc.gap),
                          stop_reason=_STOP_NAMES.get(sc.stop, "running"), device_seconds=device_s)
    res.graph_replays = replays         # trip-graph replays of this rank (0: per-phase host loop)
    return res
