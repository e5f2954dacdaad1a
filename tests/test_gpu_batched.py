"""Tensor-core (tcgen05) batched correlation GEMM vs a torch fp32 reference of the same op."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1412_4080_b200 import _native as nat  # noqa: E402


def _gemm(A, B, S, Nb):
    L = nat.lib()
    M, K = A.shape
    C = torch.empty((Nb, M), dtype=torch.float32, device=A.device)
    nat.check(L.dscr_batched_gemm_bf16(A.data_ptr(), M, K, B.data_ptr(), Nb, K, K, S, C.data_ptr(), M,
                                       nat.stream_ptr()))
    return C


@pytest.mark.parametrize("M,Nb,K,S", [(128, 256, 64, 1), (256, 512, 128, 1), (384, 256, 192, 2), (1024, 1024, 1024, 1)])
def test_gemm_matches_fp32_reference(M, Nb, K, S):
    g = torch.Generator(device="cuda").manual_seed(M + Nb + K + S)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(S * Nb, K, device="cuda", generator=g).to(torch.bfloat16)
    C = _gemm(A, B, S, Nb)
    torch.cuda.synchronize()
    ref = sum(B[s * Nb:(s + 1) * Nb].double() @ A.double().T for s in range(S))
    err = (C.double() - ref).abs().max().item()
    scale = (B.double().abs().max() * A.double().abs().max() * K * S).item()
    assert err <= 1e-6 * scale, (err, scale)


def test_gemm_c5_shape_throughput():
    M, Nb, K = 16384, 4096, 1024
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(Nb, K, device="cuda").to(torch.bfloat16)
    C = _gemm(A, B, 1, Nb)
    torch.cuda.synchronize()
    idx = torch.randint(0, M, (64,), device="cuda")
    ref = (B.float() @ A[idx].float().T)
    assert torch.allclose(C[:, idx], ref, rtol=1e-3, atol=1e-2)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        _gemm(A, B, 1, Nb)
    ev0.record()
    for _ in range(10):
        _gemm(A, B, 1, Nb)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 10
    tflops = 2 * M * Nb * K / ms / 1e9
    print(f"\nc5 D^T Theta: {ms * 1e3:.1f} us, {tflops:.0f} TFLOP/s")
    assert tflops > 200


def _corr_exact(Dt, V):
    L = nat.lib()
    K, N = Dt.shape
    B = V.shape[0]
    out = torch.empty((B, K), dtype=torch.float64, device=Dt.device)
    ws = L.dscr_corr_exact_work_size(K, N, B)
    work = torch.empty(ws, dtype=torch.uint8, device=Dt.device)
    nat.check(L.dscr_corr_exact_bf16(Dt.data_ptr(), K, N, N, V.data_ptr(), B, N, out.data_ptr(), K,
                                     work.data_ptr(), ws, nat.stream_ptr()))
    return out


def _slices(X, S):
    """Row scale 2^e (max|x| < 2^e) and S truncated 7-bit slices: x = 2^e sum_s q_s 2^-7(s+1)."""
    m = np.abs(X).max(axis=1)
    e = np.zeros(len(X), dtype=np.int64)
    nz = m > 0
    e[nz] = np.frexp(m[nz])[1]
    x = np.ldexp(X, -e[:, None])
    qs = []
    for _ in range(S):
        x = x * 128.0
        q = np.trunc(x)
        x = x - q
        qs.append(q)
    return qs, e


def _slice_emulation(D, V, S=4, T=5, dmax=5):
    """numpy restatement of the integer-slice correlation (exact int64 combination, one rounding)."""
    Ds, eD = _slices(D, S)
    Vs, eV = _slices(V, T)
    acc = np.zeros((V.shape[0], D.shape[0]), dtype=np.int64)
    for d in range(dmax + 1):
        C = np.zeros_like(acc)
        for s_ in range(S):
            t = d - s_
            if 0 <= t < T:
                C += Vs[t].astype(np.int64) @ Ds[s_].astype(np.int64).T     # exact integer products
        acc += C << (7 * (dmax - d))                                         # exact, < 2^63
    return np.ldexp(acc.astype(np.float64), eD[None, :] + eV[:, None] - 14 - 7 * dmax), eD, eV


@pytest.mark.parametrize("K,N,B,hard", [(128, 128, 128, True), (384, 256, 256, True), (1024, 1024, 512, False),
                                        (256, 2048, 128, True)])
def test_corr_exact_matches_fp64(K, N, B, hard):
    """Integer-slice tensor-core correlations: bit-identical to the numpy restatement of the
    slice algorithm, and within its rigorous error bound of fp64 (fp32 GEMM: ~2^-13)."""
    rng = np.random.default_rng(K + N + B)
    D = rng.standard_normal((K, N))
    V = rng.standard_normal((B, N))
    if hard:
        D *= np.exp(rng.uniform(-6, 6, size=(K, 1)))         # per-atom scales
        D[:, ::7] *= 1e-5                                     # entries below 2^-21 of the row max: truncated
        D[1] = 0.0                                            # empty atom
        V *= np.exp(rng.uniform(-20, 20, size=(B, 1)))
        V[:, ::5] *= 1e-7
        V[2] = 0.0
    Dt = torch.from_numpy(D).to(torch.bfloat16).cuda()
    out = _corr_exact(Dt, torch.from_numpy(V).cuda()).cpu().numpy()
    Dh = Dt.double().cpu().numpy()
    emu, eD, eV = _slice_emulation(Dh, V)
    assert np.array_equal(out, emu)
    ref = V @ Dh.T
    # |err| <= 2^(E_i - 28) ||v_j||_1 + 2^(F_j - 35) ||d_i||_1 (+ dropped pairs, fp64 rounding)
    bound = (np.ldexp(1.0, eD - 28)[None, :] * np.abs(V).sum(1)[:, None]
             + np.ldexp(1.0, eV - 35)[:, None] * np.abs(Dh).sum(1)[None, :])
    err = np.abs(out - ref)
    assert np.all(err <= 1.01 * bound + 1e-12 * np.abs(ref) + 1e-300)
    if hard:
        assert np.all(out[2] == 0.0) and np.all(out[:, 1] == 0.0)
    else:   # unit-scale Gaussian dictionary (every bf16 entry sliced exactly): ~fp64 accuracy
        rel = err / (np.abs(V) @ np.abs(Dh).T)
        assert rel.max() < 2.0 ** -30, rel.max()


def test_corr_exact_rejects_bad_shapes():
    L = nat.lib()
    assert L.dscr_corr_exact_bf16(None, 128, 128, 128, None, 128, 128, None, 128, None, 0, None) == nat.DSCR_EINVAL
    assert L.dscr_corr_exact_work_size(0, 128, 128) == 0


# ---------------------------------------------------------------- batched solver vs oracle

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402
from paper_1412_4080_b200.batched import solve_batched  # noqa: E402
from oracle import batched_oracle as bo  # noqa: E402
from oracle import screen_oracle as so  # noqa: E402


def _batch_problem(n, k, b, ratio, seed=0):
    w = wl.config5(seed=seed, n=n, k=k, batch=b, nnz=8, ratio=ratio)
    dic = ds.Dictionary(w.D, check_unit_norms=False, dtype="bf16")
    D64 = dic.as_float64()
    L = float(np.linalg.norm(D64, 2) ** 2 * (1 + 1e-6))
    return w, dic, D64, L


@pytest.mark.parametrize("ratio,splits", [(0.4, 1), (0.4, 2), (0.85, 1), (0.85, 2)])
def test_batched_fista_matches_oracle(ratio, splits):
    """Per observation: the same screened set as the operand-precision oracle (theta rounded to
    one / two bf16 terms, everything else fp64: oracle/batched_oracle.py), objective to 1e-7
    and x to 1e-3 of it (fp32 accumulation in the tensor cores; x after 100 iterations is far
    from converged, measured 3e-7 .. 8e-4); against the reference's fp64
    algorithm the objective agrees to 1e-6 and the screened set is a subset of its set (the
    dual scaling's correlation bound carries the rigorous bf16/fp32 error term, so the device
    never screens more)."""
    w, dic, D64, L = _batch_problem(128, 1024, 256, ratio)
    res = solve_batched(dic, w.y, w.lam, L, iterations=100, test="dst3", splits=splits, masks=True)
    assert res.iterations == 100
    worst_f, worst_fr = 0.0, 0.0
    for j in range(0, 256, 17):
        y, lam = w.y[:, j], float(w.lam[j])
        emu = bo.solve_bf16(D64, y, lam, L, 100, splits=splits)
        ref = so.solve(so.make_problem(D64, y, lam), so.Config(algorithm="fista", strategy="dynamic", test="dst3",
                                                                max_iters=100, rel_tol=1e-300, L0=L, norm_aware=True))
        x = res.x_dense(j, 1024)
        worst_f = max(worst_f, abs(res.objective[j] - emu.objective) / emu.objective)
        worst_fr = max(worst_fr, abs(res.objective[j] - ref.final_objective) / ref.final_objective)
        assert np.linalg.norm(x - emu.x) <= 1e-3 * max(np.linalg.norm(emu.x), 0.1)
        elim = res.eliminated(j)
        assert np.array_equal(elim, emu.eliminated), j
        assert np.all(np.isin(elim, ref.eliminated)), j
    assert worst_f <= 1e-7, worst_f
    assert worst_fr <= 1e-6, worst_fr
    if ratio > 0.5:
        assert res.kept.min() < 1024      # screening fired somewhere


def test_batched_c5_shape_runs():
    w, dic, D64, L = _batch_problem(1024, 16384, 512, 0.4, seed=1)
    res = solve_batched(dic, w.y, w.lam, L, iterations=100, test="dst3", splits=1)
    assert res.iterations == 100 and np.all(res.status == 0)
    for j in (0, 255):
        op = so.make_problem(D64, w.y[:, j], w.lam[j])
        ref = so.solve(op, so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=100,
                                     rel_tol=1e-300, L0=L, norm_aware=True))
        assert abs(res.objective[j] - ref.final_objective) <= 1e-6 * ref.final_objective
    print(f"\nc5-shape batch of 512: {res.device_seconds * 1e3:.1f} ms for 100 iterations")


@pytest.mark.parametrize("ratio", [0.4, 0.85])
def test_fused_epilogue_matches_dense_update(ratio):
    """Hot-entry epilogue (no dense C round trip) == dense C + full per-atom update."""
    w, dic, D64, L = _batch_problem(256, 2048, 512, ratio, seed=3)
    a = solve_batched(dic, w.y, w.lam, L, iterations=60, test="dst3", splits=2, fused=True)
    b = solve_batched(dic, w.y, w.lam, L, iterations=60, test="dst3", splits=2, fused=False)
    np.testing.assert_allclose(a.objective, b.objective, rtol=1e-13)
    assert np.array_equal(a.kept, b.kept) and np.array_equal(a.nnz, b.nnz)
    for j in range(0, 512, 37):
        assert np.array_equal(a.x_idx[j], b.x_idx[j])
        np.testing.assert_allclose(a.x_val[j], b.x_val[j], rtol=1e-13, atol=1e-15)
    if ratio > 0.5:
        assert a.kept.min() < 2048


@pytest.mark.parametrize("ratio", [0.4, 0.85])
@pytest.mark.parametrize("setup,test", [("", "dst3"), ("oz2", "dst3"), ("", "safe"), ("oz2", "safe")])
def test_integer_slice_setup_matches_fp64_setup(ratio, setup, test, monkeypatch):
    """Setup correlations on the integer tensor cores -- the default single exact product D^T Z of
    the test centres after an approximate argmax, and the two exact products D^T Y, D^T A_*
    (DSCR_BATCHED_SETUP=oz2) -- vs the fp64 FMA path: same lambda_*, screening decisions, support
    and trace (centres differ by < 2^-28 of their scale, far inside the test slack)."""
    w, dic, D64, L = _batch_problem(256, 2048, 512, ratio, seed=5)
    if setup:
        monkeypatch.setenv("DSCR_BATCHED_SETUP", setup)
    a = solve_batched(dic, w.y, w.lam, L, iterations=60, test=test, splits=2)
    monkeypatch.setenv("DSCR_BATCHED_SETUP", "fp64")
    b = solve_batched(dic, w.y, w.lam, L, iterations=60, test=test, splits=2)
    np.testing.assert_allclose(a.lambda_max, b.lambda_max, rtol=1e-12)
    assert np.array_equal(a.kept, b.kept) and np.array_equal(a.nnz, b.nnz)
    np.testing.assert_allclose(a.objective, b.objective, rtol=1e-12)
    np.testing.assert_allclose(a.gap, b.gap, rtol=1e-9, atol=1e-12)
    for j in range(0, 512, 41):
        assert np.array_equal(a.x_idx[j], b.x_idx[j])


@pytest.mark.parametrize("ratio", [0.4, 0.85])
def test_warp_update_matches_cta_update(ratio, monkeypatch):
    """Warp-per-observation update (<= 64 hot/list entries) vs the CTA update for every
    observation: same lists, screening and trace (penalty sums differ only in reduction order)."""
    w, dic, D64, L = _batch_problem(256, 2048, 512, ratio, seed=9)
    a = solve_batched(dic, w.y, w.lam, L, iterations=60, test="dst3", splits=2)
    monkeypatch.setenv("DSCR_BATCHED_UPDATE", "cta")
    b = solve_batched(dic, w.y, w.lam, L, iterations=60, test="dst3", splits=2)
    assert np.array_equal(a.kept, b.kept) and np.array_equal(a.nnz, b.nnz)
    np.testing.assert_allclose(a.objective, b.objective, rtol=1e-13)
    for j in range(0, 512, 23):
        assert np.array_equal(a.x_idx[j], b.x_idx[j])
        np.testing.assert_allclose(a.x_val[j], b.x_val[j], rtol=1e-13, atol=1e-15)


def test_block_sort_matches_device_sort(monkeypatch):
    """Screening order by the per-observation shared-memory sort == the segmented device sort."""
    w, dic, D64, L = _batch_problem(256, 2048, 512, 0.85, seed=13)
    a = solve_batched(dic, w.y, w.lam, L, iterations=60, test="dst3", splits=2)
    monkeypatch.setenv("DSCR_BATCHED_SORT", "device")
    b = solve_batched(dic, w.y, w.lam, L, iterations=60, test="dst3", splits=2)
    assert np.array_equal(a.kept, b.kept) and np.array_equal(a.nnz, b.nnz)
    assert np.array_equal(a.objective, b.objective)
    assert a.kept.min() < 2048
    for j in range(0, 512, 29):
        assert np.array_equal(a.x_idx[j], b.x_idx[j])


def test_batched_max_rows_matches_oracle():
    """N = 2048 (the largest row count of the register-resident residual kernels and of the
    integer-slice setup)."""
    w, dic, D64, L = _batch_problem(2048, 1024, 256, 0.5, seed=17)
    res = solve_batched(dic, w.y, w.lam, L, iterations=40, test="dst3", splits=2)
    for j in (0, 77, 255):
        ref = so.solve(so.make_problem(D64, w.y[:, j], w.lam[j]),
                       so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=40, rel_tol=1e-300,
                                 L0=L, norm_aware=True))
        assert abs(res.objective[j] - ref.final_objective) <= 1e-4 * ref.final_objective
        x = res.x_dense(j, 1024)
        assert np.linalg.norm(x - ref.x_star) <= 1e-3 * max(np.linalg.norm(ref.x_star), 1e-12)


@pytest.mark.parametrize("n,splits", [(2112, 2), (2176, 1), (4160, 1), (8192, 2)])
def test_batched_tall_dictionaries_match_oracle(n, splits):
    """Dictionaries taller than 2048 rows (the register-resident residual kernels' limit): the
    chunked residual pass with theta in shared memory, setup on the integer tensor cores when the
    row count is a multiple of 128 (2176, 8192) and on the fp64 path otherwise, against the
    oracle (objective, x, screened set a subset of the reference's) and the operand-precision
    oracle (identical screened set)."""
    w, dic, D64, L = _batch_problem(n, 1024, 256, 0.6, seed=41)
    res = solve_batched(dic, w.y, w.lam, L, iterations=40, test="dst3", splits=splits, masks=True)
    assert res.iterations == 40 and np.all(res.status == 0)
    for j in (0, 131, 255):
        y, lam = w.y[:, j], float(w.lam[j])
        ref = so.solve(so.make_problem(D64, y, lam),
                       so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=40, rel_tol=1e-300,
                                 L0=L, norm_aware=True))
        emu = bo.solve_bf16(D64, y, lam, L, 40, splits=splits)
        assert abs(res.objective[j] - ref.final_objective) <= 1e-5 * ref.final_objective
        assert abs(res.objective[j] - emu.objective) <= 1e-6 * emu.objective
        x = res.x_dense(j, 1024)
        assert np.linalg.norm(x - emu.x) <= 1e-3 * max(np.linalg.norm(emu.x), 0.1)
        elim = res.eliminated(j)
        assert np.array_equal(elim, emu.eliminated), j
        assert np.all(np.isin(elim, ref.eliminated)), j


@pytest.mark.parametrize("n,k,b,splits", [(1000, 5000, 300, 2), (200, 1000, 37, 1), (1024, 2048, 256, 1)])
def test_batched_any_shape_matches_oracle(n, k, b, splits):
    """Row, atom and batch counts that are not multiples of the kernels' tiles (64 / 128 / 256):
    the host pads with zero rows, all-zero atoms (inactive from the start, not counted as kept)
    and trivial observations, and cuts the results back.  Per observation the result equals the
    oracle's on the unpadded problem; the batch aggregates count only the caller's observations."""
    w, dic, D64, L = _batch_problem(n, k, b, 0.6, seed=51)
    res = solve_batched(dic, w.y, w.lam, L, iterations=50, test="dst3", splits=splits, masks=True)
    assert res.objective.shape == (b,) and res.kept.shape == (b,) and res.status.shape == (b,)
    assert np.all(res.status == 0) and res.kept.max() <= k and len(res.x_idx) == b
    np.testing.assert_allclose(res.trace[-1, 0], res.objective.sum(), rtol=1e-12)
    np.testing.assert_allclose(res.trace[-1, 3], res.kept.sum(), rtol=0, atol=0.5)
    for j in sorted({0, b // 2, b - 1}):
        y, lam = w.y[:, j], float(w.lam[j])
        emu = bo.solve_bf16(D64, y, lam, L, 50, splits=splits)
        ref = so.solve(so.make_problem(D64, y, lam),
                       so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=50, rel_tol=1e-300,
                                 L0=L, norm_aware=True))
        assert abs(res.objective[j] - emu.objective) <= 1e-7 * emu.objective
        assert abs(res.objective[j] - ref.final_objective) <= 1e-6 * ref.final_objective
        x = res.x_dense(j, k)
        assert np.linalg.norm(x - emu.x) <= 1e-3 * max(np.linalg.norm(emu.x), 0.1)
        elim = res.eliminated(j)
        assert res.active_mask(j).shape == (k,)
        assert np.array_equal(elim, emu.eliminated), j
        assert np.all(np.isin(elim, ref.eliminated)), j
        assert res.kept[j] == k - elim.size


def test_batched_solver_any_shape_reuse_and_dictionary_swap():
    """BatchedSolver on a padded shape: a second batch and a swapped dictionary reuse the engine
    and equal one-shot solves."""
    from paper_1412_4080_b200.batched import BatchedSolver
    w1, dic1, _, L1 = _batch_problem(200, 1000, 37, 0.5, seed=61)
    w2, dic2, _, L2 = _batch_problem(200, 1000, 37, 0.5, seed=62)
    L = max(L1, L2)
    solver = BatchedSolver(dic1, L, iterations=40, test="dst3", splits=2)
    a1 = solver.solve(w1.y, w1.lam)
    eng = solver.eng
    a2 = solver.solve(w2.y, w2.lam, dictionary=dic2)
    assert solver.eng is eng
    solver.close()
    b1 = solve_batched(dic1, w1.y, w1.lam, L, iterations=40, test="dst3", splits=2)
    b2 = solve_batched(dic2, w2.y, w2.lam, L, iterations=40, test="dst3", splits=2)
    for a, c in ((a1, b1), (a2, b2)):
        assert np.array_equal(a.objective, c.objective) and np.array_equal(a.kept, c.kept)
        assert np.array_equal(a.x_indices, c.x_indices) and np.array_equal(a.x_values, c.x_values)


def test_batched_capacity_overflow_falls_back_to_dense_path():
    """A small lam makes supports larger than the per-observation list capacity: the solve reruns
    on the dense-update path with room for every atom (the reference has no support limit) and
    matches the oracle."""
    from paper_1412_4080_b200.batched import BatchedCapacityError, BatchedEngine
    w, dic, D64, L = _batch_problem(128, 1024, 256, 0.02, seed=71)
    eng = BatchedEngine(dic, w.y, w.lam, L, iterations=30, test="dst3", splits=2, cap=32)
    eng.setup()
    eng.run()
    eng.stream.synchronize()
    with pytest.raises(BatchedCapacityError):
        eng.result()
    eng.close()
    res = solve_batched(dic, w.y, w.lam, L, iterations=30, test="dst3", splits=2, cap=32)
    assert np.all(res.status == 0) and res.nnz.max() > 32
    for j in (0, 200):
        ref = so.solve(so.make_problem(D64, w.y[:, j], w.lam[j]),
                       so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=30, rel_tol=1e-300,
                                 L0=L, norm_aware=True))
        assert abs(res.objective[j] - ref.final_objective) <= 1e-6 * ref.final_objective
        assert res.nnz[j] == np.count_nonzero(ref.x_star)


def test_batched_rejects_more_than_16384_rows():
    with pytest.raises((ValueError, RuntimeError)):
        w, dic, D64, L = _batch_problem(16448, 128, 256, 0.6, seed=43)
        solve_batched(dic, w.y, w.lam, L, iterations=5, test="dst3", splits=1)


@pytest.mark.parametrize("n,k,b", [(64, 1024, 256), (320, 1024, 256), (640, 2048, 256), (1024, 2048, 256),
                                   (1088, 1024, 256)])
def test_group_residual_matches_cta_residual(n, k, b, monkeypatch):
    """Residual pass with 32 / 64 / 128 threads per observation (several observations per CTA, 8-row
    chunks; row counts that leave the second chunk partly or wholly empty) vs the one-CTA-per-
    observation kernel: same lists and screening, objective / gap equal up to the reduction order."""
    w, dic, D64, L = _batch_problem(n, k, b, 0.6, seed=21)
    a = solve_batched(dic, w.y, w.lam, L, iterations=50, test="dst3", splits=2)
    monkeypatch.setenv("DSCR_BATCHED_RESID", "cta")
    c = solve_batched(dic, w.y, w.lam, L, iterations=50, test="dst3", splits=2)
    assert np.all(a.status == 0) and np.all(c.status == 0)
    assert np.array_equal(a.kept, c.kept) and np.array_equal(a.nnz, c.nnz)
    np.testing.assert_allclose(a.objective, c.objective, rtol=1e-12)
    np.testing.assert_allclose(a.gap, c.gap, rtol=1e-8, atol=1e-11)
    for j in range(0, b, 19):
        assert np.array_equal(a.x_idx[j], c.x_idx[j])
        np.testing.assert_allclose(a.x_val[j], c.x_val[j], rtol=1e-11, atol=1e-14)
    ref = so.solve(so.make_problem(D64, w.y[:, 3], w.lam[3]),
                   so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=50, rel_tol=1e-300,
                             L0=L, norm_aware=True))
    assert abs(a.objective[3] - ref.final_objective) <= 1e-4 * ref.final_objective


@pytest.mark.parametrize("setup", ["", "oz2", "fp64"])
def test_setup_trivial_regime_ties_and_lambda_max(setup, monkeypatch):
    """Setup edge cases on every setup path (single exact product after the approximate argmax,
    two exact products, fp64): lambda_* equals max|D^T y_j| of the stored bf16 atoms (reference
    problems.py:75-86); observations with lam_j > lambda_* are trivial (status 1, x = 0, nothing
    kept -- solvers.py:384-397); a duplicated extremal atom (an exact tie of the two largest
    correlations) changes nothing in the outcome; the other observations match the oracle."""
    w, dic, D64, L = _batch_problem(128, 1024, 256, 0.6, seed=33)
    lmax_ref = np.max(np.abs(D64.T @ w.y), axis=0)
    lam = w.lam.copy()
    triv = np.arange(0, 256, 9)
    lam[triv] = 1.05 * lmax_ref[triv]
    # duplicate the extremal atom of observation 5 at a later index (same bf16 bits)
    Dq = np.array(dic.data, copy=True)
    i_star = int(np.argmax(np.abs(D64.T @ w.y[:, 5])))
    dup = 1000 if i_star != 1000 else 999
    Dq[:, dup] = Dq[:, i_star]
    dic2 = ds.Dictionary(Dq, check_unit_norms=False, dtype="bf16")
    D2 = dic2.as_float64()
    L2 = float(np.linalg.norm(D2, 2) ** 2 * (1 + 1e-6))
    lmax2 = np.max(np.abs(D2.T @ w.y), axis=0)
    if setup:
        monkeypatch.setenv("DSCR_BATCHED_SETUP", setup)
    res = solve_batched(dic2, w.y, lam, L2, iterations=50, test="dst3", splits=2, masks=True)
    np.testing.assert_allclose(res.lambda_max, lmax2, rtol=1e-12)
    assert np.all(res.status[triv] == 1) and np.all(res.nnz[triv] == 0) and np.all(res.kept[triv] == 0)
    ok = np.setdiff1d(np.arange(256), triv)
    assert np.all(res.status[ok] == 0)
    for j in (5, 6, 100):
        if j in triv:
            continue
        ref = so.solve(so.make_problem(D2, w.y[:, j], lam[j]),
                       so.Config(algorithm="fista", strategy="dynamic", test="dst3", max_iters=50, rel_tol=1e-300,
                                 L0=L2, norm_aware=True))
        assert abs(res.objective[j] - ref.final_objective) <= 1e-6 * ref.final_objective
        assert np.all(np.isin(res.eliminated(j), ref.eliminated)), j


def test_batched_solver_reuses_engine_across_batches_and_dictionaries():
    """BatchedSolver (engine, workspace and iteration graph reused) == one-shot solve_batched, for
    a second batch on the same dictionary and after swapping in another dictionary."""
    from paper_1412_4080_b200.batched import BatchedSolver
    w1, dic1, _, L1 = _batch_problem(128, 1024, 256, 0.5, seed=5)
    w2, _, _, _ = _batch_problem(128, 1024, 256, 0.7, seed=6)
    w3, dic3, _, _ = _batch_problem(128, 1024, 256, 0.6, seed=7)
    solver = BatchedSolver(dic1, L1, iterations=40, test="dst3")
    try:
        runs = [solver.solve(w1.y, w1.lam), solver.solve(w2.y, w2.lam), solver.solve(w3.y, w3.lam, dictionary=dic3)]
    finally:
        solver.close()
    refs = [solve_batched(dic1, w1.y, w1.lam, L1, iterations=40, test="dst3"),
            solve_batched(dic1, w2.y, w2.lam, L1, iterations=40, test="dst3"),
            solve_batched(dic3, w3.y, w3.lam, L1, iterations=40, test="dst3")]
    for got, ref in zip(runs, refs):
        assert np.array_equal(got.objective, ref.objective)
        assert np.array_equal(got.kept, ref.kept) and np.array_equal(got.x_ptr, ref.x_ptr)
        assert np.array_equal(got.x_indices, ref.x_indices) and np.array_equal(got.x_values, ref.x_values)
