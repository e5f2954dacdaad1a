"""Seeded synthetic inputs for the BASELINE configurations (host side, numpy).

Every array is produced on the host from Philox streams keyed by
``(seed, stream)`` so the GPU engine and the CPU oracle consume the same
bytes.  The generators for the reference's own families restate
``screenlab.datagen`` (reference ``pkg/src/screenlab/datagen.py:33-36`` for the
keyed Philox, ``:60-66`` for Gaussian atoms, ``:112-131`` for observations,
``:134-155`` for the Bernoulli-Gaussian planted observation and ``:158-165`` for
random partitions); the BASELINE-only families (correlated "Pnorm-style"
dictionary, planted sparse observations, the fp32 and bf16 configs) are
defined here and documented in DESIGN.md.

This module is host data preparation, not part of the screened-solver hot
path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from concurrent.futures import ThreadPoolExecutor

import numpy as np

DICT_STREAM = 0
OBS_STREAM = 1
GROUP_STREAM = 2
PLANT_STREAM = 3
NOISE_STREAM = 4
BLOCK_STREAM_BASE = 100


def make_rng(seed, stream=0):
    """Philox 4x64 generator keyed by (seed, stream) (datagen.py:33-36)."""
    seq = np.random.SeedSequence(entropy=int(seed), spawn_key=(int(stream),))
    return np.random.Generator(np.random.Philox(seq))


def unit_columns(mat):
    nrm = np.linalg.norm(mat, axis=0)
    if np.any(nrm == 0.0):
        raise ValueError("cannot normalize a zero column")
    return mat / nrm


def gaussian_dictionary(n, k, seed):
    """Unit-norm Gaussian atoms, drawn as one (n, k) block (datagen.py:60-61, 90-94)."""
    return np.asfortranarray(unit_columns(make_rng(seed, DICT_STREAM).standard_normal((n, k))))


def pnoise_dictionary(n, k, seed):
    """Spike-plus-scaled-noise atoms (datagen.py:64-70)."""
    rng = make_rng(seed, DICT_STREAM)
    kappa = rng.random(k)
    g = rng.standard_normal((n, k))
    mat = 0.1 * kappa * g
    mat[0, :] += 1.0
    return np.asfortranarray(unit_columns(mat))


def gaussian_observation(n, seed):
    """Unit-sphere observation (datagen.py:118-119)."""
    return unit_columns(make_rng(seed, OBS_STREAM).standard_normal((n, 1)))[:, 0]


def pnoise_observation(n, seed):
    rng = make_rng(seed, OBS_STREAM)
    kappa = rng.random(1)
    g = rng.standard_normal((n, 1))
    mat = 0.1 * kappa * g
    mat[0, :] += 1.0
    return unit_columns(mat)[:, 0]


def random_groups(k, group_size, seed):
    """Equal-size random partition, each group sorted (datagen.py:158-165)."""
    if group_size < 1 or k % group_size:
        raise ValueError("group_size must divide the number of columns")
    perm = make_rng(seed, GROUP_STREAM).permutation(k)
    return [np.sort(perm[i:i + group_size]) for i in range(0, k, group_size)]


def bernoulli_gaussian_observation(dic, groups, seed, p=0.05, snr_db=20.0, retries=100):
    """Group-planted observation at a target SNR (datagen.py:134-155)."""
    rng = make_rng(seed, OBS_STREAM)
    n, k = dic.shape
    for _ in range(retries):
        on = rng.random(len(groups)) < p
        if not on.any():
            continue
        x = np.zeros(k)
        for gid in np.flatnonzero(on):
            idx = groups[gid]
            x[idx] = rng.standard_normal(idx.size)
        clean = dic @ x
        c_nrm = float(np.linalg.norm(clean))
        if c_nrm == 0.0:
            continue
        g = rng.standard_normal(n)
        noise = g * (c_nrm / (np.linalg.norm(g) * 10.0 ** (snr_db / 20.0)))
        y = clean + noise
        return y / np.linalg.norm(y)
    raise RuntimeError("no active group drawn")


def lambda_star(dic, y, groups=None, weights=None):
    """max |D^T y| (or max_g ||D_g^T y|| / w_g) on the host, for building lam."""
    corr = dic.T @ y
    if groups is None:
        return float(np.max(np.abs(corr)))
    if weights is None:
        weights = np.sqrt([g.size for g in groups])
    return float(max(np.linalg.norm(corr[g]) / w for g, w in zip(groups, weights)))


# ---------------------------------------------------------------------------
# BASELINE configurations
# ---------------------------------------------------------------------------


@dataclass
class Workload:
    """Host arrays of one BASELINE configuration."""

    name: str
    D: np.ndarray                  # (N, K) column-major; fp64, fp32 or bf16-as-uint16 (c5)
    y: np.ndarray                  # (N,) fp64 unit norm, or (N, B) for c5
    lam: object                    # float, or (B,) array for c5
    algorithm: str = "fista"
    test: str = "dst3"
    gap_tol: float = 1e-6
    max_iters: int = 10000
    groups: list | None = None
    dtype: str = "f64"
    meta: dict = field(default_factory=dict)


def config1(seed=0, ratio=0.5, n=1000, k=5000):
    """c1: Gaussian N=1000 x K=5000 fp64, ISTA + dynamic ST3, 0.5 lam*."""
    D = gaussian_dictionary(n, k, seed)
    y = gaussian_observation(n, seed)
    lam = ratio * lambda_star(D, y)
    return Workload("c1", D, y, lam, algorithm="ista", test="dst3", gap_tol=1e-6)


def correlated_dictionary(n, k, seed, rho=0.5):
    """c2 dictionary: N(0,1) columns, then d_i <- d_i + rho*d_{i-1} applied
    simultaneously (right-hand side uses the original draws), then unit norm."""
    raw = make_rng(seed, DICT_STREAM).standard_normal((n, k))
    mixed = raw.copy()
    mixed[:, 1:] = raw[:, 1:] + rho * raw[:, :-1]
    return np.asfortranarray(unit_columns(mixed))


def planted_observation(D, seed, nnz=20, noise=0.01):
    n, k = D.shape
    rng = make_rng(seed, PLANT_STREAM)
    pos = np.sort(rng.choice(k, size=nnz, replace=False))
    x0 = np.zeros(k)
    x0[pos] = rng.standard_normal(nnz)
    y = D @ x0 + noise * make_rng(seed, NOISE_STREAM).standard_normal(n)
    return y / np.linalg.norm(y), x0


def config2(seed=0, ratio=0.5, n=2000, k=10000, test="dst3"):
    """c2: correlated N=2000 x K=10000 fp64, FISTA + dynamic SAFE/ST3, ratio sweep."""
    D = correlated_dictionary(n, k, seed)
    y, x0 = planted_observation(D, seed)
    lam = ratio * lambda_star(D, y)
    return Workload("c2", D, y, lam, algorithm="fista", test=test, gap_tol=1e-6,
                    meta={"ratio": ratio, "x0_support": np.flatnonzero(x0)})


def config3(seed=0, ratio=0.3, n=2000, k=10000, group_size=10, n_active=10, test="gst3"):
    """c3: Gaussian N=2000 x K=10000 fp64 in contiguous groups of 10; lam* uses
    the reference's weighted definition max_g ||D_g^T y|| / sqrt(|g|)."""
    D = gaussian_dictionary(n, k, seed)
    groups = [np.arange(g, g + group_size) for g in range(0, k, group_size)]
    rng = make_rng(seed, PLANT_STREAM)
    on = rng.choice(len(groups), size=n_active, replace=False)
    x0 = np.zeros(k)
    for g in np.sort(on):
        x0[groups[g]] = rng.standard_normal(group_size)
    y = D @ x0 + 0.01 * make_rng(seed, NOISE_STREAM).standard_normal(n)
    y = y / np.linalg.norm(y)
    lam = ratio * lambda_star(D, y, groups)
    return Workload("c3", D, y, lam, algorithm="fista", test=test, gap_tol=1e-6, groups=groups)


def _fp32_gaussian_block(args):
    n, cols, seed, b = args
    blk = make_rng(seed, BLOCK_STREAM_BASE + b).standard_normal((n, cols))
    return (blk / np.linalg.norm(blk, axis=0)).astype(np.float32)


def gaussian_dictionary_f32(n, k, seed, block=4096, threads=8):
    """Column-blocked fp32 Gaussian atoms (block b from stream 100+b), each
    column normalised in fp64 then rounded to fp32.  Used for c4 and its
    proxies; blocking keeps host generation parallel and bounded in memory."""
    out = np.empty((n, k), dtype=np.float32, order="F")
    jobs = [(n, min(block, k - c0), seed, b) for b, c0 in enumerate(range(0, k, block))]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        for (job, blk) in zip(jobs, pool.map(_fp32_gaussian_block, jobs)):
            c0 = job[3] * block
            out[:, c0:c0 + blk.shape[1]] = blk
    return out


def config4(seed=0, ratio=0.2, n=8192, k=262144, gap_tol=1e-5):
    """c4: N=8192 x K=262144 fp32 dictionary (8 GiB), Gaussian unit-norm y, 0.2 lam*,
    FISTA + dynamic ST3, gap 1e-5.  y and all solver state stay fp64."""
    D = gaussian_dictionary_f32(n, k, seed)
    y = gaussian_observation(n, seed)
    corr = np.empty(k)
    for c0 in range(0, k, 16384):
        corr[c0:c0 + 16384] = D[:, c0:c0 + 16384].astype(np.float64).T @ y
    lam = ratio * float(np.max(np.abs(corr)))
    return Workload("c4", D, y, lam, algorithm="fista", test="dst3", gap_tol=gap_tol, dtype="f32")


def bf16_round(a):
    """Round-to-nearest-even fp64/fp32 -> bf16 bit patterns (uint16)."""
    f = np.asarray(a, dtype=np.float32)
    bits = f.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_to_f64(bits):
    return (np.asarray(bits, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)


def config5(seed=0, n=1024, k=16384, batch=4096, nnz=32, noise=0.05, ratio=0.4):
    """c5: shared bf16 dictionary, `batch` planted observations, lam_j = 0.4 max|D^T y_j|.

    Observations are built from the bf16-rounded dictionary (upcast), so the
    solver and the oracle see the same atoms."""
    Dq = bf16_round(gaussian_dictionary(n, k, seed))
    D = bf16_to_f64(Dq).reshape(n, k)
    rng = make_rng(seed, PLANT_STREAM)
    X = np.zeros((k, batch))
    for j in range(batch):
        pos = rng.choice(k, size=nnz, replace=False)
        X[pos, j] = rng.standard_normal(nnz)
    Y = D @ X + noise * make_rng(seed, NOISE_STREAM).standard_normal((n, batch))
    Y /= np.linalg.norm(Y, axis=0)
    lam = ratio * np.max(np.abs(D.T @ Y), axis=0)
    return Workload("c5", np.asfortranarray(Dq.reshape(n, k)), Y, lam, algorithm="fista",
                    test="dst3", gap_tol=0.0, max_iters=100, dtype="bf16")
