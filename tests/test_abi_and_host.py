"""CPU tests: the C ABI library loads and exports every declared symbol; host-side
validation mirrors the reference (solvers.py:65-85, problems.py:33-45,
dictionary.py:17-27, 192-216, screening.py:104-112, instrument.py:21-57)."""

import os
import re

import numpy as np
import pytest

import paper_1412_4080_b200 as ds
from paper_1412_4080_b200 import _native as nat
from paper_1412_4080_b200 import workloads as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "dynscreen.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(dscr_\w+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(nat.LIB_PATH):
        from paper_1412_4080_b200 import build
        build.build()
    return nat.load_library()


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) <= set(nat.ABI_FUNCTIONS) | {"dscr_apply_work_size"}
    assert lib.dscr_abi_version() == 1


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", nat.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_ctypes_struct_layouts_match_header(tmp_path):
    """Compile a C probe against include/dynscreen.h and compare every field offset."""
    import ctypes as C
    import subprocess
    structs = {"dscr_problem_desc": nat.ProblemDesc, "dscr_config": nat.Config,
               "dscr_scalars": nat.Scalars, "dscr_solver_buffers": nat.Buffers}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "dynscreen.h"', "int main(void){"]
    for sname, cls in structs.items():
        lines.append(f'printf("{sname} size %zu\\n", sizeof({sname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{sname} {fname} %zu\\n", offsetof({sname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            parts = ln.split()
            got[(parts[0], parts[1])] = int(parts[2])
    for sname, cls in structs.items():
        assert got[(sname, "size")] == C.sizeof(cls), sname
        for fname, _ in cls._fields_:
            assert got[(sname, fname)] == getattr(cls, fname).offset, (sname, fname)


def test_config_validation_messages():
    with pytest.raises(ValueError, match="unknown algorithm"):
        ds.SolverConfig(algorithm="sgd").validate("lasso")
    with pytest.raises(ValueError, match="unknown strategy"):
        ds.SolverConfig(strategy="sometimes").validate("lasso")
    with pytest.raises(ValueError, match="test kind"):
        ds.SolverConfig(strategy="dynamic").validate("lasso")
    with pytest.raises(ValueError, match="does not apply"):
        ds.SolverConfig(strategy="dynamic", test="gsafe").validate("lasso")
    with pytest.raises(ValueError, match="does not apply"):
        ds.SolverConfig(strategy="static", test="dome").validate("group")
    with pytest.raises(ValueError, match="cp_step_safety"):
        ds.SolverConfig(algorithm="cp", cp_step_safety=1.0).validate("lasso")
    with pytest.raises(ValueError, match="max_iters"):
        ds.SolverConfig(max_iters=0).validate("lasso")
    ds.SolverConfig(algorithm="fista", strategy="dynamic", test="dst3").validate("lasso")


def test_problem_validation():
    D = wl.gaussian_dictionary(12, 30, 3)
    y = wl.gaussian_observation(12, 3)
    dic = ds.Dictionary(D)
    with pytest.raises(ValueError, match="unit l2 norm"):
        ds.Problem(dic, 2 * y, 0.1)
    with pytest.raises(ValueError, match="strictly positive"):
        ds.Problem(dic, y, 0.0)
    with pytest.raises(ValueError, match="match the dictionary rows"):
        ds.Problem(dic, np.ones(5) / np.sqrt(5), 0.1)
    with pytest.raises(ValueError, match="unit l2 norm"):
        ds.Dictionary(2 * D)
    p = ds.Problem(dic, y, 0.1)
    assert p.kind == "lasso" and p.n_rows == 12 and p.n_cols == 30


def test_dictionary_dtypes_and_layout():
    D32 = wl.gaussian_dictionary_f32(64, 100, 1)
    dic = ds.Dictionary(D32, check_unit_norms=False, dtype="f32")
    assert ds.Dictionary(D32, check_unit_norms=False).dtype == "f64"   # reference upcast by default
    assert dic.dtype == "f32" and dic.data is D32 and dic.ldd == 64
    dic2 = ds.Dictionary(wl.gaussian_dictionary(1000, 3, 0))
    assert dic2.ldd == 1008
    bits = wl.bf16_round(D32)
    dic3 = ds.Dictionary(np.asfortranarray(bits), check_unit_norms=False, dtype="bf16")
    np.testing.assert_allclose(dic3.as_float64(), wl.bf16_to_f64(bits))
    assert np.max(np.abs(dic3.as_float64() - D32)) < 1e-2


def test_group_partition_validation():
    dic = ds.Dictionary(np.eye(4))
    with pytest.raises(ValueError, match="disjoint"):
        ds.GroupPartition.build(dic, [[0, 1], [1, 2, 3]], spectral_norms=np.ones(2))
    with pytest.raises(ValueError, match="cover"):
        ds.GroupPartition.build(dic, [[0, 1], [2]], spectral_norms=np.ones(2))
    with pytest.raises(ValueError, match="nonempty"):
        ds.GroupPartition.build(dic, [[0, 1, 2, 3], []], spectral_norms=np.ones(2))
    part = ds.GroupPartition.build(dic, [[0, 2], [1, 3]], spectral_norms=np.ones(2))
    assert np.allclose(part.weights, np.sqrt(2)) and part.n_groups == 2 and part.size == 4


def test_index_set_and_expand():
    with pytest.raises(ValueError, match="strictly increasing"):
        ds.index_set([2, 1])
    with pytest.raises(ValueError):
        ds.index_set([0, 5], size=5)
    assert np.array_equal(ds.expand([1.0, 2.0], [1, 3], 5), [0, 1, 0, 2, 0])


def test_screen_state_algebra():
    st = ds.ScreenState.initial(6)
    m1 = np.array([True, False, False, True, False, False])
    m2 = np.array([False, True, False, True])
    two = ds.screen_update(ds.screen_update(st, m1), m2)
    one = ds.screen_update(st, np.array([True, False, True, True, False, True]))
    assert np.array_equal(two.eliminated, one.eliminated) and np.array_equal(two.kept, one.kept)
    assert ds.screen_update(st, np.zeros(6, bool)) is st
    with pytest.raises(ValueError, match="align"):
        ds.screen_update(st, np.zeros(3, bool))


def test_flops_model_worked_values():
    assert ds.flops_iteration("lasso", "none", 10, 5, 10, 2) == 105
    assert ds.flops_iteration("lasso", "dynamic", 10, 5, 6, 2) == 101
    assert ds.flops_iteration("group", "dynamic", 10, 5, 6, 2, 3) == 122
    assert ds.flops_static_init(7, 3) == 21


def test_workload_generators_deterministic():
    a = wl.config2(seed=3, n=50, k=200)
    b = wl.config2(seed=3, n=50, k=200)
    assert a.D.tobytes() == b.D.tobytes() and np.array_equal(a.y, b.y) and a.lam == b.lam
    assert np.allclose(np.linalg.norm(a.D, axis=0), 1.0) and abs(np.linalg.norm(a.y) - 1) < 1e-12
    c = wl.config3(seed=1, n=40, k=100, group_size=10, n_active=2)
    assert len(c.groups) == 10 and c.lam < wl.lambda_star(c.D, c.y, c.groups)
    f = wl.gaussian_dictionary_f32(32, 9000, 2)
    assert f.dtype == np.float32 and f.flags.f_contiguous
    assert np.max(np.abs(np.linalg.norm(f.astype(np.float64), axis=0) - 1)) < 1e-6


def test_reference_generators_match_reference_bytes():
    """workloads restates screenlab.datagen; pin against the committed golden inputs."""
    from tests.golden_cases import load
    cases = {c["name"]: c for c in load()}
    c = cases["lasso_s3_12x30_r0.7"]
    assert np.array_equal(wl.gaussian_dictionary(12, 30, 3), c["D"])
    assert np.array_equal(wl.gaussian_observation(12, 3), c["y"])
    g = cases["group_s12_12x30_r0.5"]
    groups = wl.random_groups(30, 3, 12)
    got = np.empty(30, dtype=np.int64)
    for gid, grp in enumerate(groups):
        got[grp] = gid
    want = np.empty(30, dtype=np.int64)
    for gid, grp in enumerate(g["groups"]):
        want[grp] = gid
    assert np.array_equal(got, want)
    D = wl.gaussian_dictionary(12, 30, 12)
    assert np.array_equal(wl.bernoulli_gaussian_observation(D, groups, 12, p=0.2), g["y"])


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = ds.Problem(ds.Dictionary(np.eye(2)), np.array([1.0, 0.0]), 0.5)
    with pytest.raises(RuntimeError, match="CUDA device"):
        ds.run(p, ds.SolverConfig())


def test_peer_buffer_size_is_flags_plus_two_receive_areas(lib):
    """Host-only sizing of the native exchange buffer: 64 uint64 flags + [2][world][len] doubles,
    len = SUM scalars + 2 * ldd residual partials + 8 slot doubles per rank."""
    for world, ldd in ((1, 1024), (2, 8192), (8, 8192), (64, 16)):
        length = (nat.CM_VEC - nat.CM_SUM) + 2 * ldd + nat.OC_SLOT * world
        assert lib.dscr_peer_buffer_bytes(world, ldd) == 64 * 8 + 2 * world * length * 8
    assert lib.dscr_peer_buffer_bytes(0, 1024) == 0
    assert lib.dscr_peer_buffer_bytes(65, 1024) == 0
    assert lib.dscr_peer_buffer_bytes(2, 0) == 0
