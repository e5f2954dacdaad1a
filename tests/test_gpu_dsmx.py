"""DSMX ingestion straight to the device: bit-identical to the in-memory Dictionary path."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import dsmx  # noqa: E402
from paper_1412_4080_b200 import workloads as wl  # noqa: E402


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
@pytest.mark.parametrize("shape", [(37, 100), (64, 33), (200, 1000)])
def test_load_dictionary_matches_in_memory(tmp_path, dtype, shape):
    rng = np.random.default_rng(shape[0] + shape[1])
    D = rng.standard_normal(shape)
    D /= np.linalg.norm(D, axis=0)
    p = tmp_path / "d.dsmx"
    dsmx.write_dsmx(p, D)
    dev = torch.device("cuda", 0)
    got = dsmx.load_dictionary(p, dtype=dtype, check_unit_norms=(dtype == "f64"), stage_bytes=24 * shape[1] * 8)
    if dtype == "f64":
        ref = ds.Dictionary(D)
    elif dtype == "f32":
        ref = ds.Dictionary(D.astype(np.float32), check_unit_norms=False, dtype="f32")
    else:
        ref = ds.Dictionary(wl.bf16_round(D), check_unit_norms=False, dtype="bf16")
    assert np.array_equal(got.data, ref.data)                       # host copy of the stored values
    assert torch.equal(got.device_data(dev), ref.device_data(dev))  # engine layout, padding rows zero
    got.drop_device()
    assert torch.equal(got.device_data(dev), ref.device_data(dev))  # pinned re-upload path


def test_loaded_dictionary_solves_identically(tmp_path):
    w = wl.config1()
    p = tmp_path / "c1.dsmx"
    dsmx.write_dsmx(p, w.D)
    dic = dsmx.load_dictionary(p)
    a = ds.run(ds.Problem(dic, w.y, w.lam), ds.SolverConfig(algorithm="ista", strategy="dynamic", test="dst3",
                                                             max_iters=50, rel_tol=1e-300))
    b = ds.run(ds.Problem(ds.Dictionary(w.D), w.y, w.lam),
               ds.SolverConfig(algorithm="ista", strategy="dynamic", test="dst3", max_iters=50, rel_tol=1e-300))
    assert a.iterations == b.iterations and np.array_equal(a.x_star, b.x_star)
    with pytest.raises(ValueError, match="unit l2 norm"):
        bad = w.D.copy()
        bad[:, 3] *= 1.01
        dsmx.write_dsmx(p, bad)
        dsmx.load_dictionary(p)
