"""DSMX container (dictionary.py:304-335): byte-compatible writer/reader, header validation."""

import os
import struct

import numpy as np
import pytest

from paper_1412_4080_b200 import dsmx

HERE = os.path.join(os.path.dirname(__file__), "golden")


def test_writer_matches_reference_bytes(tmp_path):
    M = np.load(os.path.join(HERE, "small_dsmx_matrix.npy"))
    ref = open(os.path.join(HERE, "small.dsmx"), "rb").read()
    p = tmp_path / "ours.dsmx"
    dsmx.write_dsmx(p, M)
    assert p.read_bytes() == ref
    assert np.array_equal(dsmx.read_dsmx(os.path.join(HERE, "small.dsmx")), M)
    assert dsmx.read_dsmx_header(p) == (5, 7, 24)


def test_header_validation(tmp_path):
    good = open(os.path.join(HERE, "small.dsmx"), "rb").read()
    cases = {
        "truncated DSMX header": good[:10],
        "not a DSMX file": b"XXXX" + good[4:],
        "unsupported DSMX version 2": good[:4] + struct.pack("<I", 2) + good[8:],
        "payload bytes": good[:-8],
    }
    for msg, blob in cases.items():
        p = tmp_path / "bad.dsmx"
        p.write_bytes(blob)
        with pytest.raises(ValueError, match=msg):
            dsmx.read_dsmx_header(p)
