"""A small DSMX file written by the reference's own writer (dictionary.py:304-318).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_dsmx_golden.py
"""
import os

import numpy as np

from screenlab.dictionary import write_dsmx

rng = np.random.default_rng(42)
M = rng.standard_normal((5, 7))
write_dsmx(os.path.join(os.path.dirname(__file__), "small.dsmx"), M)
np.save(os.path.join(os.path.dirname(__file__), "small_dsmx_matrix.npy"), M)
