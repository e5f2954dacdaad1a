"""DSMX ingestion throughput vs the host path (read + transpose + upload): python scripts/time_dsmx.py [dir]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4080_b200 as ds  # noqa: E402
from paper_1412_4080_b200 import dsmx  # noqa: E402

d = sys.argv[1] if len(sys.argv) > 1 else "/tmp"
n, k = 8192, 32768
path = os.path.join(d, "bench.dsmx")
rng = np.random.default_rng(0)
D = rng.standard_normal((n, k), dtype=np.float64)
dsmx.write_dsmx(path, D)
del D
gb = n * k * 8 / 1e9
dev = torch.device("cuda", 0)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dic = dsmx.load_dictionary(path, dtype="f32", check_unit_norms=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    host = dsmx.read_dsmx(path).astype(np.float32)
    ref = ds.Dictionary(host, check_unit_norms=False, dtype="f32")
    ref.device_data(dev)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    same = torch.equal(dic.device_data(dev), ref.device_data(dev))
    print(f"{gb:.2f} GB fp64 file -> fp32 device: ingest {t1 - t0:.2f} s ({gb / (t1 - t0):.1f} GB/s), "
          f"host read+transpose+upload {t2 - t1:.2f} s, identical={same}", flush=True)
    del dic, ref, host
os.remove(path)
