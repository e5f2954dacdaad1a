"""DSMX dictionaries straight to the device.

The reference's container (dictionary.py:304-335): magic ``DSMX``, u32 version 1,
u64 rows, u64 cols, then a row-major little-endian fp64 payload.  ``write_dsmx`` /
``read_dsmx`` restate it (byte-compatible with the reference).  ``load_dictionary``
ingests a file without a host-side transpose or fp64 host copy: the payload is
memory-mapped, row blocks stream through two pinned staging buffers to the device
(copy stream, double-buffered), and a kernel (``dscr_ingest_rows_f64``) transposes
each block into the column-major padded engine layout in the storage dtype (fp64 /
fp32 / bf16, the rounding of ``workloads.bf16_round``).  The host copy the
``Dictionary`` keeps is one device-to-host transfer of the stored values into
pinned memory (which is also its re-upload source).
"""

from __future__ import annotations

import struct

import numpy as np

from . import _native as nat
from .problem import UNIT_NORM_TOL, Dictionary, _pad16

DSMX_MAGIC = b"DSMX"
DSMX_VERSION = 1
_HEADER = struct.Struct("<4sIQQ")


def write_dsmx(path, matrix):
    """Dense float64 matrix in the DSMX container (dictionary.py:304-318)."""
    arr = np.ascontiguousarray(matrix, dtype="<f8")
    if arr.ndim == 1:
        arr = arr[:, None]
    if arr.ndim != 2:
        raise ValueError("DSMX stores 2-D matrices")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(DSMX_MAGIC, DSMX_VERSION, arr.shape[0], arr.shape[1]))
        fh.write(arr.tobytes(order="C"))


def read_dsmx_header(path):
    """(rows, cols, payload offset); the reference's validation (dictionary.py:321-335)."""
    with open(path, "rb") as fh:
        header = fh.read(_HEADER.size)
        if len(header) != _HEADER.size:
            raise ValueError(f"{path}: truncated DSMX header")
        magic, version, rows, cols = _HEADER.unpack(header)
        if magic != DSMX_MAGIC:
            raise ValueError(f"{path}: not a DSMX file")
        if version != DSMX_VERSION:
            raise ValueError(f"{path}: unsupported DSMX version {version}")
        fh.seek(0, 2)
        payload = fh.tell() - _HEADER.size
    if payload != rows * cols * 8:
        raise ValueError(f"{path}: expected {rows * cols * 8} payload bytes, got {payload}")
    return int(rows), int(cols), _HEADER.size


def read_dsmx(path):
    """Host read, (rows, cols) float64 (dictionary.py:321-335)."""
    rows, cols, off = read_dsmx_header(path)
    return np.array(np.memmap(path, dtype="<f8", mode="r", offset=off, shape=(rows, cols)), dtype=np.float64)


_TORCH_DTYPES = {"f64": "float64", "f32": "float32", "bf16": "uint16"}


def load_dictionary(path, dtype="f64", device=None, check_unit_norms=True, stage_bytes=256 << 20):
    """Dictionary from a DSMX file, ingested on the device (see the module docstring)."""
    import torch
    if dtype not in _TORCH_DTYPES:
        raise ValueError(f"unknown dictionary dtype {dtype!r}")
    rows, cols, off = read_dsmx_header(path)
    if rows < 1 or cols < 1:
        raise ValueError("dictionary must have at least one row and one column")
    L = nat.lib()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    code = {"f64": nat.F64, "f32": nat.F32, "bf16": nat.BF16}[dtype]
    tdt = getattr(torch, _TORCH_DTYPES[dtype])
    ldd = _pad16(rows)
    mm = np.memmap(path, dtype="<f8", mode="r", offset=off, shape=(rows, cols))
    D = torch.zeros((cols, ldd), dtype=tdt, device=dev)
    R = max(1, min(rows, stage_bytes // (cols * 8)))
    stage = [torch.empty((R, cols), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    dstage = [torch.empty((R, cols), dtype=torch.float64, device=dev) for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    compute = torch.cuda.current_stream(dev)
    h2d = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]
    sptr = nat.C.c_void_p(compute.cuda_stream)
    for bi, r0 in enumerate(range(0, rows, R)):
        b = bi & 1
        nr = min(R, rows - r0)
        if used[b]:
            h2d[b].synchronize()                     # pinned buffer b free again
        np.copyto(stage[b].numpy()[:nr], mm[r0:r0 + nr])
        with torch.cuda.stream(copy_stream):
            if used[b]:
                copy_stream.wait_event(done[b])      # device buffer b consumed by its kernel
            dstage[b][:nr].copy_(stage[b][:nr], non_blocking=True)
            h2d[b].record(copy_stream)
        compute.wait_event(h2d[b])
        nat.check(L.dscr_ingest_rows_f64(dstage[b].data_ptr(), nr, cols, r0, code, D.data_ptr(), ldd, sptr))
        done[b].record(compute)
        used[b] = True
    torch.cuda.synchronize(dev)
    if check_unit_norms:      # on the stored values' fp64 upcast, like Dictionary(...)
        if dtype == "bf16":
            up = (D[:, :rows].to(torch.int32) << 16).view(torch.float32).double()
        else:
            up = D[:, :rows].double()
        worst = float((torch.linalg.vector_norm(up, dim=1) - 1.0).abs().max())
        if worst > UNIT_NORM_TOL:
            raise ValueError(f"columns must have unit l2 norm (worst deviation {worst:.3e})")
    host = torch.empty((cols, rows), dtype=tdt, pin_memory=True)
    host.copy_(D[:, :rows])
    dic = Dictionary(host.numpy().T, check_unit_norms=False, dtype=dtype)    # F-contiguous view, no copy
    dic.col_norm_checked = bool(check_unit_norms)
    dic._host_tensor = host
    dic._dev[(str(dev), None)] = D
    return dic
