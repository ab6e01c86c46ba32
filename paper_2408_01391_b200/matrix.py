"""Matrix plumbing: dtypes, validation, the Gaussian-blob workload, row norms.

``gaussian_mixture`` reproduces the reference generator (matrix.py:86-110)
bit for bit -- same Generator draw order -- but never materialises the
reference's k x k x D float64 temporary and draws the noise in row chunks, so
configs with k = 4096 or N = 1e8 fit in host memory.  ``row_sq_norms`` runs on
the GPU (bit-identical left-to-right sum, _kernels.py:106-114).
"""

from __future__ import annotations

import struct
import sys

import numpy as np

from .errors import FormatError

PRECISIONS = {"single": np.float32, "double": np.float64}
_MAGIC = b"FTKM"
_VERSION = 1
HEADER_SIZE = 28  # magic(4) u32 version u8 precision 3 reserved u64 rows u64 cols


def dtype_of(precision):
    if isinstance(precision, str):
        if precision not in PRECISIONS:
            raise ValueError(f"unknown precision {precision!r}")
        return np.dtype(PRECISIONS[precision])
    dt = np.dtype(precision)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"unsupported dtype {dt}")
    return dt


def precision_of(arr):
    dt = np.dtype(arr.dtype if hasattr(arr, "dtype") else arr)
    if dt == np.float32:
        return "single"
    if dt == np.float64:
        return "double"
    raise ValueError(f"unsupported dtype {dt}")


def as_matrix(x, precision=None):
    """2-D C-contiguous float32/float64 numpy matrix (other dtypes -> float64)."""
    dt = dtype_of(precision) if precision is not None else None
    a = np.ascontiguousarray(x, dtype=dt)
    if a.dtype not in (np.float32, np.float64):
        a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={a.ndim}")
    return a


def _min_pairwise_sq(centers, chunk=256):
    """min_{i != j} sum((c_i - c_j)^2) with the reference's per-pair reduction
    (numpy pairwise sum over the feature axis), computed in row chunks."""
    k = centers.shape[0]
    best = np.inf
    for i0 in range(0, k, chunk):
        blk = ((centers[i0:i0 + chunk, None, :] - centers[None, :, :]) ** 2).sum(axis=2)
        idx = np.arange(blk.shape[0])
        blk[idx, i0 + idx] = np.inf
        best = min(best, float(blk.min()))
    return best


def gaussian_mixture(rows, cols, k, spread, precision="single", seed=0, chunk_rows=1 << 18):
    """(x, labels, centers): k centers in the unit cube rescaled so the minimum
    pairwise distance is >= 20 * spread, uniform labels, isotropic noise."""
    if rows < 1 or cols < 1:
        raise ValueError(f"matrix dimensions must be >= 1, got {rows}x{cols}")
    if k < 1 or k > rows:
        raise ValueError(f"need 1 <= k <= rows, got k={k}, rows={rows}")
    dt = dtype_of(precision)
    rng = np.random.default_rng(seed)
    centers = rng.random((k, cols))
    if k > 1:
        min_dist = np.sqrt(_min_pairwise_sq(centers))
        target = 20.0 * spread
        if min_dist < target:
            centers *= target / max(min_dist, 1e-12)
    labels = rng.integers(0, k, size=rows)
    x = np.empty((rows, cols), dtype=dt)
    for r0 in range(0, rows, chunk_rows):
        r1 = min(rows, r0 + chunk_rows)
        x[r0:r1] = centers[labels[r0:r1]] + spread * rng.standard_normal((r1 - r0, cols))
    return x, labels.astype(np.int64), centers


def mat_load_pinned(path):
    """ftkm-binary -> a page-locked host tensor in the file's precision, the
    payload read straight into pinned memory (one copy less than mat_load,
    and the H2D copy of the fit runs at full PCIe rate).  Same header checks
    and FormatError messages as mat_load (matrix.py:123-172)."""
    import torch

    with open(path, "rb") as fh:
        head = fh.read(HEADER_SIZE)
        if len(head) < HEADER_SIZE or head[:4] != _MAGIC:
            raise FormatError(f"{path}: not an ftkm-binary file")
        version, code = struct.unpack("<IB", head[4:9])
        if version != _VERSION:
            raise FormatError(f"{path}: unsupported version {version}")
        if code not in (4, 8):
            raise FormatError(f"{path}: bad precision code {code}")
        rows, cols = struct.unpack("<QQ", head[12:28])
        if rows < 1 or cols < 1 or rows * cols > 2**48:
            raise FormatError(f"{path}: implausible dimensions {rows}x{cols}")
        x = torch.empty((rows, cols), dtype=torch.float32 if code == 4 else torch.float64,
                        pin_memory=torch.cuda.is_available())
        view = x.numpy().reshape(-1).view(np.uint8)
        got = fh.readinto(memoryview(view))
    if got != view.nbytes:
        raise FormatError(f"{path}: truncated payload")
    if sys.byteorder != "little":
        x.copy_(torch.from_numpy(x.numpy().byteswap()))
    if not bool(torch.isfinite(x).all()):
        i, j = (int(v) for v in torch.nonzero(~torch.isfinite(x))[0])
        raise FormatError(f"{path}: non-finite value at ({i + 1},{j + 1})", i + 1, j + 1)
    return x


def mat_random(rows, cols, precision="single", seed=0, distribution="uniform"):
    if rows < 1 or cols < 1:
        raise ValueError(f"matrix dimensions must be >= 1, got {rows}x{cols}")
    dt = dtype_of(precision)
    if distribution == "uniform":
        return np.ascontiguousarray(np.random.default_rng(seed).random((rows, cols)), dtype=dt)
    if isinstance(distribution, str) and distribution.startswith("gm:"):
        parts = distribution.split(":")
        if len(parts) != 3:
            raise ValueError(f"bad mixture spec {distribution!r}, want gm:k:spread")
        distribution = ("gm", int(parts[1]), float(parts[2]))
    if isinstance(distribution, tuple) and distribution[0] == "gm":
        return gaussian_mixture(rows, cols, distribution[1], distribution[2], dt, seed)[0]
    raise ValueError(f"unknown distribution {distribution!r}")


def row_sq_norms(x):
    """Squared row norms, left-to-right in the row's dtype, on the GPU."""
    from . import _engine

    return _engine.row_sq_norms(as_matrix(x))


def mat_store(x, path, format="ftkm-binary"):
    x = as_matrix(x)
    if format == "ftkm-binary":
        with open(path, "wb") as fh:
            fh.write(_MAGIC + struct.pack("<IB3x", _VERSION, 4 if x.dtype == np.float32 else 8))
            fh.write(struct.pack("<QQ", *x.shape))
            fh.write(np.ascontiguousarray(x, dtype=x.dtype.newbyteorder("<")).tobytes())
    elif format == "csv":
        np.savetxt(path, x, fmt="%.17g", delimiter=",")
    else:
        raise ValueError(f"unknown format {format!r}")


def _csv_cell(path, tok, line_no, col_no):
    """One CSV token -> a finite float, or FormatError at its 1-based
    (file line, column) position (matrix.py:175-212)."""
    try:
        v = float(tok)
    except ValueError:
        raise FormatError(f"{path}: bad value {tok.strip()!r} at ({line_no},{col_no})",
                          row=line_no, col=col_no) from None
    if not np.isfinite(v):
        raise FormatError(f"{path}: non-finite value at ({line_no},{col_no})",
                          row=line_no, col=col_no)
    return v


def _csv_rows(path, dt):
    """The reference's CSV reader semantics: positions are 1-based FILE line
    numbers (blank lines are skipped but still counted), every row must have
    the first row's column count, '#' is an ordinary (bad) token."""
    out, width = [], None
    with open(path, "r") as fh:
        for line_no, raw in enumerate(fh, start=1):
            text = raw.strip()
            if not text:
                continue
            cells = text.split(",")
            width = len(cells) if width is None else width
            if len(cells) != width:
                raise FormatError(f"{path}: row {line_no} has {len(cells)} columns, expected {width}",
                                  row=line_no, col=len(cells))
            out.append([_csv_cell(path, c, line_no, i) for i, c in enumerate(cells, start=1)])
    if not out:
        raise FormatError(f"{path}: empty matrix")
    return np.ascontiguousarray(np.array(out, dtype=np.float64), dtype=dt)


def mat_load(path, format="ftkm-binary", precision="double"):
    if format == "csv":
        return _csv_rows(path, dtype_of(precision))
    if format != "ftkm-binary":
        raise ValueError(f"unknown format {format!r}")
    with open(path, "rb") as fh:
        head = fh.read(HEADER_SIZE)
        if len(head) < HEADER_SIZE or head[:4] != _MAGIC:
            raise FormatError(f"{path}: not an ftkm-binary file")
        version, code = struct.unpack("<IB", head[4:9])
        if version != _VERSION:
            raise FormatError(f"{path}: unsupported version {version}")
        if code not in (4, 8):
            raise FormatError(f"{path}: bad precision code {code}")
        rows, cols = struct.unpack("<QQ", head[12:28])
        if rows < 1 or cols < 1 or rows * cols > 2**48:
            raise FormatError(f"{path}: implausible dimensions {rows}x{cols}")
        dt = np.dtype("<f4") if code == 4 else np.dtype("<f8")
        payload = fh.read(rows * cols * dt.itemsize)
    if len(payload) != rows * cols * dt.itemsize:
        raise FormatError(f"{path}: truncated payload")
    x = np.frombuffer(payload, dtype=dt).reshape(rows, cols)
    x = np.ascontiguousarray(x, dtype=np.float32 if code == 4 else np.float64)
    if not np.isfinite(x).all():
        i, j = np.argwhere(~np.isfinite(x))[0]
        raise FormatError(f"{path}: non-finite value at ({i + 1},{j + 1})", i + 1, j + 1)
    return x
