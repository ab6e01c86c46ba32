"""Fused nearest-centroid assignment (reference gemm.py).

``fused_assign`` / ``gemm_tiled`` keep the reference signatures, validation
and results; the work runs on the B200 through ``ftk_assign`` / ``ftk_gemm``
(include/ftk_b200.h).  ``min_dists`` holds ``|y|^2 - 2 x.y`` at the winner,
bit-identical to the reference (the exact kernel evaluates it in the same
order; the tensor-core variant certifies the argmin and recomputes the winner
exactly).  ``threads`` is accepted for compatibility and validated; the GPU
does not use it.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _engine as E
from .matrix import as_matrix
from .tiles import TileConfig, default_config

_VARIANT = os.environ.get("FTK_VARIANT", "auto")


def set_variant(name):
    """Select the assign kernel family: 'auto' (variants.resolve: the
    measured variant table, else tensor cores where they apply), 'exact',
    'tc', or a family of variants.FAMILIES ('pair', 'narrow', 'dmma',
    'dfma')."""
    global _VARIANT
    E.variant_code(name)
    _VARIANT = name


def get_variant():
    return _VARIANT


@dataclass
class AssignResult:
    assignments: np.ndarray
    min_dists: np.ndarray


def resolve_threads(threads):
    """Reference semantics (gemm.py:32-40): arg > FTKM_THREADS > cpu count."""
    if threads is not None:
        n = int(threads)
    else:
        env = os.environ.get("FTKM_THREADS")
        n = int(env) if env else (os.cpu_count() or 1)
    if n < 1:
        raise ValueError(f"threads must be >= 1, got {n}")
    return n


def _is_torch(a):
    try:
        import torch
    except ImportError:
        return False
    return isinstance(a, torch.Tensor)


def _as_operand(a):
    if _is_torch(a):
        if a.dim() != 2:
            raise ValueError(f"expected a 2-D matrix, got ndim={a.dim()}")
        if E.ndtype(a.dtype) not in (np.float32, np.float64):
            raise ValueError(f"unsupported dtype {a.dtype}")
        return a
    return as_matrix(a)


def _dtype(a):
    return E.ndtype(a.dtype) if _is_torch(a) else a.dtype


def _check_pair(a, b, cfg):
    a, b = _as_operand(a), _as_operand(b)
    if _dtype(a) != _dtype(b):
        raise ValueError(f"operand dtypes differ: {_dtype(a)} vs {_dtype(b)}")
    if a.shape[1] != b.shape[1]:
        raise ValueError(f"inner dimensions differ: {a.shape[1]} vs {b.shape[1]} "
                         "(second operand is indexed transposed)")
    if cfg is None:
        cfg = default_config(_dtype(a))
    elif isinstance(cfg, TileConfig):
        cfg.validate()
    else:
        raise ValueError(f"cfg must be a TileConfig or None, got {type(cfg)!r}")
    return a, b, cfg


def _ynorms_dev(y_t, y_norms, dtype, k):
    if y_norms is None:
        return E.row_sq_norms_dev(y_t)
    if _is_torch(y_norms):
        yn = y_norms.to(device=y_t.device, dtype=y_t.dtype).contiguous()
    else:
        yn = E.to_dev(np.ascontiguousarray(y_norms, dtype=dtype))
    if tuple(yn.shape) != (k,):
        raise ValueError(f"y_norms must have length {k}")
    return yn


def gemm_tiled(a, b, cfg=None, threads=None):
    """``a @ b.T`` (materialised), same bits as the reference's tiled kernel."""
    a, b, cfg = _check_pair(a, b, cfg)
    resolve_threads(threads)
    if a.shape[0] == 0 or b.shape[0] == 0:
        return np.empty((a.shape[0], b.shape[0]), dtype=_dtype(a))
    out = E.gemm_dev(E.to_dev(a), E.to_dev(b), cfg.block)
    return E.to_host(out)


def fused_assign(x, y, y_norms=None, cfg=None, threads=None, hook=None, iteration=0):
    """Nearest row of ``y`` for every row of ``x`` (ties -> lowest index)."""
    x, y, cfg = _check_pair(x, y, cfg)
    dt = _dtype(x)
    resolve_threads(threads)
    m, k = x.shape[0], y.shape[0]
    x_t, y_t = E.to_dev(x), E.to_dev(y)
    yn_t = _ynorms_dev(y_t, y_norms, dt, k)
    if m == 0:
        return AssignResult(np.empty(0, np.int64), np.empty(0, dt))
    inj = E.injection_for(hook, iteration, dt)
    from .variants import resolve

    idx, val = E.assign_dev(x_t, y_t, yn_t, cfg.block, variant=resolve((m, x.shape[1], k), dt),
                            inj=inj)
    labels = E.to_host(idx).astype(np.int64)
    md = E.to_host(val)
    if inj is not None:
        inj.finish()
    if hook is not None:
        arrs = inj.host if inj is not None else None
        if arrs is not None:
            hook.absorb_kernel_results(iteration, arrs[5], arrs[6], arrs[7])
        else:
            hook.absorb_kernel_results(iteration, np.zeros(0, np.int64), np.zeros(0),
                                       np.zeros(0))
    return AssignResult(assignments=labels, min_dists=md)


def true_sq_dists(result, x):
    """min_dists + |x|^2 in float64 (gemm.py:144-146)."""
    from .matrix import row_sq_norms

    return result.min_dists.astype(np.float64) + row_sq_norms(x).astype(np.float64)
