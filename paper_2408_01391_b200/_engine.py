"""Device-side driver: torch owns device memory and the stream, the C ABI
(libftkb200.so) does every numeric operation.  No CPU fallback exists; every
entry point raises when CUDA or the extension is missing.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

_CTX = {}
_ROWS_OWNER = {}  # device -> id of the RowInfo registered on its context
_VARIANT = {"auto": N.VARIANT_AUTO, "exact": N.VARIANT_EXACT, "tc": N.VARIANT_TC,
            "pair": N.VARIANT_TC_PAIR, "narrow": N.VARIANT_TC_NARROW,
            "dmma": N.VARIANT_F64_DMMA, "dfma": N.VARIANT_F64_DFMA}


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 engine has no CPU fallback")
    return torch


def device():
    t = _torch()
    return t.device("cuda", t.cuda.current_device())


def ctx():
    t = _torch()
    dev = t.cuda.current_device()
    if dev not in _CTX:
        lib = N.load()
        c = lib.ftk_ctx_create(dev)
        if not c:
            raise N.FTKError("ftk_ctx_create failed: " + lib.ftk_last_error().decode())
        _CTX[dev] = c
    return _CTX[dev]


def stream():
    return _torch().cuda.current_stream().cuda_stream


def code(dtype):
    return N.FTK_F32 if np.dtype(dtype) == np.float32 else N.FTK_F64


def tdtype(dtype):
    t = _torch()
    return t.float32 if np.dtype(dtype) == np.float32 else t.float64


def ndtype(tensor_dtype):
    t = _torch()
    return np.dtype(np.float32) if tensor_dtype == t.float32 else np.dtype(np.float64)


def ptr(t):
    return None if t is None else (t.data_ptr() or None)


def to_dev(a, dtype=None, copy=False):
    """numpy / torch (any device) -> contiguous CUDA tensor (`copy`: never
    alias a CUDA input, e.g. for a buffer that outlives the call)."""
    t = _torch()
    if isinstance(a, t.Tensor):
        out = a.to(device=device(), dtype=tdtype(dtype) if dtype is not None else a.dtype,
                   non_blocking=True, copy=copy)
        return out.contiguous()
    arr = np.ascontiguousarray(a, dtype=dtype)
    if arr.nbytes < _H2D_MIN:
        return t.from_numpy(arr).to(device(), non_blocking=False)
    out = t.empty(arr.shape, dtype=t.from_numpy(arr[:0]).dtype, device=device())
    upload_into(out, arr)
    return out


_H2D_MIN = 8 << 20  # below this the driver's own pageable copy is as fast


def upload_into(dst_t, arr):
    """Copy a C-contiguous host numpy array into the device tensor `dst_t`
    (same bytes) through the staged pageable uploader (ftk_h2d); the current
    stream is ordered behind it.  The source may be reused on return."""
    arr = np.ascontiguousarray(arr)
    assert dst_t.is_contiguous() and dst_t.numel() * dst_t.element_size() == arr.nbytes
    N.check(N.load().ftk_h2d(ctx(), ptr(dst_t), arr.ctypes.data, arr.nbytes, stream()), "ftk_h2d")


def to_host(tensor):
    return tensor.detach().cpu().numpy()


def variant_code(variant):
    if variant not in _VARIANT:
        raise ValueError(f"unknown kernel variant {variant!r}")
    return _VARIANT[variant]


# ------------------------------------------------------------- hooks -----
class DevInjection:
    """FaultHook.kernel_arrays (8 host arrays) mirrored on the device."""

    def __init__(self, arrs):
        t = _torch()
        bi, bj, ei, ej, bit, applied, before, after = arrs
        n = len(bi)
        self.n = n
        self.host = arrs
        idx = np.stack([np.asarray(v, np.int64) for v in (bi, bj, ei, ej, bit)]) if n else \
            np.zeros((5, 0), np.int64)
        self.idx = t.from_numpy(np.ascontiguousarray(idx)).to(device())
        self.applied = t.zeros(max(n, 1), dtype=t.int64, device=device())
        self.ba = t.zeros((2, max(n, 1)), dtype=t.float64, device=device())
        base = self.idx.data_ptr()
        self.struct = N.Injection(
            n, *(base + 8 * n * c for c in range(5)), self.applied.data_ptr(),
            self.ba[0].data_ptr(), self.ba[1].data_ptr())

    def ref(self):
        import ctypes

        return ctypes.byref(self.struct)

    def finish(self):
        """Copy applied/before/after back into the hook's host arrays."""
        if self.n == 0:
            return
        applied = to_host(self.applied)[: self.n]
        ba = to_host(self.ba)[:, : self.n]
        self.host[5][:] = applied
        self.host[6][:] = ba[0]
        self.host[7][:] = ba[1]


class StaticInjection:
    """Fixed-address injection arrays with the live count on the device
    (ftk_injection.n_dev), for CUDA-graph replay of injected passes: `load`
    stages one pass's schedule (pinned host -> device, stream-ordered before
    the replay), the captured graph copies applied/before/after back into
    pinned host memory, `finish` hands them to the hook after the step's
    synchronisation."""

    def __init__(self, cap):
        t = _torch()
        self.cap = int(cap)
        self.idx = t.zeros((5, self.cap), dtype=t.int64, device=device())
        self.n_dev = t.zeros(1, dtype=t.int64, device=device())
        self.applied = t.zeros(self.cap, dtype=t.int64, device=device())
        self.ba = t.zeros((2, self.cap), dtype=t.float64, device=device())
        self.idx_h = t.zeros((5, self.cap), dtype=t.int64).pin_memory()
        self.n_h = t.zeros(1, dtype=t.int64).pin_memory()
        self.applied_h = t.zeros(self.cap, dtype=t.int64).pin_memory()
        self.ba_h = t.zeros((2, self.cap), dtype=t.float64).pin_memory()
        base = self.idx.data_ptr()
        self.struct = N.Injection(self.cap, *(base + 8 * self.cap * c for c in range(5)),
                                  self.applied.data_ptr(), self.ba[0].data_ptr(),
                                  self.ba[1].data_ptr(), self.n_dev.data_ptr())
        self.n = 0
        self.host = None

    def ref(self):
        import ctypes

        return ctypes.byref(self.struct)

    def load(self, arrs):
        """Stage the pass's schedule (None: no flips); False if over capacity."""
        n = 0 if arrs is None else len(arrs[0])
        if n > self.cap:
            return False
        self.n, self.host = n, arrs
        if n:
            self.idx_h[:, :n] = torch_from(np.stack([np.asarray(v, np.int64) for v in arrs[:5]]))
        self.n_h[0] = n
        self.idx.copy_(self.idx_h, non_blocking=True)
        self.n_dev.copy_(self.n_h, non_blocking=True)
        return True

    def copy_back(self):
        """Captured with the pass: device outputs -> pinned host."""
        self.applied_h.copy_(self.applied, non_blocking=True)
        self.ba_h.copy_(self.ba, non_blocking=True)

    def finish(self):
        if self.n == 0 or self.host is None:
            return
        n = self.n
        self.host[5][:] = self.applied_h.numpy()[:n]
        self.host[6][:] = self.ba_h.numpy()[0, :n]
        self.host[7][:] = self.ba_h.numpy()[1, :n]


def torch_from(a):
    return _torch().from_numpy(np.ascontiguousarray(a))


def ctx_generation():
    return int(N.load().ftk_ctx_generation(ctx()))


def injection_for(hook, iteration, dtype):
    if hook is None:
        return None
    arrs = hook.kernel_arrays(iteration, np.dtype(dtype))
    if arrs is None:
        return None
    return DevInjection(arrs)


class DevEvents:
    """Detection-event ring on the device (abft.py:281-294)."""

    def __init__(self, cap, storage=None):
        t = _torch()
        self.cap = int(cap)
        self.storage = max(self.cap, int(storage or 0), 1)
        self.gen = 0  # bumped when the buffers move (captured CUDA graphs go stale)
        self.rec = t.zeros((self.storage, 7), dtype=t.int64, device=device())
        self.delta = t.zeros(self.storage, dtype=t.float64, device=device())
        self.count = t.zeros(1, dtype=t.int64, device=device())
        self.struct = N.Events(self.cap, self.rec.data_ptr(), self.delta.data_ptr(),
                               self.count.data_ptr())

    def set_cap(self, cap):
        """Logical capacity of the next launch (the overflow rule of
        abft.py:315-316); the buffers only move when `cap` exceeds storage."""
        cap = int(cap)
        if cap > self.storage:
            t = _torch()
            self.storage = max(cap, 2 * self.storage)
            self.rec = t.zeros((self.storage, 7), dtype=t.int64, device=device())
            self.delta = t.zeros(self.storage, dtype=t.float64, device=device())
            self.count = t.zeros(1, dtype=t.int64, device=device())
            self.gen += 1
        self.cap = cap
        self.struct = N.Events(cap, self.rec.data_ptr(), self.delta.data_ptr(),
                               self.count.data_ptr())

    def ref(self):
        import ctypes

        return ctypes.byref(self.struct)

    def reset(self):
        self.count.zero_()

    def read(self, n=None, cap=None):
        """-> (overflowed, [(rec7..., delta)]); `n` = the count if the caller
        already copied it to the host (saves a synchronisation), `cap` the
        logical capacity when the launch ran with a larger one (graphs)."""
        n = int(self.count.item()) if n is None else int(n)
        cap = self.cap if cap is None else min(int(cap), self.storage)
        m = min(n, cap)
        if m == 0:
            return n > cap, []
        rec = to_host(self.rec[:m])
        delta = to_host(self.delta[:m])
        return n > cap, [(tuple(int(v) for v in rec[i]), float(delta[i])) for i in range(m)]


# ------------------------------------------------------------ kernels ----
def set_label_hint(labels_t, m):
    """Previous-iteration labels as the assignment's speed hint
    (ftk_ctx_set_label_hint); None clears it."""
    N.check(N.load().ftk_ctx_set_label_hint(ctx(), None if labels_t is None else ptr(labels_t),
                                            int(m) if labels_t is not None else 0),
            "ftk_ctx_set_label_hint")


def set_inj_replay(on):
    """FTK_OPT_INJ_REPLAY: exact replay of blocks with scheduled flips (default on)."""
    N.check(N.load().ftk_ctx_set_option(ctx(), 1, 1 if on else 0), "ftk_ctx_set_option")


def row_sq_norms_dev(x_t):
    t = _torch()
    out = t.empty(x_t.shape[0], dtype=x_t.dtype, device=x_t.device)
    N.check(N.load().ftk_row_sq_norms(ctx(), code(ndtype(x_t.dtype)), ptr(x_t), x_t.shape[0],
                                      x_t.shape[1], ptr(out), stream()), "ftk_row_sq_norms")
    return out


class RowInfo:
    """Per-fit screening bounds of the data matrix (ftk_row_info; float64
    data also keep the fp32 copy the tensor cores screen, ftk_row_info64),
    registered on the context for the lifetime of a fit (ftk_ctx_set_rows /
    ftk_ctx_set_rows64); ``close`` unregisters them before the data can be
    freed or modified."""

    def __init__(self, x_t):
        t = _torch()
        self.x_t = x_t
        self.info = None
        self.x32 = None
        if x_t.dtype not in (t.float32, t.float64) or x_t.shape[0] == 0:
            return
        m, d = x_t.shape
        if x_t.dtype == t.float64:
            if d % 4 or d > 256:  # no tensor-core screen for this shape (tc64.cu)
                return
            self.x32 = t.empty((m, d), dtype=t.float32, device=x_t.device)
        self.info = t.empty((m, 4), dtype=t.float32, device=x_t.device)
        self._compute()

    def _compute(self):
        m, d = self.x_t.shape
        lib = N.load()
        if self.x32 is None:
            N.check(lib.ftk_row_info(ctx(), ptr(self.x_t), m, d, ptr(self.info), stream()), "ftk_row_info")
            N.check(lib.ftk_ctx_set_rows(ctx(), ptr(self.x_t), m, d, ptr(self.info)), "ftk_ctx_set_rows")
        else:
            N.check(lib.ftk_row_info64(ctx(), ptr(self.x_t), m, d, ptr(self.x32), ptr(self.info), stream()),
                    "ftk_row_info64")
            N.check(lib.ftk_ctx_set_rows64(ctx(), ptr(self.x_t), m, d, ptr(self.x32), ptr(self.info)),
                    "ftk_ctx_set_rows64")
        _ROWS_OWNER[self.x_t.device.index] = id(self)

    def refresh(self):
        """Recompute the bounds in place after x_t's contents changed (same
        buffers, so captured graphs stay valid) and register them again."""
        if self.info is None:
            return
        self._compute()

    def close(self):
        if self.info is not None:
            dev = self.x_t.device.index
            if _ROWS_OWNER.get(dev) == id(self):  # a later fit may own the slot now
                N.load().ftk_ctx_set_rows(ctx(), None, 0, 0, None)
                _ROWS_OWNER.pop(dev, None)
            self.info = None
            self.x32 = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kpp_buffers(m, k, dev):
    """(d2 f64[m], picks i64[k], total f64[1], pick i64[1], replays u64[1])."""
    t = _torch()
    return (t.empty(m, dtype=t.float64, device=dev), t.zeros(k, dtype=t.int64, device=dev),
            t.empty(1, dtype=t.float64, device=dev), t.zeros(1, dtype=t.int64, device=dev),
            t.zeros(1, dtype=t.int64, device=dev))


def kpp_update_dev(x_t, host_pick, pick_dev, first, d2, picks, c):
    """k-means++ D^2 update (ftk_kpp_update); the pick is `host_pick` if >= 0,
    else the device scalar `pick_dev`; picks[c] records it."""
    m, d = x_t.shape
    N.check(N.load().ftk_kpp_update(ctx(), code(ndtype(x_t.dtype)), ptr(x_t), m, d, int(host_pick),
                                    ptr(pick_dev), int(bool(first)), ptr(d2), ptr(picks), int(c),
                                    stream()), "ftk_kpp_update")


def kpp_search_dev(d2, r, pick_dev, n_replays):
    """pick_dev <- min(searchsorted(cumsum(d2), r, 'right'), m - 1), bit-exact."""
    N.check(N.load().ftk_kpp_search(ctx(), ptr(d2), d2.shape[0], float(r), ptr(pick_dev),
                                    ptr(n_replays), stream()), "ftk_kpp_search")


def row_sq_norms(x):
    if x.shape[0] == 0:
        return np.empty(0, dtype=x.dtype)
    return to_host(row_sq_norms_dev(to_dev(x)))


def assign_dev(x_t, y_t, yn_t, block, variant="auto", inj=None, checked=False, delta_rel=0.0,
               abs_tol=0.0, iteration=0, events=None, out_idx=None, out_val=None):
    """Launch the fused assignment; returns (labels int32 tensor, min_dists tensor)."""
    t = _torch()
    m, d = x_t.shape
    k = y_t.shape[0]
    dt = ndtype(x_t.dtype)
    if out_idx is None:
        out_idx = t.empty(m, dtype=t.int32, device=x_t.device)
    if out_val is None:
        out_val = t.empty(m, dtype=x_t.dtype, device=x_t.device)
    bm, bn, bk = (int(v) for v in block)
    lib = N.load()
    injp = inj.ref() if inj is not None else None
    if checked:
        rc = lib.ftk_checked_assign(ctx(), code(dt), variant_code(variant), ptr(x_t), ptr(y_t),
                                    ptr(yn_t), m, k, d, bm, bn, bk, float(delta_rel),
                                    float(abs_tol), int(iteration), ptr(out_idx), ptr(out_val),
                                    injp, events.ref(), stream())
        N.check(rc, "ftk_checked_assign")
    else:
        rc = lib.ftk_assign(ctx(), code(dt), variant_code(variant), ptr(x_t), ptr(y_t),
                            ptr(yn_t), m, k, d, bm, bn, bk, ptr(out_idx), ptr(out_val), injp,
                            stream())
        N.check(rc, "ftk_assign")
    return out_idx, out_val


def gemm_dev(x_t, y_t, block, inj=None, checked=False, delta_rel=0.0, abs_tol=0.0, iteration=0,
             events=None):
    t = _torch()
    m, d = x_t.shape
    k = y_t.shape[0]
    out = t.empty((m, k), dtype=x_t.dtype, device=x_t.device)
    bm, bn, bk = (int(v) for v in block)
    rc = N.load().ftk_gemm(ctx(), code(ndtype(x_t.dtype)), ptr(x_t), ptr(y_t), m, k, d, bm, bn,
                           bk, float(delta_rel), float(abs_tol), int(iteration), ptr(out),
                           inj.ref() if inj is not None else None,
                           events.ref() if (checked and events is not None) else None, stream())
    N.check(rc, "ftk_gemm")
    return out


def update_sums_dev(x_t, labels_i32, k, dmr=False):
    t = _torch()
    m, d = x_t.shape
    dev = x_t.device
    sums_a = t.empty((k, d), dtype=t.float64, device=dev)
    counts_a = t.empty(k, dtype=t.int64, device=dev)
    sums_b = t.empty((k, d), dtype=t.float64, device=dev) if dmr else None
    counts_b = t.empty(k, dtype=t.int64, device=dev) if dmr else None
    rc = N.load().ftk_update_sums(ctx(), code(ndtype(x_t.dtype)), ptr(x_t), ptr(labels_i32), m, d,
                                  k, ptr(sums_a), ptr(counts_a), ptr(sums_b), ptr(counts_b),
                                  stream())
    N.check(rc, "ftk_update_sums")
    return sums_a, counts_a, sums_b, counts_b


def dmr_mismatch_dev(sa, ca, sb, cb, flag):
    k, d = sa.shape
    N.check(N.load().ftk_dmr_compare(ctx(), ptr(sa), ptr(ca), ptr(sb), ptr(cb), k, d, ptr(flag),
                                     stream()), "ftk_dmr_compare")


def finalize_dev(sums, counts, dtype, out=None, n_empty=None):
    t = _torch()
    k, d = sums.shape
    if out is None:
        out = t.empty((k, d), dtype=tdtype(dtype), device=sums.device)
    N.check(N.load().ftk_update_finalize(ctx(), code(dtype), ptr(sums), ptr(counts), k, d,
                                         ptr(out), ptr(n_empty), stream()), "ftk_update_finalize")
    return out


def reseed_dev(x_t, counts, sq, cent):
    m, d = x_t.shape
    N.check(N.load().ftk_reseed_empty(ctx(), code(ndtype(x_t.dtype)), ptr(x_t), m, d,
                                      ptr(counts), counts.shape[0], ptr(sq), ptr(cent), stream()),
            "ftk_reseed_empty")


def sq_dists_dev(md, xsq, out):
    N.check(N.load().ftk_sq_dists(ctx(), code(ndtype(md.dtype)), ptr(md), ptr(xsq), md.shape[0],
                                  ptr(out), stream()), "ftk_sq_dists")
    return out


def pairwise_sum_dev(a, out):
    N.check(N.load().ftk_pairwise_sum(ctx(), ptr(a), a.shape[0], ptr(out), stream()),
            "ftk_pairwise_sum")
    return out


def movement_dev(new_c, old_c, eps, out):
    k, d = new_c.shape
    N.check(N.load().ftk_movement(ctx(), code(ndtype(new_c.dtype)), ptr(new_c), ptr(old_c), k, d,
                                  float(eps), ptr(out), stream()), "ftk_movement")
    return out


def labels_equal_dev(a, b, out):
    N.check(N.load().ftk_labels_equal(ctx(), ptr(a), ptr(b), a.shape[0], ptr(out), stream()),
            "ftk_labels_equal")
    return out


def flip_f64_dev(a, i, j, bit, ba):
    N.check(N.load().ftk_flip_f64(ctx(), ptr(a), a.shape[1], int(i), int(j), int(bit), ptr(ba),
                                  stream()), "ftk_flip_f64")


def own_sq_dists_dev(x_t, labels_i32, cent64, out):
    m, d = x_t.shape
    N.check(N.load().ftk_own_sq_dists(ctx(), code(ndtype(x_t.dtype)), ptr(x_t), ptr(labels_i32),
                                      ptr(cent64), m, d, ptr(out), stream()), "ftk_own_sq_dists")
    return out

def tc_fallback_rows():
    """(rows the 1xTF32 screen left uncertified, rows the 3xTF32 re-screen
    left for the exact kernel, rows whose TC row checksum failed) of the last
    TC assignment."""
    import ctypes

    v = (ctypes.c_int64 * 3)()
    N.check(N.load().ftk_tc_fallback_rows(ctx(), v, stream()), "ftk_tc_fallback_rows")
    return int(v[0]), int(v[1]), int(v[2])


def abft_flags_total(reset=False):
    """Rows whose screened row checksum failed, summed over every checked
    assignment on this device since the last reset (ftk_abft_flags_total)."""
    import ctypes

    v = ctypes.c_int64(0)
    N.check(N.load().ftk_abft_flags_total(ctx(), ctypes.byref(v), int(bool(reset)), stream()),
            "ftk_abft_flags_total")
    return int(v.value)


def tc_last_kernel_ms():
    """Device time of the last tensor-core screen launch (ms, -1 if none)."""
    import ctypes

    v = ctypes.c_float(-1.0)
    N.check(N.load().ftk_tc_last_kernel_ms(ctx(), ctypes.byref(v)), "ftk_tc_last_kernel_ms")
    return float(v.value)


def tc_raw_dots(x_t, y_t, yn_t, split=False):
    """Raw tensor-core screened dot products (m x k) + the assignment."""
    t = _torch()
    m, d = x_t.shape
    k = y_t.shape[0]
    raw = t.zeros((m, k), dtype=t.float32, device=x_t.device)
    idx = t.empty(m, dtype=t.int32, device=x_t.device)
    val = t.empty(m, dtype=t.float32, device=x_t.device)
    N.check(N.load().ftk_tc_raw_dots(ctx(), int(bool(split)), ptr(x_t), ptr(y_t), ptr(yn_t), m, k,
                                     d, ptr(raw), ptr(idx), ptr(val), stream()), "ftk_tc_raw_dots")
    return raw, idx, val
