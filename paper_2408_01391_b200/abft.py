"""Checksum-protected assignment and the detection report (reference abft.py).

``checked_assign`` / ``checked_gemm`` run ``ftk_checked_assign`` /
``ftk_gemm``: per logical tile the kernel verifies the e1 column checksum
against the encoded-input reference in float64 with the reference tolerance
``delta_rel * max(1, max|x_block| * max|y_block|) * k + abs_tol``, and on a
violation locates (scan + e2/e1 quotients), corrects and rechecks the tile
exactly like _checked_range/_diagnose (_kernels.py:479-612, 321-405).  Events
come back through a device ring and are reported here in the reference's
order.  The small helpers at the bottom (encode/locate/correct/ChecksumSet/
dmr_reduce) are the reference's standalone host utilities.
"""

from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, field

import numpy as np

from . import _engine as E
from .errors import FaultEscalationError
from .gemm import AssignResult, _check_pair, _dtype, _ynorms_dev, get_variant, resolve_threads

EV_CORRECTED, EV_UNCORRECTABLE = 0, 1
KIND_NAMES = {0: "detected-corrected", 1: "detected-uncorrectable", 2: "dmr-mismatch"}
KIND_CODES = {v: k for k, v in KIND_NAMES.items()}
REPORT_HEADER = ["iteration", "tile_i", "tile_j", "kind", "loc_i", "loc_j", "delta"]


@dataclass(frozen=True)
class Threshold:
    """Relative: delta_rel * max(1, amax_x * amax_y) * k_acc; absolute: delta_rel."""

    delta_rel: float
    mode: str = "relative"

    def __post_init__(self):
        if not self.delta_rel > 0:
            raise ValueError(f"delta_rel must be positive, got {self.delta_rel}")
        if self.mode not in ("relative", "absolute"):
            raise ValueError(f"unknown threshold mode {self.mode!r}")

    @staticmethod
    def default_for(dtype):
        return Threshold(1e-4 if np.dtype(dtype) == np.float32 else 1e-10)

    def kernel_params(self):
        """(delta_rel, abs_tol) as the checked kernel consumes them."""
        if self.mode == "relative":
            return float(self.delta_rel), 0.0
        return 0.0, float(self.delta_rel)


@dataclass
class DetectionEvent:
    iteration: int
    tile: tuple
    kind: str
    loc: tuple
    delta: float
    interval: int = 0


@dataclass
class DetectionReport:
    events: list = field(default_factory=list)
    false_alarms: int = 0

    @property
    def detections(self):
        return len(self.events)

    @property
    def corrections(self):
        return sum(e.kind == "detected-corrected" for e in self.events)

    @property
    def uncorrectable(self):
        return sum(e.kind == "detected-uncorrectable" for e in self.events)

    @property
    def dmr_mismatches(self):
        return sum(e.kind == "dmr-mismatch" for e in self.events)

    def merge(self, other):
        self.events.extend(other.events)
        self.false_alarms += other.false_alarms
        return self

    def to_csv(self, path_or_file):
        own = isinstance(path_or_file, (str, bytes)) or hasattr(path_or_file, "__fspath__")
        fh = open(path_or_file, "w", newline="") if own else path_or_file
        try:
            w = csv.writer(fh)
            w.writerow(REPORT_HEADER)
            for e in self.events:
                w.writerow([e.iteration, e.tile[0], e.tile[1], e.kind, e.loc[0], e.loc[1],
                            repr(e.delta)])
        finally:
            if own:
                fh.close()

    @staticmethod
    def from_csv(path):
        with open(path, newline="") as fh:
            rows = list(csv.reader(fh))[1:]
        return DetectionReport([DetectionEvent(int(r[0]), (int(r[1]), int(r[2])), r[3],
                                               (int(r[4]), int(r[5])), float(r[6])) for r in rows])

    def to_csv_text(self):
        buf = io.StringIO()
        self.to_csv(buf)
        return buf.getvalue()


def events_from_ring(raw, iteration_filter=None):
    out = []
    for rec, delta in raw:
        it, ti, tj, kind, li, lj, interval = rec
        out.append(DetectionEvent(it, (ti, tj), KIND_NAMES[kind], (li, lj), delta, interval))
    out.sort(key=lambda e: (e.iteration, e.tile, e.interval))
    return out


def split_ranges(n_blocks, threads):
    """Contiguous [lo, hi) row-block ranges, one per reference worker
    (_kernels.py:615-619): each worker owns an event buffer of its own."""
    threads = max(1, min(int(threads), n_blocks)) if n_blocks else 1
    step = max(1, (n_blocks + threads - 1) // threads)
    return [(lo, min(lo + step, n_blocks)) for lo in range(0, n_blocks, step)]


def worker_overflow(raw, n_inj, nbi, threads):
    """The reference's overflow rule (abft.py:280-316): every worker's buffer
    holds n_inj + 64 events and ANY worker exceeding it raises.  The device
    ring holds the sum of the worker capacities, so a ring overflow implies a
    worker overflow, and otherwise every event is present to count per range."""
    cap = n_inj + 64
    ranges = split_ranges(nbi, threads)
    if len(ranges) <= 1:
        return len(raw) > cap
    los = np.array([lo for lo, _ in ranges], np.int64)
    bi = np.array([rec[1] for rec, _ in raw], np.int64)
    per = np.bincount(np.searchsorted(los, bi, side="right") - 1, minlength=len(ranges))
    return bool((per > cap).any())


def _scheduled_tiles(inj):
    if inj is None or inj.n == 0:
        return set()
    bi, bj = inj.host[0], inj.host[1]
    return {(int(a), int(b)) for a, b in zip(bi, bj)}


def _checked_run(a, b, cfg, thr, hook, iteration, threads, y_norms, materialize):
    threads = resolve_threads(threads)
    dt = _dtype(a)
    if thr is None:
        thr = Threshold.default_for(dt)
    delta_rel, abs_tol = thr.kernel_params()
    m, k = a.shape[0], b.shape[0]
    bm = cfg.block[0]
    nbi = (m + bm - 1) // bm
    inj = E.injection_for(hook, iteration, dt)
    n_inj = inj.n if inj is not None else 0
    # the reference gives every worker an event buffer of n_inj + 64
    cap = (n_inj + 64) * max(1, min(threads, nbi))
    a_t, b_t = E.to_dev(a), E.to_dev(b)
    events = E.DevEvents(cap)
    if m == 0:
        if inj is not None:
            inj.finish()
        if hook is not None:
            hook.absorb_kernel_results(iteration, *(inj.host[5:8] if inj is not None else
                                                    (np.zeros(0, np.int64), np.zeros(0), np.zeros(0))))
        out = (np.empty((0, k), dt) if materialize
               else AssignResult(np.empty(0, np.int64), np.empty(0, dt)))
        return out, DetectionReport()
    if materialize:
        res_t = E.gemm_dev(a_t, b_t, cfg.block, inj=inj, checked=True, delta_rel=delta_rel,
                           abs_tol=abs_tol, iteration=iteration, events=events)
    else:
        yn_t = _ynorms_dev(b_t, y_norms, dt, k)
        from .variants import resolve

        idx, val = E.assign_dev(a_t, b_t, yn_t, cfg.block,
                                variant=resolve((m, a_t.shape[1], k), dt, ft_on=True), inj=inj,
                                checked=True, delta_rel=delta_rel, abs_tol=abs_tol,
                                iteration=iteration, events=events)
    overflow, raw = events.read()
    if overflow or worker_overflow(raw, n_inj, nbi, threads):
        raise RuntimeError("detection event buffer overflow; threshold likely miscalibrated")
    evs = events_from_ring(raw)
    report = DetectionReport(events=evs)
    sched = _scheduled_tiles(inj)
    report.false_alarms = sum(1 for e in evs if e.tile not in sched)
    if inj is not None:
        inj.finish()
    if hook is not None:
        if inj is not None:
            hook.absorb_kernel_results(iteration, inj.host[5], inj.host[6], inj.host[7])
        else:
            hook.absorb_kernel_results(iteration, np.zeros(0, np.int64), np.zeros(0), np.zeros(0))
    if materialize:
        return E.to_host(res_t), report
    return AssignResult(E.to_host(idx).astype(np.int64), E.to_host(val)), report


def checked_gemm(a, b, cfg=None, thr=None, hook=None, iteration=0, threads=None):
    """Checksum-protected ``a @ b.T``; fault-free output equals gemm_tiled bitwise."""
    a, b, cfg = _check_pair(a, b, cfg)
    return _checked_run(a, b, cfg, thr, hook, iteration, threads, None, True)


def checked_assign(x, y, y_norms=None, cfg=None, thr=None, hook=None, iteration=0, threads=None):
    """Fused assignment over checksum-protected distance tiles -> (AssignResult, report)."""
    x, y, cfg = _check_pair(x, y, cfg)
    return _checked_run(x, y, cfg, thr, hook, iteration, threads, y_norms, False)


# ------------------------------------------------ standalone helpers ------
def encode_cols(tile):
    t = np.asarray(tile, dtype=np.float64)
    if t.ndim != 2 or t.size == 0:
        raise ValueError("tile must be a non-empty 2-D array")
    return t.sum(axis=0), np.arange(1, t.shape[0] + 1, dtype=np.float64) @ t


def encode_rows(tile):
    t = np.asarray(tile, dtype=np.float64)
    if t.ndim != 2 or t.size == 0:
        raise ValueError("tile must be a non-empty 2-D array")
    return t.sum(axis=1), t @ np.arange(1, t.shape[1] + 1, dtype=np.float64)


def locate(d_c1, d_c2, d_r1, d_r2, tol, tile_shape=None):
    """(i, j, delta) from the four divergences, or None (abft.py:209-232)."""
    if not all(math.isfinite(v) for v in (d_c1, d_c2, d_r1, d_r2)):
        return None
    if abs(d_c1 - d_r1) > max(tol, 0.05 * abs(d_c1)) or d_c1 == 0.0 or d_r1 == 0.0:
        return None
    qi, qj = d_r2 / d_r1, d_c2 / d_c1
    i, j = int(math.floor(qi + 0.5)), int(math.floor(qj + 0.5))
    if abs(qi - i) > 0.05 or abs(qj - j) > 0.05 or i < 1 or j < 1:
        return None
    if tile_shape is not None and (i > tile_shape[0] or j > tile_shape[1]):
        return None
    return i - 1, j - 1, d_c1


def correct(tile, i, j, delta):
    if not (0 <= i < tile.shape[0] and 0 <= j < tile.shape[1]):
        raise ValueError(f"({i},{j}) outside tile {tile.shape}")
    tile[i, j] -= tile.dtype.type(delta)


@dataclass
class ChecksumSet:
    colsum1: np.ndarray
    colsum2: np.ndarray
    rowsum1: np.ndarray
    rowsum2: np.ndarray
    outsum_c1: np.ndarray
    outsum_c2: np.ndarray
    outsum_r1: np.ndarray
    outsum_r2: np.ndarray

    @staticmethod
    def from_tiles(x_tile, y_tile):
        x64 = np.asarray(x_tile, dtype=np.float64)
        y64 = np.asarray(y_tile, dtype=np.float64)
        c1, c2 = encode_cols(x64)
        r1, r2 = encode_rows(y64.T)
        return ChecksumSet(c1, c2, r1, r2, y64 @ c1, y64 @ c2, x64 @ r1, x64 @ r2)

    def verify(self, d_tile, tol):
        d64 = np.asarray(d_tile, dtype=np.float64)
        return (bool(np.all(np.abs(d64.sum(axis=0) - self.outsum_c1) <= tol)),
                bool(np.all(np.abs(d64.sum(axis=1) - self.outsum_r1) <= tol)))


def dmr_reduce(values, init=0.0, op="sum", hook=None, iteration=0, site=(0, 0), _chunk=4096):
    """Duplicated reduction with bitwise compare, one retry, then escalation."""
    if op != "sum":
        raise ValueError(f"unsupported reduction op {op!r}")
    v = np.asarray(values, dtype=np.float64).ravel()

    def once():
        a = b = np.float64(init)
        for lo in range(0, v.size, _chunk):
            s = np.add.reduce(v[lo:lo + _chunk], dtype=np.float64)
            a += s
            b += s
        if hook is not None:
            buf = np.array([[a]], dtype=np.float64)
            hook.maybe_corrupt(iteration, site, buf)
            a = buf[0, 0]
        return a, b

    a, b = once()
    first = a
    if a.tobytes() == b.tobytes():
        return float(a), False
    a, b = once()
    if a.tobytes() != b.tobytes():
        raise FaultEscalationError(
            f"DMR mismatch persisted after retry at site {site} (got {first!r} then {a!r})")
    return float(a), True
