"""Kernel-variant selector: the B200 counterpart of the reference's tile tuner.

The reference tunes CPU cache tiles per shape and keeps the winners in a
``TuneTable`` keyed by (M bucket, N, K, precision), with nearest-shape lookup
and a CSV file format (tuner.py:230-293), filled by ``select`` which
benchmarks every feasible candidate and keeps the fastest (tuner.py:296-351).
On the GPU the choice that matters is the *kernel family* of the fused
assignment, so this module keeps the same structure for it:

  single precision   "pair"    CTA-pair tcgen05 screen (tc_pair.cu; X resident up to d = 256,
                               streamed with the centroid stages above)
                     "narrow"  streamed-X tcgen05 screen (tc_narrow.cu, k + 4 <= 256)
                     "exact"   SIMT kernel in the reference's evaluation order (exact.cu)
  double precision   "pair"    tf32 CTA-pair screen of the fp32 copy, certified in float64
                               (tc64.cu; uncertified rows go to the DMMA screen)
                     "dmma"    FP64 tensor-core screen (dscreen.cu)
                     "dfma"    SIMT DFMA screen (dscreen.cu)
                     "exact"

Every family returns the reference's bits, so the choice is speed only.
``select`` measures each feasible family on the device (synthetic blobs of the
shape, one warm pass, then the median of ``reps`` CUDA-event-timed steady-state
passes with the previous labels as the narrow screen's hint) and records the
GFLOP/s.  ``resolve`` is what the package calls: an explicit
``gemm.set_variant`` wins, else the loaded table (``set_table`` /
``FTK_VARIANT_TABLE``, default: the table measured on a B200 shipped in
``data/variants_b200.csv`` when the device is a B200), else the built-in rule.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

PRECISIONS = ("single", "double")
FAMILIES = {"single": ("pair", "narrow", "exact"), "double": ("pair", "dmma", "dfma", "exact")}
HEADER = "# M_bucket,D,K,precision,variant,gflops,reps\n"
DEFAULT_TABLE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data",
                             "variants_b200.csv")


def precision_of(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "single"
    if dt == np.float64:
        return "double"
    raise ValueError(f"unsupported dtype {dt}")


def m_bucket(m):
    """Power-of-two floor, as the reference buckets M (tuner.py:229-230)."""
    return 1 << int(math.floor(math.log2(max(int(m), 1))))


def feasible(variant, shape, precision, ft_on=False):
    """Can this family run the shape (m, d, k)?  Mirrors the library's own
    checks (tc.cu tc_supported / narrow_supported, dscreen.cu)."""
    m, d, k = (int(v) for v in shape)
    if variant == "exact":
        return True
    if precision == "single":
        if d < 4 or d % 4 or m >= (1 << 31) or k >= (1 << 24):
            return False
        if variant == "pair":
            return d <= 8192  # X resident up to d = 256, streamed through the stages above
        if variant == "narrow":
            return k + (4 if ft_on else 0) <= 256
        return False
    if variant in ("dmma", "dfma"):
        return k < 65536 and m < (1 << 31)
    if variant == "pair":  # tf32 screen of the fp32 copy, certified in float64 (tc64.cu)
        return 4 <= d <= 256 and d % 4 == 0 and k < 65536 and m < (1 << 31)
    return False


def builtin(shape, precision, ft_on=False):
    """The rule used without a table: the tensor cores wherever they apply
    (pair screen up to d = 256; above, the narrow screen when it takes k,
    else the pair screen with streamed X), DMMA for float64, the exact
    kernel otherwise."""
    if precision == "double":
        if shape[0] >= 65536 and feasible("pair", shape, precision, ft_on):
            return "pair"
        return "dmma" if feasible("dmma", shape, precision, ft_on) else "exact"
    _, d, _ = shape
    if d > 256 and feasible("narrow", shape, precision, ft_on):
        return "narrow"
    if feasible("pair", shape, precision, ft_on):
        return "pair"
    return "exact"


@dataclass
class VariantEntry:
    variant: str
    gflops: float
    reps: int


@dataclass
class VariantTable:
    """Per-shape kernel-family selections keyed by (M bucket, D, K, precision)."""

    entries: dict = field(default_factory=dict)
    measured: dict = field(default_factory=dict)  # every candidate's gflops (not serialised)

    def put(self, shape, precision, variant, gflops, reps):
        m, d, k = shape
        self.entries[(m_bucket(m), int(d), int(k), precision)] = VariantEntry(variant, float(gflops),
                                                                              int(reps))

    def lookup(self, shape, dtype, ft_on=False):
        """Stored family for the shape, else the nearest stored (D, K) by
        log-distance among entries whose family can run this shape, else the
        built-in rule (tuner.py:248-262)."""
        prec = precision_of(dtype)
        m, d, k = shape
        key = (m_bucket(m), int(d), int(k), prec)
        e = self.entries.get(key)
        if e is not None and feasible(e.variant, shape, prec, ft_on):
            return e.variant
        cands = [c for c, v in self.entries.items()
                 if c[3] == prec and feasible(v.variant, shape, prec, ft_on)]
        if cands:
            ld, lk = math.log2(max(d, 1)), math.log2(max(k, 1))
            best = min(cands, key=lambda c: ((math.log2(c[1]) - ld) ** 2 +
                                             (math.log2(max(c[2], 1)) - lk) ** 2,
                                             abs(math.log2(c[0]) - math.log2(max(m, 1)))))
            return self.entries[best].variant
        return builtin(shape, prec, ft_on)

    def save(self, path):
        with open(path, "w") as fh:
            fh.write(HEADER)
            for (mb, d, k, prec), e in sorted(self.entries.items()):
                fh.write(f"{mb},{d},{k},{prec},{e.variant},{e.gflops!r},{e.reps}\n")

    @staticmethod
    def load(path):
        table = VariantTable()
        with open(path) as fh:
            for line in fh:
                line = line.strip()
                if not line or line.startswith("#"):
                    continue
                parts = line.split(",")
                if len(parts) != 7:
                    raise ValueError(f"bad variant-table row: {line!r}")
                mb, d, k = int(parts[0]), int(parts[1]), int(parts[2])
                prec, var = parts[3], parts[4]
                if prec not in PRECISIONS or var not in FAMILIES[prec]:
                    raise ValueError(f"bad variant-table row: {line!r}")
                table.entries[(mb, d, k, prec)] = VariantEntry(var, float(parts[5]), int(parts[6]))
        return table


# ------------------------------------------------------------ measuring --
def _blobs(m, d, k, precision, seed):
    """Gaussian blobs on the device (k centers, sigma 0.5) and k sampled rows
    as centroids: the near-converged regime Lloyd spends its time in."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    dt = torch.float32 if precision == "single" else torch.float64
    c = torch.randn((k, d), generator=g, device="cuda", dtype=torch.float64)
    lab = torch.randint(0, k, (m,), generator=g, device="cuda")
    x = (c[lab] + 0.5 * torch.randn((m, d), generator=g, device="cuda", dtype=torch.float64)).to(dt)
    y = x[torch.randperm(m, generator=g, device="cuda")[:k]].contiguous()
    return x.contiguous(), y


def measure(variant, shape, precision="single", ft_mode="off", reps=5, seed=0):
    """GFLOP/s (2 m d k per pass) of one family on the device: the median of
    `reps` steady-state passes, the previous pass's labels as the hint."""
    import torch

    from . import _engine as E
    from .abft import Threshold

    m, d, k = (int(v) for v in shape)
    x_t, y_t = _blobs(m, d, k, precision, seed)
    yn = E.row_sq_norms_dev(y_t)
    checked = ft_mode != "off"
    ev = E.DevEvents(64) if checked else None
    d_rel, a_tol = Threshold.default_for(E.ndtype(x_t.dtype)).kernel_params()
    labels = [torch.full((m,), -1, dtype=torch.int32, device=x_t.device) for _ in range(2)]
    times = []
    for r in range(reps + 1):
        E.set_label_hint(labels[(r + 1) % 2], m)
        try:
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if ev is not None:
                ev.reset()
            s0.record()
            E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant=variant, checked=checked,
                         delta_rel=d_rel, abs_tol=a_tol, events=ev, out_idx=labels[r % 2])
            s1.record()
            torch.cuda.synchronize()
        finally:
            E.set_label_hint(None, 0)
        if r:
            times.append(s0.elapsed_time(s1))
    ms = float(np.median(times))
    return 2.0 * m * d * k / (ms * 1e-3) / 1e9


def select(shapes, precision="single", ft_mode="off", reps=5, probe_m=1 << 20, seed=0,
           progress=None):
    """Measure every feasible family per shape and keep the fastest
    (tuner.py:296-351); the probe runs min(M, probe_m) rows."""
    if not shapes:
        raise ValueError("no shapes to tune")
    table = VariantTable()
    ft_on = ft_mode != "off"
    for shape in shapes:
        m, d, k = (int(v) for v in shape)
        probe = (min(m, probe_m), d, k)
        best = None
        for var in FAMILIES[precision]:
            if not feasible(var, probe, precision, ft_on):
                continue
            gf = measure(var, probe, precision, ft_mode, reps, seed)
            table.measured[(m_bucket(m), d, k, precision, var)] = gf
            if progress:
                progress(shape, var, gf)
            if best is None or gf > best[1]:
                best = (var, gf)
        table.put(shape, precision, best[0], best[1], reps)
    return table


# ------------------------------------------------------------- resolving --
_TABLE = None
_TABLE_LOADED = False


def set_table(table):
    """Use `table` (a VariantTable, a path, or None for the built-in rule)."""
    global _TABLE, _TABLE_LOADED
    _TABLE = VariantTable.load(table) if isinstance(table, str) else table
    _TABLE_LOADED = True


def get_table():
    global _TABLE, _TABLE_LOADED
    if not _TABLE_LOADED:
        _TABLE_LOADED = True
        env = os.environ.get("FTK_VARIANT_TABLE")
        if env == "0":
            _TABLE = None
        elif env:
            _TABLE = VariantTable.load(env)
        elif os.path.exists(DEFAULT_TABLE) and _on_b200():
            _TABLE = VariantTable.load(DEFAULT_TABLE)
    return _TABLE


def _on_b200():
    try:
        import torch

        return torch.cuda.is_available() and "B200" in torch.cuda.get_device_name()
    except Exception:
        return False


def resolve(shape, dtype, ft_on=False):
    """The family an assignment of this shape runs: gemm.set_variant's
    explicit choice ('auto' defers), else the table, else the built-in rule."""
    from . import gemm

    v = gemm.get_variant()
    prec = precision_of(dtype)
    if v == "tc":
        return "pair" if feasible("pair", shape, prec, ft_on) else \
            ("narrow" if feasible("narrow", shape, prec, ft_on) else "tc")
    if v != "auto":
        return v
    t = get_table()
    if t is not None:
        return t.lookup(shape, dtype, ft_on)
    return builtin(shape, prec, ft_on)
