"""Lloyd's iteration on the B200 (reference kmeans.py).

Same entry points, config/result types, stopping rules and fault-campaign
planning as the reference; the data stays resident in HBM for the whole fit
and each iteration is: assign (fused or checksum-protected kernel) -> inertia
(device pairwise sum) -> label comparison -> update (ordered float64 member
chains, optional DMR) -> finalize -> movement, with ONE small device->host
control readback per iteration for the host-side stopping decision
(kmeans.py:277, 295-297).  Results are bit-identical to the reference.
"""

from __future__ import annotations

import dataclasses
import gc
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _engine as E
from . import _native as N
from .abft import DetectionEvent, DetectionReport, Threshold, checked_assign, events_from_ring
from .abft import _scheduled_tiles, worker_overflow
from .errors import FaultEscalationError
from .faults import NOOP_HOOK, FaultHook, FaultSpec, ScheduledFaultHook, plan_faults
from .gemm import _as_operand, _dtype, _is_torch, fused_assign, get_variant, resolve_threads
from .matrix import as_matrix
from .tiles import TileConfig, default_config

FT_MODES = ("off", "abft", "abft+dmr")
INIT_METHODS = ("random-sample", "kmeanspp")


@dataclass
class KMeansConfig:
    k: int
    max_iters: int = 300
    tol: float = 1e-4
    seed: int = 0
    ft_mode: str = "off"
    init: str = "kmeanspp"
    tile: object = "auto"
    threshold: Threshold = None
    threads: int = None
    tune_table: object = None

    def validate(self):
        if self.k < 1:
            raise ValueError(f"k must be >= 1, got {self.k}")
        if self.max_iters < 0:
            raise ValueError(f"max_iters must be >= 0, got {self.max_iters}")
        if self.tol < 0:
            raise ValueError(f"tol must be >= 0, got {self.tol}")
        if self.ft_mode not in FT_MODES:
            raise ValueError(f"ft_mode must be one of {FT_MODES}, got {self.ft_mode!r}")
        if self.init not in INIT_METHODS:
            raise ValueError(f"init must be one of {INIT_METHODS}, got {self.init!r}")
        return self


@dataclass
class KMeansResult:
    centroids: np.ndarray
    assignments: np.ndarray
    inertia: float
    iters: int
    converged: bool
    report: DetectionReport
    timings: dict = field(default_factory=dict)
    inertia_history: list = field(default_factory=list)


def init_centroids(x, k, seed=0, method="kmeanspp"):
    """Deterministic seeding with the reference's Generator draws
    (kmeans.py:69-103).  random-sample is a gather of the reference's
    ``rng.choice`` rows; kmeanspp runs its D^2 seeding on the device
    (_kmeanspp_dev) for every D.  numpy in -> numpy out (data dtype)."""
    if _is_torch(x) and x.is_cuda:
        x_t, x_h = x, None
        m = x.shape[0]
    else:
        x_h = as_matrix(E.to_host(x) if _is_torch(x) else x)
        x_t, m = None, x_h.shape[0]
    if k > m:
        raise ValueError(f"k={k} exceeds the number of samples {m}")
    if method not in INIT_METHODS:
        raise ValueError(f"unknown init method {method!r}")
    rng = np.random.default_rng(seed)
    if method == "random-sample":
        idx = rng.choice(m, size=k, replace=False)
        if x_h is not None:
            return np.ascontiguousarray(x_h[idx])
        return E.to_host(x_t[E._torch().as_tensor(idx, device=x_t.device)])
    if x_t is None:
        x_t = E.to_dev(x_h)
    picks = _kmeanspp_dev(x_t, k, rng)
    if x_h is not None:
        return np.ascontiguousarray(x_h[picks])
    return E.to_host(x_t[E._torch().as_tensor(picks, device=x_t.device)])


def _kmeanspp_dev(x_t, k, rng):
    """k-means++ D^2 seeding with the reference's draws (kmeans.py:86-103),
    on the device: the D^2 updates (ftk_kpp_update: float64, numpy's
    pairwise feature reduce, np.minimum), ``d2.sum()`` (device pairwise sum)
    and ``searchsorted(cumsum(d2), r, "right")`` (ftk_kpp_search: bit-exact
    against numpy's sequential cumsum).  Per pick the host reads one scalar
    -- the total its ``rng.random()`` draw is scaled by -- and nothing else.
    Returns the k picked row indices (int64)."""
    t = E._torch()
    m = x_t.shape[0]
    if m == 0 or k == 0:
        return np.zeros(0, dtype=np.int64)
    d2, picks, tot, pick_dev, n_rep = E.kpp_buffers(m, k, x_t.device)
    tot_h = t.empty(1, dtype=t.float64).pin_memory()
    stream = t.cuda.current_stream()
    E.kpp_update_dev(x_t, int(rng.integers(0, m)), None, True, d2, picks, 0)
    for c in range(1, k):
        E.pairwise_sum_dev(d2, tot)
        tot_h.copy_(tot, non_blocking=True)
        stream.synchronize()
        total = float(tot_h[0])
        if total <= 0:
            E.kpp_update_dev(x_t, int(rng.integers(0, m)), None, False, d2, picks, c)
        else:
            E.kpp_search_dev(d2, rng.random() * total, pick_dev, n_rep)
            E.kpp_update_dev(x_t, -1, pick_dev, False, d2, picks, c)
    return E.to_host(picks)


def _resolve_tile(tile, x, k, tune_table):
    if isinstance(tile, TileConfig):
        return tile.validate()
    if tile == "auto":
        if tune_table is not None:
            return tune_table.lookup((x.shape[0], x.shape[1], k), _dtype(x))
        return default_config(_dtype(x))
    raise ValueError(f"tile must be a TileConfig or 'auto', got {tile!r}")


def assign_step(x, y, cfg=None, ft_mode="off", hook=NOOP_HOOK, thr=None, iteration=0,
                threads=None):
    """ft_mode 'off' -> fused kernel; otherwise the checksum-protected one."""
    if ft_mode == "off":
        return fused_assign(x, y, cfg=cfg, threads=threads, hook=hook, iteration=iteration), None
    return checked_assign(x, y, cfg=cfg, thr=thr, hook=hook, iteration=iteration, threads=threads)


def _site_pending(hook, iteration, tile=(0, 0)):
    if hook is None or hook is NOOP_HOOK:
        return False
    probe = getattr(hook, "has_pending_site", None)
    return probe(iteration, tile) if probe is not None else True


def _corrupt_on_host(hook, iteration, sums_t):
    """Run the hook's maybe_corrupt on a host copy of the device sums (the
    reference's array fault site, kmeans.py:172-173) and write it back."""
    host = E.to_host(sums_t).copy()
    before = host.copy()
    hook.maybe_corrupt(iteration, (0, 0), host)
    if host.tobytes() != before.tobytes():
        sums_t.copy_(E._torch().from_numpy(host).to(sums_t.device))


def _update_dev(x_t, labels_i32, k, dtype, ft_mode, hook, iteration, ctl_i32):
    """Sums/counts (+DMR) -> float64 sums and counts on the device, events."""
    dmr = ft_mode == "abft+dmr"
    events = []

    def accumulate():
        sa, ca, sb, cb = E.update_sums_dev(x_t, labels_i32, k, dmr=dmr)
        if _site_pending(hook, iteration):
            _corrupt_on_host(hook, iteration, sa)
        return sa, ca, sb, cb

    sa, ca, sb, cb = accumulate()
    if dmr:
        E.dmr_mismatch_dev(sa, ca, sb, cb, ctl_i32[2:3])
        if int(ctl_i32[2].item()):
            events.append(DetectionEvent(iteration=iteration, tile=(0, 0), kind="dmr-mismatch",
                                         loc=(-1, -1), delta=0.0))
            sa, ca, sb, cb = accumulate()
            E.dmr_mismatch_dev(sa, ca, sb, cb, ctl_i32[2:3])
            if int(ctl_i32[2].item()):
                raise FaultEscalationError(
                    f"update-phase DMR mismatch persisted after retry (iteration {iteration})")
    return sa, ca, events


def update_step(x, assignments, k, ft_mode="off", hook=NOOP_HOOK, iteration=0, sq_dists=None):
    """Per-cluster means, float64 sums in ascending sample order; empty
    clusters take successive farthest points.  -> (centroids, counts, events)."""
    t = E._torch()
    x = _as_operand(x)
    dtype = _dtype(x)
    lab = E.to_host(assignments) if _is_torch(assignments) else np.asarray(assignments)
    m, n = x.shape
    if lab.shape != (m,):
        raise ValueError(f"assignments must have shape ({m},)")
    if lab.size and (lab.min() < 0 or lab.max() >= k):
        raise ValueError("assignments out of range")
    x_t = E.to_dev(x)
    lab_t = E.to_dev(lab.astype(np.int32))
    ctl_i32 = t.zeros(8, dtype=t.int32, device=x_t.device)
    sums, counts, events = _update_dev(x_t, lab_t, k, dtype, ft_mode, hook, iteration, ctl_i32)
    cent = E.finalize_dev(sums, counts, dtype, n_empty=ctl_i32[1:2])
    if int(ctl_i32[1].item()):
        if sq_dists is None:
            c64 = E.finalize_dev(sums, counts, np.float64)
            sq = t.empty(m, dtype=t.float64, device=x_t.device)
            E.own_sq_dists_dev(x_t, lab_t, c64, sq)
        else:
            sq = E.to_dev(np.asarray(sq_dists, dtype=np.float64)).clone()
        E.reseed_dev(x_t, counts, sq, cent)
    return E.to_host(cent), E.to_host(counts), events


def _plan_hooks(fault_spec, cfg, m, n, k, max_iters, dtype):
    if isinstance(fault_spec, str):
        fault_spec = FaultSpec.parse(fault_spec)
    gemm_hook = update_hook = NOOP_HOOK
    if fault_spec is not None and fault_spec.mode != "none":
        bm, bn = cfg.block[0], cfg.block[1]
        grid = ((m + bm - 1) // bm, (k + bn - 1) // bn)
        horizon = max(max_iters, 1)
        if fault_spec.target in ("gemm-accumulator", "both"):
            gemm_hook = ScheduledFaultHook(plan_faults(fault_spec, horizon, grid, (bm, bn),
                                                       dtype=dtype, shape=(m, k)))
        if fault_spec.target in ("update-accumulator", "both"):
            spec = dataclasses.replace(fault_spec, seed=fault_spec.seed + 1)
            update_hook = ScheduledFaultHook(plan_faults(spec, horizon, (1, 1), (k, n),
                                                         dtype=np.float64, shape=(k, n)))
    return gemm_hook, update_hook


class _DeviceAssign:
    """One assignment pass on resident data (fused or checked), hook protocol
    and event decoding included."""

    def __init__(self, x_t, m, k, dtype, cfg, ft_mode, thr, threads):
        t = E._torch()
        self.x_t, self.m, self.k, self.dtype, self.cfg = x_t, m, k, dtype, cfg
        self.checked = ft_mode != "off"
        from .variants import resolve

        # kernel family (variants.py: explicit choice, measured table, rule)
        self.variant = resolve((m, x_t.shape[1], k), dtype, ft_on=self.checked)
        self.delta_rel, self.abs_tol = (thr.kernel_params() if thr is not None else (0.0, 0.0))
        self.nbi = (m + cfg.block[0] - 1) // cfg.block[0]
        self.threads = threads
        # per buffer parity: min_dists and the event ring, so the next step can
        # run while the host still reads this one's (LloydEngine._graph_step)
        self._md = [t.empty(m, dtype=x_t.dtype, device=x_t.device) for _ in range(2)]
        # -1: no label yet (the first pass has no hint for the narrow screen)
        self.labels = [t.full((m,), -1, dtype=t.int32, device=x_t.device) for _ in range(2)]
        mult = max(1, min(threads, self.nbi))
        # storage for a few hundred injected flips per pass, so eager injected
        # steps do not move the ring that captured graph replays write into
        self._rings = [E.DevEvents(64 * mult, storage=(64 + 256) * mult) if self.checked else None
                       for _ in range(2)]
        self.bind(0)

    def bind(self, par):
        self.md, self.events = self._md[par], self._rings[par]

    def ring_gen(self):
        return sum(r.gen for r in self._rings) if self.checked else 0

    def run(self, cent_t, yn_t, hook, iteration, slot, sinj=None):
        """`sinj`: a StaticInjection (device-count schedule, graph capture)
        used instead of the hook's arrays for this pass."""
        inj = sinj if sinj is not None else E.injection_for(hook, iteration, self.dtype)
        if self.checked:
            self.events.set_cap(self.ev_cap(inj.cap if sinj is not None else (inj.n if inj else 0)))
            self.events.reset()
        # the other parity holds the previous iteration's labels: the narrow
        # screen's exact-chain hint (a speed hint only, results never depend on it)
        E.set_label_hint(self.labels[1 - slot], self.m)
        try:
            E.assign_dev(self.x_t, cent_t, yn_t, self.cfg.block, variant=self.variant, inj=inj,
                         checked=self.checked, delta_rel=self.delta_rel, abs_tol=self.abs_tol,
                         iteration=iteration, events=self.events, out_idx=self.labels[slot],
                         out_val=self.md)
        finally:
            E.set_label_hint(None, 0)
        return inj

    def ev_cap(self, n_inj):
        """Event capacity of a pass with n_inj flips: the reference gives
        every worker n_inj + 64 (abft.py); finish() applies the per-worker rule."""
        return (n_inj + 64) * max(1, min(self.threads, self.nbi))

    def finish(self, hook, iteration, inj, n_events=None, replayed=False):
        """Host side of the pass: events -> report, applied flips -> hook.
        `replayed`: the pass ran from a CUDA graph, whose launch carries the
        iteration number of its capture; the records get the real one."""
        report = None
        if self.checked:
            n_inj = inj.n if inj else 0
            overflow, raw = self.events.read(n_events, cap=self.ev_cap(n_inj))
            if replayed:
                raw = [((iteration,) + tuple(rec[1:]), d) for rec, d in raw]
            if overflow or worker_overflow(raw, n_inj, self.nbi, self.threads):
                raise RuntimeError("detection event buffer overflow; threshold likely "
                                   "miscalibrated")
            evs = events_from_ring(raw)
            report = DetectionReport(events=evs)
            sched = _scheduled_tiles(inj)
            report.false_alarms = sum(1 for e in evs if e.tile not in sched)
        if inj is not None:
            inj.finish()
            hook.absorb_kernel_results(iteration, inj.host[5], inj.host[6], inj.host[7])
        elif hook is not None and hook is not NOOP_HOOK:
            hook.absorb_kernel_results(iteration, np.zeros(0, np.int64), np.zeros(0), np.zeros(0))
        return report


class _StepGraph:
    """One captured step: the assignment graph and the update graph, replayed
    back to back with timing events around each (phase times on every graph
    step, from events recorded between the replays on the stream)."""

    def __init__(self, parts, launches):
        self.parts = parts
        self.launches = launches

    def replay(self, ev):
        ev[0].record()
        self.parts[0].replay()
        ev[1].record()
        self.parts[1].replay()
        ev[2].record()
        N.load().ftk_add_launches(self.launches)


def _graphable_shape(d, k):
    """fp32 shapes whose screened assignment is free of host synchronisation:
    the CTA-pair screen (X resident up to d = 256, streamed up to 8192) and
    the narrow screen, both with d % 4 == 0."""
    return d % 4 == 0 and 8 <= d <= 8192


class LloydEngine:
    """Device-resident Lloyd state: one ``step`` per iteration (assign ->
    inertia -> label compare -> update -> finalize -> movement) with a single
    control readback.  ``lloyd`` drives it with the reference's stopping
    rules; bench.py times exact step counts through it."""

    def __init__(self, x_t, c0, k, dtype, cfg, ft_mode, thr, threads, gemm_hook=NOOP_HOOK,
                 update_hook=NOOP_HOOK, dist=None, graph=False):
        t = E._torch()
        self.t = t
        self.dist = dist  # parallel.ShardComm for row-sharded multi-GPU runs
        self.x_t, self.k, self.dtype, self.cfg = x_t, k, np.dtype(dtype), cfg
        self.ft_mode = ft_mode
        self.gemm_hook, self.update_hook = gemm_hook, update_hook
        m = x_t.shape[0]
        dev = x_t.device
        self.xsq = E.row_sq_norms_dev(x_t).to(t.float64)
        self.rows = E.RowInfo(x_t)  # per-fit screening bounds (X is constant)
        self._sq = [t.empty(m, dtype=t.float64, device=dev) for _ in range(2)]
        self.ctl_f64 = t.zeros(4, dtype=t.float64, device=dev)   # inertia, moved
        self.ctl_i32 = t.zeros(8, dtype=t.int32, device=dev)     # equal, n_empty, dmr flag
        self._ctl_host = [t.zeros(4, dtype=t.float64).pin_memory() for _ in range(2)]
        self._ctl_i32_host = [t.zeros(8, dtype=t.int32).pin_memory() for _ in range(2)]
        self._evc_host = [t.zeros(1, dtype=t.int64).pin_memory() for _ in range(2)]  # event count
        self.cent = E.to_dev(c0) if not _is_torch(c0) else c0.to(dev).contiguous()
        self.eps = float(np.finfo(self.dtype).eps)
        self.A = _DeviceAssign(x_t, m, k, self.dtype, cfg, ft_mode,
                               thr if ft_mode != "off" else None, threads)
        self.report = DetectionReport()
        self.slot = 0
        self.ev = [t.cuda.Event(enable_timing=True) for _ in range(3)]
        self.assign_ms = 0.0
        self.update_ms = 0.0
        # CUDA-graph replay of the device part of a step (one graph per label /
        # centroid buffer parity); static centroid and count buffers carry the
        # state across replays.  Eager steps remain for iterations with
        # scheduled flips, DMR, update-site hooks or multi-GPU.
        # (only the fp32 CTA-pair assignment is free of host synchronisation)
        self.use_graph = bool(graph) and (dist is None or dist.capturable) and \
            update_hook is NOOP_HOOK and self.dtype == np.float32 and \
            _graphable_shape(x_t.shape[1], k) and self.A.variant in ("pair", "narrow", "tc")
        self.graphs = [None, None]
        # injected passes replay their own graphs, the schedule staged into
        # fixed device arrays (count on the device) before the replay
        self.sinj = E.StaticInjection(64) if self.use_graph and self.A.checked and \
            getattr(gemm_hook, "schedule", None) is not None else None
        self.inj_graphs = [None, None]
        self.graph_gen = self.A.ring_gen()
        self.ctx_gen = None
        self.cent_buf = [t.empty_like(self.cent), t.empty_like(self.cent)]
        self.cent_buf[0].copy_(self.cent)
        self.cent = self.cent_buf[0]
        self.cbuf = 0
        self._counts_buf = [t.zeros(k, dtype=t.int64, device=dev) for _ in range(2)]
        self._done = [t.cuda.Event(), t.cuda.Event()]  # end of the last replay, per parity
        # per parity: around the assign graph and the update graph of a replay
        self._gev = [[t.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(2)]
        self._ahead = None  # iteration already replayed ahead of its step() call
        self._cent_prev = None
        self.bind(0)
        self._pool = None
        self._cap_stream = None
        self._side = None  # graph branch: inertia + label compare

    def bind(self, par):
        """Point the per-parity buffers (min_dists, sq_dists, counts, event
        ring, pinned control block) at parity `par`."""
        self.A.bind(par)
        self.sq, self.counts_buf = self._sq[par], self._counts_buf[par]
        self.ctl_host, self.ctl_i32_host = self._ctl_host[par], self._ctl_i32_host[par]
        self.evc_host = self._evc_host[par]

    def _graph_ok(self, it):
        """Graph replay is used from the second step on: clean steps replay
        the step graph of their buffer parity, steps with scheduled flips
        (up to the static capacity) the injected-pass graph."""
        if not self.use_graph or it < 1:
            return False
        if self.gemm_hook is NOOP_HOOK or type(self.gemm_hook) is FaultHook:
            return True  # the no-op hook never injects
        sched = getattr(self.gemm_hook, "schedule", None)
        if sched is None:
            return False
        n = len(sched.for_iteration(it))
        return n == 0 or (self.sinj is not None and n <= self.sinj.cap)

    def _part_assign(self, it, sinj=None):
        """First half of a graph step (capturable): centroid norms and the
        assignment pass (+ the injected pass's applied/before/after copy)."""
        yn = E.row_sq_norms_dev(self.cent)
        self.A.run(self.cent, yn, NOOP_HOOK, it, self.slot, sinj=sinj)
        if sinj is not None:
            sinj.copy_back()

    def _part_update(self):
        """Second half (capturable, no host synchronisation): inertia + label
        compare on a side-stream branch, update sums, finalize into the other
        static centroid buffer, movement, control copies."""
        A = self.A
        # inertia and the label compare only read the assignment: a graph
        # branch on a side stream, concurrent with the update chain
        cur = self.t.cuda.current_stream()
        if self._side is None:
            self._side = self.t.cuda.Stream()
        side = self._side
        side.wait_stream(cur)
        with self.t.cuda.stream(side):
            E.sq_dists_dev(A.md, self.xsq, self.sq)
            E.pairwise_sum_dev(self.sq, self.ctl_f64[0:1])
            E.labels_equal_dev(A.labels[self.slot], A.labels[1 - self.slot], self.ctl_i32[0:1])
        dmr = self.ft_mode == "abft+dmr"
        sa, ca, sb, cb = E.update_sums_dev(self.x_t, A.labels[self.slot], self.k, dmr=dmr)
        if dmr:  # duplicated accumulators compared on the device; the host reads the flag
            E.dmr_mismatch_dev(sa, ca, sb, cb, self.ctl_i32[2:3])
        if self.dist is not None:
            # row shards: ONE packed all-reduce of the partial sums, counts,
            # inertia and changed-label count (NCCL, captured in the graph)
            cur.wait_stream(side)
            self.dist.reduce_partials(sa, ca, self.ctl_f64, self.ctl_i32)
        new_cent = self.cent_buf[1 - self.cbuf]
        E.finalize_dev(sa, ca, self.dtype, out=new_cent, n_empty=self.ctl_i32[1:2])
        self.counts_buf.copy_(ca)
        E.movement_dev(new_cent, self.cent, self.eps, self.ctl_f64[1:2])
        cur.wait_stream(side)
        self.ctl_host.copy_(self.ctl_f64, non_blocking=True)
        self.ctl_i32_host.copy_(self.ctl_i32, non_blocking=True)
        if A.checked:
            self.evc_host.copy_(A.events.count, non_blocking=True)

    def _capture(self, it):
        """Capture the step graphs of BOTH buffer parities (captured, not
        run), so an eager injected step never leaves a capture for later."""
        t = self.t
        if self.sinj is not None and self.inj_graphs[self.slot] is None:
            # size the injected pass's scratch before capture (a capture cannot
            # allocate): one eager pass with an empty schedule into this
            # step's own outputs, which the replay overwrites
            self.sinj.load(None)
            self.A.run(self.cent, E.row_sq_norms_dev(self.cent), NOOP_HOOK, it, self.slot,
                       sinj=self.sinj)
        t.cuda.synchronize()
        gen0 = E.ctx_generation()
        state = (self.slot, self.cbuf, self.cent)
        todo = [(self.graphs, None)] + ([(self.inj_graphs, self.sinj)] if self.sinj else [])
        for store, sinj in todo:
            for par in (self.slot, 1 - self.slot):
                if store[par] is not None:
                    continue
                self.slot = self.cbuf = par
                self.cent = self.cent_buf[par]
                self.bind(par)
                l0 = N.launch_count()
                try:
                    parts = (self._record(lambda: self._part_assign(it, sinj)),
                             self._record(self._part_update))
                except Exception:
                    # a launch path that needs the host mid-step: stay eager
                    t.cuda.synchronize()
                    self.use_graph = False
                    N.load().ftk_add_launches(-(N.launch_count() - l0))
                    self.slot, self.cbuf, self.cent = state
                    self.bind(self.slot)
                    return False
                store[par] = _StepGraph(parts, N.launch_count() - l0)
                N.load().ftk_add_launches(-store[par].launches)  # captured, not run
        self.slot, self.cbuf, self.cent = state
        self.bind(self.slot)
        if E.ctx_generation() != gen0:  # a capture grew a scratch buffer: redo
            self._drop_graphs()
            return False
        self.ctx_gen = gen0
        return True

    def _record(self, fn):
        """Stream capture of `fn`'s launches into a new graph on a side stream.
        Unlike torch.cuda.graph this does not empty the caching allocator
        (whose cudaFree/cudaMalloc churn cost more than the capture itself);
        the graphs share one private memory pool and replay one at a time."""
        t = self.t
        g = t.cuda.CUDAGraph()
        cur = t.cuda.current_stream()
        if self._cap_stream is None:
            self._cap_stream = t.cuda.Stream()
        s = self._cap_stream
        s.wait_stream(cur)
        with t.cuda.stream(s):
            if self._pool is None:
                g.capture_begin()
            else:
                g.capture_begin(pool=self._pool)
            try:
                fn()
            finally:
                g.capture_end()
        cur.wait_stream(s)
        if self._pool is None:
            self._pool = g.pool()
        return g

    def reset(self, x, c0, gemm_hook=NOOP_HOOK, update_hook=NOOP_HOOK):
        """Start a new fit of the same shape on this engine: X copied into the
        resident buffer, per-fit row bounds and ||x||^2 recomputed in place,
        centroids and step state reset.  Every buffer keeps its address, so
        the captured step graphs are reused (no allocation, no capture)."""
        t = self.t
        if self._ahead is not None:
            t.cuda.current_stream().synchronize()
            self._ahead = None
        if _is_torch(x):
            self.x_t.copy_(x, non_blocking=True)
        else:  # numpy (pageable): the staged parallel uploader
            E.upload_into(self.x_t, np.ascontiguousarray(x, dtype=self.dtype))
        self.xsq.copy_(E.row_sq_norms_dev(self.x_t).to(t.float64))
        self.rows.refresh()
        self.cent_buf[0].copy_(E.to_dev(c0) if not _is_torch(c0) else c0)
        self.cbuf = self.slot = 0
        self.cent = self.cent_buf[0]
        self.bind(0)
        self.gemm_hook, self.update_hook = gemm_hook, update_hook
        self.report = DetectionReport()
        self.assign_ms = self.update_ms = 0.0

    def warm_graphs(self, it=1):
        """Capture the step graphs now (they are otherwise captured at the
        first graph-eligible step); a no-op when graphs are off or ready."""
        if self.use_graph and it >= 1 and (self.graphs[self.slot] is None or (
                self.sinj is not None and self.inj_graphs[self.slot] is None)):
            self._capture(it)

    def _drop_graphs(self):
        self.graphs = [None, None]
        self.inj_graphs = [None, None]

    def _can_run_ahead(self, it):
        """Step `it` may be replayed before the host has read the previous
        step: a clean graph step whose graph is ready and current."""
        if not self._graph_ok(it) or self.graphs[1 - self.slot] is None:
            return False
        sched = getattr(self.gemm_hook, "schedule", None)
        if sched is not None and sched.for_iteration(it):
            return False
        if self.A.ring_gen() != self.graph_gen:
            return False
        return self.ctx_gen is not None and E.ctx_generation() == self.ctx_gen

    def _graph_step(self, it, more=None):
        t, A = self.t, self.A
        self.bind(self.slot)
        inj = None
        if self._ahead == it:
            self._ahead = None  # already replayed behind the previous step
        else:
            self._ahead = None
            if (A.checked and A.ring_gen() != self.graph_gen) or \
                    (self.ctx_gen is not None and E.ctx_generation() != self.ctx_gen):
                self._drop_graphs()  # the event ring or a scratch buffer moved: recapture
                self.graph_gen = A.ring_gen()
                self.ctx_gen = None
            arrs = None
            if self.sinj is not None:
                arrs = self.gemm_hook.kernel_arrays(it, self.dtype)
            store = self.graphs
            if arrs is not None and len(arrs[0]):
                store, inj = self.inj_graphs, self.sinj
            if store[self.slot] is None and not self._capture(it):
                return self.step(it, eager=True)
            self.bind(self.slot)
            if inj is not None:
                inj.load(arrs)  # stream-ordered before the replay
            store[self.slot].replay(self._gev[self.slot])
            self._done[self.slot].record()
        # one step queued ahead: the next replay (the other parity's buffers)
        # goes out before the host reads this step, so the GPU does not idle
        # through the host turnaround.  If this step turns out to be the last,
        # the extra replay only touched buffers nothing reads any more.
        if more is not None and inj is None and self._can_run_ahead(it + 1) and more():
            # the queued step overwrites this step's input centroids; keep a
            # copy for a host-side reseed (movement against the old centroids)
            if self._cent_prev is None:
                self._cent_prev = t.empty_like(self.cent)
            self._cent_prev.copy_(self.cent, non_blocking=True)
            self.graphs[1 - self.slot].replay(self._gev[1 - self.slot])
            self._done[1 - self.slot].record()
            self._ahead = it + 1
        self._done[self.slot].synchronize()
        ge = self._gev[self.slot]  # phase times of this step's replay
        self.assign_ms = ge[0].elapsed_time(ge[1])
        self.update_ms = ge[1].elapsed_time(ge[2])
        n_ev = int(self.evc_host[0]) if A.checked else None
        rep = A.finish(self.gemm_hook, it, inj, n_events=n_ev, replayed=True)
        if rep is not None:
            self.report.merge(rep)
        new_cent = self.cent_buf[1 - self.cbuf]
        if self.ft_mode == "abft+dmr" and self._dmr_flagged():
            self._dmr_retry(it, new_cent)
        if int(self.ctl_i32_host[1]):
            old = self.cent
            if self._ahead is not None:
                # the queued step read the centroids before this reseed: rerun it
                t.cuda.current_stream().synchronize()
                self._ahead = None
                old = self._cent_prev
            if self.dist is not None:
                self.dist.reseed(self.x_t, self.counts_buf, self.sq, new_cent)
            else:
                E.reseed_dev(self.x_t, self.counts_buf, self.sq, new_cent)
            E.movement_dev(new_cent, old, self.eps, self.ctl_f64[1:2])
            # movement only: ctl_f64[0] may already hold the queued step's inertia
            self.ctl_host[1:2].copy_(self.ctl_f64[1:2])
        unchanged = bool(int(self.ctl_i32_host[0]))
        self.cbuf = 1 - self.cbuf
        self.cent = self.cent_buf[self.cbuf]
        self.slot = 1 - self.slot
        return max(0.0, float(self.ctl_host[0])), unchanged, float(self.ctl_host[1])

    def _dmr_flagged(self):
        """The graph step's device DMR compare flag (read after the step)."""
        return bool(int(self.ctl_i32_host[2]))

    def _dmr_retry(self, it, new_cent):
        """A graph step's duplicated update disagreed (kmeans.py:176-189):
        record the mismatch, drop the replay queued on its centroids, and
        redo this iteration's update eagerly -- recomputed sums that disagree
        again raise FaultEscalationError."""
        t = self.t
        if self._ahead is not None:
            # the queued replay overwrote this step's input centroids: restore them
            t.cuda.current_stream().synchronize()
            self._ahead = None
            self.cent.copy_(self._cent_prev)
        self.report.events.append(DetectionEvent(iteration=it, tile=(0, 0), kind="dmr-mismatch",
                                                 loc=(-1, -1), delta=0.0))
        sa, ca, sb, cb = E.update_sums_dev(self.x_t, self.A.labels[self.slot], self.k, dmr=True)
        E.dmr_mismatch_dev(sa, ca, sb, cb, self.ctl_i32[2:3])
        if int(self.ctl_i32[2].item()):
            raise FaultEscalationError(
                f"update-phase DMR mismatch persisted after retry (iteration {it})")
        E.finalize_dev(sa, ca, self.dtype, out=new_cent, n_empty=self.ctl_i32[1:2])
        self.counts_buf.copy_(ca)
        E.movement_dev(new_cent, self.cent, self.eps, self.ctl_f64[1:2])
        self.ctl_host[1:2].copy_(self.ctl_f64[1:2])
        self.ctl_i32_host[1:2].copy_(self.ctl_i32[1:2])

    def step(self, it, eager=False, more=None):
        """One Lloyd iteration; returns (inertia, unchanged, moved), and the
        step's device phase times in assign_ms / update_ms (eager steps: CUDA
        events around the phases; graph steps: events between the assignment
        and update graph replays).
        `more()`: the caller may run step it+1 (lets graph steps keep one
        replay queued ahead)."""
        if self._ahead is not None and (self._ahead != it or eager):
            self.t.cuda.current_stream().synchronize()  # a queued replay nobody reads
            self._ahead = None
        if not eager and (self._ahead == it or (self._graph_ok(it) and self.slot == self.cbuf)):
            return self._graph_step(it, more)
        self.bind(self.slot)
        t, A, ev = self.t, self.A, self.ev
        ev[0].record()
        yn = E.row_sq_norms_dev(self.cent)
        inj = A.run(self.cent, yn, self.gemm_hook, it, self.slot)
        ev[1].record()
        E.sq_dists_dev(A.md, self.xsq, self.sq)
        E.pairwise_sum_dev(self.sq, self.ctl_f64[0:1])
        if it > 0:
            E.labels_equal_dev(A.labels[self.slot], A.labels[1 - self.slot], self.ctl_i32[0:1])
        if inj is not None or (A.checked and self.dist is not None):
            # scheduled flips: the hook needs the applied/before/after arrays
            rep = A.finish(self.gemm_hook, it, inj)
            if rep is not None:
                self.report.merge(rep)
            pending = None
        else:
            pending = A  # events read after the single control readback
        sums, counts, ev_upd = _update_dev(self.x_t, A.labels[self.slot], self.k, self.dtype,
                                          self.ft_mode, self.update_hook, it, self.ctl_i32)
        if self.dist is not None:
            self.dist.reduce_partials(sums, counts, self.ctl_f64, self.ctl_i32, it)
        new_cent = self.cent_buf[1 - self.cbuf]
        E.finalize_dev(sums, counts, self.dtype, out=new_cent, n_empty=self.ctl_i32[1:2])
        E.movement_dev(new_cent, self.cent, self.eps, self.ctl_f64[1:2])
        ev[2].record()
        self.ctl_host.copy_(self.ctl_f64, non_blocking=True)
        self.ctl_i32_host.copy_(self.ctl_i32, non_blocking=True)
        if pending is not None and A.checked:
            self.evc_host.copy_(A.events.count, non_blocking=True)
        t.cuda.current_stream().synchronize()
        if pending is not None:
            rep = A.finish(self.gemm_hook, it, None,
                           n_events=int(self.evc_host[0]) if A.checked else None)
            if rep is not None:
                self.report.merge(rep)
        if int(self.ctl_i32_host[1]):
            if self.dist is not None:
                self.dist.reseed(self.x_t, counts, self.sq, new_cent)
            else:
                E.reseed_dev(self.x_t, counts, self.sq, new_cent)  # sq is free after the sum
            E.movement_dev(new_cent, self.cent, self.eps, self.ctl_f64[1:2])
            self.ctl_host.copy_(self.ctl_f64)
        self.assign_ms = ev[0].elapsed_time(ev[1])
        self.update_ms = ev[1].elapsed_time(ev[2])
        self.report.events.extend(ev_upd)
        unchanged = it > 0 and bool(int(self.ctl_i32_host[0]))
        self.cbuf = 1 - self.cbuf
        self.cent = self.cent_buf[self.cbuf]
        self.slot = 1 - self.slot
        return max(0.0, float(self.ctl_host[0])), unchanged, float(self.ctl_host[1])

    def labels_view(self):
        """Device int32 labels of the last completed step (no copy)."""
        return self.A.labels[1 - self.slot]

    def close(self):
        """Unregister the per-fit row bounds (X may be freed afterwards)."""
        self.rows.close()

    def final(self, iteration):
        """Final assignment against the current centroids -> (labels, inertia)."""
        self._ahead = None  # a queued replay runs before this, on buffers final() does not read
        self.bind(self.slot)
        A = self.A
        yn = E.row_sq_norms_dev(self.cent)
        inj = A.run(self.cent, yn, self.gemm_hook, iteration, self.slot)
        E.sq_dists_dev(A.md, self.xsq, self.sq)
        E.pairwise_sum_dev(self.sq, self.ctl_f64[0:1])
        rep = A.finish(self.gemm_hook, iteration, inj)
        if rep is not None:
            self.report.merge(rep)
        if self.dist is not None:  # the inertia of every shard
            self.dist.all_reduce_(self.ctl_f64[0:1])
        # int64 on the device, one D2H into page-locked memory (the pageable
        # copy plus a host-side astype cost ~2 ms at c2)
        t = self.t
        lab64 = A.labels[self.slot].to(t.int64)
        host = t.empty(lab64.shape[0], dtype=t.int64, pin_memory=True)
        host.copy_(lab64, non_blocking=True)
        inertia = max(0.0, float(self.ctl_f64[0].item()))  # synchronises the stream
        return host.numpy(), inertia


def lloyd(x, config, fault_spec=None):
    """Lloyd's iteration until labels repeat, movement < tol, or max_iters,
    then one final assignment (kmeans.py:210-319)."""
    x = _as_operand(x)
    config.validate()
    m, n = x.shape
    dtype = _dtype(x)
    k = config.k
    if k > m:
        raise ValueError(f"k={k} exceeds the number of samples {m}")
    threads = resolve_threads(config.threads)
    cfg = _resolve_tile(config.tile, x, k, config.tune_table)
    thr = config.threshold or Threshold.default_for(dtype)
    E._torch()
    gemm_hook, update_hook = _plan_hooks(fault_spec, cfg, m, n, k, config.max_iters, dtype)

    # a full cyclic-GC pass over the torch-sized heap stalls the launching
    # thread for tens of ms; the fit allocates no reference cycles
    gc_on = gc.isenabled()
    gc.disable()
    try:
        return _lloyd_fit(x, config, dtype, k, cfg, thr, threads, gemm_hook, update_hook)
    finally:
        if gc_on:
            gc.enable()


# One resident fit workspace (the most recent shape): repeated fits of the same
# shape reuse its buffers and captured graphs (tools/prof_lloyd_e2e.py).
_FIT_CACHE = {}


def _fit_cache_clear():
    eng = _FIT_CACHE.pop("eng", None)
    _FIT_CACHE.pop("key", None)
    if eng is not None:
        eng.close()


def clear_fit_cache():
    """Release the resident fit workspace (device memory of the last shape)."""
    _fit_cache_clear()


def _fit_key(x, k, dtype, cfg, ft_mode, threads, gemm_hook, update_hook, graph, thr):
    """Cache key of a reusable workspace, or None (graph steps only, no
    update-site hook; FTK_FIT_CACHE=0 disables)."""
    if not graph or update_hook is not NOOP_HOOK or os.environ.get("FTK_FIT_CACHE", "1") == "0":
        return None
    sched = getattr(gemm_hook, "schedule", None) is not None
    dev = E._torch().cuda.current_device()
    return (dev, tuple(x.shape), int(k), np.dtype(dtype).str, ft_mode, tuple(cfg.block), int(threads),
            sched, type(gemm_hook).__name__, get_variant(),
            tuple(thr.kernel_params()) if ft_mode != "off" else None)


def _lloyd_fit(x, config, dtype, k, cfg, thr, threads, gemm_hook, update_hook):
    timings = {"init_ns": 0, "assign_ns": 0, "update_ns": 0, "total_ns": 0}
    t_total = time.perf_counter_ns()
    t0 = time.perf_counter_ns()
    src = x
    if config.init == "kmeanspp" and not (_is_torch(x) and x.is_cuda):
        # the D^2 seeding runs on the device: upload once, seed from that copy
        src = E.to_dev(x)
    c0 = init_centroids(src, k, seed=config.seed, method=config.init)
    timings["init_ns"] = time.perf_counter_ns() - t0

    graph = config.max_iters >= 8
    key = _fit_key(x, k, dtype, cfg, config.ft_mode, threads, gemm_hook, update_hook, graph, thr)
    eng = None
    if key is not None and _FIT_CACHE.get("key") == key:
        eng = _FIT_CACHE["eng"]
        eng.reset(src, c0, gemm_hook, update_hook)
    else:
        _fit_cache_clear()
        own = src is not x  # our own upload: no aliasing of a caller's tensor
        eng = LloydEngine(src if own else E.to_dev(x, copy=key is not None), c0, k, dtype, cfg,
                          config.ft_mode, thr, threads, gemm_hook, update_hook, graph=graph)
        if key is not None:
            _FIT_CACHE.update(key=key, eng=eng)
    history = []
    converged = False
    iters = 0
    try:
        ahead = os.environ.get("FTK_RUN_AHEAD", "1") != "0"  # A/B knob
        for it in range(config.max_iters):
            more = (lambda it=it: it + 1 < config.max_iters) if ahead else None
            inertia, unchanged, moved = eng.step(it, more=more)
            timings["assign_ns"] += int(eng.assign_ms * 1e6)
            timings["update_ns"] += int(eng.update_ms * 1e6)
            history.append(inertia)
            iters = it + 1
            if unchanged or moved < config.tol:
                converged = True
                break
        labels, inertia = eng.final(iters)
        centroids = E.to_host(eng.cent)
    finally:
        if key is None:
            eng.close()
    timings["total_ns"] = time.perf_counter_ns() - t_total
    return KMeansResult(centroids=centroids, assignments=labels, inertia=inertia, iters=iters,
                        converged=converged, report=eng.report, timings=timings,
                        inertia_history=history)
