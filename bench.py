"""Benchmark: Lloyd iterations/s of the FT K-means hot path, one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c5] [--campaign-s S] [--c5 0|1]

Workloads (BASELINE.json configs):
  c2 (default)  N=1e6, D=128, K=1024 fp32, ABFT on, per-tile-prob fault campaign
                sized for ~50 injected errors/s.  Data: the reference
                gaussian_mixture (seed 0), random-sample init (seed 0).
  c5            N=1e8, D=128, K=4096 fp32 (the scaling config), FT off; rows
                sharded over the ranks, each rank generating its own shard on
                the device (same recipe as gaussian_mixture, torch RNG: a
                timing workload, not a parity case -- c5's shape is pinned
                against the reference at N=2e5 in tests/test_gpu_configs.py).

A step is one Lloyd iteration (assign + update) of the problem on data
resident in HBM (inputs >= 512 MB > L2: no flush needed).  For N > 1 (one
process per GPU under torchrun) rows are sharded and the per-iteration
partial sums/counts are all-reduced over NCCL ("strong": the problem is
fixed, ranks split it).  Timing: CUDA events over exactly K steps after W
warm-up steps, barrier + synchronize on both sides, max over ranks.

`--impl reference` times the reference algorithm on the host cores: the
oracle's C restatement of the reference's ``lloyd`` with its checksum-verified
assignment (oracle/, all host threads), over FULL c2 iterations (every row,
assign + update), measured -- not extrapolated.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(rows=1_000_000, dim=128, k=1024, ft="abft",
               workload="c2: N=1e6 D=128 K=1024 fp32, ABFT on, per-tile-prob campaign sized for "
                        "~50 errors/s"),
    "c4": dict(rows=10_000_000, dim=64, k=256, ft="abft",
               workload="c4: N=1e7 D=64 K=256 fp64, ABFT on (FT-off interleaved for the overhead)"),
    "c5": dict(rows=100_000_000, dim=128, k=4096, ft="off",
               workload="c5: N=1e8 D=128 K=4096 fp32, FT off, rows sharded over the ranks"),
}
ERR_PER_S = 50.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def _tf32_peak():
    """Dense TF32 denominator: a measured cuBLAS TF32 GEMM peak when
    profiles/ holds one for this box type, else MEASURED_PEAKS bf16 / 2."""
    p = os.path.join(ROOT, "profiles", "peaks_tf32_f64.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        if j.get("tf32_tflops"):
            return float(j["tf32_tflops"]), "measured cuBLAS TF32 GEMM (profiles/peaks_tf32_f64.json)"
    _, bf16, src = _peaks()
    return bf16 / 2.0, f"dense tf32 = bf16_tflops/2 from MEASURED_PEAKS.json ({src})"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """Clock + throttle-reason sampling DURING the timed region, in-process
    through NVML (a sampling thread that forked nvidia-smi every 50 ms stalled
    the launching thread for tens of ms); nvidia-smi only if NVML is absent."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nv = None
        try:
            import pynvml as nv
            import torch

            nv.nvmlInit()
            pr = torch.cuda.get_device_properties(index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            try:
                self._h = nv.nvmlDeviceGetHandleByPciBusId_v2(bus)
            except Exception:
                self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self._nv = nv
        except Exception:
            self._nv = None

    def _sample_nvml(self):
        nv, h = self._nv, self._h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nv is not None:
                    self.rows.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          "--query-gpu=" + self.Q, "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.01 if self._nv is not None else 0.05)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        self.rows = [r for r in self.rows if len(r) >= 6]  # drop nvidia-smi error lines
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm),
                "source": "nvml" if self._nv is not None else "nvidia-smi"}


def make_data(cfg, seed=0):
    from paper_2408_01391_b200.matrix import gaussian_mixture

    x, _, _ = gaussian_mixture(cfg["rows"], cfg["dim"], cfg["k"], 0.25, precision="single", seed=seed)
    return x


def make_shard_dev(cfg, lo, hi, seed=0, dtype="float32"):
    """Rows [lo, hi) of a gaussian_mixture-shaped dataset generated on the
    device: the reference's centers (numpy default_rng(seed), rescaled to a
    minimum pairwise distance of 20 * spread, matrix.py:86-110), uniform
    labels and 0.25-spread Gaussian noise from a torch CUDA generator seeded
    per shard.  Same distribution as gaussian_mixture, not the same bytes."""
    import torch

    from paper_2408_01391_b200.matrix import _min_pairwise_sq

    k, d = cfg["k"], cfg["dim"]
    rng = np.random.default_rng(seed)
    centers = rng.random((k, d))
    md = np.sqrt(_min_pairwise_sq(centers))
    if md < 20 * 0.25:
        centers *= 20 * 0.25 / max(md, 1e-12)
    cen = torch.from_numpy(centers).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed * 1_000_003 + lo)
    x = torch.empty((hi - lo, d), dtype=getattr(torch, dtype), device="cuda")
    ch = 1 << 22
    for r0 in range(0, hi - lo, ch):
        r1 = min(hi - lo, r0 + ch)
        lab = torch.randint(0, k, (r1 - r0,), generator=g, device="cuda")
        x[r0:r1] = (cen[lab] + 0.25 * torch.randn((r1 - r0, d), generator=g, device="cuda",
                                                   dtype=torch.float64)).to(x.dtype)
    # random-sample init (the first k rows of a seeded permutation of shard 0,
    # broadcast so every rank starts from the same centroids)
    return x, centers


def _campaign_schedule(p, it0, iters, m, k, seed, bm=32, bn=256):
    """Per-tile-probability campaign over iterations [it0, it0 + iters), drawn
    vectorised (same distribution as faults.plan_faults' per-tile-prob mode
    with uniform bits, not its draw order -- plan_faults walks every
    (iteration, tile) in Python, far too slow for thousands of iterations
    over 125k tiles)."""
    from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule

    rng = np.random.default_rng(seed)
    nbi, nbj = (m + bm - 1) // bm, (k + bn - 1) // bn
    n_hit = rng.binomial(iters * nbi * nbj, p)
    flat = np.unique(rng.integers(0, iters * nbi * nbj, size=n_hit))
    out = []
    for f in flat.tolist():
        it, t = divmod(f, nbi * nbj)
        bi, bj = divmod(t, nbj)
        mi, nj = min(bm, m - bi * bm), min(bn, k - bj * bn)
        out.append(FaultEntry(it0 + it, (bi, bj), (int(rng.integers(0, mi)), int(rng.integers(0, nj))),
                              int(rng.integers(0, 32))))
    return FaultSchedule(out)


# ------------------------------------------------------------- reference --
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.lib()
    return O


def cpu_lloyd_full(x, k, steps, ft_mode, threads, budget_s=150.0):
    """The oracle's restatement of the reference ``lloyd`` (kmeans.py:210-319)
    over `steps` FULL iterations of the workload (every row, assign + update;
    ft_mode "abft": the reference's checksum-verified assignment), timed.
    A first iteration sizes the run so it stays within `budget_s`."""
    O = _oracle()
    c = O.init_centroids(x, k, 0, "random-sample")
    t0 = time.perf_counter()
    r = O.lloyd(x, k, max_iters=1, tol=0.0, seed=0, init="random-sample", threads=threads,
                centroids=c, ft_mode=ft_mode)
    first = time.perf_counter() - t0
    steps = max(1, min(steps, int(budget_s / max(first, 1e-3))))
    r = O.lloyd(x, k, max_iters=steps, tol=0.0, seed=0, init="random-sample", threads=threads,
                centroids=c, ft_mode=ft_mode)
    tm = r["timings"]
    loop_ns = tm["assign_ns"] + tm["update_ns"]
    per_iter_ns = loop_ns / max(r["iters"], 1)
    return {"iters": r["iters"], "s_per_iter": per_iter_ns * 1e-9, "iter_per_s": 1e9 / per_iter_ns,
            "assign_ms": tm["assign_ns"] / max(r["iters"], 1) * 1e-6,
            "update_ms": tm["update_ns"] / max(r["iters"], 1) * 1e-6}


def cpu_c1(threads, reps=3):
    """SURVEY 8(d) CPU baseline of record: the reference lloyd on c1
    (N=1e5, D=32, K=64, 20 iterations, random-sample, FT off), median of
    `reps` after a warm-up, at `threads` threads."""
    from paper_2408_01391_b200.matrix import gaussian_mixture

    O = _oracle()
    x, _, _ = gaussian_mixture(100_000, 32, 64, 0.25, precision="single", seed=0)
    O.lloyd(x, 64, max_iters=2, tol=0.0, seed=0, init="random-sample", threads=threads)
    vals = []
    for _ in range(reps):
        r = O.lloyd(x, 64, max_iters=20, tol=0.0, seed=0, init="random-sample", threads=threads)
        tm = r["timings"]
        vals.append(r["iters"] / ((tm["total_ns"] - tm["init_ns"]) * 1e-9))
    return statistics.median(vals)


def cpu_baseline_record(x, k, steps, ft_mode):
    threads = os.cpu_count() or 1
    full = cpu_lloyd_full(x, k, steps, ft_mode, threads)
    return {"value": full["iter_per_s"], "unit": "iter/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{full['iters']} full Lloyd iterations (all {x.shape[0]} rows, assign+update, "
                      f"ft_mode={ft_mode}) of the workload through the oracle's restatement of the "
                      f"reference lloyd; measured, not extrapolated",
            "assign_ms": full["assign_ms"], "update_ms": full["update_ms"]}


def run_reference(args, rank):
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    if args.config != "c2":
        print(json.dumps({"impl": "reference", "unavailable":
                          "c5 (N=1e8) needs ~25 CPU-minutes per iteration; the reference arm runs c2"}))
        return
    x = make_data(cfg)
    cb = cpu_baseline_record(x, cfg["k"], args.steps, cfg["ft"])
    line = {"metric": "lloyd_iters_per_s", "value": cb["value"], "unit": "iter/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cb["value"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic gaussian_mixture seed 0",
            "config": {"workload": cfg["workload"] + " (CPU: reference lloyd restated in C, "
                                                     "checksum-verified assignment, no injection)"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "iter/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------- ours --
def run_ours(args, rank, world):
    import torch

    import paper_2408_01391_b200 as P
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200 import _native
    from paper_2408_01391_b200.faults import ScheduledFaultHook
    from paper_2408_01391_b200.kmeans import LloydEngine
    from paper_2408_01391_b200.tiles import default_config

    cfg = CONFIGS[args.config]
    N_ROWS, DIM, K = cfg["rows"], cfg["dim"], cfg["k"]
    # FTK_BENCH_DEVICE pins every rank to one GPU and FTK_DIST_BACKEND=gloo
    # lets the sharded path be exercised on a single-GPU box (test only)
    dev_env = os.environ.get("FTK_BENCH_DEVICE")
    torch.cuda.set_device(int(dev_env) if dev_env is not None else int(os.environ.get("LOCAL_RANK", 0)))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("FTK_DIST_BACKEND", "nccl"))
    from paper_2408_01391_b200.shard import ShardComm

    lo, hi = ShardComm.shard_bounds(N_ROWS, world, rank)
    if args.config == "c2":
        x = make_data(cfg)
        x_t = E.to_dev(x[lo:hi])
        c0 = P.init_centroids(x, K, seed=0, method="random-sample")
    else:
        x = None
        x_t, _ = make_shard_dev(cfg, lo, hi)
        # every rank starts from the same centroids: rank 0's first K rows
        c0 = x_t[:K].clone() if rank == 0 else torch.empty((K, DIM), dtype=torch.float32, device="cuda")
        if world > 1:
            torch.distributed.broadcast(c0, 0)
    tcfg = default_config(np.float32)
    thr = P.Threshold.default_for(np.float32)
    comm = ShardComm(lo) if world > 1 else None

    def engine(ft_mode, hook=None):
        return LloydEngine(x_t, c0, K, np.float32, tcfg, ft_mode, thr, 64,
                           gemm_hook=hook or P.FaultHook(), dist=comm, graph=True)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    step_stats = []
    upd_ms = []

    def time_steps(eng, steps, warmup):
        """W warm-up steps, one eager step (phase timings + the screen's own
        CUDA events), then exactly `steps` timed steps."""
        gc.collect()
        gc.disable()  # a cyclic-GC pass in the timed region stalls the launching thread
        for it in range(warmup):
            eng.step(it)
        eng.step(warmup, eager=True)
        a_ms, k_ms = eng.assign_ms, E.tc_last_kernel_ms()
        upd_ms.append(eng.update_ms)  # the update phase of the eager step (CUDA events)
        eng.warm_graphs(warmup + 1)
        barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        l0 = _native.launch_count()
        evs[0].record()
        last = warmup + steps
        for i, it in enumerate(range(warmup + 1, warmup + 1 + steps)):
            # graph steps keep one replay queued ahead, never past the last timed
            # step; per-step event gaps are then approximate, the total is exact
            eng.step(it, more=(lambda it=it: it < last))
            evs[i + 1].record()
        barrier()
        launches = _native.launch_count() - l0
        ms = max_over_ranks(evs[0].elapsed_time(evs[-1]))
        per = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(steps))
        step_stats.append({"p50": per[len(per) // 2], "max": per[-1], "min": per[0]})
        gc.enable()
        return ms / steps, a_ms, launches, (k_ms if k_ms > 0 else None)

    hbm, _, _ = _peaks()
    tf32_peak, peak_note = _tf32_peak()
    flops = 2.0 * N_ROWS * DIM * K / world

    if args.config == "c5":
        eng = engine("off")
        with ClockSampler(torch.cuda.current_device()) as cs:
            ms, a_ms, launches, k_ms = time_steps(eng, args.steps, args.warmup)
        eng.close()
        kern = k_ms or a_ms
        if rank == 0:
            print(json.dumps({
                "metric": "lloyd_iters_per_s", "value": 1e3 / ms, "unit": "iter/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic: gaussian_mixture recipe generated per shard on the device",
                "config": {"workload": cfg["workload"], "global_batch": N_ROWS,
                           "parallelism": f"dp{world} (row shards, NCCL all-reduce of partials)",
                           "l2": "inputs 51 GB > L2 (no flush)"},
                "roofline": {"bound": "tensor", "achieved": flops / (kern * 1e-3) / 1e12,
                             "peak": tf32_peak, "unit": "TFLOP/s",
                             "frac": flops / (kern * 1e-3) / 1e12 / tf32_peak, "peak_note": peak_note,
                             "kernel": "pair_screen_kernel (tcgen05 tf32 screen, fused argmin)",
                             "kernel_ms": kern, "traffic": None},
                "assign_ms": a_ms, "assign_tflops": flops / (a_ms * 1e-3) / 1e12,
                "gpu_launches": launches, "clocks": cs.summary(), "cpu_baseline": None,
                "e2e": None, "e2e_note": "c5's 51 GB input does not fit a host-buffer fit here"}))
        return

    # ---- c2: FT-off and ABFT timed runs (the line's value is the ABFT one)
    eng_off = engine("off")
    ms_off, a_off, _, k_off = time_steps(eng_off, args.steps, args.warmup)
    eng_off.close()
    n_tiles = ((hi - lo + tcfg.block[0] - 1) // tcfg.block[0]) * ((K + tcfg.block[1] - 1) // tcfg.block[1])
    p = min(1.0, ERR_PER_S * (ms_off * 1e-3) / n_tiles)
    horizon = args.warmup + args.steps + 1
    sched = _campaign_schedule(p, 0, horizon, hi - lo, K, seed=1)
    hook = ScheduledFaultHook(sched)
    eng = engine("abft", hook)
    with ClockSampler(torch.cuda.current_device()) as cs:
        ms_ft, a_ft, launches, k_ft = time_steps(eng, args.steps, args.warmup)
    eng.close()
    clocks = cs.summary()
    injected = len(hook.injected)
    rep = eng.report

    # ---- FT overhead: interleaved FT-off / ABFT-under-injection repetitions
    # (median of >= 10), both engines stepping the same iterations from the
    # same centroids.  Every flip is corrected, so the two runs stay in
    # lockstep: identical inertia at every step and identical final labels
    # ("zero label divergence"), checked here on the full campaign.
    campaign = None
    if args.campaign_s > 0:
        reps = max(10, args.reps)
        per = max(20, int(args.campaign_s / reps / max(ms_ft * 1e-3, 1e-6)))
        total = reps * per
        c_sched = _campaign_schedule(p, 1, total, hi - lo, K, seed=2)
        c_hook = ScheduledFaultHook(c_sched)
        e_off, e_ft = engine("off"), engine("abft", c_hook)
        hist = {0: [], 1: []}
        for e in (e_off, e_ft):
            e.step(0)
            e.warm_graphs(1)
        barrier()
        times = {0: [], 1: []}
        flags0 = E.abft_flags_total(reset=True)
        with ClockSampler(torch.cuda.current_device()) as ccs:
            gc.collect()
            gc.disable()
            for r in range(reps):
                for side, e in ((0, e_off), (1, e_ft)):
                    its = range(1 + r * per, 1 + (r + 1) * per)
                    last = its[-1]
                    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s0.record()
                    for it in its:
                        out = e.step(it, more=(lambda it=it: it < last))
                        hist[side].append(out[0])
                    s1.record()
                    torch.cuda.synchronize()
                    times[side].append(s0.elapsed_time(s1))
            gc.enable()
        flags = E.abft_flags_total() - flags0
        lab_off = e_off.labels_view()
        lab_ft = e_ft.labels_view()
        divergence = int((lab_off != lab_ft).sum().item())
        hist_equal = hist[0] == hist[1]
        c_rep = e_ft.report
        c_inj = len(c_hook.injected)
        ft_s = sum(times[1]) * 1e-3
        over = [100.0 * (b / a - 1.0) for a, b in zip(times[0], times[1])]
        campaign = {"reps": reps, "steps_per_rep": per, "iters": total,
                    "overhead_pct_median": statistics.median(over),
                    "overhead_pct_min": min(over), "overhead_pct_max": max(over),
                    "ft_ms_per_step": sum(times[1]) / total, "off_ms_per_step": sum(times[0]) / total,
                    "injected": c_inj, "injected_per_s": c_inj / ft_s,
                    "detections": c_rep.detections, "corrections": c_rep.corrections,
                    "uncorrectable": c_rep.uncorrectable, "false_alarms": c_rep.false_alarms,
                    "tc_checksum_flags": flags,
                    "label_divergence": divergence, "inertia_history_equal": hist_equal,
                    "p_tile": p, "clocks": ccs.summary()}
        e_off.close()
        e_ft.close()
        del e_off, e_ft

    # ---- DMR on the update (abft+dmr vs abft, fault-free), interleaved: the
    # duplicated accumulators and the device compare run inside the graph steps
    dmr = None
    if args.campaign_s > 0:
        reps, per = 5, 20
        e_a, e_d = engine("abft"), engine("abft+dmr")
        for e in (e_a, e_d):
            e.step(0)
            e.warm_graphs(1)
        barrier()
        tms = {0: [], 1: []}
        gc.collect()
        gc.disable()
        for r in range(reps):
            for side, e in ((0, e_a), (1, e_d)):
                its = range(1 + r * per, 1 + (r + 1) * per)
                last = its[-1]
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                for it in its:
                    e.step(it, more=(lambda it=it: it < last))
                s1.record()
                torch.cuda.synchronize()
                tms[side].append(s0.elapsed_time(s1))
        gc.enable()
        over = [100.0 * (b / a - 1.0) for a, b in zip(tms[0], tms[1])]
        dmr = {"reps": reps, "steps_per_rep": per, "overhead_pct_median": statistics.median(over),
               "abft_ms_per_step": sum(tms[0]) / (reps * per), "dmr_ms_per_step": sum(tms[1]) / (reps * per),
               "dmr_mismatches": e_d.report.dmr_mismatches, "graph_steps": bool(e_d.use_graph),
               "labels_equal": bool((e_a.labels_view() == e_d.labels_view()).all().item())}
        e_a.close()
        e_d.close()
        del e_a, e_d

    B_u = (hi - lo) * DIM * 4 + (hi - lo) * 8 + K * DIM * 8 + K * 8
    kern_ms = k_ft if k_ft else a_ft
    achieved = flops / (kern_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("pair_screen_kernel_chk_c2_bytes")
        if traffic is not None and world > 1:
            traffic = int(traffic * (hi - lo) / N_ROWS)

    # ---- e2e through the public API with host buffers: the reference's own
    # call (a numpy array, pageable memory) and a pinned torch tensor
    e2e = None
    if world == 1:
        conf = P.KMeansConfig(k=K, max_iters=args.steps, tol=0.0, seed=0, init="random-sample",
                              ft_mode="abft")

        def fit_wall(inp):
            # one untimed fit first: the timed fit sees a warm process, like
            # any fit after the first in a serving process
            P.lloyd(inp, conf)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = P.lloyd(inp, conf)
            torch.cuda.synchronize()
            return r, time.perf_counter() - t0

        r_np, wall_np = fit_wall(x)
        xp = torch.from_numpy(x).pin_memory()
        r_pin, wall_pin = fit_wall(xp)
        del xp
        assert np.array_equal(r_np.assignments, r_pin.assignments)
        e2e = {"value": r_np.iters / wall_np, "unit": "iter/s",
               "h2d_bytes_per_step": int(x.nbytes // max(r_np.iters, 1)),
               "d2h_bytes_per_step": int(N_ROWS * 8 // max(r_np.iters, 1)),
               "iters": r_np.iters, "wall_s": wall_np,
               "input": "numpy float32 (pageable host memory), lloyd() public API, ABFT",
               "pinned": {"value": r_pin.iters / wall_pin, "wall_s": wall_pin,
                          "input": "torch pinned host tensor"}}
        P.clear_fit_cache()

    # ---- c5 at one GPU (the scaling config's 1-GPU point, same sharded code
    # path as --config c5) and the CPU baselines
    c5 = None
    if world == 1 and args.c5:
        del eng_off, eng
        gc.collect()
        torch.cuda.empty_cache()
        c5 = c5_point(args)
    c4 = c4_point(args) if world == 1 and args.c4 else None
    cpu = None
    if rank == 0 and world == 1:
        cpu = cpu_baseline_record(x, K, 3, "abft")
        threads = os.cpu_count() or 1
        cpu["c1_reference_iter_per_s"] = {"threads_all": cpu_c1(threads), "threads_1": cpu_c1(1),
                                          "cores": threads}
    if rank != 0:
        return
    line = {
        "metric": "lloyd_iters_per_s", "value": 1e3 / ms_ft, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_ft,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference gaussian_mixture(1e6, 128, 1024 blobs, 0.25, seed 0); "
                "random-sample init seed 0",
        "config": {"workload": cfg["workload"], "global_batch": N_ROWS,
                   "parallelism": f"dp{world} (row shards)", "l2": "inputs 512 MB > L2 (no flush)",
                   "variant": P.gemm.get_variant()},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": tf32_peak,
                     "unit": "TFLOP/s", "frac": achieved / tf32_peak, "peak_note": peak_note,
                     "frac_vs_bf16_half": achieved / (_peaks()[1] / 2.0),
                     "kernel": "pair_screen_kernel<CHK> (cta_group::2 tcgen05 tf32 screen + "
                               "fused argmin/certificate/exact refine/ABFT)",
                     "kernel_ms": kern_ms, "traffic": traffic,
                     "traffic_note": "dram read+write bytes per launch, ncu --set full "
                                     "(profiles/traffic.json)"},
        "assign_ms": a_ft, "assign_tflops": flops / (a_ft * 1e-3) / 1e12,
        "update_roofline": {"bound": "hbm", "unit": "GB/s", "peak": hbm, "ms": upd_ms[-1],
                            "bytes": B_u, "achieved": B_u / (upd_ms[-1] * 1e-3) / 1e9,
                            "frac": B_u / (upd_ms[-1] * 1e-3) / 1e9 / hbm,
                            "note": "SURVEY 8(d) B_u = N*D*s + N*8 + K*D*8 + K*8 over the whole update phase "
                                    "(sort, certified segment sums, fold, finalize) of one eager step"},
        "ft_off_kernel_ms": k_off, "ft_off_ms_per_step": ms_off,
        "ft_overhead_pct": 100.0 * (ms_ft / ms_off - 1.0),
        "faults": {"injected": injected, "detections": rep.detections,
                   "corrections": rep.corrections, "uncorrectable": rep.uncorrectable, "p_tile": p},
        "ft_campaign": campaign,
        "dmr": dmr,
        "step_ms": {"ft_off": step_stats[0], "abft": step_stats[1]},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "c5_1gpu": c5,
        "c4_1gpu": c4,
    }
    print(json.dumps(line))


def c5_point(args):
    """c5 (N=1e8, D=128, K=4096 fp32, FT off) on this GPU through the
    row-sharded engine path (world 1): iterations/s and the screen's TF/s."""
    import torch

    import paper_2408_01391_b200 as P
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200.kmeans import LloydEngine

    cfg = CONFIGS["c5"]
    free, _ = torch.cuda.mem_get_info()
    if free < 70e9:
        return {"skipped": f"only {free / 1e9:.0f} GB free"}
    x_t, _ = make_shard_dev(cfg, 0, cfg["rows"])
    c0 = x_t[:cfg["k"]].clone()
    eng = LloydEngine(x_t, c0, cfg["k"], np.float32, P.default_config(np.float32), "off",
                      P.Threshold.default_for(np.float32), 64, graph=True)
    warm, steps = 2, 3
    for it in range(warm):
        eng.step(it)
    eng.step(warm, eager=True)
    k_ms, a_ms, u_ms = E.tc_last_kernel_ms(), eng.assign_ms, eng.update_ms
    eng.warm_graphs(warm + 1)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    last = warm + steps
    for it in range(warm + 1, last + 1):
        eng.step(it, more=(lambda it=it: it < last))
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / steps
    eng.close()
    del eng, x_t
    torch.cuda.empty_cache()
    flops = 2.0 * cfg["rows"] * cfg["dim"] * cfg["k"]
    peak, note = _tf32_peak()
    return {"workload": cfg["workload"] + ", 1 GPU", "iter_per_s": 1e3 / ms, "ms_per_step": ms,
            "steps": steps, "warmup": warm, "screen_ms": k_ms, "assign_ms": a_ms, "update_ms": u_ms,
            "screen_tflops": flops / (k_ms * 1e-3) / 1e12, "frac": flops / (k_ms * 1e-3) / 1e12 / peak,
            "peak": peak, "peak_note": note,
            "data": "device-generated gaussian_mixture recipe (torch RNG), random-sample init"}


def c4_point(args, reps=5, per=2):
    """c4 (N=1e7, D=64, K=256 fp64, ABFT) on this GPU: an ABFT engine and an
    FT-off engine from the same centroids, `per` steps each, interleaved
    `reps` times (median ms per step of each), the overhead and the label
    divergence between the two runs' final labels (fault-free ABFT is
    bit-identical to FT off)."""
    import torch

    import paper_2408_01391_b200 as P
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200 import variants as V
    from paper_2408_01391_b200.kmeans import LloydEngine

    cfg = CONFIGS["c4"]
    x_t, _ = make_shard_dev(cfg, 0, cfg["rows"], dtype="float64")
    c0 = x_t[:cfg["k"]].clone()
    thr = P.Threshold.default_for(np.float64)
    engs = {ft: LloydEngine(x_t, c0, cfg["k"], np.float64, P.default_config(np.float64), ft, thr, 64)
            for ft in ("off", "abft")}
    for eng in engs.values():  # warm-up: first iterations of a fit reshuffle many labels
        for it in range(2):
            eng.step(it)
    times = {"off": [], "abft": []}
    phase = {"off": [], "abft": []}
    it = 2
    for _ in range(reps):
        for ft, eng in engs.items():
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for q in range(per):
                eng.step(it + q)
            s1.record()
            torch.cuda.synchronize()
            times[ft].append(s0.elapsed_time(s1) / per)
            phase[ft].append((eng.assign_ms, eng.update_ms))
        it += per
    lab = {ft: E.to_host(eng.labels_view()) for ft, eng in engs.items()}
    rep = engs["abft"].report
    fb = E.tc_fallback_rows()
    for eng in engs.values():
        eng.close()
    del engs, x_t
    torch.cuda.empty_cache()
    ms = {ft: float(np.median(v)) for ft, v in times.items()}
    a_ms = float(np.median([p[0] for p in phase["abft"]]))
    u_ms = float(np.median([p[1] for p in phase["abft"]]))
    flops = 2.0 * cfg["rows"] * cfg["dim"] * cfg["k"]
    return {"workload": cfg["workload"] + ", 1 GPU", "iter_per_s": 1e3 / ms["abft"],
            "ms_per_step": ms["abft"], "ft_off_ms_per_step": ms["off"],
            "ft_overhead_pct": 100.0 * (ms["abft"] / ms["off"] - 1.0),
            "reps": reps, "steps_per_rep": per, "assign_ms": a_ms, "update_ms": u_ms,
            "assign_tflops_f64_equiv": flops / (a_ms * 1e-3) / 1e12,
            "variant": V.resolve((cfg["rows"], cfg["dim"], cfg["k"]), np.float64, True),
            "uncertified_rows_last_pass": int(fb[0]),
            "label_divergence": int((lab["off"] != lab["abft"]).sum()),
            "detections": rep.detections, "false_alarms": rep.false_alarms,
            "data": "device-generated gaussian_mixture recipe (torch RNG, float64), first-k-rows init"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c5"])
    ap.add_argument("--variant", default=None)
    ap.add_argument("--campaign-s", type=float, default=1.0,
                    help="seconds of ABFT iterations under ~50 injected errors/s (0: skip)")
    ap.add_argument("--reps", type=int, default=10, help="interleaved FT-off/on repetitions")
    ap.add_argument("--c5", type=int, default=1, help="also time c5 on one GPU (N=1 only)")
    ap.add_argument("--c4", type=int, default=1, help="also time c4 (fp64) on one GPU (N=1 only)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.variant:
        from paper_2408_01391_b200 import gemm

        gemm.set_variant(args.variant)
    run_ours(args, rank, world)


if __name__ == "__main__":
    main()
