"""Benchmark: Lloyd iterations/s on BASELINE configs[1] (N=1e6, D=128, K=1024,
fp32, ABFT on, ~50 injected errors/s), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one Lloyd iteration (assign + update) of the fixed problem on data
resident in HBM (inputs 512 MB > L2, so no flush is needed).  For N > 1 (one
process per GPU under torchrun) the rows are sharded across ranks and the
per-iteration partial sums/counts are all-reduced over NCCL ("strong"
scaling: the problem is fixed, ranks split it).  `--impl reference` times the
reference algorithm's CPU restatement (oracle/, multi-threaded C) on a
bounded sample of the same workload and reports the same metric.
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

N_ROWS, DIM, K = 1_000_000, 128, 1024
ERR_PER_S = 50.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


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


def make_data(seed=0):
    from paper_2408_01391_b200.matrix import gaussian_mixture

    x, _, _ = gaussian_mixture(N_ROWS, DIM, K, 0.25, precision="single", seed=seed)
    return x


def _campaign_schedule(p, iters, m, k, seed, bm=32, bn=256):
    """Per-tile-probability campaign drawn vectorised (same distribution as
    faults.plan_faults' per-tile-prob mode with uniform bits, not its draw
    order -- plan_faults walks every (iteration, tile) in Python, far too slow
    for a ~1 s campaign over 125k tiles)."""
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
        out.append(FaultEntry(it, (bi, bj), (int(rng.integers(0, mi)), int(rng.integers(0, nj))),
                              int(rng.integers(0, 32))))
    return FaultSchedule(out)


# ------------------------------------------------------------- reference --
def cpu_reference(x, threads=None, sample_rows=50_000, iters=2):
    """Times the oracle's Lloyd iteration (assign + update; C, all host
    threads) on the first `sample_rows` rows with the workload's centroids,
    scaled linearly in N to the full problem."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.lib()
    threads = threads or os.cpu_count() or 1
    xs = np.ascontiguousarray(x[:sample_rows])
    c = O.init_centroids(x, K, 0, "random-sample")
    O.assign(xs[:2000], c, threads=threads)  # warm
    t0 = time.perf_counter()
    for _ in range(iters):
        lab, md = O.assign(xs, c, threads=threads)
        O.update_step(xs, lab, K, sq_dists=md.astype(np.float64), threads=threads)
    dt = (time.perf_counter() - t0) / iters
    t_full = dt * (N_ROWS / sample_rows)
    return {"value": 1.0 / t_full, "unit": "iter/s", "cores": threads, "kind": "port",
            "sample": f"{iters} Lloyd iterations (assign+update) on {sample_rows} of {N_ROWS} rows, "
                      f"D={DIM}, K={K}, extrapolated linearly in N ({dt * 1e3:.1f} ms/sample-iter)"}


def run_reference(args, rank):
    if rank != 0:
        return
    x = make_data()
    cb = cpu_reference(x, iters=max(1, min(args.steps, 3)))
    line = {"metric": "lloyd_iters_per_s", "value": cb["value"], "unit": "iter/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / cb["value"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic gaussian_mixture seed 0",
            "config": {"workload": "c2: N=1e6 D=128 K=1024 fp32 (CPU reference restatement)"},
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
    from paper_2408_01391_b200.faults import FaultSpec, ScheduledFaultHook, plan_faults
    from paper_2408_01391_b200.kmeans import LloydEngine
    from paper_2408_01391_b200.tiles import default_config

    # FTK_BENCH_DEVICE pins every rank to one GPU and FTK_DIST_BACKEND=gloo
    # lets the sharded path be exercised on a single-GPU box (test only)
    dev_env = os.environ.get("FTK_BENCH_DEVICE")
    torch.cuda.set_device(int(dev_env) if dev_env is not None else int(os.environ.get("LOCAL_RANK", 0)))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("FTK_DIST_BACKEND", "nccl"))
    x = make_data()
    lo, hi = rank * N_ROWS // world, (rank + 1) * N_ROWS // world
    x_t = E.to_dev(x[lo:hi])
    c0 = P.init_centroids(x, K, seed=0, method="random-sample")
    cfg = default_config(np.float32)
    thr = P.Threshold.default_for(np.float32)

    comm = None
    if world > 1:
        from paper_2408_01391_b200.shard import ShardComm

        comm = ShardComm(lo)

    def engine(ft_mode, hook=None):
        return LloydEngine(x_t, c0, K, np.float32, cfg, ft_mode, thr, 64,
                           gemm_hook=hook or P.FaultHook(), dist=comm, graph=True)

    step_stats = []  # per-step device times of each timed run (min/median/max)

    def time_steps(eng, steps, warmup, sampler=None):
        gc.collect()
        gc.disable()  # a cyclic-GC pass in the timed region stalls the launching thread
        for it in range(warmup):
            eng.step(it)
        # one eager (non-graph) step: phase timings and CUDA events around the
        # screen launch on its stream (graph replays carry no events)
        eng.step(warmup, eager=True)
        a_ms, k_ms = [eng.assign_ms], [E.tc_last_kernel_ms()]
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        l0 = _native.launch_count()
        evs[0].record()
        last = warmup + steps
        for i, it in enumerate(range(warmup + 1, warmup + 1 + steps)):
            # graph steps keep one replay queued ahead, never past the last timed
            # step; per-step event gaps are then approximate, the total is exact
            eng.step(it, more=(lambda it=it: it < last))
            evs[i + 1].record()
        torch.cuda.synchronize()
        launches = _native.launch_count() - l0
        ms = evs[0].elapsed_time(evs[-1])
        per = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(steps))
        step_stats.append({"p50": per[len(per) // 2], "max": per[-1], "min": per[0]})
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        kern = [v for v in k_ms if v > 0]
        gc.enable()
        return ms / steps, statistics.median(a_ms), launches, (statistics.mean(kern) if kern else None)

    # FT-off reference timing and the per-iteration time used to size the campaign
    eng_off = engine("off")
    ms_off, a_off, _, k_off = time_steps(eng_off, args.steps, args.warmup)
    eng_off.close()
    n_tiles = ((hi - lo + cfg.block[0] - 1) // cfg.block[0]) * ((K + cfg.block[1] - 1) // cfg.block[1])
    p = min(1.0, ERR_PER_S * (ms_off * 1e-3) / n_tiles)
    horizon = args.warmup + args.steps + 1
    spec = FaultSpec(mode="per-tile-prob", prob=p, seed=1)
    sched = plan_faults(spec, horizon, ((hi - lo + 31) // 32, (K + 255) // 256), (32, 256),
                        dtype=np.float32, shape=(hi - lo, K))
    hook = ScheduledFaultHook(sched)
    eng = engine("abft", hook)
    with ClockSampler(torch.cuda.current_device()) as cs:
        ms_ft, a_ft, launches, k_ft = time_steps(eng, args.steps, args.warmup, cs)
    eng.close()
    clocks = cs.summary()
    injected = len(hook.injected)
    rep = eng.report

    # fault campaign long enough (~1 s of iterations) for tens of injected
    # errors at ~50/s: FT-on iterations under injection vs the FT-off step time
    campaign = None
    def run_long(eng, iters, sampler=None):
        """`iters` graph steps back to back after step 0 and the captures."""
        eng.step(0)
        eng.warm_graphs(1)  # capture outside the timed region
        torch.cuda.synchronize()
        gc.collect()
        gc.disable()
        cst, cen = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cst.record()
        for it in range(1, iters + 1):
            eng.step(it, more=(lambda it=it: it < iters))
        cen.record()
        torch.cuda.synchronize()
        gc.enable()
        eng.close()
        return cst.elapsed_time(cen)

    if args.campaign_s > 0:
        c_iters = max(50, int(args.campaign_s / max(ms_ft * 1e-3, 1e-6)))
        c_sched = _campaign_schedule(p, c_iters + 1, hi - lo, K, seed=2)
        c_hook = ScheduledFaultHook(c_sched)
        c_eng = engine("abft", c_hook)
        with ClockSampler(torch.cuda.current_device()) as ccs:
            c_ms = run_long(c_eng, c_iters)
        c_clocks = ccs.summary()
        # the same number of FT-off iterations from the same start: the
        # overhead compares runs of equal length (the centroids, and with them
        # the share of uncertified rows, change over a ~1 s run)
        off_ms = run_long(engine("off"), c_iters)
        c_rep = c_eng.report
        c_inj = sum(1 for e in c_hook.injected if e["iteration"] >= 1)
        campaign = {"iters": c_iters, "device_s": c_ms * 1e-3, "ms_per_step": c_ms / c_iters,
                    "injected": c_inj, "injected_per_s": c_inj / (c_ms * 1e-3),
                    "detections": c_rep.detections, "corrections": c_rep.corrections,
                    "uncorrectable": c_rep.uncorrectable,
                    "ft_off_ms_per_step": off_ms / c_iters,
                    "overhead_vs_ft_off_pct": 100.0 * (c_ms / off_ms - 1.0),
                    "p_tile": p, "clocks": c_clocks}

    flops = 2.0 * N_ROWS * DIM * K / world
    hbm, bf16, src = _peaks()
    tf32_peak = bf16 / 2.0
    assign_tflops = flops / (a_ft * 1e-3) / 1e12
    # dominant kernel: the CTA-pair screen, timed by CUDA events around its own
    # launch on the launching stream (algorithmic 2 N D K flops per launch)
    kern_ms = k_ft if k_ft else a_ft
    achieved = flops / (kern_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("pair_screen_kernel_chk_c2_bytes")
        if traffic is not None and world > 1:  # this rank's shard of the c2 rows
            traffic = int(traffic * (hi - lo) / N_ROWS)
    # e2e: public API with host buffers (H2D of X and D2H of labels inside)
    e2e = None
    if world == 1:
        xp = torch.from_numpy(x).pin_memory()
        conf = P.KMeansConfig(k=K, max_iters=args.steps, tol=0.0, seed=0, init="random-sample",
                              ft_mode="abft")
        # one untimed fit of the same configuration: the timed fit then sees a
        # warm process (lazily loaded kernels, allocator, first graph
        # instantiation), like any fit after the first in a serving process
        P.lloyd(xp, conf)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = P.lloyd(xp, conf)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e = {"value": r.iters / wall, "unit": "iter/s",
               "h2d_bytes_per_step": int(x.nbytes // max(r.iters, 1)),
               "d2h_bytes_per_step": int(N_ROWS * 8 // max(r.iters, 1)),
               "iters": r.iters, "wall_s": wall}
    cpu = cpu_reference(x) if rank == 0 and world == 1 else None
    if rank != 0:
        return
    line = {
        "metric": "lloyd_iters_per_s", "value": 1e3 / ms_ft, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_ft,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference gaussian_mixture(1e6, 128, 1024 blobs, 0.25, seed 0); "
                "random-sample init seed 0",
        "config": {"workload": "c2: N=1e6 D=128 K=1024 fp32, ABFT on, per-tile-prob campaign "
                               "sized for ~50 errors/s", "global_batch": N_ROWS,
                   "parallelism": f"dp{world} (row shards)", "l2": "inputs 512 MB > L2 (no flush)",
                   "variant": P.gemm.get_variant()},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": tf32_peak,
                     "unit": "TFLOP/s", "frac": achieved / tf32_peak,
                     "peak_note": f"dense tf32 = bf16_tflops/2 from MEASURED_PEAKS.json ({src})",
                     "kernel": "pair_screen_kernel<CHK> (cta_group::2 tcgen05 tf32 screen + "
                               "fused argmin/certificate/exact refine/ABFT)",
                     "kernel_ms": kern_ms, "traffic": traffic,
                     "traffic_note": "dram read+write bytes per launch, ncu --set full "
                                     "(profiles/traffic.json)"},
        "assign_ms": a_ft, "assign_tflops": assign_tflops,
        "ft_off_kernel_ms": k_off,
        "ft_off_ms_per_step": ms_off, "ft_overhead_pct": 100.0 * (ms_ft / ms_off - 1.0),
        "faults": {"injected": injected, "per_s": injected / (ms_ft * 1e-3 * horizon),
                   "detections": rep.detections, "corrections": rep.corrections,
                   "uncorrectable": rep.uncorrectable, "p_tile": p},
        "ft_campaign": campaign,
        "step_ms": {"ft_off": step_stats[0], "abft": step_stats[1]},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default=None)
    ap.add_argument("--campaign-s", type=float, default=1.0,
                    help="seconds of ABFT iterations under ~50 injected errors/s (0: skip)")
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
