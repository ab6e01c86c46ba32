"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

This script imports the reference package ``ftkmeans`` 0.1.0 (numba CPU) from
``$FTK_REF`` or ``/root/reference/pkg/src`` -- available only in the build
container, never on the GPU box -- and records its outputs on seeded inputs.
The committed .npz/.json files are what the oracle and the CUDA path are
pinned against.  Regenerate with:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("FTK_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from ftkmeans import faults as F  # noqa: E402
from ftkmeans.abft import Threshold, checked_assign  # noqa: E402
from ftkmeans.gemm import fused_assign  # noqa: E402
from ftkmeans.kmeans import KMeansConfig, init_centroids, lloyd, update_step  # noqa: E402
from ftkmeans.matrix import gaussian_mixture, row_sq_norms  # noqa: E402
from ftkmeans.tiles import make_config, MICRO_SINGLE  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def assign_cases():
    rng = np.random.default_rng(1001)
    rec = {}
    shapes = [(1, 1, 1), (3, 5, 2), (129, 17, 65), (37, 33, 31), (300, 64, 70), (257, 3, 300),
              (64, 128, 33), (200, 8, 257), (50, 1, 9), (513, 32, 64)]
    for t in range(40):
        if t < len(shapes):
            m, d, k = shapes[t]
        else:
            m, d, k = int(rng.integers(1, 300)), int(rng.integers(1, 96)), int(rng.integers(1, 80))
        dt = np.float32 if t % 2 == 0 else np.float64
        scale = 100.0 if t % 7 == 3 else 1.0
        x = np.ascontiguousarray(rng.standard_normal((m, d)) * scale, dtype=dt)
        y = np.ascontiguousarray(rng.standard_normal((k, d)) * scale, dtype=dt)
        if t % 5 == 4 and k > 2 and m > 2:  # exact duplicates -> ties
            y[1] = y[0]
            x[0] = y[0]
        r = fused_assign(x, y)
        rec[f"c{t}_x"], rec[f"c{t}_y"] = x, y
        rec[f"c{t}_lab"], rec[f"c{t}_val"] = r.assignments, r.min_dists
        rec[f"c{t}_yn"] = row_sq_norms(y)
        rec[f"c{t}_xn"] = row_sq_norms(x)
    # documented worked examples (test_gemm.py:66-76)
    rec["tie_x"] = np.array([[1, 0]], dtype=np.float32)
    rec["tie_y"] = np.array([[1, 0], [1, 0]], dtype=np.float32)
    rec["tie_lab"] = fused_assign(rec["tie_x"], rec["tie_y"]).assignments
    np.savez_compressed(os.path.join(OUT, "assign_cases.npz"), n=40, **rec)


def update_cases():
    rng = np.random.default_rng(1002)
    rec = {}
    for t in range(12):
        m, d, k = int(rng.integers(5, 400)), int(rng.integers(1, 40)), int(rng.integers(1, 30))
        dt = np.float32 if t % 2 == 0 else np.float64
        x = np.ascontiguousarray(rng.standard_normal((m, d)) * np.exp(rng.uniform(-20, 5, (m, d))),
                                 dtype=dt)
        lab = rng.integers(0, max(1, k - (t % 3)), m)  # some clusters empty
        sq = rng.random(m)
        c, counts, _ = update_step(x, lab, k, sq_dists=sq)
        rec[f"u{t}_x"], rec[f"u{t}_lab"], rec[f"u{t}_k"], rec[f"u{t}_sq"] = x, lab, k, sq
        rec[f"u{t}_c"], rec[f"u{t}_counts"] = c, counts
    np.savez_compressed(os.path.join(OUT, "update_cases.npz"), n=12, **rec)


def pairwise_cases():
    rng = np.random.default_rng(1003)
    rec = {}
    ns = [1, 2, 7, 8, 9, 15, 16, 17, 127, 128, 129, 130, 255, 256, 1000, 4097, 65537, 100000]
    for t, n in enumerate(ns):
        a = rng.standard_normal(n) * np.exp(rng.uniform(-25, 25, n))
        rec[f"p{t}_a"] = a
        rec[f"p{t}_s"] = np.float64(a.sum())
    for t, (r, c) in enumerate([(5, 3), (7, 8), (4, 32), (3, 129), (2, 300)]):
        a = rng.standard_normal((r, c))
        rec[f"n{t}_a"] = a
        rec[f"n{t}_norm"] = np.linalg.norm(a, axis=1)
    np.savez_compressed(os.path.join(OUT, "pairwise_cases.npz"), n=len(ns), nn=5, **rec)


def lloyd_cases():
    rec = {}
    cases = [
        # (rows, cols, blobs, spread, precision, seed, k, init, max_iters, tol)
        (2048, 8, 4, 0.2, "single", 16, 4, "kmeanspp", 300, 1e-4),
        (3000, 16, 10, 0.3, "double", 3, 10, "random-sample", 300, 1e-4),
        (5000, 32, 20, 0.25, "single", 5, 16, "random-sample", 25, 0.0),
        (1500, 6, 3, 0.1, "single", 31, 3, "kmeanspp", 300, 1e-4),
        (4000, 64, 12, 0.5, "double", 7, 12, "kmeanspp", 40, 0.0),
        (1000, 3, 50, 0.05, "single", 9, 60, "random-sample", 50, 1e-4),  # empties likely
    ]
    for t, (rows, cols, blobs, spread, prec, seed, k, init, mi, tol) in enumerate(cases):
        x, _, _ = gaussian_mixture(rows, cols, blobs, spread, precision=prec, seed=seed)
        res = lloyd(x, KMeansConfig(k=k, seed=seed, init=init, max_iters=mi, tol=tol))
        rec[f"l{t}_args"] = np.array([rows, cols, blobs, k, mi, seed], dtype=np.int64)
        rec[f"l{t}_meta"] = np.array([spread, tol], dtype=np.float64)
        rec[f"l{t}_prec"] = np.array(prec)
        rec[f"l{t}_init"] = np.array(init)
        rec[f"l{t}_xsha"] = np.array(sha(x))
        rec[f"l{t}_c"] = res.centroids
        rec[f"l{t}_lab"] = res.assignments
        rec[f"l{t}_inertia"] = np.float64(res.inertia)
        rec[f"l{t}_hist"] = np.array(res.inertia_history, dtype=np.float64)
        rec[f"l{t}_iters"] = np.int64(res.iters)
        rec[f"l{t}_conv"] = np.bool_(res.converged)
        rec[f"l{t}_init_c"] = init_centroids(x, k, seed=seed, method=init)
    np.savez_compressed(os.path.join(OUT, "lloyd_cases.npz"), n=len(cases), **rec)


def lloyd_c1():
    # BASELINE.json configs[0]: N=100k, D=32, K=64 fp32, 20 iters, FT off, seed 0
    x, _, _ = gaussian_mixture(100000, 32, 64, 0.25, precision="single", seed=0)
    res = lloyd(x, KMeansConfig(k=64, max_iters=20, tol=0.0, seed=0, init="random-sample",
                                ft_mode="off"))
    np.savez_compressed(
        os.path.join(OUT, "lloyd_c1.npz"), xsha=np.array(sha(x)),
        lab=res.assignments.astype(np.uint8), c=res.centroids, inertia=np.float64(res.inertia),
        hist=np.array(res.inertia_history), iters=np.int64(res.iters),
        conv=np.bool_(res.converged))


def gmm_cases():
    rec = {}
    for t, (r, c, k, s, p, seed) in enumerate([(50, 4, 3, 0.1, "single", 1), (40, 3, 5, 0.25,
                                                "double", 2), (30, 2, 1, 0.3, "single", 3)]):
        x, lab, cen = gaussian_mixture(r, c, k, s, precision=p, seed=seed)
        rec[f"g{t}_x"], rec[f"g{t}_lab"], rec[f"g{t}_cen"] = x, lab, cen
        rec[f"g{t}_args"] = np.array([r, c, k, seed])
        rec[f"g{t}_spread"] = np.float64(s)
        rec[f"g{t}_prec"] = np.array(p)
    shas = {}
    for (r, c, k) in [(20000, 32, 64), (10000, 128, 256)]:
        x, _, _ = gaussian_mixture(r, c, k, 0.25, precision="single", seed=0)
        shas[f"{r}_{c}_{k}"] = sha(x)
    rec["big_shas"] = np.array(json.dumps(shas))
    np.savez_compressed(os.path.join(OUT, "gmm_cases.npz"), n=3, **rec)


def fault_cases():
    out = {"flip": [], "plans": []}
    for v, b in [(1.0, 31), (0.0, 0), (1.5, 30), (-2.25, 23), (3.0, 5)]:
        out["flip"].append([v, b, float(F.flip_bit(np.float32(v), b)),
                            repr(float(F.flip_bit(np.float64(v), b + 32)))])
    specs = [("prob:0.3", 4, (5, 3), (32, 256), "float32", (150, 700)),
             ("fixed:4@exp", 3, (4, 4), (32, 256), "float32", (100, 1000)),
             ("fixed:2@sign", 5, (2, 1), (64, 64), "float64", None),
             ("prob:0.5@b7", 2, (3, 2), (16, 16), "float64", (40, 20)),
             ("sweep@any", 1, (1, 1), (2, 2), "float32", None),
             ("fixed:3", 2, (2, 2), (8, 8), "float32", (10, 12))]
    for text, iters, grid, dims, dt, shape in specs:
        sp = F.FaultSpec.parse(text, seed=11)
        plan = F.plan_faults(sp, iters, grid, dims, dtype=np.dtype(dt), shape=shape)
        out["plans"].append({
            "text": text, "iters": iters, "grid": grid, "dims": dims, "dtype": dt,
            "shape": shape,
            "entries": [[e.iteration, e.tile[0], e.tile[1], e.elem[0], e.elem[1], e.bit]
                        for e in plan.entries]})
    with open(os.path.join(OUT, "fault_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def checked_cases():
    """checked_assign / fused_assign under scheduled flips (reference events)."""
    rng = np.random.default_rng(1004)
    rec = {}
    cases = []
    x = np.ascontiguousarray(rng.random((200, 16)), dtype=np.float32)
    y = np.ascontiguousarray(rng.random((24, 16)), dtype=np.float32)
    cases.append(("a", x, y, [(0, (0, 0), (7, 3), 30)], None))
    x2, _, _ = gaussian_mixture(2000, 32, 16, 0.25, precision="single", seed=4)
    y2 = np.ascontiguousarray(x2[:40])
    ent = [(0, (i, 0), (int(rng.integers(0, 32)), int(rng.integers(0, 40))), b)
           for i, b in zip(range(0, 60, 3), [30, 31, 29, 28, 27, 26, 25, 24, 23, 22, 21, 20, 19,
                                             18, 17, 16, 10, 5, 1, 0])]
    cases.append(("b", x2, y2, ent, None))
    x3 = np.ascontiguousarray(rng.standard_normal((300, 24)), dtype=np.float64)
    y3 = np.ascontiguousarray(rng.standard_normal((70, 24)), dtype=np.float64)
    ent3 = [(0, (0, 0), (5, 60), 62), (0, (2, 1), (3, 2), 52), (0, (4, 0), (10, 10), 63)]
    cases.append(("c", x3, y3, ent3, None))
    cfg4 = make_config((32, 32, 8), (32, 32, 8), MICRO_SINGLE)
    x4 = np.ascontiguousarray(rng.random((64, 40)), dtype=np.float32)
    y4 = np.ascontiguousarray(rng.random((64, 40)), dtype=np.float32)
    cases.append(("d", x4, y4, [(0, (0, 0), (1, 2), 31), (0, (1, 1), (9, 9), 30)], cfg4))
    for name, x, y, ent, cfg in cases:
        entries = [F.FaultEntry(*e) for e in ent]
        h1 = F.ScheduledFaultHook(F.FaultSchedule(list(entries)))
        res, rep = checked_assign(x, y, cfg=cfg, hook=h1)
        h2 = F.ScheduledFaultHook(F.FaultSchedule(list(entries)))
        plain = fused_assign(x, y, cfg=cfg, hook=h2)
        clean = fused_assign(x, y, cfg=cfg)
        rec[f"{name}_x"], rec[f"{name}_y"] = x, y
        rec[f"{name}_ent"] = np.array([[e[0], e[1][0], e[1][1], e[2][0], e[2][1], e[3]]
                                       for e in ent], dtype=np.int64)
        rec[f"{name}_block"] = np.array(cfg.block if cfg else (-1, -1, -1), dtype=np.int64)
        rec[f"{name}_lab"], rec[f"{name}_val"] = res.assignments, res.min_dists
        rec[f"{name}_clean_lab"], rec[f"{name}_clean_val"] = clean.assignments, clean.min_dists
        rec[f"{name}_plain_lab"], rec[f"{name}_plain_val"] = plain.assignments, plain.min_dists
        rec[f"{name}_ev"] = np.array([[e.iteration, e.tile[0], e.tile[1],
                                       0 if e.kind == "detected-corrected" else 1,
                                       e.loc[0], e.loc[1]] for e in rep.events],
                                     dtype=np.int64).reshape(-1, 6)
        rec[f"{name}_evdelta"] = np.array([e.delta for e in rep.events], dtype=np.float64)
        rec[f"{name}_inj"] = np.array([[d["before"], d["after"]] for d in h1.injected],
                                      dtype=np.float64).reshape(-1, 2)
        rec[f"{name}_plain_inj"] = np.array([[d["before"], d["after"]] for d in h2.injected],
                                            dtype=np.float64).reshape(-1, 2)
    np.savez_compressed(os.path.join(OUT, "checked_cases.npz"), names=np.array(["a", "b", "c", "d"]),
                        **rec)


def lloyd_ft_cases():
    rec = {}
    for t, (seed, mode, spec) in enumerate([(21, "abft+dmr", "fixed:2"), (22, "abft", "fixed:3@exp"),
                                            (23, "abft+dmr", "prob:0.05")]):
        x, _, _ = gaussian_mixture(2048, 8, 4, 0.2, precision="single", seed=seed)
        base = lloyd(x, KMeansConfig(k=4, seed=seed, ft_mode="off"))
        prot = lloyd(x, KMeansConfig(k=4, seed=seed, ft_mode=mode), fault_spec=spec)
        rec[f"f{t}_seed"] = np.int64(seed)
        rec[f"f{t}_mode"] = np.array(mode)
        rec[f"f{t}_spec"] = np.array(spec)
        rec[f"f{t}_base_lab"] = base.assignments
        rec[f"f{t}_lab"] = prot.assignments
        rec[f"f{t}_iters"] = np.int64(prot.iters)
        rec[f"f{t}_counts"] = np.array([prot.report.detections, prot.report.corrections,
                                        prot.report.uncorrectable, prot.report.dmr_mismatches])
        rec[f"f{t}_ev"] = np.array([[e.iteration, e.tile[0], e.tile[1], e.loc[0], e.loc[1]]
                                    for e in prot.report.events], dtype=np.int64).reshape(-1, 5)
    np.savez_compressed(os.path.join(OUT, "lloyd_ft_cases.npz"), n=3, **rec)


def sweep_cases():
    """cli.exhaustive_sweep(8, 8, seed=303) outcome per (elem, bit) (acceptance 3)."""
    from ftkmeans.abft import checked_gemm
    from ftkmeans.gemm import gemm_tiled
    rng = np.random.default_rng(303)
    a = np.ascontiguousarray(rng.random((8, 8)), dtype=np.float32)
    b = np.ascontiguousarray(rng.random((8, 8)), dtype=np.float32)
    ref = gemm_tiled(a, b)
    rows = []
    outs = []
    for i in range(8):
        for j in range(8):
            for bit in range(32):
                hook = F.ScheduledFaultHook(F.FaultSchedule([F.FaultEntry(0, (0, 0), (i, j), bit)]))
                out, rep = checked_gemm(a, b, hook=hook)
                ev = rep.events[0] if rep.events else None
                rows.append([i, j, bit, rep.detections, rep.corrections,
                             ev.loc[0] if ev else -9, ev.loc[1] if ev else -9])
                outs.append(out)
    np.savez_compressed(os.path.join(OUT, "sweep_cases.npz"), a=a, b=b, ref=ref,
                        rows=np.array(rows, dtype=np.int64), outs=np.stack(outs))


def acceptance4_cases():
    rec = {}
    for k in (4, 128):
        x, _, _ = gaussian_mixture(65536, 8, 4, 0.25, precision="single", seed=404)
        base = lloyd(x, KMeansConfig(k=k, seed=404, max_iters=50, ft_mode="off"))
        spec = F.FaultSpec(mode="fixed-count", count=10, seed=405)
        prot = lloyd(x, KMeansConfig(k=k, seed=404, max_iters=50, ft_mode="abft+dmr"),
                     fault_spec=spec)
        rec[f"k{k}_base_lab"] = base.assignments.astype(np.uint8)
        rec[f"k{k}_base_c"] = base.centroids
        rec[f"k{k}_base_iters"] = np.int64(base.iters)
        rec[f"k{k}_base_hist"] = np.array(base.inertia_history)
        rec[f"k{k}_prot_lab"] = prot.assignments.astype(np.uint8)
        rec[f"k{k}_prot_c"] = prot.centroids
        rec[f"k{k}_prot_iters"] = np.int64(prot.iters)
        rec[f"k{k}_prot_counts"] = np.array([prot.report.detections, prot.report.corrections,
                                             prot.report.uncorrectable,
                                             prot.report.dmr_mismatches])
        rec[f"k{k}_prot_ev"] = np.array([[e.iteration, e.tile[0], e.tile[1], e.loc[0], e.loc[1],
                                          0 if e.kind == "detected-corrected" else 1]
                                         for e in prot.report.events], np.int64).reshape(-1, 6)
        rec[f"k{k}_prot_delta"] = np.array([e.delta for e in prot.report.events])
    np.savez_compressed(os.path.join(OUT, "acceptance4_cases.npz"), **rec)


def dmr_cases():
    rng = np.random.default_rng(707)
    rec = []
    arrays = {}
    for trial in range(20):
        m, n, k = 256, 6, 5
        x = np.ascontiguousarray(rng.random((m, n)), dtype=np.float32)
        assignments = rng.integers(0, k, m)
        clean, counts_clean, _ = update_step(x, assignments, k)
        bit = int(rng.integers(32, 64))
        ci, cj = int(rng.integers(0, k)), int(rng.integers(0, n))
        hook = F.ScheduledFaultHook(F.FaultSchedule([F.FaultEntry(0, (0, 0), (ci, cj), bit)]))
        got, counts, events = update_step(x, assignments, k, ft_mode="abft+dmr", hook=hook)
        hook2 = F.ScheduledFaultHook(F.FaultSchedule([F.FaultEntry(0, (0, 0), (ci, cj), bit)]))
        off, _, _ = update_step(x, assignments, k, ft_mode="off", hook=hook2)
        arrays[f"t{trial}_x"], arrays[f"t{trial}_lab"] = x, assignments
        arrays[f"t{trial}_clean"], arrays[f"t{trial}_got"], arrays[f"t{trial}_off"] = clean, got, off
        rec.append([ci, cj, bit, len(events)])
    np.savez_compressed(os.path.join(OUT, "dmr_cases.npz"), meta=np.array(rec), **arrays)


CLI_CASES = [
    # (name, generate args, cluster args)
    ("gm_off", ["--rows", "3000", "--cols", "16", "--dist", "gm:8:0.1", "--seed", "4"],
     ["--k", "8", "--max-iters", "50", "--init", "kmeanspp", "--seed", "2"]),
    ("gm_abft_inject", ["--rows", "4000", "--cols", "24", "--dist", "gm:12:0.2", "--seed", "5"],
     ["--k", "12", "--ft", "abft", "--inject", "prob:0.05@exp", "--max-iters", "30", "--tol", "0",
      "--init", "random-sample", "--seed", "1"]),
    ("uni_dmr_f64", ["--rows", "2500", "--cols", "9", "--precision", "double", "--seed", "6"],
     ["--k", "5", "--ft", "abft+dmr", "--max-iters", "20", "--init", "random-sample"]),
]


def cli_cases():
    """Reference ``ftkm cluster`` RunReports (machine-independent rows) on
    datasets written by the reference ``ftkm generate``."""
    import csv
    import tempfile

    from ftkmeans import cli

    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name, gen, clu in CLI_CASES:
            path = os.path.join(td, name + ".ftkm")
            rep = os.path.join(td, name + ".csv")
            assert cli.main(["generate", *gen, "--out", path]) == 0
            code = cli.main(["cluster", "--input", path, *clu, "--report", rep])
            with open(rep) as fh:
                rows = [r for r in csv.reader(fh)][1:]
            keep = [r for r in rows if r[0] in ("result", "ft", "summary", "config")
                    or (r[0] == "meta" and r[1] in ("precision", "rows", "cols", "schema_version"))]
            with open(path, "rb") as fh:
                data_sha = hashlib.sha256(fh.read()).hexdigest()
            out[name] = {"generate": gen, "cluster": clu, "exit": code, "rows": keep,
                         "file_sha256": data_sha}
    with open(os.path.join(OUT, "cli_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    sweep_cases()
    acceptance4_cases()
    dmr_cases()
    assign_cases()
    update_cases()
    pairwise_cases()
    gmm_cases()
    fault_cases()
    checked_cases()
    lloyd_cases()
    lloyd_ft_cases()
    lloyd_c1()
    cli_cases()
    print("golden fixtures written to", OUT)
