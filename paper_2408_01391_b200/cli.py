"""Command-line front end for the GPU path: ``generate`` and ``cluster``.

Mirrors the reference's ``ftkm generate`` / ``ftkm cluster`` (cli.py:44-151,
343-418): same arguments, the same phase,metric,value RunReport CSV (schema
version 1), the same labels / events outputs and exit codes (0 ok, 2 usage
error, 3 a detected-uncorrectable fault).  An ftkm-binary input is read
straight into pinned host memory (matrix.mat_load_pinned) and copied to the
device once per fit.  The reference's ``tune`` / ``bench`` / ``verify``
commands drive its CPU tuner and self-checks and are not part of this path.

    python -m paper_2408_01391_b200.cli cluster --input x.ftkm --k 64 --ft abft --report r.csv
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import sys

import numpy as np

from . import __version__
from .abft import Threshold
from .errors import FormatError
from .kmeans import KMeansConfig, lloyd
from .matrix import mat_load, mat_load_pinned, mat_random, mat_store, precision_of
from .tiles import TileTable, parse_tile

REPORT_SCHEMA_VERSION = 1

EXIT_OK = 0
EXIT_USAGE = 2
EXIT_UNCORRECTABLE = 3


def _write_report(path, rows):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["phase", "metric", "value"])
        w.writerow(["meta", "schema_version", REPORT_SCHEMA_VERSION])
        for phase, metric, value in rows:
            w.writerow([phase, metric, value])


def _load_input(path, precision):
    """CSV -> numpy in the requested precision; ftkm-binary -> pinned host
    tensor in the file's precision (cli.py:44-47)."""
    if str(path).endswith(".csv"):
        return mat_load(path, format="csv", precision=precision)
    return mat_load_pinned(path)


def _precision(x):
    if isinstance(x, np.ndarray):
        return precision_of(x)
    return "single" if x.element_size() == 4 else "double"


def cmd_generate(args):
    x = mat_random(args.rows, args.cols, precision=args.precision, seed=args.seed,
                   distribution=args.dist)
    mat_store(x, args.out, format="ftkm-binary")
    print(f"wrote {args.rows}x{args.cols} {precision_of(x)} matrix to {args.out}")
    return EXIT_OK


def _cluster_rows(args, x, result, gflops):
    digest = hashlib.sha256(result.assignments.tobytes()).hexdigest()
    return [
        ("meta", "command", "cluster"),
        ("meta", "version", __version__),
        ("meta", "precision", _precision(x)),
        ("meta", "rows", x.shape[0]),
        ("meta", "cols", x.shape[1]),
        ("config", "k", args.k),
        ("config", "ft", args.ft),
        ("config", "inject", args.inject or "none"),
        ("config", "seed", args.seed),
        ("config", "max_iters", args.max_iters),
        ("config", "tol", args.tol),
        ("config", "tile", args.tile),
        ("timing", "init_ns", result.timings["init_ns"]),
        ("timing", "assign_ns", result.timings["assign_ns"]),
        ("timing", "update_ns", result.timings["update_ns"]),
        ("timing", "total_ns", result.timings["total_ns"]),
        ("perf", "assign_gflops", gflops),
        ("result", "iters", result.iters),
        ("result", "converged", result.converged),
        ("result", "inertia", repr(result.inertia)),
        ("result", "assignments_sha256", digest),
        ("ft", "detections", result.report.detections),
        ("ft", "corrections", result.report.corrections),
        ("ft", "uncorrectable", result.report.uncorrectable),
        ("ft", "dmr_mismatches", result.report.dmr_mismatches),
        ("ft", "false_alarms", result.report.false_alarms),
    ]


def cmd_cluster(args):
    x = _load_input(args.input, args.precision)
    if args.inject and args.inject != "none" and args.ft == "off":
        print("warning: faults injected without protection", file=sys.stderr)
    dtype = np.float32 if _precision(x) == "single" else np.float64
    tune_table = TileTable.load(args.tune_table) if args.tune_table else None
    tile = "auto"
    if args.tile != "auto":
        tile = parse_tile(args.tile, dtype)
    elif tune_table is None:
        print("warning: --tile auto with no tune table, using default config", file=sys.stderr)
    config = KMeansConfig(
        k=args.k, max_iters=args.max_iters, tol=args.tol, seed=args.seed, ft_mode=args.ft,
        init=args.init, tile=tile, threshold=Threshold(args.delta) if args.delta else None,
        threads=args.threads, tune_table=tune_table)
    result = lloyd(x, config, fault_spec=args.inject)
    m, n = x.shape
    flops = 2.0 * m * n * args.k * (result.iters + 1)
    gflops = flops / max(result.timings["assign_ns"], 1) if result.timings["assign_ns"] else 0.0
    rows = _cluster_rows(args, x, result, gflops)
    if args.compare:
        base_cfg = KMeansConfig(k=args.k, max_iters=args.max_iters, tol=args.tol, seed=args.seed,
                                ft_mode="off", init=args.init, tile=tile, threads=args.threads)
        base = lloyd(x, base_cfg)
        t_ft, t_base = result.timings["total_ns"], base.timings["total_ns"]
        overhead = (t_ft - t_base) / t_base if t_base else float("inf")
        rows.append(("summary", "baseline_total_ns", t_base))
        rows.append(("summary", "overhead_pct", 100.0 * overhead))
        rows.append(("summary", "assignments_match_baseline",
                     bool(np.array_equal(base.assignments, result.assignments))))
    exit_code = EXIT_UNCORRECTABLE if result.report.uncorrectable else EXIT_OK
    rows.append(("summary", "exit_code", exit_code))
    if args.report:
        _write_report(args.report, rows)
    if args.labels_out:
        np.savetxt(args.labels_out, result.assignments, fmt="%d")
    if args.events_out:
        result.report.to_csv(args.events_out)
    print(f"k={args.k} iters={result.iters} converged={result.converged} "
          f"inertia={result.inertia:.6g} detections={result.report.detections} "
          f"corrections={result.report.corrections}")
    return exit_code


def build_parser():
    p = argparse.ArgumentParser(prog="ftkm-b200", description=__doc__,
                                formatter_class=argparse.RawDescriptionHelpFormatter)
    p.add_argument("--threads", type=int, default=None,
                   help="accepted for compatibility (the GPU path ignores it)")
    sub = p.add_subparsers(dest="command", required=True)

    g = sub.add_parser("generate", help="write a synthetic dataset")
    g.add_argument("--rows", type=int, required=True)
    g.add_argument("--cols", type=int, required=True)
    g.add_argument("--precision", choices=["single", "double"], default="single")
    g.add_argument("--dist", default="uniform", help='"uniform" or "gm:k:spread"')
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--out", required=True)
    g.set_defaults(fn=cmd_generate)

    c = sub.add_parser("cluster", help="run fault-tolerant K-means on the GPU")
    c.add_argument("--input", required=True)
    c.add_argument("--precision", choices=["single", "double"], default="single",
                   help="target precision for CSV inputs")
    c.add_argument("--k", type=int, required=True)
    c.add_argument("--ft", choices=["off", "abft", "abft+dmr"], default="off")
    c.add_argument("--inject", default=None,
                   help='fault spec: none | prob:P | fixed:N | sweep, with @sign/@exp/@any/@b<k>')
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--max-iters", type=int, default=300)
    c.add_argument("--tol", type=float, default=1e-4)
    c.add_argument("--tile", default="auto", help='"auto" or bm,bn,bk,sm,sn,sk')
    c.add_argument("--tune-table", default=None,
                   help="reference tune-table CSV: picks the logical tile (fault grid, event coordinates)")
    c.add_argument("--delta", type=float, default=None, help="checksum threshold scale")
    c.add_argument("--init", choices=["kmeanspp", "random-sample"], default="kmeanspp")
    c.add_argument("--report", default=None, help="write a phase,metric,value CSV")
    c.add_argument("--labels-out", default=None, help="write assignments, one per line")
    c.add_argument("--events-out", default=None, help="write the detection log CSV")
    c.add_argument("--compare", action="store_true",
                   help="also run the fault-free unprotected baseline and report overhead")
    c.set_defaults(fn=cmd_cluster)
    return p


def main(argv=None):
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code not in (0, None) else 0
    try:
        return args.fn(args)
    except (ValueError, FormatError, FileNotFoundError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
