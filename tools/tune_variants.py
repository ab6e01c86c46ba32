"""Measure the kernel-variant table on this GPU (variants.select) and write it.

  python tools/tune_variants.py [--out paper_2408_01391_b200/data/variants_b200.csv]
                                [--quick]

Shapes: the BASELINE configs plus a (D, K) grid per precision, probed at
2^18 rows (the selection is driven by D and K; the table buckets M).
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join("paper_2408_01391_b200", "data", "variants_b200.csv"))
ap.add_argument("--probe", type=int, default=1 << 18)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--quick", action="store_true")
ap.add_argument("--only", choices=["single", "double"], default=None,
                help="re-measure one precision and keep the other's rows of --out")
a = ap.parse_args()

from paper_2408_01391_b200 import variants as V  # noqa: E402

M = 1_000_000
if a.quick:
    single = [(M, 128, 1024), (M, 512, 16), (M, 32, 64), (M, 8, 4096)]
    double = [(M, 64, 256)]
else:
    single = [(M, d, k) for d in (4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048)
              for k in (8, 16, 32, 64, 128, 252, 1024, 4096)]
    double = [(M, d, k) for d in (16, 32, 64, 128, 256) for k in (16, 64, 256, 1024)]

t0 = time.time()


def show(shape, var, gf):
    print(f"{shape} {var:7s} {gf:9.1f} GFLOP/s  [{time.time() - t0:.0f} s]", flush=True)


keep = V.VariantTable.load(a.out) if a.only and os.path.exists(a.out) else V.VariantTable()
ts = V.select(single, "single", reps=a.reps, probe_m=a.probe, progress=show) \
    if a.only != "double" else V.VariantTable()
td = V.select(double, "double", reps=a.reps, probe_m=a.probe, progress=show) \
    if a.only != "single" else V.VariantTable()
for key, e in keep.entries.items():
    if key[3] != a.only:
        ts.entries[key] = e
ts.entries.update(td.entries)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
ts.save(a.out)
print("wrote", a.out, len(ts.entries), "entries")
