"""Golden fixtures at the BASELINE configs' own sizes, from the REFERENCE.

Runs the reference ``ftkmeans.kmeans.lloyd`` (numba CPU, imported from
``$FTK_REF`` or ``/root/reference/pkg/src``; build container only) on the
bench's configurations and records digests of its results in
``tests/golden/lloyd_configs.json``:

* c2      N=1e6, D=128, K=1024 f32, 20 iterations, FT off       (bench.py's workload)
* c2_ft   the same with ft_mode="abft" and 2 scheduled flips per iteration
* c3_*    the irregular sweep, K in {8,16,32} x D in {512,2048} and D in {4,8} x K=4096,
          at N=2e5 (reduced N; the per-row work is unchanged)
* c4      N=1e6, D=64, K=256 f64, 20 iterations, FT off and ABFT with flips
* c5s     c5's shape (D=128, K=4096) at N=2e5, 10 iterations

Data: the reference ``gaussian_mixture`` (seed 0, spread 0.25, blobs = K) --
except c5s, whose 4096 blobs would need the reference's k x k x D float64
temporary (17 GB); it uses the package's chunked generator, which is
bit-identical (tests/golden/gmm_cases.npz), and the digest of the data is
recorded so both sides provably start from the same bytes.

Each record holds sha256 digests of the labels (int64), centroids and
min-distance-free outputs, the inertia history, iteration count, the
detection-event list, and (for FT runs) the reference's own label divergence
from the FT-off run.  GPU tests (tests/test_gpu_configs.py) rerun each case
through the package and compare digests bitwise.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_configs.py [case ...]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("FTK_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from ftkmeans.faults import FaultSpec  # noqa: E402
from ftkmeans.kmeans import KMeansConfig, lloyd  # noqa: E402
from ftkmeans.matrix import gaussian_mixture  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lloyd_configs.json")

# name: (rows, cols, blobs, precision, k, max_iters, ft_mode, fault spec text, generator)
CASES = {
    "c2": (1_000_000, 128, 1024, "single", 1024, 20, "off", None, "ref"),
    "c2_ft": (1_000_000, 128, 1024, "single", 1024, 20, "abft", "fixed:2", "ref"),
    "c3_k8_d512": (200_000, 512, 8, "single", 8, 20, "off", None, "ref"),
    "c3_k16_d512": (200_000, 512, 16, "single", 16, 20, "off", None, "ref"),
    "c3_k32_d512": (200_000, 512, 32, "single", 32, 20, "off", None, "ref"),
    "c3_k8_d2048": (200_000, 2048, 8, "single", 8, 20, "off", None, "ref"),
    "c3_k16_d2048": (200_000, 2048, 16, "single", 16, 20, "off", None, "ref"),
    "c3_k32_d2048": (200_000, 2048, 32, "single", 32, 20, "off", None, "ref"),
    "c3_k16_d512_ft": (200_000, 512, 16, "single", 16, 20, "abft", "fixed:2", "ref"),
    "c3_k4096_d4": (200_000, 4, 4096, "single", 4096, 20, "off", None, "ref"),
    "c3_k4096_d8": (200_000, 8, 4096, "single", 4096, 20, "off", None, "ref"),
    "c4": (1_000_000, 64, 256, "double", 256, 20, "off", None, "ref"),
    "c4_ft": (1_000_000, 64, 256, "double", 256, 20, "abft", "fixed:2", "ref"),
    "c5s": (200_000, 128, 4096, "single", 4096, 10, "off", None, "pkg"),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_x(rows, cols, blobs, prec, gen):
    if gen == "pkg":
        sys.path.insert(0, ROOT)
        from paper_2408_01391_b200.matrix import gaussian_mixture as gm

        return gm(rows, cols, blobs, 0.25, precision=prec, seed=0)[0]
    return gaussian_mixture(rows, cols, blobs, 0.25, precision=prec, seed=0)[0]


def run_case(name):
    rows, cols, blobs, prec, k, mi, ft, spec, gen = CASES[name]
    x = make_x(rows, cols, blobs, prec, gen)
    cfg = KMeansConfig(k=k, max_iters=mi, tol=0.0, seed=0, init="random-sample", ft_mode=ft)
    t0 = time.perf_counter()
    fs = FaultSpec.parse(spec, seed=1) if spec else None
    r = lloyd(x, cfg, fault_spec=fs)
    wall = time.perf_counter() - t0
    rec = {"args": [rows, cols, blobs, prec, k, mi, ft, spec, gen],
           "xsha": sha(x), "lab_sha": sha(r.assignments.astype(np.int64)),
           "c_sha": sha(r.centroids), "inertia": float(r.inertia),
           "hist": [float(v) for v in r.inertia_history], "iters": int(r.iters),
           "converged": bool(r.converged),
           "lab_head": r.assignments[:64].astype(int).tolist(),
           "counts": np.bincount(r.assignments, minlength=k).astype(int).tolist(),
           "events": [[e.iteration, e.tile[0], e.tile[1], e.kind, e.loc[0], e.loc[1], float(e.delta)]
                      for e in r.report.events],
           "false_alarms": int(r.report.false_alarms),
           "ref_wall_s": wall}
    if ft != "off":
        base = lloyd(x, KMeansConfig(k=k, max_iters=mi, tol=0.0, seed=0, init="random-sample"))
        rec["label_divergence_vs_off"] = int(np.count_nonzero(base.assignments != r.assignments))
        rec["off_lab_sha"] = sha(base.assignments.astype(np.int64))
    return rec


def main(names):
    db = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            db = json.load(fh)
    for name in names or list(CASES):
        t0 = time.perf_counter()
        db[name] = run_case(name)
        print(f"{name}: iters={db[name]['iters']} inertia={db[name]['inertia']!r} "
              f"events={len(db[name]['events'])} {time.perf_counter() - t0:.1f} s", flush=True)
        with open(OUT, "w") as fh:
            json.dump(db, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
