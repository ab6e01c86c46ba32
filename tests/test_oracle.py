"""The CPU oracle is pinned to the reference's own outputs (tests/golden/)."""

import json
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN


def test_assign_matches_reference(golden):
    z = golden("assign_cases.npz")
    for t in range(int(z["n"])):
        x, y = z[f"c{t}_x"], z[f"c{t}_y"]
        lab, val = O.assign(x, y, threads=3)
        assert np.array_equal(lab, z[f"c{t}_lab"]), t
        assert val.tobytes() == z[f"c{t}_val"].tobytes(), t
        assert O.row_sq_norms(y).tobytes() == z[f"c{t}_yn"].tobytes()
        assert O.row_sq_norms(x).tobytes() == z[f"c{t}_xn"].tobytes()
    assert O.assign(z["tie_x"], z["tie_y"])[0].tolist() == z["tie_lab"].tolist() == [0]


def test_update_matches_reference(golden):
    z = golden("update_cases.npz")
    for t in range(int(z["n"])):
        c, counts = O.update_step(z[f"u{t}_x"], z[f"u{t}_lab"], int(z[f"u{t}_k"]),
                                  sq_dists=z[f"u{t}_sq"], threads=4)
        assert counts.tolist() == z[f"u{t}_counts"].tolist()
        assert c.tobytes() == z[f"u{t}_c"].tobytes(), t


def test_pairwise_sum_matches_numpy(golden):
    z = golden("pairwise_cases.npz")
    for t in range(int(z["n"])):
        assert O.pairwise_sum(z[f"p{t}_a"]) == float(z[f"p{t}_s"]), t
    for t in range(int(z["nn"])):
        assert O.row_norms(z[f"n{t}_a"]).tobytes() == z[f"n{t}_norm"].tobytes(), t


def test_lloyd_matches_reference(golden):
    z = golden("lloyd_cases.npz")
    gm = pytest.importorskip("paper_2408_01391_b200.matrix")
    for t in range(int(z["n"])):
        rows, cols, blobs, k, mi, seed = (int(v) for v in z[f"l{t}_args"])
        spread, tol = (float(v) for v in z[f"l{t}_meta"])
        x, _, _ = gm.gaussian_mixture(rows, cols, blobs, spread, precision=str(z[f"l{t}_prec"]),
                                      seed=seed)
        import hashlib
        assert hashlib.sha256(x.tobytes()).hexdigest() == str(z[f"l{t}_xsha"])
        init = str(z[f"l{t}_init"])
        c0 = O.init_centroids(x, k, seed, init)
        assert c0.tobytes() == z[f"l{t}_init_c"].tobytes()
        r = O.lloyd(x, k, max_iters=mi, tol=tol, seed=seed, init=init, threads=2)
        assert r["iters"] == int(z[f"l{t}_iters"]), t
        assert r["converged"] == bool(z[f"l{t}_conv"])
        assert np.array_equal(r["assignments"], z[f"l{t}_lab"]), t
        assert r["centroids"].tobytes() == z[f"l{t}_c"].tobytes(), t
        assert r["inertia"] == float(z[f"l{t}_inertia"])
        assert r["inertia_history"] == z[f"l{t}_hist"].tolist()


@pytest.mark.slow
def test_lloyd_c1_matches_reference(golden):
    """BASELINE configs[0] (N=100k, D=32, K=64, 20 iters): oracle == reference."""
    z = golden("lloyd_c1.npz")
    from paper_2408_01391_b200.matrix import gaussian_mixture
    x, _, _ = gaussian_mixture(100000, 32, 64, 0.25, precision="single", seed=0)
    import hashlib
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["xsha"])
    r = O.lloyd(x, 64, max_iters=20, tol=0.0, seed=0, init="random-sample")
    assert r["iters"] == int(z["iters"])
    assert np.array_equal(r["assignments"], z["lab"].astype(np.int64))
    assert r["centroids"].tobytes() == z["c"].tobytes()
    assert r["inertia_history"] == z["hist"].tolist()
    assert r["inertia"] == float(z["inertia"])


def test_exact_dot_is_the_flipped_accumulator(golden):
    """The hook's recorded 'before' value is the exact sequential dot product."""
    z = golden("checked_cases.npz")
    for n in ["a", "b", "c"]:
        x, y, ent, inj = z[f"{n}_x"], z[f"{n}_y"], z[f"{n}_ent"], z[f"{n}_plain_inj"]
        bm, bn = (32, 256) if x.dtype == np.float32 else (64, 64)
        for q, e in enumerate(ent):
            i, j = e[1] * bm + e[3], e[2] * bn + e[4]
            assert float(O.exact_dot(x[i], y[j])) == inj[q, 0]
