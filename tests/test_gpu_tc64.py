"""Float64 assignment screened on the tf32 tensor cores (tc64.cu): the
screen only proposes the argmin, a float64 certificate accepts it, and the
winner's distance is the reference's own float64 chain -- so labels and
min_dists must equal the reference's (oracle) bit for bit on every row,
including near-ties (DMMA pass 2), non-finite data and checked passes with
scheduled flips (reference-identical event records)."""

import numpy as np
import pytest

import oracle as O
from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_01391_b200")
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200 import gemm as G  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture
def pair64():
    old = G.get_variant()
    G.set_variant("pair")
    yield
    G.set_variant(old)


def _blobs(m, d, k, seed, spread=0.25):
    x, _, _ = P.gaussian_mixture(m, d, k, spread, precision="double", seed=seed)
    y = np.ascontiguousarray(x[np.random.default_rng(seed).choice(m, k, replace=False)])
    return x, y


@pytest.mark.parametrize("m,d,k", [(70000, 64, 256), (66000, 128, 1024), (3000, 4, 17),
                                   (2000, 256, 300), (1, 8, 1), (513, 12, 129), (4097, 32, 64)])
def test_tc64_random_bit_exact(m, d, k, pair64):
    rng = np.random.default_rng(m + d + k)
    x = np.ascontiguousarray(rng.standard_normal((m, d)))
    y = np.ascontiguousarray(rng.standard_normal((k, d)))
    r = P.fused_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(r.assignments, lab)
    assert r.min_dists.tobytes() == val.tobytes()


@pytest.mark.parametrize("ctab", ["0", "1"])
@pytest.mark.parametrize("m,d,k", [(70000, 64, 256), (40000, 32, 500), (30000, 48, 7)])
def test_tc64_refine_centroid_table_both_ways(m, d, k, ctab, pair64, monkeypatch):
    """The float64 refine with the centroids in shared memory (K*D*8 <= 128 KB,
    d % 16 == 0; swizzled 16-byte chunks) and gathered from L2 (FTK_T64_CTAB=0)
    give the oracle's labels and distances bit for bit."""
    monkeypatch.setenv("FTK_T64_CTAB", ctab)
    x, y = _blobs(m, d, k, 5)
    r = P.fused_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(r.assignments, lab)
    assert r.min_dists.tobytes() == val.tobytes()


@pytest.mark.parametrize("m,d,k", [(100000, 64, 256), (70000, 128, 64)])
def test_tc64_blobs_certified_and_exact(m, d, k, pair64):
    """Near-converged blobs: almost every row is certified by the screen."""
    x, y = _blobs(m, d, k, seed=3)
    r = P.fused_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(r.assignments, lab)
    assert r.min_dists.tobytes() == val.tobytes()
    unc = E.tc_fallback_rows()[0]
    assert unc < m // 4  # the DMMA pass sees only the uncertified rows


def test_tc64_ties_and_nonfinite_go_to_dmma(pair64):
    """Duplicated centroids (exact ties: lowest index wins), a row of huge
    values (fp32 overflow in the screen) and a NaN row."""
    rng = np.random.default_rng(9)
    y = rng.standard_normal((40, 16))
    y[7] = y[3]
    y[20] = y[3]
    x = np.ascontiguousarray(y[rng.integers(0, 40, 5000)] + 1e-9 * rng.standard_normal((5000, 16)))
    x[10] = y[3]
    x[11] = 1e300
    x[12, 5] = np.nan
    x[13] = 3e38 * np.sign(rng.standard_normal(16))
    y = np.ascontiguousarray(y)
    r = P.fused_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(r.assignments, lab)
    assert r.min_dists.tobytes() == val.tobytes()
    assert E.tc_fallback_rows()[0] >= 3


def test_tc64_checked_with_flips_matches_exact_variant():
    """ABFT pass with scheduled flips: results, events and the hook's
    before/after equal the exact checked kernel's (the reference's)."""
    x, y = _blobs(70000, 64, 256, seed=5)
    entries = [FaultEntry(0, (3, 0), (5, 7), 62), FaultEntry(0, (100, 0), (0, 0), 40),
               FaultEntry(0, (2000, 0), (31, 255), 51)]
    old = G.get_variant()
    try:
        out = {}
        for v in ("exact", "pair"):
            G.set_variant(v)
            h = ScheduledFaultHook(FaultSchedule(list(entries)))
            res, rep = P.checked_assign(x, y, hook=h)
            out[v] = (res, rep, h.injected)
    finally:
        G.set_variant(old)
    (ra, pa, ia), (rb, pb, ib) = out["exact"], out["pair"]
    assert np.array_equal(ra.assignments, rb.assignments)
    assert ra.min_dists.tobytes() == rb.min_dists.tobytes()
    assert [(e.iteration, e.tile, e.kind, e.loc, e.delta, e.interval) for e in pa.events] == \
        [(e.iteration, e.tile, e.kind, e.loc, e.delta, e.interval) for e in pb.events]
    assert ia == ib
    assert pa.detections > 0


def test_tc64_lloyd_matches_oracle(pair64):
    """A float64 Lloyd fit through the tf32-screened family
    equals the oracle's restatement of the reference lloyd bitwise."""
    x, _ = _blobs(80000, 64, 32, seed=11)
    cfg = P.KMeansConfig(k=32, max_iters=8, seed=0, init="random-sample", ft_mode="abft")
    res = P.lloyd(x, cfg)
    ref = O.lloyd(x, 32, max_iters=8, seed=0, init="random-sample", ft_mode="abft")
    assert np.array_equal(res.assignments, ref["assignments"])
    assert res.centroids.tobytes() == ref["centroids"].tobytes()
    assert res.inertia == ref["inertia"]
    assert res.iters == ref["iters"]


def test_tc64_candidate_overflow_goes_to_dmma(pair64):
    """Rows whose pass-2 candidate set exceeds its cap (300 identical
    centroids tie for every row) fall through to the DMMA screen; rows with a
    few close centroids are resolved by the float64 candidate pass."""
    rng = np.random.default_rng(12)
    base = rng.standard_normal((1, 64))
    y = np.ascontiguousarray(np.vstack([np.repeat(base, 300, axis=0), rng.standard_normal((20, 64)) * 5]))
    x = np.ascontiguousarray(np.vstack([base + 1e-3 * rng.standard_normal((700, 64)),
                                        y[300:310] + 1e-9 * rng.standard_normal((10, 64))]))
    r = P.fused_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(r.assignments, lab)
    assert r.min_dists.tobytes() == val.tobytes()
    assert E.tc_fallback_rows()[1] > 0  # rows reached the DMMA screen


@pytest.mark.parametrize("m,d,k", [(70000, 4, 1), (66000, 8, 5), (70000, 6, 33), (70000, 300, 40)])
def test_tc64_auto_edge_shapes(m, d, k):
    """The default family choice for float64 at edge shapes (k = 1, tiny d,
    d % 4 != 0 and d > 256 -- the last two outside the tf32 path) stays
    bit-exact."""
    rng = np.random.default_rng(m + d + k)
    x = np.ascontiguousarray(rng.standard_normal((m, d)) * 2.0)
    y = np.ascontiguousarray(x[rng.choice(m, k, replace=False)] + 0.01)
    r = P.fused_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(r.assignments, lab)
    assert r.min_dists.tobytes() == val.tobytes()


def test_tc64_estimator_fit_matches_oracle():
    """FTKMeans on float64 data (default variant selection, ABFT) against the
    oracle's restatement of the reference lloyd."""
    x, _ = _blobs(90000, 32, 64, seed=21)
    km = P.FTKMeans(n_clusters=64, init="random-sample", max_iter=6, random_state=3, ft_mode="abft").fit(x)
    ref = O.lloyd(x, 64, max_iters=6, seed=3, init="random-sample", ft_mode="abft")
    assert np.array_equal(km.labels_, ref["assignments"])
    assert km.cluster_centers_.tobytes() == ref["centroids"].tobytes()
    assert km.inertia_ == ref["inertia"]
