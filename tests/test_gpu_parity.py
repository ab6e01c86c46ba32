"""Parity of the CUDA path (through the C ABI) with the reference and the oracle.

Every comparison is bitwise: labels, min_dists, centroids, inertia, counts,
corrected values and detection events must equal the reference's bits.
"""

import hashlib

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_01391_b200")
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200 import gemm as G  # noqa: E402
from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook  # noqa: E402
from paper_2408_01391_b200.tiles import MICRO_SINGLE, make_config  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


VARIANTS = ["exact", "auto"]


@pytest.fixture(params=VARIANTS)
def variant(request):
    old = G.get_variant()
    G.set_variant(request.param)
    yield request.param
    G.set_variant(old)


def _hook(entries):
    return ScheduledFaultHook(FaultSchedule([FaultEntry(*e) for e in entries]))


def test_row_sq_norms_golden(golden):
    z = golden("assign_cases.npz")
    for t in range(int(z["n"])):
        assert P.row_sq_norms(z[f"c{t}_y"]).tobytes() == z[f"c{t}_yn"].tobytes()
        assert P.row_sq_norms(z[f"c{t}_x"]).tobytes() == z[f"c{t}_xn"].tobytes()


def test_fused_assign_golden(golden, variant):
    z = golden("assign_cases.npz")
    for t in range(int(z["n"])):
        r = P.fused_assign(z[f"c{t}_x"], z[f"c{t}_y"])
        assert r.assignments.dtype == np.int64
        assert np.array_equal(r.assignments, z[f"c{t}_lab"]), t
        assert r.min_dists.tobytes() == z[f"c{t}_val"].tobytes(), t
    assert P.fused_assign(z["tie_x"], z["tie_y"]).assignments.tolist() == [0]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_fused_assign_vs_oracle(dt, variant):
    rng = np.random.default_rng(77)
    for m, d, k in [(1000, 128, 1024), (4097, 32, 64), (777, 7, 300), (2048, 256, 33),
                    (513, 1, 5), (1, 3, 1), (300, 513, 17), (5000, 4, 4096)]:
        x = np.ascontiguousarray(rng.standard_normal((m, d)), dtype=dt)
        y = np.ascontiguousarray(rng.standard_normal((k, d)), dtype=dt)
        r = P.fused_assign(x, y)
        lab, val = O.assign(x, y)
        assert np.array_equal(r.assignments, lab), (m, d, k)
        assert r.min_dists.tobytes() == val.tobytes(), (m, d, k)


def test_custom_tiles_same_result():
    rng = np.random.default_rng(5)
    x = np.ascontiguousarray(rng.standard_normal((333, 40)), dtype=np.float32)
    y = np.ascontiguousarray(rng.standard_normal((70, 40)), dtype=np.float32)
    lab, val = O.assign(x, y)
    for blk in [(128, 64, 16), (32, 32, 8), (16, 16, 4), (64, 128, 32), (8, 8, 8), (2, 4, 2),
                (256, 256, 64), (1, 1, 1)]:
        r = _assign_block(x, y, blk)
        assert np.array_equal(r[0], lab), blk
        assert r[1].tobytes() == val.tobytes(), blk


def _assign_block(x, y, blk):
    from paper_2408_01391_b200 import _engine as E
    x_t, y_t = E.to_dev(x), E.to_dev(y)
    idx, val = E.assign_dev(x_t, y_t, E.row_sq_norms_dev(y_t), blk, variant="exact")
    return E.to_host(idx).astype(np.int64), E.to_host(val)


def test_gemm_tiled_exact():
    rng = np.random.default_rng(9)
    a = np.ascontiguousarray(rng.standard_normal((70, 37)), dtype=np.float32)
    b = np.ascontiguousarray(rng.standard_normal((45, 37)), dtype=np.float32)
    out = P.gemm_tiled(a, b)
    for i in range(0, 70, 7):
        for j in range(0, 45, 5):
            assert out[i, j] == O.exact_dot(a[i], b[j])
    assert P.gemm_tiled(np.eye(2, dtype=np.float32),
                        np.array([[5, 6], [7, 8]], np.float32)).tolist() == [[5, 7], [6, 8]]


def test_update_golden(golden):
    z = golden("update_cases.npz")
    for t in range(int(z["n"])):
        c, counts, ev = P.update_step(z[f"u{t}_x"], z[f"u{t}_lab"], int(z[f"u{t}_k"]),
                                      sq_dists=z[f"u{t}_sq"])
        assert counts.tolist() == z[f"u{t}_counts"].tolist(), t
        assert c.tobytes() == z[f"u{t}_c"].tobytes(), t
        assert ev == []


def test_update_empty_cluster_own_dists():
    rng = np.random.default_rng(4)
    x = np.ascontiguousarray(rng.random((50, 3)), dtype=np.float32)
    lab = np.zeros(50, dtype=np.int64)
    c, counts, _ = P.update_step(x, lab, 2)
    ref, _ = O.update_step(x, lab, 2)
    assert counts.tolist() == [50, 0]
    assert c.tobytes() == ref.tobytes()


def _lloyd_case(z, t):
    rows, cols, blobs, k, mi, seed = (int(v) for v in z[f"l{t}_args"])
    spread, tol = (float(v) for v in z[f"l{t}_meta"])
    x, _, _ = P.gaussian_mixture(rows, cols, blobs, spread, precision=str(z[f"l{t}_prec"]),
                                 seed=seed)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z[f"l{t}_xsha"])
    return x, P.KMeansConfig(k=k, seed=seed, init=str(z[f"l{t}_init"]), max_iters=mi, tol=tol)


def test_lloyd_golden(golden, variant):
    z = golden("lloyd_cases.npz")
    for t in range(int(z["n"])):
        x, cfg = _lloyd_case(z, t)
        r = P.lloyd(x, cfg)
        assert r.iters == int(z[f"l{t}_iters"]), t
        assert r.converged == bool(z[f"l{t}_conv"]), t
        assert np.array_equal(r.assignments, z[f"l{t}_lab"]), t
        assert r.centroids.tobytes() == z[f"l{t}_c"].tobytes(), t
        assert r.inertia == float(z[f"l{t}_inertia"]), t
        assert r.inertia_history == z[f"l{t}_hist"].tolist(), t


def test_lloyd_c1_golden(golden, variant):
    """BASELINE configs[0]: N=100k, D=32, K=64 f32, 20 iterations, seed 0."""
    z = golden("lloyd_c1.npz")
    x, _, _ = P.gaussian_mixture(100000, 32, 64, 0.25, precision="single", seed=0)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(z["xsha"])
    r = P.lloyd(x, P.KMeansConfig(k=64, max_iters=20, tol=0.0, seed=0, init="random-sample"))
    assert r.iters == int(z["iters"]) == 20
    assert np.array_equal(r.assignments, z["lab"].astype(np.int64))
    assert r.centroids.tobytes() == z["c"].tobytes()
    assert r.inertia_history == z["hist"].tolist()
    assert r.inertia == float(z["inertia"])


def test_checked_assign_golden(golden):
    z = golden("checked_cases.npz")
    for n in [str(v) for v in z["names"]]:
        x, y, ent = z[f"{n}_x"], z[f"{n}_y"], z[f"{n}_ent"]
        blk = tuple(int(v) for v in z[f"{n}_block"])
        cfg = None if blk[0] < 0 else make_config(blk, blk, MICRO_SINGLE)
        entries = [(int(e[0]), (int(e[1]), int(e[2])), (int(e[3]), int(e[4])), int(e[5]))
                   for e in ent]
        h1 = _hook(entries)
        res, rep = P.checked_assign(x, y, cfg=cfg, hook=h1)
        assert np.array_equal(res.assignments, z[f"{n}_lab"]), n
        assert res.min_dists.tobytes() == z[f"{n}_val"].tobytes(), n
        ev = np.array([[e.iteration, e.tile[0], e.tile[1],
                        0 if e.kind == "detected-corrected" else 1, e.loc[0], e.loc[1]]
                       for e in rep.events], np.int64).reshape(-1, 6)
        assert ev.tolist() == z[f"{n}_ev"].tolist(), n
        assert [e.delta for e in rep.events] == z[f"{n}_evdelta"].tolist(), n
        inj = np.array([[d["before"], d["after"]] for d in h1.injected]).reshape(-1, 2)
        assert inj.tobytes() == z[f"{n}_inj"].tobytes(), n
        # unprotected: corruption flows to the result exactly like the reference
        h2 = _hook(entries)
        plain = P.fused_assign(x, y, cfg=cfg, hook=h2)
        assert np.array_equal(plain.assignments, z[f"{n}_plain_lab"]), n
        assert plain.min_dists.tobytes() == z[f"{n}_plain_val"].tobytes(), n
        clean = P.fused_assign(x, y, cfg=cfg)
        assert np.array_equal(clean.assignments, z[f"{n}_clean_lab"]), n


def test_fault_free_checked_is_bit_identical_and_silent():
    rng = np.random.default_rng(202)
    for case in range(120):
        m, n, k = int(rng.integers(1, 192)), int(rng.integers(1, 64)), int(rng.integers(1, 80))
        dt = np.float32 if case % 2 == 0 else np.float64
        scale = 100.0 if case % 5 == 0 else 1.0
        x = np.ascontiguousarray(rng.standard_normal((m, n)) * scale, dtype=dt)
        y = np.ascontiguousarray(rng.standard_normal((k, n)), dtype=dt)
        out, rep = P.checked_gemm(x, y)
        assert rep.detections == 0, case
        assert out.tobytes() == P.gemm_tiled(x, y).tobytes(), case
        res, rep2 = P.checked_assign(x, y)
        plain = P.fused_assign(x, y)
        assert rep2.detections == 0
        assert np.array_equal(res.assignments, plain.assignments)
        assert res.min_dists.tobytes() == plain.min_dists.tobytes()


def test_exhaustive_single_error_sweep(golden):
    """Acceptance 3: every (element, bit) flip of an 8x8 f32 tile -> same
    outcome, location and corrected output bits as the reference."""
    z = golden("sweep_cases.npz")
    a, b, ref = z["a"], z["b"], z["ref"]
    assert P.gemm_tiled(a, b).tobytes() == ref.tobytes()
    rows, outs = z["rows"], z["outs"]
    silent = 0
    for q, (i, j, bit, det, corr, li, lj) in enumerate(rows.tolist()):
        out, rep = P.checked_gemm(a, b, hook=_hook([(0, (0, 0), (i, j), bit)]))
        assert (rep.detections, rep.corrections) == (det, corr), (i, j, bit)
        if rep.events:
            assert rep.events[0].loc == (li, lj)
        assert out.tobytes() == outs[q].tobytes(), (i, j, bit)
        err = float(np.abs(out.astype(np.float64) - ref.astype(np.float64)).max())
        silent += not ((corr == 1 or det == 0) and err <= 1e-4 * 8)
    assert silent == 0


def test_lloyd_ft_transparency_golden(golden):
    z = golden("lloyd_ft_cases.npz")
    for t in range(int(z["n"])):
        seed = int(z[f"f{t}_seed"])
        x, _, _ = P.gaussian_mixture(2048, 8, 4, 0.2, precision="single", seed=seed)
        base = P.lloyd(x, P.KMeansConfig(k=4, seed=seed))
        prot = P.lloyd(x, P.KMeansConfig(k=4, seed=seed, ft_mode=str(z[f"f{t}_mode"])),
                       fault_spec=str(z[f"f{t}_spec"]))
        assert np.array_equal(base.assignments, z[f"f{t}_base_lab"])
        assert np.array_equal(prot.assignments, z[f"f{t}_lab"])
        assert prot.iters == int(z[f"f{t}_iters"])
        r = prot.report
        assert [r.detections, r.corrections, r.uncorrectable, r.dmr_mismatches] == \
            z[f"f{t}_counts"].tolist()
        ev = np.array([[e.iteration, e.tile[0], e.tile[1], e.loc[0], e.loc[1]]
                       for e in r.events], np.int64).reshape(-1, 5)
        assert ev.tolist() == z[f"f{t}_ev"].tolist()


@pytest.mark.slow
def test_acceptance4_ft_transparency(golden):
    z = golden("acceptance4_cases.npz")
    x, _, _ = P.gaussian_mixture(65536, 8, 4, 0.25, precision="single", seed=404)
    for k in (4, 128):
        base = P.lloyd(x, P.KMeansConfig(k=k, seed=404, max_iters=50))
        prot = P.lloyd(x, P.KMeansConfig(k=k, seed=404, max_iters=50, ft_mode="abft+dmr"),
                       fault_spec=P.FaultSpec(mode="fixed-count", count=10, seed=405))
        assert np.array_equal(base.assignments, z[f"k{k}_base_lab"].astype(np.int64))
        assert base.centroids.tobytes() == z[f"k{k}_base_c"].tobytes()
        assert base.inertia_history == z[f"k{k}_base_hist"].tolist()
        assert np.array_equal(prot.assignments, z[f"k{k}_prot_lab"].astype(np.int64))
        assert prot.centroids.tobytes() == z[f"k{k}_prot_c"].tobytes()
        assert prot.iters == int(z[f"k{k}_prot_iters"])
        r = prot.report
        assert [r.detections, r.corrections, r.uncorrectable, r.dmr_mismatches] == \
            z[f"k{k}_prot_counts"].tolist()
        ev = np.array([[e.iteration, e.tile[0], e.tile[1], e.loc[0], e.loc[1],
                        0 if e.kind == "detected-corrected" else 1] for e in r.events
                       if e.kind != "dmr-mismatch"], np.int64).reshape(-1, 6)
        assert ev.tolist() == z[f"k{k}_prot_ev"].tolist()


def test_dmr_update_golden(golden):
    z = golden("dmr_cases.npz")
    for t, (ci, cj, bit, nev) in enumerate(z["meta"].tolist()):
        x, lab = z[f"t{t}_x"], z[f"t{t}_lab"]
        got, _, ev = P.update_step(x, lab, 5, ft_mode="abft+dmr",
                                   hook=_hook([(0, (0, 0), (ci, cj), bit)]))
        assert len(ev) == nev and all(e.kind == "dmr-mismatch" for e in ev)
        assert got.tobytes() == z[f"t{t}_got"].tobytes() == z[f"t{t}_clean"].tobytes()
        off, _, _ = P.update_step(x, lab, 5, hook=_hook([(0, (0, 0), (ci, cj), bit)]))
        assert off.tobytes() == z[f"t{t}_off"].tobytes()


def test_dmr_graph_steps_match_and_retry():
    """abft+dmr runs in the CUDA-graph steps (duplicated accumulators compared
    on the device): same results as abft, and a flagged step redoes its update
    eagerly (kmeans.py:176-189) without changing the outcome."""
    old = G.get_variant()
    G.set_variant("pair")  # a graph-step family (the variant table may pick exact here)
    try:
        _dmr_graph_case()
    finally:
        G.set_variant(old)


def _dmr_graph_case():
    from paper_2408_01391_b200.kmeans import LloydEngine

    x, _, _ = P.gaussian_mixture(60000, 32, 16, 0.25, precision="single", seed=8)
    cfg = dict(k=16, seed=1, max_iters=12, init="random-sample")
    base = P.lloyd(x, P.KMeansConfig(ft_mode="abft", **cfg))
    dmr = P.lloyd(x, P.KMeansConfig(ft_mode="abft+dmr", **cfg))
    assert np.array_equal(base.assignments, dmr.assignments)
    assert base.centroids.tobytes() == dmr.centroids.tobytes()
    assert base.inertia_history == dmr.inertia_history
    assert dmr.report.dmr_mismatches == 0
    c0 = P.init_centroids(x, 16, seed=1, method="random-sample")
    thr = P.Threshold.default_for(np.float32)
    runs = []
    for flag_at in (None, 3):
        eng = LloydEngine(E.to_dev(x), c0, 16, np.float32, P.default_config(np.float32), "abft+dmr",
                          thr, 1, graph=True)
        assert eng.use_graph
        hist = []
        for it in range(6):
            if it == flag_at:
                eng._dmr_flagged = lambda: True
            hist.append(eng.step(it, more=lambda: True))
            eng.__dict__.pop("_dmr_flagged", None)
        runs.append((hist, E.to_host(eng.cent).tobytes(), eng.report))
        eng.close()
    assert runs[0][0] == runs[1][0] and runs[0][1] == runs[1][1]
    assert runs[1][2].dmr_mismatches == 1 and runs[0][2].dmr_mismatches == 0


def test_dmr_persistent_escalates():
    class AlwaysCorrupt:
        def maybe_corrupt(self, iteration, tile, acc):
            acc[0, 0] += 1.0

    x = np.ones((8, 2), dtype=np.float32)
    with pytest.raises(P.FaultEscalationError):
        P.update_step(x, np.zeros(8, dtype=np.int64), 1, ft_mode="abft+dmr",
                      hook=AlwaysCorrupt())


def test_estimator_surface():
    from sklearn.base import clone
    from sklearn.metrics import adjusted_rand_score

    x, labels, _ = P.gaussian_mixture(1500, 6, 3, 0.1, precision="single", seed=31)
    est = P.FTKMeans(n_clusters=3, random_state=2).fit(x)
    assert est.cluster_centers_.shape == (3, 6) and est.labels_.dtype == np.int64
    assert est.converged_ and est.detection_report_.detections == 0
    assert adjusted_rand_score(labels, est.labels_) >= 0.99
    assert np.array_equal(est.predict(x), est.labels_)
    assert est.score(x) == pytest.approx(-est.inertia_, rel=1e-5)
    ref = O.lloyd(x, 3, seed=2)
    assert np.array_equal(est.labels_, ref["assignments"])
    assert est.cluster_centers_.tobytes() == ref["centroids"].tobytes()
    prot = P.FTKMeans(n_clusters=3, random_state=6, ft_mode="abft+dmr", inject="fixed:2").fit(x)
    clean = P.FTKMeans(n_clusters=3, random_state=6).fit(x)
    assert prot.detection_report_.corrections > 0
    assert np.array_equal(prot.labels_, clean.labels_)
    assert clone(est).get_params() == est.get_params()
    d64 = P.FTKMeans(n_clusters=3, random_state=7).fit(x.astype(np.float64))
    assert d64.cluster_centers_.dtype == np.float64
    with pytest.raises(ValueError):
        bad = x.copy()
        bad[3, 1] = np.nan
        P.FTKMeans(n_clusters=2).fit(bad)


def test_native_library_is_the_one_loaded():
    from paper_2408_01391_b200 import _native

    before = _native.launch_count()
    P.fused_assign(np.ones((8, 4), np.float32), np.ones((2, 4), np.float32))
    assert _native.launch_count() > before
    import os
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libftkb200.so" in maps


@pytest.mark.parametrize("m,d,k,dt,tiny", [
    (60000, 32, 2048, np.float32, False),   # segment partials + certified fold (K*D/32 > one wave)
    (60000, 32, 2048, np.float32, True),    # + tiny values: uncertified chains replayed in order
    (40000, 96, 5, np.float32, True),       # few long chains: pipelined ordered chains
    (30000, 24, 7, np.float64, False),      # float64 data: pipelined ordered chains
    (200000, 8, 8192, np.float32, False),   # counting sort at its largest K (2 warps, 64 KB smem)
    (120000, 64, 256, np.float64, False),   # float64: warp-specialised ordered chains (c4 shape)
    (20000, 130, 9, np.float64, True),      # float64, partial last consumer warp, long chains
    (50000, 16, 9000, np.float32, True),    # K beyond the counting sort: radix-sort member lists
])
def test_update_paths_bit_exact(m, d, k, dt, tiny):
    """Every update path (segment partials with the exactness certificate,
    the ordered replay of uncertified chains, the pipelined chain kernel)
    reproduces numpy.bincount's float64 sums bit for bit."""
    rng = np.random.default_rng(m + d + k)
    x = rng.standard_normal((m, d)) * 3.0
    if tiny:  # magnitudes ~1e-9 next to O(1e3) sums force roundings in the reference chain
        x[rng.integers(0, m, 200), rng.integers(0, d, 200)] = 1e-9
    x = np.ascontiguousarray(x, dtype=dt)
    lab = rng.integers(0, k, m).astype(np.int64)
    lab[:m // 3] = 0  # one long chain
    c, counts, _ = P.update_step(x, lab, k)
    ref, ref_counts = O.update_step(x, lab, k)
    assert counts.tolist() == ref_counts.tolist()
    assert c.tobytes() == ref.tobytes()


@pytest.mark.parametrize("m,d,k,dt,env", [
    (50000, 64, 37, np.float64, {}),                          # warp-specialised chains, one 512-byte slab
    (40000, 130, 5, np.float64, {}),                          # partial last slab (2 features)
    (30000, 7, 5, np.float64, {}),                            # rows not 16-byte aligned: cp.async chains
    (40000, 64, 37, np.float64, {"FTK_UPD_CHAIN": "0"}),      # cp.async chains forced
    (40000, 200, 9, np.float32, {"FTK_UPD_PATH": "pipe"}),    # float32 data through the ordered chains
    (40000, 100, 9, np.float64, {"FTK_CS_SLAB": "128"}),      # 128-byte slabs, partial last slab
    (40000, 72, 9, np.float64, {"FTK_CS_SLAB": "256"}),       # 256-byte slabs
    (30000, 36, 5, np.float32, {"FTK_UPD_PATH": "pipe", "FTK_CS_SLAB": "128"}),
])
@pytest.mark.parametrize("dmr", [False, True])
def test_ordered_chain_kernels_bit_exact(m, d, k, dt, env, dmr, monkeypatch):
    """The ordered float64 chains (warp-specialised and cp.async kernels, with and
    without the DMR duplicate) equal numpy.bincount's sums bit for bit."""
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(m + d + k)
    x = np.ascontiguousarray(rng.standard_normal((m, d)) * 3.0, dtype=dt)
    lab = rng.integers(0, k, m).astype(np.int64)
    lab[: m // 2] = 1  # one long chain
    lab[-5:] = k - 1
    c, counts, ev = P.update_step(x, lab, k, ft_mode="abft+dmr" if dmr else "off")
    ref, ref_counts = O.update_step(x, lab, k)
    assert counts.tolist() == ref_counts.tolist()
    assert c.tobytes() == ref.tobytes()
    assert ev == []


@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("dmr", [False, True])
def test_update_fused_fold_bit_exact(fused, dmr, monkeypatch):
    """The segment fold fused into the partials kernel (the last segment block
    of a cluster folds its chains) and the separate fold pass give
    numpy.bincount's bits, with empty clusters (zero sums written by the
    surplus blocks), one long chain, and tiny values whose chains the replay
    walks in 32-member sub-segments."""
    monkeypatch.setenv("FTK_UPD_FUSED_FOLD", fused)
    rng = np.random.default_rng(77)
    m, d, k = 50000, 128, 1024
    x = rng.standard_normal((m, d)) * 3.0 + 20.0
    x[rng.integers(0, m, 300), rng.integers(0, d, 300)] = 1e-9
    x = np.ascontiguousarray(x, dtype=np.float32)
    lab = 2 * rng.integers(0, k // 2, m).astype(np.int64)  # odd clusters empty
    lab[: m // 4] = 6  # one long chain (49 segments)
    c, counts, ev = P.update_step(x, lab, k, ft_mode="abft+dmr" if dmr else "off")
    ref, ref_counts = O.update_step(x, lab, k)
    assert counts.tolist() == ref_counts.tolist()
    assert c.tobytes() == ref.tobytes()
    assert ev == []


def test_candidate_overflow_rows_go_exact():
    """Rows whose pass-2 candidate set exceeds its cap (300 identical
    centroids tie for every row) are resolved by the exact row kernel."""
    rng = np.random.default_rng(12)
    base = rng.standard_normal((1, 64)).astype(np.float32)
    y = np.ascontiguousarray(np.vstack([np.repeat(base, 300, axis=0),
                                        rng.standard_normal((20, 64)).astype(np.float32) * 5]))
    x = np.ascontiguousarray(base + 1e-3 * rng.standard_normal((700, 64)).astype(np.float32))
    res = P.fused_assign(x, y)
    from paper_2408_01391_b200 import _engine as E

    assert E.tc_fallback_rows()[1] > 0  # the exact row kernel ran
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(res.assignments, ref_lab)
    assert res.min_dists.tobytes() == ref_val.tobytes()


@pytest.mark.parametrize("m,d,k,prec", [(20000, 32, 64, "single"), (5000, 100, 40, "double"),
                                        (3000, 5, 17, "single"), (4000, 300, 24, "single"),
                                        (2500, 1030, 9, "double"), (200000, 16, 128, "single")])
def test_kmeanspp_seeding_matches_reference(m, d, k, prec):
    """GPU D^2 seeding (float64 pairwise feature reduce for any D, device
    pairwise total, bit-exact device searchsorted over numpy's sequential
    cumsum; only the reference's Generator draws on the host) picks exactly
    the reference's centroids (kmeans.py:86-103)."""
    x, _, _ = P.gaussian_mixture(m, d, k, 0.3, precision=prec, seed=5)
    got = P.init_centroids(x, k, seed=9, method="kmeanspp")
    ref = O.init_centroids(x, k, 9, "kmeanspp")
    assert got.tobytes() == ref.tobytes()


def test_kmeanspp_search_ambiguity_replay():
    """ftk_kpp_search on adversarial prefixes: r placed exactly on, and one
    ulp around, sequential-cumsum boundaries (the certified scan cannot
    decide these; the exact replay must) -- against numpy's searchsorted."""
    import torch

    from paper_2408_01391_b200 import _engine as E

    rng = np.random.default_rng(3)
    d2 = rng.random(300_001) * rng.choice([1e-8, 1.0, 1e8], 300_001)
    d2[1000:1100] = 0.0  # a flat stretch of the cumsum
    cs = np.cumsum(d2)
    dev = torch.from_numpy(d2).cuda()
    pick = torch.zeros(1, dtype=torch.int64, device="cuda")
    nrep = torch.zeros(1, dtype=torch.int64, device="cuda")
    rs = [0.0, cs[0], cs[999], cs[1050], cs[150_000], np.nextafter(cs[150_000], 0),
          np.nextafter(cs[150_000], np.inf), cs[-1], cs[-1] * 2, float(rng.random() * cs[-1])]
    for r in rs:
        E.kpp_search_dev(dev, float(r), pick, nrep)
        want = min(int(np.searchsorted(cs, r, side="right")), len(d2) - 1)
        assert int(pick.item()) == want, (r, int(pick.item()), want)
    assert int(nrep.item()) >= 1  # the on-boundary draws went through the exact replay


@pytest.mark.parametrize("ft", ["off", "abft"])
def test_graph_replay_equals_eager(ft):
    """CUDA-graph replay of the Lloyd step gives the eager step's bits
    (inertia, label-change flag, movement, centroids) every iteration."""
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200.kmeans import LloydEngine

    x, _, _ = P.gaussian_mixture(20000, 64, 96, 0.3, precision="single", seed=3)
    x_t = E.to_dev(x)
    c0 = P.init_centroids(x, 96, seed=1, method="random-sample")
    runs = []
    for graph in (False, True):
        eng = LloydEngine(x_t, c0, 96, np.float32, P.default_config(np.float32), ft,
                          P.Threshold.default_for(np.float32), 8, graph=graph)
        outs = [eng.step(it) for it in range(9)]
        runs.append((outs, E.to_host(eng.cent).copy(), eng.graphs[0] is not None))
        eng.close()
    assert runs[1][2], "graph mode did not capture"
    assert runs[0][0] == runs[1][0]
    assert runs[0][1].tobytes() == runs[1][1].tobytes()


def test_graph_replay_with_injections_equals_eager():
    """Injected passes replayed from the device-count injection graph give the
    eager path's bits: per-step outputs, centroids, detection events (with
    their real iteration numbers) and the hook's record of landed flips."""
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook
    from paper_2408_01391_b200.kmeans import LloydEngine

    x, _, _ = P.gaussian_mixture(20010, 64, 96, 0.3, precision="single", seed=3)
    x_t = E.to_dev(x)
    c0 = P.init_centroids(x, 96, seed=1, method="random-sample")
    # duplicate blocks, an unsorted schedule, the partial last block (625:
    # 10 rows), a flip past its live rows and a low mantissa bit
    ents = [FaultEntry(2, (5, 0), (3, 7), 30), FaultEntry(4, (600, 0), (2, 2), 27),
            FaultEntry(4, (17, 0), (0, 1), 29), FaultEntry(4, (17, 0), (9, 40), 31),
            FaultEntry(7, (625, 0), (5, 95), 30), FaultEntry(7, (625, 0), (20, 3), 30),
            FaultEntry(7, (3, 0), (31, 95), 30), FaultEntry(8, (1, 0), (1, 1), 2)]
    runs = []
    for graph in (False, True):
        hook = ScheduledFaultHook(FaultSchedule(list(ents)))
        eng = LloydEngine(x_t, c0, 96, np.float32, P.default_config(np.float32), "abft",
                          P.Threshold.default_for(np.float32), 8, gemm_hook=hook, graph=graph)
        outs = [eng.step(it) for it in range(10)]
        evs = [(e.iteration, e.tile, e.kind, e.loc, e.delta) for e in eng.report.events]
        runs.append((outs, E.to_host(eng.cent).copy(), evs, hook.injected,
                     eng.inj_graphs[0] is not None or eng.inj_graphs[1] is not None))
        eng.close()
    assert runs[1][4], "injected passes were not replayed from a graph"
    assert runs[0][0] == runs[1][0]
    assert runs[0][1].tobytes() == runs[1][1].tobytes()
    assert runs[0][2] == runs[1][2]
    assert len(runs[0][2]) >= 4
    assert runs[0][3] == runs[1][3]


@pytest.mark.parametrize("ft", ["off", "abft"])
def test_run_ahead_steps_equal_plain_steps(ft):
    """Graph steps with one replay queued ahead (more=...) give the plain
    steps' bits: per-step outputs, centroids, detections and hook records,
    with scheduled flips interleaved and an empty-cluster reseed (which
    discards and reruns the queued step)."""
    from paper_2408_01391_b200 import _engine as E
    from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook
    from paper_2408_01391_b200.kmeans import LloydEngine

    x, _, _ = P.gaussian_mixture(30000, 64, 96, 0.3, precision="single", seed=5)
    x_t = E.to_dev(x)
    c0 = P.init_centroids(x, 96, seed=3, method="random-sample")
    c0[5] = 1e6  # a far centroid: empty at step 0, reseeded on the host
    ents = [FaultEntry(3, (7, 0), (2, 9), 30), FaultEntry(6, (100, 0), (1, 50), 29)]
    runs = []
    for ahead in (False, True):
        hook = ScheduledFaultHook(FaultSchedule(list(ents))) if ft == "abft" else P.FaultHook()
        eng = LloydEngine(x_t, c0, 96, np.float32, P.default_config(np.float32), ft,
                          P.Threshold.default_for(np.float32), 8, gemm_hook=hook, graph=True)
        outs = [eng.step(it, more=(lambda it=it: it + 1 < 14) if ahead else None)
                for it in range(14)]
        evs = [(e.iteration, e.tile, e.kind, e.loc, e.delta) for e in eng.report.events]
        lab, inertia = eng.final(14)
        runs.append((outs, E.to_host(eng.cent).tobytes(), evs,
                     getattr(hook, "injected", None), lab.tolist(), inertia))
        eng.close()
    assert runs[0] == runs[1]


@pytest.mark.parametrize("ft,inject", [("off", None), ("abft", "prob:0.02@exp")])
def test_fit_workspace_reuse_equals_fresh(ft, inject, monkeypatch):
    """Back-to-back fits of one shape reuse the resident workspace (buffers and
    captured graphs): each result equals a fit on a fresh engine."""
    from paper_2408_01391_b200 import kmeans as K

    xs = [P.gaussian_mixture(6000, 32, 20, 0.3, precision="single", seed=s)[0] for s in (1, 2, 3)]
    cfg = P.KMeansConfig(k=20, max_iters=12, tol=0.0, seed=4, init="random-sample", ft_mode=ft)

    def fits():
        out = []
        for x in xs:
            r = P.lloyd(x, cfg, fault_spec=inject)
            out.append((r.assignments.tolist(), r.centroids.tobytes(), r.inertia, r.iters,
                        r.inertia_history, [(e.iteration, e.tile, e.kind, e.loc, e.delta)
                                            for e in r.report.events]))
        return out

    K.clear_fit_cache()
    cached = fits()
    assert K._FIT_CACHE.get("eng") is not None
    monkeypatch.setenv("FTK_FIT_CACHE", "0")
    K.clear_fit_cache()
    fresh = fits()
    assert cached == fresh


def test_graph_steps_measure_phase_times():
    """timings_ on graph steps are measured per step (events around the
    assignment and update graph replays), not copies of an eager step's."""
    from paper_2408_01391_b200.kmeans import LloydEngine

    x, _, _ = P.gaussian_mixture(50_000, 64, 64, 0.25, precision="single", seed=4)
    c0 = P.init_centroids(x, 64, seed=4, method="random-sample")
    eng = LloydEngine(P._engine.to_dev(x), c0, 64, np.float32, P.default_config(np.float32), "off",
                      P.Threshold.default_for(np.float32), 8, graph=True)
    seen = []
    for it in range(12):
        eng.step(it, more=(lambda it=it: it < 11))
        seen.append((eng.assign_ms, eng.update_ms))
    eng.close()
    graph = seen[2:]
    assert all(a > 0 and u > 0 for a, u in graph)
    assert len(set(graph)) > 1  # measured each step, not repeated
    r = P.lloyd(x, P.KMeansConfig(k=64, max_iters=12, tol=0.0, seed=4, init="random-sample"))
    assert 0 < r.timings["assign_ns"] + r.timings["update_ns"] < r.timings["total_ns"]


@pytest.mark.parametrize("nbytes", [(8 << 20) + 4, (48 << 20) + 12, (200 << 20) - 4])
def test_staged_pageable_upload(nbytes):
    """ftk_h2d (parallel pinned staging, chunked DMA) delivers every byte of a
    pageable numpy buffer, and work queued after it sees the data."""
    import torch

    from paper_2408_01391_b200 import _engine as E

    a = np.random.default_rng(nbytes).standard_normal(nbytes // 4).astype(np.float32)
    dst = torch.empty(a.shape, dtype=torch.float32, device="cuda")
    E.upload_into(dst, a)
    s = dst.sum()  # queued behind the upload on the current stream
    assert np.array_equal(dst.cpu().numpy(), a)
    assert abs(float(s) - float(a.astype(np.float64).sum())) < 1e-2 * a.size ** 0.5
    t = E.to_dev(a)
    assert np.array_equal(t.cpu().numpy(), a)
