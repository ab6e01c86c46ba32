"""tcgen05 screened assignment: bit-identical to the reference on every row
(certified rows via the exact winner recomputation, the rest via the 3xTF32
re-screen and the exact fallback), plus the screening error model the
certification relies on."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_01391_b200")
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200 import gemm as G  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _tc(x, y):
    x_t, y_t = E.to_dev(x), E.to_dev(y)
    idx, val = E.assign_dev(x_t, y_t, E.row_sq_norms_dev(y_t), (32, 256, 16), variant="tc")
    fb = E.tc_fallback_rows()
    return E.to_host(idx).astype(np.int64), E.to_host(val), fb


SHAPES = [(1000, 32, 64), (4096, 128, 1024), (333, 40, 70), (129, 8, 5), (2000, 256, 300),
          (5000, 64, 16), (257, 12, 129), (1, 32, 1), (640, 100, 33), (3000, 200, 40),
          (3000, 4, 700), (2000, 4, 4096)]


@pytest.mark.parametrize("m,d,k", SHAPES)
def test_tc_matches_reference_random(m, d, k):
    rng = np.random.default_rng(m * 7 + d * 3 + k)
    x = np.ascontiguousarray(rng.standard_normal((m, d)), dtype=np.float32)
    y = np.ascontiguousarray(rng.standard_normal((k, d)), dtype=np.float32)
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab)
    assert val.tobytes() == ref_val.tobytes()
    assert 0 <= fb[1] <= fb[0] <= m


@pytest.mark.parametrize("d,k", [(128, 256), (32, 64), (64, 1000)])
def test_tc_blobs(d, k):
    x, _, _ = P.gaussian_mixture(20000, d, k, 0.25, precision="single", seed=0)
    rng = np.random.default_rng(1)
    y = np.ascontiguousarray(x[rng.choice(20000, k, replace=False)])
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab)
    assert val.tobytes() == ref_val.tobytes()
    assert fb[1] < 0.01 * 20000, fb  # the 3xTF32 re-screen certifies nearly every tie


def test_tc_ties_resolved_exactly():
    rng = np.random.default_rng(3)
    y = np.ascontiguousarray(rng.standard_normal((40, 32)), dtype=np.float32)
    y[7] = y[3]  # exact duplicate centroid: every row nearest to it is a tie
    x = np.ascontiguousarray(np.repeat(y[3:4], 50, axis=0) + 1e-3 * rng.standard_normal((50, 32)),
                             dtype=np.float32)
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab) and set(lab.tolist()) == {3}
    assert val.tobytes() == ref_val.tobytes()
    # no screen can certify an exact tie: every row takes the exact path
    # (the candidate evaluation of the CTA-pair pass 2, or the exact kernel)
    assert fb[0] >= 50


def _tf32(a):
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("split", [False, True])
def test_screen_error_model(split):
    """Raw tensor-core dots vs exact float64: the error stays inside the bound
    the certification uses (and well below it)."""
    rng = np.random.default_rng(11)
    m, d, k = 512, 128, 256
    x = np.ascontiguousarray(rng.standard_normal((m, d)) * np.exp(rng.uniform(-3, 3, (m, 1))),
                             dtype=np.float32)
    y = np.ascontiguousarray(rng.standard_normal((k, d)), dtype=np.float32)
    x_t, y_t = E.to_dev(x), E.to_dev(y)
    raw, idx, val = E.tc_raw_dots(x_t, y_t, E.row_sq_norms_dev(y_t), split=split)
    raw = E.to_host(raw).astype(np.float64)
    exact = x.astype(np.float64) @ y.astype(np.float64).T
    s = np.abs(x.astype(np.float64)) @ np.abs(y.astype(np.float64)).T
    if split:
        bound = (3 * 2.0**-20 + 6 * d * 2.0**-24) * s
    else:
        bound = (2.0**-9 + 2.0**-20 + 2 * d * 2.0**-24) * s
    err = np.abs(raw - exact)
    assert (err <= bound).all(), float((err / np.maximum(bound, 1e-300)).max())
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(E.to_host(idx), ref_lab)
    assert E.to_host(val).tobytes() == ref_val.tobytes()
    print("max err/bound", float((err / bound).max()), "split", split)


def test_tc_checked_matches_reference_events(golden):
    """Checksum-protected TC path: fault-free -> same bits as the unprotected
    reference and no TC checksum alarm; injected -> the reference's labels,
    min_dists, events and hook records (golden fixtures)."""
    from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook
    from paper_2408_01391_b200.tiles import MICRO_SINGLE, make_config

    rng = np.random.default_rng(5)
    x = np.ascontiguousarray(rng.standard_normal((3000, 64)), dtype=np.float32)
    y = np.ascontiguousarray(rng.standard_normal((300, 64)), dtype=np.float32)
    res, rep = P.checked_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(res.assignments, lab) and res.min_dists.tobytes() == val.tobytes()
    assert rep.detections == 0 and E.tc_fallback_rows()[2] == 0
    z = golden("checked_cases.npz")
    for n in ["a", "b", "d"]:
        xx, yy, ent = z[f"{n}_x"], z[f"{n}_y"], z[f"{n}_ent"]
        if xx.shape[1] % 4:
            continue
        blk = tuple(int(v) for v in z[f"{n}_block"])
        cfg = None if blk[0] < 0 else make_config(blk, blk, MICRO_SINGLE)
        entries = [FaultEntry(int(e[0]), (int(e[1]), int(e[2])), (int(e[3]), int(e[4])), int(e[5]))
                   for e in ent]
        h = ScheduledFaultHook(FaultSchedule(entries))
        old = G.get_variant()
        G.set_variant("tc")  # the tensor-core screen, whatever the variant table prefers
        try:
            r2, rep2 = P.checked_assign(xx, yy, cfg=cfg, hook=h)
        finally:
            G.set_variant(old)
        assert np.array_equal(r2.assignments, z[f"{n}_lab"]), n
        assert r2.min_dists.tobytes() == z[f"{n}_val"].tobytes(), n
        ev = np.array([[e.iteration, e.tile[0], e.tile[1],
                        0 if e.kind == "detected-corrected" else 1, e.loc[0], e.loc[1]]
                       for e in rep2.events], np.int64).reshape(-1, 6)
        assert ev.tolist() == z[f"{n}_ev"].tolist(), n
        inj = np.array([[d["before"], d["after"]] for d in h.injected]).reshape(-1, 2)
        assert inj.tobytes() == z[f"{n}_inj"].tobytes(), n
        # the tensor-core checksum itself saw the above-threshold flips
        assert E.tc_fallback_rows()[2] >= 1, n


@pytest.mark.parametrize("m,d,k", [(3000, 512, 16), (1500, 2048, 8), (2000, 300, 200),
                                   (700, 260, 256), (4100, 1024, 33)])
def test_tc_streamed_x_matches_reference(m, d, k, monkeypatch):
    """d > 256 with k <= 256 (experimental, FTK_TC_SX=1): the pair screen
    streams X through its stages and the refine reads the row from global
    memory -- still the reference's bits."""
    monkeypatch.setenv("FTK_TC_SX", "1")
    rng = np.random.default_rng(m + d + k)
    x = np.ascontiguousarray(rng.standard_normal((m, d)), dtype=np.float32)
    y = np.ascontiguousarray(x[rng.choice(m, k, replace=False)] +
                             0.3 * rng.standard_normal((k, d)).astype(np.float32))
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab)
    assert val.tobytes() == ref_val.tobytes()
    assert fb[0] < m  # the screen certified rows itself (the TC path ran)


def test_tc_streamed_x_checked_with_flips(monkeypatch):
    """ABFT on the streamed-X screen: fault-free -> no alarm and the reference's
    bits; scheduled flips -> the exact checked kernel's events and records."""
    monkeypatch.setenv("FTK_TC_SX", "1")
    from paper_2408_01391_b200 import gemm as G
    from paper_2408_01391_b200.faults import FaultEntry, FaultSchedule, ScheduledFaultHook

    rng = np.random.default_rng(21)
    x = np.ascontiguousarray(rng.standard_normal((2500, 640)), dtype=np.float32)
    y = np.ascontiguousarray(rng.standard_normal((24, 640)), dtype=np.float32)
    res, rep = P.checked_assign(x, y)
    lab, val = O.assign(x, y)
    assert np.array_equal(res.assignments, lab) and res.min_dists.tobytes() == val.tobytes()
    assert rep.detections == 0 and E.tc_fallback_rows()[2] == 0
    ents = [FaultEntry(0, (3, 0), (5, 7), 30), FaultEntry(0, (40, 0), (0, 23), 29),
            FaultEntry(0, (78, 0), (3, 1), 27)]
    outs = []
    for variant in ("exact", "auto"):
        old = G.get_variant()
        G.set_variant(variant)
        try:
            h = ScheduledFaultHook(FaultSchedule(list(ents)))
            r2, rep2 = P.checked_assign(x, y, hook=h)
        finally:
            G.set_variant(old)
        outs.append((r2.assignments.tolist(), r2.min_dists.tobytes(),
                     [(e.iteration, e.tile, e.kind, e.loc, e.delta) for e in rep2.events],
                     h.injected))
    assert outs[0] == outs[1]
    assert len(outs[1][2]) >= 2


@pytest.mark.parametrize("d,k", [(32, 64), (128, 16), (512, 16), (64, 200)])
def test_tc_small_k_rows_certify(d, k, monkeypatch):
    """K < 256 leaves whole 32-column chunks without a centroid; they must not
    demote the running winner to runner-up (which failed every row's
    certificate and sent the whole pass to the exact fallback)."""
    monkeypatch.setenv("FTK_TC_SX", "1")  # d = 512 runs the streamed-X screen
    x, _, _ = P.gaussian_mixture(20000, d, k, 0.25, precision="single", seed=0)
    rng = np.random.default_rng(2)
    y = np.ascontiguousarray(x[rng.choice(20000, k, replace=False)])
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab)
    assert val.tobytes() == ref_val.tobytes()
    assert fb[0] < 0.05 * 20000, fb
