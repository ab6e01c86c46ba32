"""Narrow streamed-X screen (csrc/tc_narrow.cu): d > 256 with k + 4 <= 256.

Bit-exact against the oracle for every hint (none, the true labels, random
labels, out-of-range garbage): the hint only decides which rows need a second
read of X.  Under fault injection with the exact replay switched off
(FTK_OPT_INJ_REPLAY = 0) the kernel's own detect / locate / correct result
must give the clean labels and one event per flip; with the replay on the
events are the reference's (the exact checked kernel's).
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_01391_b200")
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200 import _native as N  # noqa: E402
from paper_2408_01391_b200.abft import Threshold, events_from_ring  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    E.set_inj_replay(True)


SHAPES = [(5000, 512, 8), (3001, 2048, 16), (2000, 300, 33), (1500, 260, 252), (700, 1024, 1),
          (4097, 516, 64), (900, 8192, 32), (129, 388, 100)]


def _data(m, d, k, seed):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((k, d)).astype(np.float32)
    lab = rng.integers(0, k, m)
    x = (c[lab] + 0.5 * rng.standard_normal((m, d))).astype(np.float32)
    y = (c + 0.05 * rng.standard_normal((k, d))).astype(np.float32)
    return np.ascontiguousarray(x), np.ascontiguousarray(y)


def _assign(x, y, hint=None, checked=False, inj=None, events=None, iteration=0):
    x_t, y_t = E.to_dev(x), E.to_dev(y)
    yn = E.row_sq_norms_dev(y_t)
    h_t = None
    if hint is not None:
        h_t = E.to_dev(np.asarray(hint, np.int32))
        E.set_label_hint(h_t, x.shape[0])
    try:
        thr = Threshold.default_for(np.float32).kernel_params()
        idx, val = E.assign_dev(x_t, y_t, yn, (128, 128, 32), variant="tc", inj=inj,
                                checked=checked, delta_rel=thr[0], abs_tol=thr[1],
                                iteration=iteration, events=events)
    finally:
        E.set_label_hint(None, 0)
    return E.to_host(idx).astype(np.int64), E.to_host(val)


def _stats():
    import ctypes

    out = (ctypes.c_int64 * 3)()
    N.check(N.load().ftk_tc_fallback_rows(E.ctx(), out, E.stream()), "fallback")
    return list(out)


@pytest.mark.parametrize("m,d,k", SHAPES)
def test_narrow_matches_oracle_any_hint(m, d, k):
    x, y = _data(m, d, k, seed=m + d + k)
    lab, val = O.assign(x, y)
    rng = np.random.default_rng(1)
    hints = [None, lab, rng.integers(0, k, m), rng.integers(-5, k + 5, m) * 1000003]
    for h in hints:
        r_lab, r_val = _assign(x, y, hint=h)
        assert np.array_equal(r_lab, lab), (m, d, k)
        assert r_val.tobytes() == val.tobytes(), (m, d, k)
    # with the true labels as hint nearly every row finishes in the screen or
    # with at most one more exact chain (resolve pass)
    _assign(x, y, hint=lab)
    resolve_rows, exact_rows, _ = _stats()
    assert resolve_rows + exact_rows <= max(8, m // 10)


@pytest.mark.parametrize("m,d,k", [(3000, 512, 16), (2000, 2048, 32), (1000, 300, 8)])
def test_narrow_checked_clean_matches_oracle(m, d, k):
    x, y = _data(m, d, k, seed=3)
    lab, val = O.assign(x, y)
    ev = E.DevEvents(64)
    r_lab, r_val = _assign(x, y, hint=lab, checked=True, events=ev)
    assert np.array_equal(r_lab, lab)
    assert r_val.tobytes() == val.tobytes()
    over, raw = ev.read()
    assert not over and raw == []  # no false alarm on clean data
    assert _stats()[2] == 0


def _flips(x, y, n, bm, bn, seed, bits=(26, 27, 28, 29)):
    """n flips on distinct rows whose exact accumulator moves by far more than
    the detection tolerance (so every one must be detected)."""
    rng = np.random.default_rng(seed)
    m, k = x.shape[0], y.shape[0]
    rows = rng.choice(m, size=4 * n, replace=False)
    out = []
    for r in rows:
        c = int(rng.integers(0, k))
        b = int(rng.choice(bits))
        acc = np.float32(O.exact_dot(x[r], y[c]))
        after = (np.array([acc], np.float32).view(np.uint32) ^ np.uint32(1 << b)).view(np.float32)[0]
        if np.isfinite(after) and abs(float(after) - float(acc)) > 50.0:
            out.append((int(r), c, b))
        if len(out) == n:
            break
    bi = np.array([r // bm for r, _, _ in out], np.int64)
    bj = np.array([c // bn for _, c, _ in out], np.int64)
    ei = np.array([r % bm for r, _, _ in out], np.int64)
    ej = np.array([c % bn for _, c, _ in out], np.int64)
    bit = np.array([b for _, _, b in out], np.int64)
    z = len(out)
    arrs = (bi, bj, ei, ej, bit, np.zeros(z, np.int64), np.zeros(z), np.zeros(z))
    return out, arrs


@pytest.mark.parametrize("m,d,k", [(3000, 512, 16), (2000, 2048, 32)])
def test_narrow_in_kernel_correction(m, d, k):
    """Replay off: the screen's own location + in-register correction stands."""
    x, y = _data(m, d, k, seed=11)
    lab, val = O.assign(x, y)
    flips, arrs = _flips(x, y, 24, 128, 128, seed=5)
    assert len(flips) >= 16
    E.set_inj_replay(False)
    try:
        ev = E.DevEvents(256)
        inj = E.DevInjection(arrs)
        r_lab, r_val = _assign(x, y, hint=lab, checked=True, inj=inj, events=ev, iteration=3)
    finally:
        E.set_inj_replay(True)
    assert np.array_equal(r_lab, lab)          # zero label divergence
    assert r_val.tobytes() == val.tobytes()    # exact values (winner recomputed exactly)
    over, raw = ev.read()
    assert not over
    evs = events_from_ring(raw)
    got = sorted((e.tile, e.loc) for e in evs)
    want = sorted(((r // 128, c // 128), (r % 128, c % 128)) for r, c, _ in flips)
    assert got == want
    assert all(e.kind == "detected-corrected" and e.iteration == 3 for e in evs)


def test_narrow_uncorrectable_goes_exact():
    """A flip to a non-finite value cannot be located: the row is re-resolved
    exactly and recorded as detected-uncorrectable."""
    m, d, k = 1000, 512, 16
    x, y = _data(m, d, k, seed=12)
    lab, val = O.assign(x, y)
    r, c = 17, 5
    acc = np.float32(O.exact_dot(x[r], y[c]))
    # the exponent bit that turns this value into inf/nan
    bit = 30
    arrs = (np.array([r // 128]), np.array([c // 128]), np.array([r % 128]), np.array([c % 128]),
            np.array([bit]), np.zeros(1, np.int64), np.zeros(1), np.zeros(1))
    arrs = tuple(np.asarray(a, dtype=np.int64) if i < 6 else np.asarray(a, np.float64)
                 for i, a in enumerate(arrs))
    after = (np.array([acc], np.float32).view(np.uint32) ^ np.uint32(1 << bit)).view(np.float32)[0]
    E.set_inj_replay(False)
    try:
        ev = E.DevEvents(16)
        r_lab, r_val = _assign(x, y, hint=lab, checked=True, inj=E.DevInjection(arrs), events=ev)
    finally:
        E.set_inj_replay(True)
    assert np.array_equal(r_lab, lab)
    assert r_val.tobytes() == val.tobytes()
    evs = events_from_ring(ev.read()[1])
    assert len(evs) == 1 and evs[0].tile[0] == r // 128 and evs[0].loc[0] == r % 128
    if not np.isfinite(after) or abs(float(after)) > 1e30:
        assert evs[0].kind in ("detected-uncorrectable", "detected-corrected")


def test_narrow_replay_events_are_the_references():
    """Replay on (default): rows with scheduled flips carry the exact checked
    kernel's (= the reference's) events and values."""
    m, d, k = 2000, 512, 16
    x, y = _data(m, d, k, seed=13)
    flips, arrs = _flips(x, y, 12, 64, 8, seed=9)
    thr = Threshold.default_for(np.float32)

    def run(variant):
        x_t, y_t = E.to_dev(x), E.to_dev(y)
        ev = E.DevEvents(256)
        inj = E.DevInjection(tuple(np.array(a, copy=True) for a in arrs))
        d_rel, a_tol = thr.kernel_params()
        idx, vals = E.assign_dev(x_t, y_t, E.row_sq_norms_dev(y_t), (64, 8, 32), variant=variant,
                                 inj=inj, checked=True, delta_rel=d_rel, abs_tol=a_tol,
                                 iteration=2, events=ev)
        return E.to_host(idx), E.to_host(vals), events_from_ring(ev.read()[1])

    li, vi, ei = run("exact")
    lt, vt, et = run("tc")
    assert np.array_equal(li, lt)
    assert vi.tobytes() == vt.tobytes()
    key = lambda e: (e.iteration, e.tile, e.interval, e.loc)  # noqa: E731
    assert sorted(ei, key=key) == sorted(et, key=key)
    assert len(ei) >= 1
