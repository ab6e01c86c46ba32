"""Online ABFT of the CTA-pair tensor-core screen (csrc/tc_pair.cu).

With the exact replay of scheduled blocks switched off (FTK_OPT_INJ_REPLAY=0)
the screen's own result stands: every flip far above the tolerance must be
detected by the row checksum, located to its 128-column group by the
group-weighted checksum, corrected (exact values of j1 and of the group's
columns, certified against the runner-up) and recorded as a
detected-corrected event -- with labels and min_dists bit-identical to the
clean pass.  Clean data raises no event.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_01391_b200")
from paper_2408_01391_b200 import _engine as E  # noqa: E402
from paper_2408_01391_b200.abft import Threshold, events_from_ring  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    E.set_inj_replay(True)


def _data(m, d, k, seed):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((k, d)).astype(np.float32)
    lab = rng.integers(0, k, m)
    x = (c[lab] + 0.5 * rng.standard_normal((m, d))).astype(np.float32)
    y = (c + 0.05 * rng.standard_normal((k, d))).astype(np.float32)
    return np.ascontiguousarray(x), np.ascontiguousarray(y)


def _checked(x, y, block, inj=None, iteration=0, cap=256):
    x_t, y_t = E.to_dev(x), E.to_dev(y)
    ev = E.DevEvents(cap)
    d_rel, a_tol = Threshold.default_for(np.float32).kernel_params()
    idx, val = E.assign_dev(x_t, y_t, E.row_sq_norms_dev(y_t), block, variant="tc", inj=inj,
                            checked=True, delta_rel=d_rel, abs_tol=a_tol, iteration=iteration,
                            events=ev)
    over, raw = ev.read()
    assert not over
    return E.to_host(idx).astype(np.int64), E.to_host(val), events_from_ring(raw)


def _flips(x, y, n, bm, bn, seed):
    rng = np.random.default_rng(seed)
    m, k = x.shape[0], y.shape[0]
    out = []
    for r in rng.choice(m, size=6 * n, replace=False):
        c = int(rng.integers(0, k))
        b = int(rng.choice([26, 27, 28, 29]))
        acc = np.float32(O.exact_dot(x[r], y[c]))
        after = (np.array([acc], np.float32).view(np.uint32) ^ np.uint32(1 << b)).view(np.float32)[0]
        if np.isfinite(after) and 50.0 < abs(float(after) - float(acc)) < 1e6:
            out.append((int(r), c, b))
        if len(out) == n:
            break
    cols = [np.array(v, np.int64) for v in zip(*[(r // bm, c // bn, r % bm, c % bn, b)
                                                 for r, c, b in out])]
    z = len(out)
    return out, tuple(cols) + (np.zeros(z, np.int64), np.zeros(z), np.zeros(z))


@pytest.mark.parametrize("m,d,k", [(4000, 128, 1024), (3000, 64, 300), (2500, 256, 77)])
def test_pair_clean_no_events(m, d, k):
    x, y = _data(m, d, k, seed=21)
    lab, val = O.assign(x, y)
    r_lab, r_val, evs = _checked(x, y, (128, 128, 32))
    assert np.array_equal(r_lab, lab)
    assert r_val.tobytes() == val.tobytes()
    assert evs == []


@pytest.mark.parametrize("m,d,k", [(4000, 128, 1024), (3000, 64, 300)])
def test_pair_in_kernel_location_and_correction(m, d, k):
    x, y = _data(m, d, k, seed=22)
    lab, val = O.assign(x, y)
    bm, bn = 128, 64
    flips, arrs = _flips(x, y, 20, bm, bn, seed=3)
    assert len(flips) >= 12
    E.set_inj_replay(False)
    try:
        r_lab, r_val, evs = _checked(x, y, (bm, bn, 32), inj=E.DevInjection(arrs), iteration=5)
    finally:
        E.set_inj_replay(True)
    assert np.array_equal(r_lab, lab)        # zero label divergence
    assert r_val.tobytes() == val.tobytes()  # the reference's bits
    got = sorted((e.tile[0], e.loc[0], e.kind) for e in evs)
    want = sorted((r // bm, r % bm, "detected-corrected") for r, _, _ in flips)
    assert got == want
    # located to the flipped column's 128-column group
    group_of = {r: c // 128 for r, c, _ in flips}
    for e in evs:
        r = e.tile[0] * bm + e.loc[0]
        assert e.tile[1] == (group_of[r] * 128) // bn and e.iteration == 5


@pytest.mark.parametrize("m,d,k", [(2000, 512, 600), (1200, 1024, 300)])
def test_pair_streamed_x_checked_with_replay(m, d, k):
    """d > 256 with several column tiles (X streamed through the stages and
    re-read per tile): clean pass = oracle, injected pass = the exact checked
    kernel's values and events (the reference's)."""
    x, y = _data(m, d, k, seed=23)
    lab, val = O.assign(x, y)
    r_lab, r_val, evs = _checked(x, y, (32, 256, 16))
    assert np.array_equal(r_lab, lab) and r_val.tobytes() == val.tobytes() and evs == []
    flips, arrs = _flips(x, y, 8, 32, 256, seed=4)

    def run(variant):
        x_t, y_t = E.to_dev(x), E.to_dev(y)
        ev = E.DevEvents(256)
        d_rel, a_tol = Threshold.default_for(np.float32).kernel_params()
        inj = E.DevInjection(tuple(np.array(a, copy=True) for a in arrs))
        idx, v = E.assign_dev(x_t, y_t, E.row_sq_norms_dev(y_t), (32, 256, 16), variant=variant,
                              inj=inj, checked=True, delta_rel=d_rel, abs_tol=a_tol, iteration=1,
                              events=ev)
        return E.to_host(idx), E.to_host(v), events_from_ring(ev.read()[1])

    li, vi, ei = run("exact")
    lp, vp, ep = run("pair")
    assert np.array_equal(li, lp) and vi.tobytes() == vp.tobytes()
    key = lambda e: (e.iteration, e.tile, e.interval, e.loc)  # noqa: E731
    assert sorted(ei, key=key) == sorted(ep, key=key) and len(ei) >= 1
