"""tcgen05 screened assignment: bit-identical to the reference on every row
(certified rows via the exact winner recomputation, the rest via the exact
fallback), across shapes that exercise partial tiles and near-ties."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_01391_b200")
from paper_2408_01391_b200 import _engine as E  # noqa: E402


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


@pytest.mark.parametrize("m,d,k", [(1000, 32, 64), (4096, 128, 1024), (333, 40, 70),
                                   (129, 8, 5), (2000, 256, 300), (5000, 64, 16),
                                   (257, 12, 129), (1, 32, 1), (640, 100, 33)])
def test_tc_matches_reference_random(m, d, k):
    rng = np.random.default_rng(m * 7 + d * 3 + k)
    x = np.ascontiguousarray(rng.standard_normal((m, d)), dtype=np.float32)
    y = np.ascontiguousarray(rng.standard_normal((k, d)), dtype=np.float32)
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab)
    assert val.tobytes() == ref_val.tobytes()
    assert 0 <= fb <= m


def test_tc_blobs_certify_almost_everything():
    x, _, _ = P.gaussian_mixture(20000, 128, 256, 0.25, precision="single", seed=0)
    rng = np.random.default_rng(1)
    y = np.ascontiguousarray(x[rng.choice(20000, 256, replace=False)])
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab)
    assert val.tobytes() == ref_val.tobytes()
    assert fb < 0.05 * 20000, fb


def test_tc_ties_go_to_fallback():
    rng = np.random.default_rng(3)
    y = np.ascontiguousarray(rng.standard_normal((40, 32)), dtype=np.float32)
    y[7] = y[3]  # exact duplicate centroid: every row nearest to it is a tie
    x = np.ascontiguousarray(np.repeat(y[3:4], 50, axis=0) + 1e-3 * rng.standard_normal((50, 32)),
                             dtype=np.float32)
    lab, val, fb = _tc(x, y)
    ref_lab, ref_val = O.assign(x, y)
    assert np.array_equal(lab, ref_lab) and set(lab.tolist()) == {3}
    assert val.tobytes() == ref_val.tobytes()
    assert fb >= 50
