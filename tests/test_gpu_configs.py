"""Lloyd parity at the BASELINE configs' own shapes (GPU).

Every case of tests/golden/lloyd_configs.json was produced by the REFERENCE
``lloyd`` (kmeans.py:210-319) in the build container
(tests/golden/make_golden_configs.py).  Here the same data (digest-checked)
and configuration run through this package's ``lloyd`` on the B200, and the
results must be bit-identical: labels, centroids, inertia and its history,
iteration count, convergence flag and -- for the ABFT runs with scheduled
flips -- the detection-event list.  The FT runs also check the north_star
gate "errors detected and corrected with zero label divergence": the labels
of the protected, injected run equal those of the FT-off run exactly when the
reference's do.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2408_01391_b200 as P
from paper_2408_01391_b200.faults import FaultSpec

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "lloyd_configs.json")) as _fh:
    DB = json.load(_fh)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_XCACHE = {}


def _data(rows, cols, blobs, prec):
    key = (rows, cols, blobs, prec)
    if key not in _XCACHE:
        _XCACHE.clear()
        _XCACHE[key] = P.gaussian_mixture(rows, cols, blobs, 0.25, precision=prec, seed=0)[0]
    return _XCACHE[key]


@pytest.fixture(autouse=True, scope="module")
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    yield
    P.clear_fit_cache()


def _fit(case, ft=None, spec="keep"):
    rows, cols, blobs, prec, k, mi, ft0, spec0, _gen = DB[case]["args"]
    x = _data(rows, cols, blobs, prec)
    assert _sha(x) == DB[case]["xsha"], "input data differs from the reference's"
    ft = ft0 if ft is None else ft
    spec = spec0 if spec == "keep" else spec
    fs = FaultSpec.parse(spec, seed=1) if spec else None
    cfg = P.KMeansConfig(k=k, max_iters=mi, tol=0.0, seed=0, init="random-sample", ft_mode=ft)
    return P.lloyd(x, cfg, fault_spec=fs)


@pytest.mark.parametrize("case", sorted(DB))
def test_lloyd_config_matches_reference(case):
    z = DB[case]
    r = _fit(case)
    assert r.iters == z["iters"]
    assert r.converged == z["converged"]
    assert r.assignments[:64].tolist() == z["lab_head"]
    assert np.bincount(r.assignments, minlength=z["args"][4]).tolist() == z["counts"]
    assert _sha(r.assignments.astype(np.int64)) == z["lab_sha"]
    assert _sha(r.centroids) == z["c_sha"]
    assert r.inertia_history == z["hist"]
    assert r.inertia == z["inertia"]
    evs = [[e.iteration, e.tile[0], e.tile[1], e.kind, e.loc[0], e.loc[1], float(e.delta)]
           for e in r.report.events]
    assert evs == [list(e) for e in z["events"]]
    assert r.report.false_alarms == z["false_alarms"]
    if z["args"][6] != "off":
        # protected + injected run vs the FT-off run of the same data
        base = _fit(case, ft="off", spec=None)
        assert _sha(base.assignments.astype(np.int64)) == z["off_lab_sha"]
        div = int(np.count_nonzero(base.assignments != r.assignments))
        assert div == z["label_divergence_vs_off"]
