"""CPU-only checks: host logic pinned to the reference, and the C ABI surface."""

import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

from paper_2408_01391_b200 import faults as F
from paper_2408_01391_b200.matrix import gaussian_mixture
from paper_2408_01391_b200.tiles import TileConfig, default_config, make_config, parse_tile


def test_abi_exports_every_declared_symbol():
    from paper_2408_01391_b200 import _native

    hdr = open(os.path.join(ROOT, "include", "ftk_b200.h")).read()
    declared = set(re.findall(r"\b(ftk_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = _native.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.PROTOTYPES), declared ^ set(_native.PROTOTYPES)
    assert lib.ftk_version() == 1


def test_flip_bit_golden():
    cases = json.load(open(os.path.join(GOLDEN, "fault_cases.json")))
    for v, b, f32, f64 in cases["flip"]:
        got = float(F.flip_bit(np.float32(v), b))
        assert got == f32 or (np.isnan(got) and np.isnan(f32))
        assert repr(float(F.flip_bit(np.float64(v), b + 32))) == f64
    assert F.flip_bit(np.float32(1.0), 31) == -1.0
    with pytest.raises(ValueError):
        F.flip_bit(np.float32(1.0), 32)


def test_plan_faults_golden():
    cases = json.load(open(os.path.join(GOLDEN, "fault_cases.json")))
    for c in cases["plans"]:
        sp = F.FaultSpec.parse(c["text"], seed=11)
        plan = F.plan_faults(sp, c["iters"], tuple(c["grid"]), tuple(c["dims"]),
                             dtype=np.dtype(c["dtype"]),
                             shape=tuple(c["shape"]) if c["shape"] else None)
        got = [[e.iteration, *e.tile, *e.elem, e.bit] for e in plan.entries]
        assert got == c["entries"], c["text"]


def test_fault_spec_parse_errors():
    for bad in ["bogus", "fixed:2@zzz", "prob:x"]:
        with pytest.raises(ValueError):
            F.FaultSpec.parse(bad)
    with pytest.raises(ValueError):
        F.FaultSpec(mode="per-tile-prob", prob=2.0)


def test_hook_protocol_roundtrip():
    h = F.ScheduledFaultHook(F.FaultSchedule([F.FaultEntry(0, (0, 0), (1, 2), 62)]))
    assert h.kernel_arrays(1, np.float32) is None
    arrs = h.kernel_arrays(0, np.float32)
    assert [a.dtype for a in arrs] == [np.int64] * 6 + [np.float64] * 2
    arrs[5][0] = 1
    arrs[6][0], arrs[7][0] = 1.0, 3.0
    h.absorb_kernel_results(0, arrs[5], arrs[6], arrs[7])
    assert h.injected[0]["delta"] == 2.0
    acc = np.ones((3, 3))
    assert h.has_pending_site(0, (0, 0))
    h.maybe_corrupt(0, (0, 0), acc)
    assert acc[1, 2] != 1.0 and not h.has_pending_site(0, (0, 0))


def test_tiles_validation():
    assert default_config(np.float32).block == (32, 256, 16)
    assert default_config(np.float64).block == (64, 64, 16)
    assert parse_tile("128,64,16,32,64,16", np.float32).block == (128, 64, 16)
    with pytest.raises(ValueError, match="sub.k"):
        TileConfig((64, 64, 16), (32, 32, 8), (16, 8, 4)).validate()
    with pytest.raises(ValueError):
        make_config((48, 64, 16), (16, 64, 16), (16, 8, 4))


def test_gaussian_mixture_golden(golden):
    z = golden("gmm_cases.npz")
    for t in range(int(z["n"])):
        r, c, k, seed = (int(v) for v in z[f"g{t}_args"])
        x, lab, cen = gaussian_mixture(r, c, k, float(z[f"g{t}_spread"]),
                                       precision=str(z[f"g{t}_prec"]), seed=seed)
        assert x.tobytes() == z[f"g{t}_x"].tobytes()
        assert np.array_equal(lab, z[f"g{t}_lab"])
        assert cen.tobytes() == z[f"g{t}_cen"].tobytes()
    import hashlib
    shas = json.loads(str(z["big_shas"]))
    for key, want in shas.items():
        r, c, k = (int(v) for v in key.split("_"))
        x, _, _ = gaussian_mixture(r, c, k, 0.25, precision="single", seed=0, chunk_rows=3000)
        assert hashlib.sha256(x.tobytes()).hexdigest() == want, key


def test_public_api_surface():
    import inspect

    import paper_2408_01391_b200 as P

    for name in ["FTKMeans", "lloyd", "KMeansConfig", "KMeansResult", "fused_assign",
                 "checked_assign", "update_step", "row_sq_norms", "FaultSpec", "plan_faults",
                 "ScheduledFaultHook", "FaultHook", "Threshold", "DetectionReport",
                 "FaultEscalationError", "init_centroids", "gaussian_mixture", "TileConfig"]:
        assert hasattr(P, name), name
    sig = inspect.signature(P.fused_assign)
    assert list(sig.parameters) == ["x", "y", "y_norms", "cfg", "threads", "hook", "iteration"]
    sig = inspect.signature(P.checked_assign)
    assert list(sig.parameters) == ["x", "y", "y_norms", "cfg", "thr", "hook", "iteration",
                                    "threads"]
    sig = inspect.signature(P.update_step)
    assert list(sig.parameters) == ["x", "assignments", "k", "ft_mode", "hook", "iteration",
                                    "sq_dists"]
    est = P.FTKMeans()
    assert sorted(est.get_params()) == sorted(["n_clusters", "init", "max_iter", "tol",
                                               "random_state", "ft_mode", "tile", "delta_rel",
                                               "inject", "threads", "tune_table"])


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2408_01391_b200 as P

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        P.fused_assign(np.ones((4, 2), np.float32), np.ones((2, 2), np.float32))


def test_config_validation():
    import paper_2408_01391_b200 as P

    x = np.ones((16, 2), np.float32)
    with pytest.raises(ValueError):
        P.lloyd(x, P.KMeansConfig(k=0))
    with pytest.raises(ValueError):
        P.lloyd(x, P.KMeansConfig(k=2, ft_mode="huh"))
    with pytest.raises(ValueError):
        P.lloyd(x, P.KMeansConfig(k=32))
    with pytest.raises(ValueError, match="inner dimensions"):
        P.fused_assign(np.zeros((4, 3), np.float32), np.zeros((2, 5), np.float32))
    with pytest.raises(ValueError, match="dtypes"):
        P.fused_assign(np.zeros((4, 3), np.float32), np.zeros((2, 3), np.float64))
