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


def test_tile_table_reads_reference_tune_table(tmp_path):
    """tiles.TileTable parses the reference's tune-table CSV (tuner.py:268-293)
    and looks shapes up with its rule: exact key, else nearest (N, K) in log2
    distance within the precision, else the default tiles."""
    from paper_2408_01391_b200.tiles import TileTable, default_config, make_config

    p = tmp_path / "tt.csv"
    p.write_text("# M_bucket,N,K,precision,bm,bn,bk,sm,sn,sk,um,un,uk,gflops,reps\n"
                 "65536,32,64,single,64,128,32,32,32,32,16,8,4,12.5,3\n"
                 "65536,128,1024,single,32,256,16,32,64,16,16,8,4,40.0,3\n"
                 "1024,64,256,double,128,64,16,32,32,16,8,8,4,3.0,2\n")
    t = TileTable.load(str(p))
    f32, f64 = np.float32, np.float64
    assert t.lookup((100_000, 32, 64), f32) == make_config((64, 128, 32), (32, 32, 32), (16, 8, 4))
    # nearest in (log2 N, log2 K): (100, 800) is closer to (128, 1024) than to (32, 64)
    assert t.lookup((5, 100, 800), f32).block == (32, 256, 16)
    assert t.lookup((5, 40, 50), f32).block == (64, 128, 32)
    assert t.lookup((7, 3, 3), f64).block == (128, 64, 16)
    assert TileTable().lookup((7, 3, 3), f64) == default_config(f64)
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2,3,single,1\n")
    with pytest.raises(ValueError, match="bad tune-table row"):
        TileTable.load(str(bad))


def test_event_overflow_is_per_worker():
    """The reference raises when ANY worker's n_inj + 64 buffer overflows
    (abft.py:280-316), not only when the total does."""
    from paper_2408_01391_b200.abft import split_ranges, worker_overflow

    assert split_ranges(10, 4) == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert split_ranges(0, 8) == []
    ev = lambda bi: ((0, bi, 0, 0, 0, 0, 0), 0.0)  # noqa: E731
    burst = [ev(0)] * 65  # 65 events in worker 0's rows, total well under 4 * 64
    assert worker_overflow(burst, 0, 10, 4)
    assert not worker_overflow(burst, 1, 10, 4)
    spread = [ev(b) for b in (0, 3, 6, 9)] * 64
    assert not worker_overflow(spread, 0, 10, 4)
    assert worker_overflow([ev(0)] * 65, 0, 10, 1)
