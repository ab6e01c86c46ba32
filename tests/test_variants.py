"""Kernel-variant selector (variants.py): the TuneTable-shaped table, its
file format and lookup rules (CPU), and on the GPU that every family gives
the reference's bits and `select` keeps the fastest measured one."""

import numpy as np
import pytest

from paper_2408_01391_b200 import variants as V


def test_feasibility_matches_library_limits():
    assert V.feasible("pair", (10, 128, 1024), "single")
    assert V.feasible("pair", (10, 512, 16), "single")  # streamed X
    assert not V.feasible("pair", (10, 8196, 16), "single")
    assert V.feasible("narrow", (10, 512, 252), "single", ft_on=True)
    assert not V.feasible("narrow", (10, 512, 253), "single", ft_on=True)
    assert V.feasible("narrow", (10, 512, 256), "single", ft_on=False)
    assert not V.feasible("pair", (10, 130, 16), "single")  # d % 4
    assert V.feasible("exact", (10, 130, 16), "single")
    assert not V.feasible("dmma", (10, 64, 256), "single")
    assert V.feasible("dmma", (10, 64, 256), "double")


def test_builtin_rule():
    assert V.builtin((1000, 128, 1024), "single") == "pair"
    assert V.builtin((1000, 2048, 32), "single") == "narrow"
    assert V.builtin((1000, 2048, 1024), "single") == "pair"
    assert V.builtin((1000, 10000, 1024), "single") == "exact"
    assert V.builtin((1000, 7, 16), "single") == "exact"
    assert V.builtin((1000, 64, 256), "double") == "dmma"


def test_table_roundtrip_and_nearest_lookup(tmp_path):
    t = V.VariantTable()
    t.put((1_000_000, 512, 16), "single", "narrow", 5000.0, 5)
    t.put((1_000_000, 128, 1024), "single", "pair", 450000.0, 5)
    t.put((1_000_000, 64, 256), "double", "dfma", 12000.0, 5)
    p = tmp_path / "t.csv"
    t.save(str(p))
    assert p.read_text().startswith(V.HEADER)
    u = V.VariantTable.load(str(p))
    assert u.entries == t.entries
    # exact key
    assert u.lookup((1_000_000, 512, 16), np.float32) == "narrow"
    # nearest (D, K) whose family can run the shape
    assert u.lookup((1_000_000, 1024, 8), np.float32) == "narrow"
    assert u.lookup((1_000_000, 96, 900), np.float32) == "pair"
    # the nearest entry's family cannot run it: the next feasible one
    assert u.lookup((1_000_000, 1024, 1024), np.float32) == "pair"
    assert u.lookup((5, 64, 256), np.float64) == "dfma"


def test_table_rejects_bad_rows(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text(V.HEADER + "1024,64,256,single,dmma,1.0,5\n")
    with pytest.raises(ValueError):
        V.VariantTable.load(str(p))
    p.write_text(V.HEADER + "1024,64,256,single\n")
    with pytest.raises(ValueError):
        V.VariantTable.load(str(p))


def test_resolve_explicit_choice_wins():
    from paper_2408_01391_b200 import gemm

    old = gemm.get_variant()
    try:
        gemm.set_variant("exact")
        assert V.resolve((1000, 128, 1024), np.float32) == "exact"
        gemm.set_variant("auto")
        t = V.VariantTable()
        t.put((1000, 128, 254), "single", "narrow", 1.0, 1)
        V.set_table(t)
        assert V.resolve((1000, 128, 254), np.float32) == "narrow"
        # narrow cannot take k = 254 with the 4 checksum rows: the rule decides
        assert V.resolve((1000, 128, 254), np.float32, ft_on=True) == "pair"
        V.set_table(None)
        assert V.resolve((1000, 128, 254), np.float32) == "pair"
    finally:
        gemm.set_variant(old)
        V.set_table(None)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_every_family_gives_the_reference_bits(dt):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle as O

    from paper_2408_01391_b200 import _engine as E

    rng = np.random.default_rng(3)
    prec = V.precision_of(dt)
    for m, d, k in [(3000, 128, 60), (2000, 64, 250), (1500, 512, 16), (999, 32, 8),
                    (1200, 520, 700)]:
        x = np.ascontiguousarray(rng.standard_normal((m, d)), dtype=dt)
        y = np.ascontiguousarray(rng.standard_normal((k, d)), dtype=dt)
        lab, val = O.assign(x, y)
        x_t, y_t = E.to_dev(x), E.to_dev(y)
        yn = E.row_sq_norms_dev(y_t)
        for var in V.FAMILIES[prec]:
            if not V.feasible(var, (m, d, k), prec):
                with pytest.raises(ValueError):
                    E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant=var)
                continue
            idx, v = E.assign_dev(x_t, y_t, yn, (32, 256, 16), variant=var)
            assert np.array_equal(E.to_host(idx).astype(np.int64), lab), (var, m, d, k)
            assert E.to_host(v).tobytes() == val.tobytes(), (var, m, d, k)


@pytest.mark.gpu
def test_select_keeps_the_fastest():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    t = V.select([(50_000, 512, 16), (50_000, 64, 64)], "single", reps=2)
    for (mb, d, k, prec), e in t.entries.items():
        cands = {v: g for (mb2, d2, k2, p2, v), g in t.measured.items() if (d2, k2) == (d, k)}
        assert e.variant == max(cands, key=cands.get)
        assert e.gflops == max(cands.values())
    assert set(c[4] for c in t.measured if c[1] == 512) == {"pair", "narrow", "exact"}
