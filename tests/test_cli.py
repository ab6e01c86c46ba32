"""The ``generate`` / ``cluster`` CLI (reference cli.py:44-151, 343-418) and the
ftkm-binary -> pinned-host loader, against RunReports of the reference CLI
(tests/golden/cli_cases.json, written by make_golden.cli_cases)."""

import csv
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

cli = pytest.importorskip("paper_2408_01391_b200.cli")
from paper_2408_01391_b200 import matrix as M  # noqa: E402
from paper_2408_01391_b200.errors import FormatError  # noqa: E402

CASES = json.load(open(os.path.join(GOLDEN, "cli_cases.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_generate_matches_reference_file(name, tmp_path):
    case = CASES[name]
    out = tmp_path / "x.ftkm"
    assert cli.main(["generate", *case["generate"], "--out", str(out)]) == 0
    assert hashlib.sha256(out.read_bytes()).hexdigest() == case["file_sha256"]


def test_pinned_loader_matches_mat_load(tmp_path):
    for prec in ("single", "double"):
        x = M.mat_random(333, 7, prec, seed=11)
        p = tmp_path / f"{prec}.ftkm"
        M.mat_store(x, str(p))
        y = M.mat_load_pinned(str(p))
        assert y.numpy().dtype == x.dtype and y.numpy().tobytes() == x.tobytes()
        assert M.mat_load(str(p)).tobytes() == x.tobytes()


def test_pinned_loader_errors(tmp_path):
    x = M.mat_random(20, 4, "single", seed=1)
    x[3, 2] = np.inf
    bad = tmp_path / "bad.ftkm"
    M.mat_store(x, str(bad))
    with pytest.raises(FormatError, match=r"non-finite value at \(4,3\)"):
        M.mat_load_pinned(str(bad))
    trunc = tmp_path / "trunc.ftkm"
    trunc.write_bytes(bad.read_bytes()[:-5])
    with pytest.raises(FormatError, match="truncated"):
        M.mat_load_pinned(str(trunc))
    junk = tmp_path / "junk.ftkm"
    junk.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(FormatError, match="not an ftkm-binary"):
        M.mat_load_pinned(str(junk))


def test_usage_errors_exit_2(tmp_path):
    assert cli.main(["bogus"]) == 2
    assert cli.main(["cluster", "--k", "3"]) == 2  # --input missing
    assert cli.main(["cluster", "--input", str(tmp_path / "none.ftkm"), "--k", "3"]) == 2
    junk = tmp_path / "junk.ftkm"
    junk.write_bytes(b"NOPE" + bytes(40))
    assert cli.main(["cluster", "--input", str(junk), "--k", "3"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_cluster_report_matches_reference(name, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    case = CASES[name]
    data = tmp_path / "x.ftkm"
    rep = tmp_path / "r.csv"
    labels = tmp_path / "l.txt"
    assert cli.main(["generate", *case["generate"], "--out", str(data)]) == 0
    code = cli.main(["cluster", "--input", str(data), *case["cluster"], "--report", str(rep),
                     "--labels-out", str(labels)])
    assert code == case["exit"]
    with open(rep) as fh:
        rows = [r for r in csv.reader(fh)][1:]
    keep = [r for r in rows if r[0] in ("result", "ft", "summary", "config")
            or (r[0] == "meta" and r[1] in ("precision", "rows", "cols", "schema_version"))]
    assert keep == case["rows"]
    lab = np.loadtxt(labels, dtype=np.int64)
    sha = [r[2] for r in keep if r[1] == "assignments_sha256"][0]
    assert hashlib.sha256(lab.tobytes()).hexdigest() == sha


@pytest.mark.parametrize("text,row,col", [
    ("1,2\nabc,3\n", 2, 1),          # bad cell: 1-based file position
    ("1,2\n\n3,inf\n", 3, 2),        # blank line still counts as a file line
    ("# c\n1,2\n", 1, 1),            # '#' is not a comment in the reference reader
    ("1,2\n3\n", 2, 1),              # ragged row: (line, its column count)
])
def test_csv_loader_error_positions(tmp_path, text, row, col):
    """mat_load(format="csv") reports the reference reader's positions
    (matrix.py:175-212): 1-based file lines and columns."""
    from paper_2408_01391_b200.errors import FormatError
    from paper_2408_01391_b200.matrix import mat_load

    p = tmp_path / "m.csv"
    p.write_text(text)
    with pytest.raises(FormatError) as ei:
        mat_load(str(p), format="csv")
    assert (ei.value.row, ei.value.col) == (row, col)


def test_csv_loader_values(tmp_path):
    from paper_2408_01391_b200.matrix import mat_load

    p = tmp_path / "m.csv"
    p.write_text("1, 2.5\n\n-3,4e-3\n")
    a = mat_load(str(p), format="csv", precision="single")
    assert a.dtype == np.float32 and a.tolist() == [[1.0, 2.5], [-3.0, np.float32(4e-3)]]
