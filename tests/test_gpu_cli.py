"""`cli wp` on the GPU against the reference CLI's own CSV
(tests/golden/wp_ref.csv from make_golden_cli.py): every column but
runtime_ns identical, per-solve (batch 1) and batched (one launch of 256
copies per cell).  Plus the reference's solve/scaling CLI tests."""

import csv
import io
import json
import os

import pytest

from paper_2403_16341_b200 import cli

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(__file__), "golden", "wp_ref.csv")
GRID = ["--problems", "quadratic,test23/rosenbrock,test23/wood,test23/helical-valley,"
        "test23/trigonometric,test23/boggs,generalized_rosenbrock?N=10",
        "--algorithms", "newton-raphson,trust-region,broyden,klement,newton-backtracking",
        "--tols", "1e-2..1e-10"]


def _strip(rows):
    return [{k: v for k, v in r.items() if k != "runtime_ns"} for r in rows]


@pytest.mark.parametrize("batch", [1, 256])
def test_wp_matches_reference_csv(tmp_path, batch):
    out = tmp_path / "wp.csv"
    assert cli.main(["wp", *GRID, "--reps", "1", "--batch", str(batch), "--out", str(out)]) == 0
    ours = list(csv.DictReader(open(out)))
    ref = list(csv.DictReader(open(REF)))
    assert open(out).readline() == open(REF).readline()
    assert _strip(ours) == _strip(ref)
    assert all(int(r["runtime_ns"]) > 0 for r in ours)


def test_solve_json(capsys):  # test_cli.py:21-36
    assert cli.main(["solve", "quadratic", "newton-raphson"]) == 0
    payload = json.loads(capsys.readouterr().out)
    assert payload["retcode"] == "Success" and payload["resid_inf_measured"] <= 1e-8
    assert cli.main(["solve", "generalized_rosenbrock?N=10", "newton-raphson"]) == 1
    assert json.loads(capsys.readouterr().out)["retcode"] != "Success"


def test_scaling_csv(tmp_path):  # test_cli.py:103-115
    out = tmp_path / "scaling.csv"
    assert cli.main(["scaling", "--family", "generalized_rosenbrock", "--sizes", "4,8",
                     "--algorithms", "trust-region,newton-backtracking", "--batch", "64",
                     "--out", str(out)]) == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert out.read_text().splitlines()[0] == "size,algorithm,runtime_ns,resid_inf,retcode"
    assert len(rows) == 4
