"""Golden work-precision CSV from the UNMODIFIED reference CLI (nlkit/cli.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cli.py

Writes tests/golden/wp_ref.csv: `nlkit wp` over a small grid, one rep.
Everything but runtime_ns is deterministic and is compared by
tests/test_gpu_cli.py against `paper_2403_16341_b200.cli wp`.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("NLKIT_REF", "/root/reference/pkg/src"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from nlkit import cli  # noqa: E402

ARGS = ["wp", "--problems", "quadratic,test23/rosenbrock,test23/wood,test23/helical-valley,"
        "test23/trigonometric,test23/boggs,generalized_rosenbrock?N=10",
        "--algorithms", "newton-raphson,trust-region,broyden,klement,newton-backtracking",
        "--tols", "1e-2..1e-10", "--reps", "1"]

if __name__ == "__main__":
    sys.exit(cli.main(ARGS + ["--out", os.path.join(HERE, "wp_ref.csv")]))
