"""The divisions of paper_2403_16341_b200/csrc/nlk_div.cuh -- the
hoisted-reciprocal division (div_with_rcp), the zero-dividend shortcut
used on the solve path (ddiv) and the fast Newton kernels' flagged fast path
(FlagDiv, wherever it does not flag) -- are bit-identical to nvcc's `b / d` on 10^8
random operands (any bit pattern, moderate and extreme exponents, zeros,
subnormals, infinities, NaN)."""

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_hoisted_division_matches_ieee_division(tmp_path):
    src = os.path.join(ROOT, "tests", "cuda", "division_check.cu")
    exe = tmp_path / "division_check"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                    "-I", os.path.join(ROOT, "paper_2403_16341_b200", "csrc"), src, "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
