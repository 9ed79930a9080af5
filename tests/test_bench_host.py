"""bench.py's host-side pieces without a GPU: the stratified sample, the
reference arm's per-step samples, the roofline bound choice, and the parity
leg's comparison logic (the GPU outputs stood in for by the oracle's, which
are bit-identical to the reference's on these inputs; one field is then
corrupted to check that a mismatch is counted and named)."""

import os

import numpy as np
import pytest
import torch

import bench
from conftest import ROOT


def test_stratified_rows():
    idx = bench.stratified_rows(1000, 7)
    assert len(idx) == 7 and idx[0] == 0 and np.all(np.diff(idx) > 100) and idx[-1] < 1000
    assert list(bench.stratified_rows(5, 10)) == [0, 1, 2, 3, 4]
    assert np.array_equal(bench.stratified_rows(1000, 7, 3), idx + 3)


def test_reference_arm_samples_shift_per_step():
    s = bench.reference_arm_samples("c4", 4096, 5, 3)
    assert len(s) == 3 and all(len(step) == 1 for step in s)
    u = [step[0][3].u0 for step in s]
    (pid, n, alg, b), = bench.jobs_for("c4", 0, 4096)
    for k in range(3):
        assert np.array_equal(u[k], b.u0[bench.stratified_rows(4096, 5, k)])


def test_rank_rows():
    assert bench.rank_rows(10, None, 4, 2) == (20, 30)
    parts = [bench.rank_rows(0, 10, 4, r) for r in range(4)]
    assert parts == [(0, 3), (3, 6), (6, 8), (8, 10)]


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "nlkit")),
                    reason="reference not installed in oracle/_ref")
def test_parity_leg_counts_mismatches():
    from oracle import oracle as O
    prepared = []
    for idx in (5, 22):
        from paper_2403_16341_b200 import workloads as W
        b = W.c2_suite(idx, 0, 64, 0.1)
        alg = "newton-raphson"
        r = O.solve_batch(b.problem_id, alg, b.u0)
        out = {"u": torch.from_numpy(r["u"].T.copy()), "resid": torch.from_numpy(r["resid"]),
               "retcode": torch.from_numpy(r["retcode"]),
               "counters": torch.from_numpy(np.stack([r["nsteps"], r["nf"], r["njac"],
                                                      r["nlinsolve"]]))}
        prepared.append((b.problem_id, b.n, 0, alg, 0, out["u"], None, out, b))
    cb, parity = bench.cpu_baseline_and_parity(prepared, 8)
    assert parity["systems"] == 16 and parity["mismatches"] == 0, parity
    assert cb["kind"] == "reference" and cb["value"] > 0
    assert parity["host"]["cores"] >= 1 and "glibc" in parity["host"]
    prepared[1][7]["counters"][1, 0] += 1  # nf of system 0 of the boggs job
    _cb, parity = bench.cpu_baseline_and_parity(prepared, 8)
    assert parity["mismatches"] == 1 and parity["mismatches_by_field"]["nf"] == 1
    assert parity["examples"][0]["problem"] == "test23/boggs"
