"""Single-process sharding of one host batch over several GPUs
(sharding.solve_batch_devices): contiguous slices, one asynchronous
host-buffer call per device, results written straight to host memory.  On a
one-GPU box the same device is listed several times, which exercises the
split and the reassembly; every field must equal the one-call solve."""

import numpy as np
import pytest
import torch

from paper_2403_16341_b200 import sharding, solvers, workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices", [[0], [0, 0, 0], [0] * 7])
@pytest.mark.parametrize("case", ["trig-tr", "quadratic-nr", "rosenbrock16-klement"])
def test_sharded_equals_single_call(devices, case):
    if case == "trig-tr":
        b, alg = W.c2_suite(11, 0, 20011, 0.1), "trust-region"
    elif case == "quadratic-nr":
        b, alg = W.c1_quadratic(0, 30001), "newton-raphson"
    else:
        b, alg = W.c3_rosenbrock(16, 0, 25013), "klement"
    ref = solvers.solve_batch(b.problem_id, b.u0, b.p, alg, n=b.n).to_numpy()
    got = sharding.solve_batch_devices(b.problem_id, b.u0, b.p, alg, devices=devices, n=b.n)
    for k in sharding.FIELDS:
        a, r = np.asarray(got[k]), np.asarray(ref[k])
        if a.dtype.kind == "f":
            assert np.array_equal(a.view(np.int64), r.view(np.int64)), k
        else:
            assert np.array_equal(a, r), k


def test_sharded_devices_default_and_empty():
    b = W.c1_quadratic(0, 1000)
    got = sharding.solve_batch_devices(b.problem_id, b.u0, b.p, "newton-raphson", n=b.n)
    assert got["u"].shape == (1000, 2) and (got["retcode"] == 0).all()
    with pytest.raises(ValueError):
        sharding.solve_batch_devices(b.problem_id, b.u0, b.p, "newton-raphson", devices=[], n=b.n)


def test_sharded_c4_full_size():
    """C4 as BASELINE.json states it: 10 M broyden-tridiagonal n = 16 systems,
    SimpleDFSane, sharded over a device list (here the one GPU listed 4 and 8
    times: the split and reassembly of the 2/4/8-GPU runs); every field of
    every system equals the one-call solve."""
    b = W.c4_tridiagonal(0, 10_000_000)
    ref = solvers.solve_batch(b.problem_id, b.u0, None, "dfsane", n=16).to_numpy()
    for devices in ([0] * 4, [0] * 8):
        got = sharding.solve_batch_devices(b.problem_id, b.u0, None, "dfsane", devices=devices, n=16)
        for k in sharding.FIELDS:
            a, r = np.asarray(got[k]), np.asarray(ref[k])
            if a.dtype.kind == "f":
                assert np.array_equal(a.view(np.int64), r.view(np.int64)), k
            else:
                assert np.array_equal(a, r), k
        del got
