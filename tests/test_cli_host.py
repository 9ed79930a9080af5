"""CLI contract checks that need no GPU (reference: tests/test_cli.py)."""

import pytest

from paper_2403_16341_b200 import cli


def test_parse_tols_range_and_list():  # test_cli.py:53-59
    assert cli._parse_tols("1e-2..1e-4") == [1e-2, 1e-3, 1e-4]
    assert cli._parse_tols("1e-3,1e-6") == [1e-3, 1e-6]
    with pytest.raises(ValueError):
        cli._parse_tols("1e-6..1e-2")
    with pytest.raises(ValueError):
        cli._parse_tols("1e-6,1e-2")


def test_headers_match_reference():  # cli.py:33-35
    assert ",".join(cli.WP_HEADER) == "problem,algorithm,abstol,runtime_ns,resid_inf,retcode,nf,njac,nlinsolve"
    assert ",".join(cli.SCALING_HEADER) == "size,algorithm,runtime_ns,resid_inf,retcode"


def test_bench_config_validation():  # test_cli.py:152-156
    with pytest.raises(ValueError):
        cli.BenchConfig(("quadratic",), ("newton-raphson",), (1e-8, 1e-2))
    with pytest.raises(ValueError):
        cli.BenchConfig(("quadratic",), ("newton-raphson",), (1e-2,), reps=0)
    with pytest.raises(ValueError):
        cli.BenchConfig(("quadratic",), ("newton-raphson",), (1e-2,), batch=0)


def test_list_outputs(capsys):  # test_cli.py:137-149
    assert cli.main(["list", "problems"]) == 0
    out = capsys.readouterr().out
    assert "test23/rosenbrock" in out and "quadratic" in out
    assert cli.main(["list", "algorithms"]) == 0
    out = capsys.readouterr().out
    assert "newton-raphson" in out and "polyalgorithm" in out


def test_unknown_family_and_problem(capsys):  # test_cli.py:126-130, 46-50
    assert cli.main(["scaling", "--family", "bogus", "--sizes", "4",
                     "--algorithms", "newton-raphson"]) == 2
    assert cli.main(["solve", "nope", "newton-raphson"]) == 2
    assert "unknown" in capsys.readouterr().err


def test_reference_only_presets_are_not_ported(capsys):
    """A reference preset / problem with no batched kernel is reported as not
    ported (exit 3), not as unknown (exit 2); names match nlkit's presets."""
    import os
    import sys
    assert cli.main(["solve", "test23/rosenbrock", "levenberg-marquardt"]) == cli.EXIT_NOT_PORTED
    assert "not ported" in capsys.readouterr().err
    assert cli.main(["solve", "brusselator2d?N=8", "newton-raphson"]) == cli.EXIT_NOT_PORTED
    assert cli.main(["solve", "test23/rosenbrock", "no-such-preset"]) == 2
    src = os.environ.get("NLKIT_REF", "/root/reference/pkg/src")
    if os.path.isdir(src):
        sys.path.insert(0, src)
        from nlkit import solvers as ns
        from paper_2403_16341_b200 import solvers
        ref = set(ns.list_algorithms())
        ours = set(solvers.ALGORITHM_PRESETS) | {"polyalgorithm"}
        assert set(cli.REFERENCE_ONLY_PRESETS) == ref - ours - {"dfsane"}
