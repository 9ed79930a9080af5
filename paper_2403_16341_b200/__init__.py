"""B200-native batched Simple* nonlinear solvers — a drop-in for nlkit's solve path.

The public surface mirrors the reference package ``nlkit``
(/root/reference/pkg/src/nlkit/__init__.py:3-17): ``Problem``,
``SolveOptions``, ``SolveResult``, ``Stats``, ``RetCode``, ``solve``,
``run_preset``, ``ALGORITHM_PRESETS`` ..., plus the paper's names
(``NonlinearProblem``, ``SimpleNewtonRaphson``, ``SimpleTrustRegion``,
``SimpleBroyden``, ``SimpleKlement``, ``SimpleDFSane``) and the batched entry
point ``solve_batch``.  All solving happens in the CUDA library
``libnlk_b200.so`` (include/nlk_b200.h); importing this package does not load
it, the first solve does, and fails loudly if it is missing.
"""

from .core import (NonlinearProblem, Problem, RetCode, SolveOptions, SolveResult, Stats,
                   check_convergence, result_to_json)
from .errors import NlkitError, NonFiniteValue, SingularMatrix
from .problems import DeviceResidual, get_problem
from .sensitivity import (SensitivityResult, ift_adjoint, ift_adjoint_batch, ift_forward,
                          ift_forward_batch)
from .solvers import (ALGORITHM_PRESETS, AlgorithmSpec, BatchResult, SimpleBroyden,
                      SimpleDFSane, SimpleKlement, SimpleNewtonRaphson, SimpleTrustRegion,
                      list_algorithms, run_algorithm, run_polyalgorithm, run_preset, solve,
                      solve_batch, solve_batch_soa)

__all__ = [
    "Problem", "NonlinearProblem", "RetCode", "SolveOptions", "SolveResult", "Stats",
    "check_convergence", "result_to_json", "solve", "run_preset", "run_algorithm",
    "run_polyalgorithm", "list_algorithms", "ALGORITHM_PRESETS", "AlgorithmSpec",
    "SimpleNewtonRaphson", "SimpleTrustRegion", "SimpleBroyden", "SimpleKlement",
    "SimpleDFSane", "solve_batch", "solve_batch_soa", "BatchResult", "DeviceResidual",
    "get_problem", "ift_forward", "ift_adjoint", "ift_forward_batch", "ift_adjoint_batch",
    "SensitivityResult", "NlkitError", "NonFiniteValue", "SingularMatrix",
]

__version__ = "0.1.0"
