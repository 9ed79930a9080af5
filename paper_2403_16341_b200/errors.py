"""Exception types of the reference (nlkit/errors.py:4-49) that the batched
path can raise.  Per-system numerical failures of a batch are reported as
codes (retcodes, sensitivity status), never raised; the single-system
wrappers (`solve`, `ift_forward`, `ift_adjoint`) raise these like nlkit."""


class NlkitError(Exception):
    """Base class (errors.py:4-5)."""


class NonFiniteValue(NlkitError):
    """A residual, iterate, or derivative contained NaN or Inf (errors.py:8-9)."""


class SingularMatrix(NlkitError):
    """A direct factorization hit a pivot too small to trust (errors.py:12-13)."""


class IncompatibleSpec(NlkitError):
    """An algorithm specification combines incompatible blocks (errors.py:44-45)."""
