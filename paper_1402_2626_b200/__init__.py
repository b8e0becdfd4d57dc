"""B200-native Gauss-Newton hot path for sparse polynomial systems in
complex/real double, double-double and quad-double arithmetic.

Drop-in for the hot path of the reference package ``polynewt``
(arxiv 1402.2626, Verschelde & Yu): the same names and signatures
(``evaluate_system``, ``least_squares_solve``, ``mgs_qr``, ``newton_step``,
``run_newton``, ...), executed by hand-written sm_100a CUDA kernels behind the
C ABI in ``include/polynewt_b200.h``.  There is no CPU fallback.
"""

from .xprec import (Complex, DomainError, DoubleDouble, PrecisionLevel, QuadDouble,
                    precision_level)
from .polyrep import (Monomial, PackedSystem, PolySystem, SystemParseError, decompose, parse_system,
                      serialize_system)
from .evaldiff import OpCounter, PreparedSystem, SystemEvaluation, evaluate_system
from .mgs import (AugmentedMatrix, LeastSquaresResult, MgsBreakdownError, QRFactors,
                  SingularMatrixError, TilingConfig, back_substitute, back_substitute_staged,
                  least_squares_solve, mgs_qr, mgs_qr_delayed)
from .newton import (IterationTrace, NewtonConfig, TraceEntry, convergence_ratio,
                     homotopy_start_system, inf_norm, newton_step, run_newton)
from .varith import VecContext, promote

__all__ = [
    "AugmentedMatrix", "Complex", "DomainError", "DoubleDouble", "IterationTrace",
    "LeastSquaresResult", "MgsBreakdownError", "Monomial", "NewtonConfig", "OpCounter",
    "PackedSystem", "PolySystem", "PrecisionLevel", "PreparedSystem", "QRFactors",
    "QuadDouble", "SingularMatrixError", "SystemEvaluation", "TilingConfig", "TraceEntry",
    "VecContext", "back_substitute", "back_substitute_staged", "convergence_ratio",
    "decompose", "evaluate_system", "homotopy_start_system", "inf_norm",
    "least_squares_solve", "mgs_qr", "mgs_qr_delayed", "newton_step", "parse_system", "precision_level",
    "promote", "run_newton", "serialize_system", "SystemParseError",
]

__version__ = "0.1.0"
