"""B200-native superfast Tikhonov-Toeplitz solver.

Drop-in for the reference package's solve path (toepreg 0.1.0,
``toepreg.solve_tikhonov(problem, config) -> SolveReport``): same problem
containers and generator conventions, same report, computed by hand-written
sm_100a kernels in ``libtoepreg_b200.so`` behind a C ABI
(``include/toepreg_b200.h``).  There is no CPU fallback.
"""

from .toeplitz import (HermitianToeplitzSpec, ProblemSpec, ToeplitzSpec, adjoint_spec,
                       identity_spec, spec_from_json, spec_to_json, vector_from_json,
                       vector_to_json)
from .solver import (DeviceBatch, SingularSystemError, SolveReport, SolverConfig,
                     TanIntDiagnostics, plan_info, solve_tikhonov, solve_tikhonov_batch)
from .iterative import CGConfig, NormalOperator, apply_normal_operator, cg_solve, cg_solve_batch

__version__ = "0.1.0"

__all__ = [
    "ToeplitzSpec", "HermitianToeplitzSpec", "ProblemSpec", "identity_spec", "adjoint_spec",
    "SolverConfig", "SolveReport", "TanIntDiagnostics", "SingularSystemError",
    "solve_tikhonov", "solve_tikhonov_batch", "DeviceBatch", "plan_info", "__version__",
    "spec_to_json", "spec_from_json", "vector_to_json", "vector_from_json",
    "NormalOperator", "apply_normal_operator", "CGConfig", "cg_solve", "cg_solve_batch",
]
