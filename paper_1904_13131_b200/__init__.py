"""B200-native matrix-free finite-strain hyperelasticity hot path (arXiv:1904.13131).

Drop-in for the reference ``hyperfree`` operator API on the GPU: the classes
and functions below mirror the reference names and semantics; all numerics
run in the sm_100a library ``libhf.so`` (include/hf.h) through ctypes.
"""

from .material import NeoHookeanParams, NonPositiveJacobian
from .mesh import MeshHierarchy, build_benchmark_mesh, refine_globally
from .operators import (STRATEGIES, AssembledTangent, Material, MatrixFreeTangent, Problem, build_problem_hierarchy,
                        compute_residual, energy, jacobian_range, make_tangent)
from .multigrid import (ChebyshevSettings, GMGPreconditioner, LevelOperator, TransferOperator, build_gmg,
                        build_level_operators, build_transfers, chebyshev_apply, coarse_solve,
                        estimate_eigenvalue_range, restrict_solution, v_cycle)
from .solver import (CGReport, IndefiniteOperator, LoadSpec, MaxNewtonIterations, NewtonSettings, cg,
                     newton_solve, newton_solve_prescribed)

__all__ = [
    "NeoHookeanParams", "NonPositiveJacobian", "MeshHierarchy", "build_benchmark_mesh", "refine_globally",
    "STRATEGIES", "AssembledTangent", "Material", "MatrixFreeTangent", "Problem", "build_problem_hierarchy", "compute_residual", "energy",
    "jacobian_range", "make_tangent", "ChebyshevSettings", "GMGPreconditioner", "LevelOperator", "TransferOperator",
    "build_gmg", "build_level_operators", "build_transfers", "chebyshev_apply", "coarse_solve",
    "estimate_eigenvalue_range", "restrict_solution", "v_cycle", "CGReport", "IndefiniteOperator", "LoadSpec",
    "MaxNewtonIterations", "NewtonSettings", "cg", "newton_solve", "newton_solve_prescribed",
]
