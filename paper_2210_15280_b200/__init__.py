"""B200-native (sm_100a) surrogate ILU(0) smoother for hybrid tetrahedral grids.

Drop-in for the hot path of arXiv 2210.15280's reference (``tetilu``): the
matrix-free ILU(0) smoothing sweep on refined macro-tetrahedra, with the factor
stencil weights evaluated on the fly from fitted polynomial surrogates.  Every sweep runs in
hand-written CUDA kernels behind the C ABI in include/tilu.h; the setup's factorization runs on
the CPU or the GPU (same rows bitwise), sampling and the least-squares fit on the CPU.  Around the
path: a GPU multigrid V-cycle on one macro-tet (``Hierarchy``), the Schur inner solve and the
interface stages of the hybrid multi-tet smoother (``HybridSmoother``).

Public names mirror the reference's (tetilu/__init__.py:4-18) where they exist.
"""

from .fitting import (EmptySampleSet, FactorizationResult, PivotBreakdown, RankDeficientFit,
                      SurrogatePolynomial, factorize_tet, factorize_tet_device, lsq_fit, nddf_row_evaluate,
                      sample_coords)
from .hybrid import HybridHierarchy, HybridSmoother, InterfaceStage
from .lattice import grid_size, interior_size, kuhn_mesh, rank_tables
from .multigrid import Hierarchy, InnerSolveError, schur_inner_solve
from .partition import MacroMeshSmoother, allreduce_norms, partition
from .smoother import (CellILU, DevicePlan, SmootherConfig, SurrogateILU, SurrogateILUSmoother,
                       build_surrogate_ilu)
from .stencil import CoefficientField, StencilSource, stencil_source

__all__ = [
    "build_surrogate_ilu", "SurrogateILU", "CellILU", "factorize_tet", "stencil_source",
    "CoefficientField", "StencilSource", "SmootherConfig", "nddf_row_evaluate", "lsq_fit",
    "sample_coords", "SurrogatePolynomial", "FactorizationResult", "RankDeficientFit",
    "EmptySampleSet", "PivotBreakdown", "SurrogateILUSmoother", "MacroMeshSmoother", "DevicePlan",
    "partition", "allreduce_norms", "grid_size", "interior_size", "rank_tables", "kuhn_mesh",
    "factorize_tet_device", "Hierarchy", "schur_inner_solve", "InnerSolveError", "HybridSmoother", "HybridHierarchy", "InterfaceStage",
]
