"""B200-native (sm_100a) surrogate ILU(0) smoother for hybrid tetrahedral grids.

Drop-in for the hot path of arXiv 2210.15280's reference (``tetilu``): the
matrix-free ILU(0) smoothing sweep on refined macro-tetrahedra, with the factor
stencil weights evaluated on the fly from fitted polynomial surrogates.  Host setup
(factorization, sampling, least-squares fit) runs on the CPU; every sweep runs in
hand-written CUDA kernels behind the C ABI in include/tilu.h.

Public names mirror the reference's (tetilu/__init__.py:4-18) where they exist.
"""

from .fitting import (EmptySampleSet, FactorizationResult, PivotBreakdown, RankDeficientFit,
                      SurrogatePolynomial, factorize_tet, lsq_fit, nddf_row_evaluate, sample_coords)
from .lattice import grid_size, interior_size, kuhn_mesh, rank_tables
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
]
