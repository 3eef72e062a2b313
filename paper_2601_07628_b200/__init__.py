"""paper_2601_07628_b200 — B200-native distributed PDHG LP solver (gridlp drop-in).

Hot path: FP64 CSR products A·x̄ / Aᵀ·y over a 2D grid partition of A fused
with the restarted-Halpern PDHG update and the KKT / restart reductions, as
hand-written sm_100a kernels (libgridlp_b200.so, include/gridlp_b200.h).
Public API mirrors the reference package `gridlp`
(/root/reference/pkg/src/gridlp/__init__.py:6-71) for that path.
"""

from .api import (
    KktReport,
    SolveResult,
    SolverConfig,
    StepSizes,
    reference_solve,
    solve,
    warmup,
)
from .comm import CollectiveError, CollectiveMismatch, CollectiveTimeout, WorkerError
from .generators import GeneratorSpec, box_lp_optimum, generate
from .layout import (
    GridTopology,
    PartitionLayout,
    Permutation,
    block_random_permutation,
    build_layout,
    layout_summary,
    nnz_balanced_cuts,
    select_grid,
    uniform_cuts,
    unpermute_solution,
)
from .mps import MpsParseError, load_mps, parse_mps, write_mps
from .problem import LpProblem, SparseMatrix, objective_value, reported_objective

__version__ = "0.1.0"

__all__ = [
    "CollectiveError", "CollectiveMismatch", "CollectiveTimeout", "WorkerError",
    "GeneratorSpec", "GridTopology", "KktReport", "LpProblem", "MpsParseError", "PartitionLayout",
    "Permutation", "SolveResult", "SolverConfig", "SparseMatrix", "StepSizes",
    "block_random_permutation", "box_lp_optimum", "build_layout", "generate",
    "layout_summary", "load_mps", "nnz_balanced_cuts", "objective_value", "parse_mps", "reference_solve",
    "reported_objective", "select_grid", "solve", "uniform_cuts", "unpermute_solution", "warmup", "write_mps",
]
