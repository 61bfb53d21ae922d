"""B200-native DOPE hot path (arXiv 1704.03116): block min cuts + consensus
ADMM on sm_100a, behind the reference package's API names
(/root/reference/pkg/src/dope/__init__.py:10-33, hot-path subset, plus the
step-level functions of admm.py / blockform.py / solvers.py).

Importing is cheap and works without a GPU; the first device call loads
libdope_b200.so and fails loudly if it (or the GPU) is missing.
"""
from .admm import (AdmmConfig, AdmmState, BlockProblems, BlockSolveError, TraceRecord,
                   assemble_block_problems, binarize, block_residuals, consensus_objective,
                   init_state, run, solve_global, update_blocks, update_global, update_multipliers)
from .blockform import BlockProblem, block_objective
from .energy import EnergyModel, NonSubmodularError, SparseWeights, evaluate_energy
from .grid import GridShape, coords_of, index_of
from .maxflow import FlowGraph, backend_name, bk_maxflow, build_graph, min_cut, solve_binary
from .partition import Block, Partition, make_partition, scatter_add, select
from .solvers import (EXHAUSTIVE, EXHAUSTIVE_MAX_VARS, ICM, MAXFLOW, BlockSolverKind,
                      exhaustive_minimize, pairwise_energy, solve_block)

__version__ = "0.2.0"

__all__ = [
    "AdmmConfig", "AdmmState", "Block", "BlockProblem", "BlockProblems", "BlockSolveError",
    "BlockSolverKind", "EXHAUSTIVE", "EXHAUSTIVE_MAX_VARS", "EnergyModel", "FlowGraph", "GridShape",
    "ICM", "MAXFLOW", "NonSubmodularError", "Partition", "SparseWeights", "TraceRecord",
    "assemble_block_problems", "backend_name", "binarize", "bk_maxflow", "block_objective",
    "block_residuals", "build_graph", "consensus_objective", "coords_of", "evaluate_energy",
    "exhaustive_minimize", "index_of", "init_state", "make_partition", "min_cut", "pairwise_energy",
    "run", "scatter_add", "select", "solve_binary", "solve_block", "solve_global", "update_blocks",
    "update_global", "update_multipliers",
]
