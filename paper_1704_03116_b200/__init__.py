"""B200-native DOPE hot path (arXiv 1704.03116): block min cuts + consensus
ADMM on sm_100a, behind the reference package's API names
(/root/reference/pkg/src/dope/__init__.py:10-33, hot-path subset).

Importing is cheap and works without a GPU; the first device call loads
libdope_b200.so and fails loudly if it (or the GPU) is missing.
"""
from .admm import (EXHAUSTIVE, ICM, MAXFLOW, AdmmConfig, AdmmState, BlockProblems,
                   BlockSolveError, BlockSolverKind, TraceRecord, assemble_block_problems,
                   binarize, block_residuals, init_state, run, update_blocks, update_global,
                   update_multipliers)
from .energy import EnergyModel, NonSubmodularError, SparseWeights, evaluate_energy
from .grid import GridShape
from .maxflow import FlowGraph, backend_name, bk_maxflow, build_graph, min_cut, solve_binary
from .partition import Block, Partition, make_partition, scatter_add, select

__version__ = "0.1.0"

__all__ = [
    "AdmmConfig", "AdmmState", "Block", "BlockProblems", "BlockSolveError", "BlockSolverKind",
    "EXHAUSTIVE", "EnergyModel", "FlowGraph", "GridShape", "ICM", "MAXFLOW",
    "NonSubmodularError", "Partition", "SparseWeights", "TraceRecord",
    "assemble_block_problems", "backend_name", "binarize", "bk_maxflow", "block_residuals",
    "build_graph", "evaluate_energy", "init_state", "make_partition", "min_cut", "run",
    "scatter_add", "select", "solve_binary", "update_blocks", "update_global",
    "update_multipliers",
]
