"""B200-native MERIT transform operator (arXiv 1911.03458 hot path).

The product is the C-ABI library ``libmerit_dev.so`` (include/merit_dev.h)
with four sm_100a kernels; this package is its Python mirror of the
reference's operator API (``merit.py``) plus the workload templates and the
BASELINE configurations (``workloads.py``).
"""
from .merit import (AluInstr, Boundary, Dst, Dtype, Error, ErrorCode, Kernel, LookupTable, Op,
                    Operand, Plan, PlanGroup, StrategyProgram, ViewSpec, ViewTerm, Workload, run_full,
                    run_full_argmin, run_full_many, run_tiled, FLAG_ARGMIN, FLAG_EXACT, FLAG_FAST_BF16, FLAG_NO_MAP)
from . import workloads

__all__ = ["AluInstr", "Boundary", "Dst", "Dtype", "Error", "ErrorCode", "Kernel", "LookupTable",
           "Op", "Operand", "Plan", "PlanGroup", "StrategyProgram", "ViewSpec", "ViewTerm", "Workload",
           "run_full", "run_full_argmin", "run_full_many", "run_tiled", "workloads", "FLAG_ARGMIN", "FLAG_EXACT",
           "FLAG_FAST_BF16", "FLAG_NO_MAP"]
