"""B200-native inner Newton step of the PBM solver for the dual VTS problem.

Drop-in for the reference package's PBM path (`vtsopt.pbm` and what it calls,
SURVEY.md §8): same call signatures, CUDA fp64 tensors instead of numpy
arrays, and every array operation a hand-written sm_100a kernel behind the
C ABI of `include/vts_b200.h` (built in-tree as `_build/libvts_b200.so`).
"""

from .problem import CONFIGS, MeshLevel, Problem, StructuredTransfer, build_config, build_problem
from .fem import DensityBounds, ElementOps, quad_stiffness
from .penalty import PenaltyBarrier
from .linalg import (
    ComplementarityTolerance,
    FixedTolerance,
    MinresConfig,
    MinresError,
    MinresResult,
    NewtonMatrix,
    StagnationTolerance,
    StiffnessMatrix,
    minres_solve,
)
from .multigrid import MgPreconditioner
from .pbm import (
    HessianBlocks,
    LagrangianEval,
    NewtonOutcome,
    PbmConfig,
    PbmState,
    SolveReport,
    al_value,
    eval_lagrangian,
    newton_inner,
    reconstruct_nu,
    schur_system,
    solve_pbm,
)
from .doc import DocConfig, bisect_volume, doc_update, solve_doc

__version__ = "0.1.0"

__all__ = [
    "CONFIGS",
    "MeshLevel",
    "Problem",
    "StructuredTransfer",
    "build_config",
    "build_problem",
    "DensityBounds",
    "ElementOps",
    "quad_stiffness",
    "PenaltyBarrier",
    "MinresConfig",
    "MinresError",
    "MinresResult",
    "NewtonMatrix",
    "StiffnessMatrix",
    "FixedTolerance",
    "ComplementarityTolerance",
    "StagnationTolerance",
    "minres_solve",
    "MgPreconditioner",
    "HessianBlocks",
    "LagrangianEval",
    "NewtonOutcome",
    "PbmConfig",
    "PbmState",
    "SolveReport",
    "al_value",
    "eval_lagrangian",
    "newton_inner",
    "reconstruct_nu",
    "schur_system",
    "solve_pbm",
    "DocConfig",
    "doc_update",
    "bisect_volume",
    "solve_doc",
]
