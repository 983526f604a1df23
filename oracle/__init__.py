"""CPU oracle for the PBM inner Newton step on structured 2D Q1 meshes.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_1904_06556_b200/`) imports this package; only `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs of
`bench.py` use it, and only as the checker or as the timed CPU baseline.

What it is: a plain numpy/scipy (+ one small C file for the sequential
Gauss-Seidel loops) restatement of the reference package `vtsopt`
(`/root/reference/pkg/src/vtsopt`) on the 2D bilinear-Q1 plane-stress
discretisation that every BASELINE.json configuration uses.  Each function
cites the reference file:line it restates.  The reference is 3D-only; the
2D pieces (mesh hierarchy, per-dof Dirichlet masks, quad stiffness,
element connectivity) follow SURVEY.md Appendix A.

How it is pinned: `tests/golden/make_golden.py` imports the *unmodified*
reference solver modules (`pbm`, `linalg`, `multigrid`, `penalty`, `model`)
in this container, plugs in the 2D discretisation of `oracle.mesh2d` /
`oracle.fem2d` (the only new code on that side), and writes seeded
input/output fixtures to `tests/golden/`.  `tests/test_oracle_golden.py`
checks this restatement against those fixtures (and against the survey's
recorded C1/C2 run records) on every CPU test run.
"""

from .mesh2d import CONFIGS, Level2D, Problem2D, build_config, build_problem2d
from .fem2d import DensityBounds, ElementOps2D, quad_stiffness
from .phi import PenaltyBarrier
from .krylov import (
    BorderedMatrix,
    MinresConfig,
    MinresError,
    MinresResult,
    StagnationTolerance,
    minres_solve,
)
from .vcycle import MgPreconditioner
from .newton import (
    LagrangianEval,
    NewtonOutcome,
    PbmConfig,
    PbmState,
    SolveReport,
    compliance,
    dual_objective,
    duality_gap,
    eval_lagrangian,
    al_value,
    newton_inner,
    reconstruct_nu,
    schur_system,
    solve_pbm,
)

__all__ = [
    "CONFIGS",
    "Level2D",
    "Problem2D",
    "build_config",
    "build_problem2d",
    "DensityBounds",
    "ElementOps2D",
    "quad_stiffness",
    "PenaltyBarrier",
    "BorderedMatrix",
    "MinresConfig",
    "MinresError",
    "MinresResult",
    "StagnationTolerance",
    "minres_solve",
    "MgPreconditioner",
    "LagrangianEval",
    "NewtonOutcome",
    "PbmConfig",
    "PbmState",
    "SolveReport",
    "compliance",
    "dual_objective",
    "duality_gap",
    "eval_lagrangian",
    "al_value",
    "newton_inner",
    "reconstruct_nu",
    "schur_system",
    "solve_pbm",
]
