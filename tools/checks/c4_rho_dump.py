"""Run the C4 full PBM solve on the GPU and save rho / counts to gpurun_out/ (diagnostic)."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
import paper_1904_06556_b200 as vts  # noqa: E402

rep = vts.solve_pbm(vts.build_config(sys.argv[1] if len(sys.argv) > 1 else "C4"))
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(REPO, "gpurun_out", "c4_gpu.npz"), rho=rep.rho.cpu().numpy(),
                    minres_per_newton=np.array(rep.extras["minres_per_newton"]), objective=rep.objective,
                    rows=np.array(rep.rows, dtype=float))
print(rep.objective, rep.outer_iterations, rep.totals())
