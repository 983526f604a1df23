#!/bin/bash
# V-cycle / C4 parity diagnostics at the target size
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/checks/diag_vcycle_levels.py > gpurun_out/diag_levels.log 2>&1
for v in VTS_NO_OVERLAP VTS_NO_PAIR VTS_UNFUSED_BOTTOM VTS_DENSE_APPLY; do
  echo "== $v=1" >> gpurun_out/diag_levels_env.log
  env $v=1 timeout 300 python tools/checks/diag_vcycle_levels.py --quick 2>&1 | tail -2 >> gpurun_out/diag_levels_env.log
done
timeout 300 python tools/checks/c4_rho_dump.py > gpurun_out/c4_dump.log 2>&1
