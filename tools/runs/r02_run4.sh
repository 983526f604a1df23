#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "4 2 2" "8 4 2" "4 2 4" "4 2 6"; do timeout 300 python tools/checks/diag_smooth.py $cfg >> gpurun_out/diag_smooth.log 2>&1; done
