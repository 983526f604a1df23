#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/checks/diag_smooth.py 4 2 9 > gpurun_out/diag_smooth9.log 2>&1
VTS_NO_PAIR=1 timeout 600 python tools/checks/diag_smooth.py 4 2 9 > gpurun_out/diag_smooth9_nopair.log 2>&1
