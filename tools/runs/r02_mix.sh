#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/mix
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_1904_06556_b200 as vts
p = vts.build_config(sys.argv[1]); rep = vts.solve_pbm(p); torch.cuda.synchronize(); print(rep.outer_iterations if hasattr(rep, "outer_iterations") else rep)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/c1.csv python /tmp/one.py C1 > gpurun_out/mix/c1.log 2>&1
python tools/checks/kernel_mix.py /tmp/c1.csv > gpurun_out/mix/c1_mix.txt 2>&1
