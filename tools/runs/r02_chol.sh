#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/chol
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_step.py -x -q -p no:cacheprovider > gpurun_out/chol/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chol/pytest.log
for k in C1 C2; do timeout 300 python tools/checks/profile_pbm.py $k 3 2>&1 | head -4 > gpurun_out/chol/pbm_$k.txt; done
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_1904_06556_b200 as vts
p = vts.build_config(sys.argv[1]); rep = vts.solve_pbm(p); torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/c1.csv python /tmp/one.py C1 > gpurun_out/chol/c1.log 2>&1
python tools/checks/kernel_mix.py /tmp/c1.csv > gpurun_out/chol/c1_mix.txt 2>&1
