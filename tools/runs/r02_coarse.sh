#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/coarse
timeout 600 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/coarse/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/coarse/pytest.log
for k in C1 C2; do timeout 300 python tools/checks/profile_pbm.py $k 3 2>&1 | head -4 > gpurun_out/coarse/pbm_$k.txt; done
timeout 120 python tools/checks/quick_time.py c1 C1 > gpurun_out/coarse/quick_c1.json 2>&1
