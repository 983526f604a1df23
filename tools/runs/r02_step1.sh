#!/bin/bash
# device-resident Newton step: conditional-graph probe, bitwise tests vs the host path, timings
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/step1
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -p no:cacheprovider > gpurun_out/step1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/step1/pytest.log
for k in C1 C2 C4; do
  VTS_HOST_NEWTON=1 timeout 600 python tools/checks/run_config.py $k 2>&1 | head -3 > gpurun_out/step1/host_$k.txt
  timeout 600 python tools/checks/run_config.py $k 2>&1 | head -3 > gpurun_out/step1/dev_$k.txt
done
