#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/div3
for r in 1 2 3; do
  timeout 120 python tools/checks/quick_time.py div6 >> gpurun_out/div3/times.jsonl 2>> gpurun_out/div3/err.log
  VTS_DOVL_DIV=8 timeout 120 python tools/checks/quick_time.py div8 >> gpurun_out/div3/times.jsonl 2>> gpurun_out/div3/err.log
done
timeout 600 python -m pytest tests/test_gpu_properties.py tests/test_gpu_determinism.py -x -q -p no:cacheprovider > gpurun_out/div3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/div3/pytest.log
