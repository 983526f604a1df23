#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/quarter3
for r in 1 2 3; do
  timeout 120 python tools/checks/quick_time.py descq >> gpurun_out/quarter3/times.jsonl 2>> gpurun_out/quarter3/err.log
  VTS_LIB=$PWD/_ab/lib_noq.so timeout 120 python tools/checks/quick_time.py window >> gpurun_out/quarter3/times.jsonl 2>> gpurun_out/quarter3/err.log
done
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/quarter3/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quarter3/pytest.log
