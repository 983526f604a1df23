#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/pub
for r in 1 2 3; do timeout 120 python tools/checks/quick_time.py pubfold >> gpurun_out/pub/times.jsonl 2>> gpurun_out/pub/err.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_step.py tests/test_gpu_doc.py -x -q -p no:cacheprovider > gpurun_out/pub/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pub/pytest.log
