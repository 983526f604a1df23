#!/bin/bash
# padding CTAs leave early: determinism/properties/parity + quick timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/check1
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/check1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check1/pytest.log
timeout 300 python tools/checks/quick_time.py pad >> gpurun_out/check1/times.jsonl 2>> gpurun_out/check1/err.log
timeout 600 python tools/checks/run_config.py C5 >> gpurun_out/check1/c5.txt 2>&1
