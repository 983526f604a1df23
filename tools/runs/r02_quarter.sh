#!/bin/bash
# quarter-window band handoff: timing A/B first (bounded), then bitwise tests and the band timeline
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/quarter
for r in 1 2; do
  timeout 120 python tools/checks/quick_time.py quarter >> gpurun_out/quarter/times.jsonl 2>> gpurun_out/quarter/err.log; echo "q rc=$?" >> gpurun_out/quarter/status.txt
  VTS_LIB=$PWD/_ab/lib_noq.so timeout 120 python tools/checks/quick_time.py window >> gpurun_out/quarter/times.jsonl 2>> gpurun_out/quarter/err.log
done
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py tests/test_gpu_parity.py tests/test_gpu_target.py -x -q -p no:cacheprovider > gpurun_out/quarter/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/quarter/status.txt
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_GS_PROBE -o gs_probe_t gs_probe.cu -lcuda > ../../gpurun_out/quarter/build.log 2>&1; cd ../..
timeout 200 ./tools/probe/gs_probe_t 9 > gpurun_out/quarter/bands.txt 2>&1
