#!/bin/bash
# sweep B of the pairs offset by half a band: timing A/B first (bounded), then the bitwise tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/offset
for r in 1 2; do
  timeout 120 python tools/checks/quick_time.py offset >> gpurun_out/offset/times.jsonl 2>> gpurun_out/offset/err.log; echo "q rc=$?" >> gpurun_out/offset/status.txt
  VTS_PAIR_OFFSET=0 timeout 120 python tools/checks/quick_time.py aligned >> gpurun_out/offset/times.jsonl 2>> gpurun_out/offset/err.log
done
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py tests/test_gpu_parity.py tests/test_gpu_target.py -x -q -p no:cacheprovider > gpurun_out/offset/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/offset/status.txt
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../gpurun_out/offset/build.log 2>&1; cd ../..
timeout 200 ./tools/probe/gs_probe_tl 9 > gpurun_out/offset/timeline.txt 2>&1
