#!/bin/bash
# streamed band handoff: quick timing A/B first (bounded), then determinism/parity tests, probe timeline
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/stream1
timeout 120 python tools/checks/quick_time.py stream > gpurun_out/stream1/times.jsonl 2> gpurun_out/stream1/err.log; echo "quick rc=$?" >> gpurun_out/stream1/status.txt
VTS_LIB=$PWD/_ab/libnostream.so timeout 120 python tools/checks/quick_time.py nostream >> gpurun_out/stream1/times.jsonl 2>> gpurun_out/stream1/err.log
timeout 120 python tools/checks/quick_time.py stream >> gpurun_out/stream1/times.jsonl 2>> gpurun_out/stream1/err.log
VTS_LIB=$PWD/_ab/libnostream.so timeout 120 python tools/checks/quick_time.py nostream >> gpurun_out/stream1/times.jsonl 2>> gpurun_out/stream1/err.log
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py tests/test_gpu_parity.py tests/test_gpu_target.py -x -q -p no:cacheprovider > gpurun_out/stream1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/stream1/status.txt
cd tools/probe && timeout 200 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_GS_PROBE -o gs_probe_t gs_probe.cu -lcuda > ../../gpurun_out/stream1/build.log 2>&1; cd ../..
timeout 120 ./tools/probe/gs_probe_t 9 > gpurun_out/stream1/bands.txt 2>&1
