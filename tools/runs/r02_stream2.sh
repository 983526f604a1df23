#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/stream2
timeout 120 python tools/checks/quick_time.py stream > gpurun_out/stream2/times.jsonl 2> gpurun_out/stream2/err.log; echo "quick rc=$?" >> gpurun_out/stream2/status.txt
cd tools/probe && timeout 200 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_GS_PROBE -o gs_probe_t gs_probe.cu -lcuda > ../../gpurun_out/stream2/build.log 2>&1; cd ../..
timeout 120 ./tools/probe/gs_probe_t 9 > gpurun_out/stream2/bands.txt 2>&1
