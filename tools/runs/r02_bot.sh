#!/bin/bash
# time marks of the fused V-cycle bottom (C3 hierarchy)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/bot
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_BOT_PROBE -o gs_probe_bot gs_probe.cu -lcuda > ../../gpurun_out/bot/build.log 2>&1; cd ../..
VTS_DET_REPS=2 timeout 200 ./tools/probe/gs_probe_bot 9 > gpurun_out/bot/c3.txt 2>&1
grep bottom gpurun_out/bot/c3.txt
