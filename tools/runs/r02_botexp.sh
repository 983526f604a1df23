#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/botexp
cd tools/probe
for e in 0 1 2; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_BOT_PROBE -DVTS_BOT_EXP=$e -o gs_probe_bot$e gs_probe.cu -lcuda > ../../gpurun_out/botexp/build$e.log 2>&1
VTS_DET_REPS=2 timeout 200 ./gs_probe_bot$e 3 16 > ../../gpurun_out/botexp/probe$e.txt 2>&1
done
