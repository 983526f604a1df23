#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/items
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -o gs_probe_tl gs_probe.cu -lcuda > ../../gpurun_out/items/build.log 2>&1; cd ../..
timeout 200 ./tools/probe/gs_probe_tl 9 > gpurun_out/items/timeline.txt 2>&1
