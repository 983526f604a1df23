#!/bin/bash
# session-5 start: current V-cycle timeline + a quick bench on the restored tree
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/s5tl
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../gpurun_out/s5tl/build.log 2>&1; cd ../..
timeout 200 ./tools/probe/gs_probe_tl 9 > gpurun_out/s5tl/timeline.txt 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/s5tl/bench.json 2> gpurun_out/s5tl/bench.err
head -c 400 gpurun_out/s5tl/bench.json; tail -40 gpurun_out/s5tl/timeline.txt
