#!/bin/bash
# V-cycle kernel timeline (probe build with -DVTS_TIMELINE -DVTS_GS_PROBE) + MINRES launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/tl
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../gpurun_out/tl/build.log 2>&1; cd ../..
timeout 300 ./tools/probe/gs_probe_tl 9 > gpurun_out/tl/timeline.txt 2>&1
timeout 300 python tools/checks/quick_time.py base > gpurun_out/tl/quick.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|vts" -s 2000 -c 120 --csv --log-file gpurun_out/tl/launches.csv python tools/checks/quick_time.py ncu > gpurun_out/tl/ncu.log 2>&1
