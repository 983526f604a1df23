#!/bin/bash
# end of round: C5 wall time, V-cycle timeline (instrumented build), step probe
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5final; mkdir -p $O
timeout 600 python tools/checks/run_config.py C5 > $O/c5.txt 2>&1
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../$O/build.log 2>&1
timeout 100 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -ffp-contract=off -o step_probe3 step_probe3.cu >> ../../$O/build.log 2>&1; cd ../..
VTS_DET_REPS=20 timeout 200 ./tools/probe/gs_probe_tl 9 > $O/tl.txt 2>&1
timeout 60 ./tools/probe/step_probe3 > $O/step_probe3.txt 2>&1
head -4 $O/c5.txt; grep -A 24 "timeline rep 1" $O/tl.txt; tail -2 $O/tl.txt
