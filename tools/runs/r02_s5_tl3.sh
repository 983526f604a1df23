#!/bin/bash
# band timelines of the single sweep and the standalone ascent pair, and the V-cycle timeline, after the half-warp change
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5tl3; mkdir -p $O
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../$O/build.log 2>&1; cd ../..
VTS_DET_REPS=2 timeout 200 ./tools/probe/gs_probe_tl 9 > $O/tl.txt 2>&1
grep -A3 "W 17" $O/tl.txt; grep "band 16\|band 32" $O/tl.txt | head; grep -A 24 "timeline rep 1" $O/tl.txt
