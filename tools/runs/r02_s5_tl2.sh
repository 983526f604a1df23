#!/bin/bash
# per-band waits of the overlapped ascent pairs (finest and L7), default clusters and cap 4
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5tl2; mkdir -p $O
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../$O/build.log 2>&1; cd ../..
VTS_DET_REPS=2 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | sed -n '/timeline rep 1/,$p' > $O/tl_cs16_L8.txt
VTS_DET_REPS=2 VTS_PAIR_CS_ASC=4,4,4,4,4 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | sed -n '/timeline rep 1/,$p' > $O/tl_cs4_L8.txt
VTS_DET_REPS=2 VTS_PROBE_LEVEL=7 VTS_PAIR_CS_ASC=4,4,4,4,4 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | sed -n '/timeline rep 1/,$p' > $O/tl_cs4_L7.txt
VTS_DET_REPS=2 VTS_PROBE_LEVEL=6 VTS_PAIR_CS_ASC=4,4,4,4,4 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | sed -n '/timeline rep 1/,$p' > $O/tl_cs4_L6.txt
