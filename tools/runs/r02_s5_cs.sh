#!/bin/bash
# ascent pairs: smaller clusters (GPC fragmentation) and A/B cluster interleave -- timing A/B + timelines
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5cs; mkdir -p $O
run() { # label, env...
  local label=$1; shift
  env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt
}
for r in 1 2; do
  run base VTS_PAIR_INTERLEAVE=0
  run il16 VTS_PAIR_INTERLEAVE=1
  run il6 VTS_PAIR_CS_ASC=6,6,6,6,6
  run il4 VTS_PAIR_CS_ASC=4,4,4,4,4
  run il3 VTS_PAIR_CS_ASC=3,3,3,3,3
  run il4top VTS_PAIR_CS_ASC=4
  run ni4 VTS_PAIR_INTERLEAVE=0 VTS_PAIR_CS_ASC=4,4,4,4,4
  run il4d6 VTS_PAIR_CS_ASC=4,4,4,4,4 VTS_PAIR_CS_DESC=0,5,5,5,5
done
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../$O/build.log 2>&1; cd ../..
VTS_PAIR_CS_ASC=4,4,4,4,4 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | grep -A 24 "timeline rep 1" > $O/timeline_il4.txt
VTS_PAIR_CS_ASC=3,3,3,3,3 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | grep -A 24 "timeline rep 1" > $O/timeline_il3.txt
cat $O/times.jsonl | cut -c1-260
