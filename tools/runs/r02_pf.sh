#!/bin/bash
# L2 prefetch in the overlap passes: A/B (alternating) + bitwise check
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/pf
for rep in 1 2 3; do
  timeout 300 python tools/checks/quick_time.py pf >> gpurun_out/pf/times.jsonl 2>> gpurun_out/pf/err.log
  VTS_LIB=$PWD/_ab/libnopf.so timeout 300 python tools/checks/quick_time.py nopf >> gpurun_out/pf/times.jsonl 2>> gpurun_out/pf/err.log
done
