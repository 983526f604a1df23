#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/stream3
for v in arm1 arm2 nsa8 noarm; do
  VTS_LIB=$PWD/_ab/lib_$v.so timeout 120 python tools/checks/quick_time.py $v >> gpurun_out/stream3/times.jsonl 2>> gpurun_out/stream3/err.log
done
