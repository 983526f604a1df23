#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/stream4
for v in ps40 ps200; do
  VTS_LIB=$PWD/_ab/lib_$v.so timeout 120 python tools/checks/quick_time.py $v >> gpurun_out/stream4/times.jsonl 2>> gpurun_out/stream4/err.log
done
