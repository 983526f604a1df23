#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/seg
run() { env "$@" timeout 120 python tools/checks/quick_time.py "$*" >> gpurun_out/seg/times.jsonl 2>> gpurun_out/seg/err.log; }
for r in 1 2; do
  run VTS_KSEG=8
  run VTS_LIB=$PWD/_ab/lib_seg16.so
  run VTS_LIB=$PWD/_ab/lib_seg16.so VTS_DOVL_BLOCKS=48,36,20,12
  run VTS_LIB=$PWD/_ab/lib_seg12.so
  run VTS_LIB=$PWD/_ab/lib_seg12.so VTS_DOVL_BLOCKS=48,36,20,12
done
