#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/chunk
for r in 1 2; do
  timeout 120 python tools/checks/quick_time.py ch128 >> gpurun_out/chunk/times.jsonl 2>> gpurun_out/chunk/err.log
  VTS_LIB=$PWD/_ab/lib_ch64.so VTS_OVL_BLOCKS=16,16,6,2 timeout 120 python tools/checks/quick_time.py ch64 >> gpurun_out/chunk/times.jsonl 2>> gpurun_out/chunk/err.log
  VTS_LIB=$PWD/_ab/lib_ch64.so timeout 120 python tools/checks/quick_time.py ch64dflt >> gpurun_out/chunk/times.jsonl 2>> gpurun_out/chunk/err.log
  VTS_LIB=$PWD/_ab/lib_ch32.so VTS_OVL_BLOCKS=16,16,6,2 timeout 120 python tools/checks/quick_time.py ch32 >> gpurun_out/chunk/times.jsonl 2>> gpurun_out/chunk/err.log
done
