#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/quarter2
for r in 1 2; do
  timeout 120 python tools/checks/quick_time.py desc >> gpurun_out/quarter2/times.jsonl 2>> gpurun_out/quarter2/err.log
  VTS_GS_QUARTERS=none timeout 120 python tools/checks/quick_time.py none >> gpurun_out/quarter2/times.jsonl 2>> gpurun_out/quarter2/err.log
  VTS_GS_QUARTERS=all timeout 120 python tools/checks/quick_time.py all >> gpurun_out/quarter2/times.jsonl 2>> gpurun_out/quarter2/err.log
done
