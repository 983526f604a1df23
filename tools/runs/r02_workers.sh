#!/bin/bash
# overlap pass block counts (prolongation / residual-restriction workers) after the padding change
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/workers
for ow in 8 12 16 24; do
  VTS_OVL_WORKERS=$ow timeout 300 python tools/checks/quick_time.py ow$ow >> gpurun_out/workers/times.jsonl 2>> gpurun_out/workers/err.log
done
for dw in 32 40 56 64; do
  VTS_DOVL_WORKERS=$dw timeout 300 python tools/checks/quick_time.py dw$dw >> gpurun_out/workers/times.jsonl 2>> gpurun_out/workers/err.log
done
