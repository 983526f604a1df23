#!/bin/bash
# MINRES it/s on C3 with each Newton-apply variant (quick_time)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/apply4
for rep in 1 2; do
VTS_APPLY_KERNEL=tile timeout 300 python tools/checks/quick_time.py tile >> gpurun_out/apply4/times.jsonl 2>> gpurun_out/apply4/err.log
VTS_APPLY_WK=16x1 timeout 300 python tools/checks/quick_time.py 16x1 >> gpurun_out/apply4/times.jsonl 2>> gpurun_out/apply4/err.log
VTS_APPLY_WK=16x1 VTS_APPLY_SPLIT=1 timeout 300 python tools/checks/quick_time.py 16x1s >> gpurun_out/apply4/times.jsonl 2>> gpurun_out/apply4/err.log
VTS_APPLY_WK=8x2 VTS_APPLY_SPLIT=1 timeout 300 python tools/checks/quick_time.py 8x2s >> gpurun_out/apply4/times.jsonl 2>> gpurun_out/apply4/err.log
done
