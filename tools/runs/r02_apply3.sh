#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/apply3
VTS_TIME_FLOOR=1 VTS_APPLY_WK=16x1 VTS_APPLY_SPLIT=1 timeout 300 python tools/checks/apply_ab.py f /tmp >> gpurun_out/apply3/times.jsonl 2>> gpurun_out/apply3/err.log
VTS_TIME_FLOOR=1 VTS_APPLY_KERNEL=tile timeout 300 python tools/checks/apply_ab.py ft /tmp >> gpurun_out/apply3/times.jsonl 2>> gpurun_out/apply3/err.log
