#!/bin/bash
# Newton-apply: acq_rel last-block reduce vs split y_alpha kernel, cold/warm timing on C3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/apply2
for v in tile 8x2 16x1 8x1; do
  for sp in 0 1; do
    if [ $v = tile ]; then export VTS_APPLY_KERNEL=tile; else unset VTS_APPLY_KERNEL; export VTS_APPLY_WK=$v; fi
    export VTS_APPLY_SPLIT=$sp
    timeout 300 python tools/checks/apply_ab.py ${v}_s$sp /tmp >> gpurun_out/apply2/times.jsonl 2>> gpurun_out/apply2/err.log
  done
done
