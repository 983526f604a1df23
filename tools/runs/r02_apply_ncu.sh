#!/bin/bash
# ncu of the Newton-apply variants (tile vs register rows) on C3 + fp64 throughput probe
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/ncu
make -s -C tools/probe fp64_tput > /dev/null 2>&1 && ./tools/probe/fp64_tput > gpurun_out/ncu/fp64_tput.txt 2>&1
export VTS_APPLY_WK=16x1
python tools/checks/apply_ab.py p16 /tmp > gpurun_out/ncu/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:newton_apply -s 3 -c 1 -o gpurun_out/ncu/rows16x1 python tools/checks/apply_ab.py p16 /tmp > gpurun_out/ncu/ncu1.log 2>&1
export VTS_APPLY_KERNEL=tile
ncu --set full --clock-control none --import-source on -k regex:newton_apply -s 3 -c 1 -o gpurun_out/ncu/tile python tools/checks/apply_ab.py pt /tmp > gpurun_out/ncu/ncu2.log 2>&1
echo done
