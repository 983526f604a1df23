#!/bin/bash
# items per block of the overlap passes: prolongation (VTS_OVL_DIV) and residual/restriction (VTS_DOVL_DIV)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/div
run() { env "$@" timeout 120 python tools/checks/quick_time.py "$*" >> gpurun_out/div/times.jsonl 2>> gpurun_out/div/err.log; }
run VTS_OVL_DIV=4
run VTS_OVL_DIV=8
run VTS_OVL_DIV=16
run VTS_OVL_DIV=12
run VTS_DOVL_DIV=12
run VTS_DOVL_DIV=16
run VTS_OVL_DIV=16 VTS_DOVL_DIV=12
run VTS_OVL_DIV=4
