#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/div2
run() { env "$@" timeout 120 python tools/checks/quick_time.py "$*" >> gpurun_out/div2/times.jsonl 2>> gpurun_out/div2/err.log; }
run VTS_DOVL_DIV=8
run VTS_DOVL_DIV=6
run VTS_DOVL_DIV=4
run VTS_DOVL_DIV=4 VTS_DOVL_WORKERS=44
run VTS_DOVL_DIV=8 VTS_DOVL_WORKERS=44
run VTS_DOVL_DIV=6 VTS_DOVL_WORKERS=44
