#!/bin/bash
# descent: tapered column segments (narrow last segment); ascent: 64-column prolongation chunks
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5taper; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2 3; do
  run base A=1
  run taper1 VTS_LIB=$PWD/_ab/lib_taper1.so
  run taper2 VTS_LIB=$PWD/_ab/lib_taper2.so
  run chunk64 VTS_LIB=$PWD/_ab/lib_chunk64.so
  run chunk64b VTS_LIB=$PWD/_ab/lib_chunk64.so VTS_OVL_DIV=8
  run c64t1 VTS_LIB=$PWD/_ab/lib_chunk64_taper1.so
done
cut -c1-200 $O/times.jsonl
