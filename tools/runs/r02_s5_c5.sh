#!/bin/bash
# C5 (2048x1024, 10 levels): iteration counts and compliance of the current build (twice), the build at the start of the
# session and the current build with each of the session's switches off
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5c5; mkdir -p $O
r() { local label=$1; shift; env "$@" timeout 300 python tools/checks/run_config.py C5 2>&1 | grep "wall_s\|compliance" | tr '\n' ' ' > $O/$label.txt; echo "$label: $(cat $O/$label.txt)"; }
r cur1 A=1
r cur2 A=1
r old VTS_LIB=$PWD/_ab/lib_old.so
r close VTS_LIB=$PWD/_ab/lib_close.so
r noshift VTS_LIB=$PWD/_ab/lib_noshift.so
r fullwarp VTS_LIB=$PWD/_ab/lib_fullwarp.so
