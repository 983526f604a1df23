#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/phi3
for b in 3 4; do
  VTS_LIB=$PWD/_ab/lib_phi$b.so timeout 200 python tools/checks/phi_ab.py minb$b > /dev/null 2>&1 && \
  VTS_LIB=$PWD/_ab/lib_phi$b.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_phi" --csv --log-file gpurun_out/phi3/launches_$b.csv python tools/checks/phi_ab.py minb$b > /dev/null 2>&1
done
