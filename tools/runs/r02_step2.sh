#!/bin/bash
# device-resident Newton step vs host path: repeated full solves (wall time per solve)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/step2
for k in C1 C2 C4; do
  VTS_HOST_NEWTON=1 timeout 600 python tools/checks/profile_pbm.py $k 4 2>&1 | grep "^solve" > gpurun_out/step2/host_$k.txt
  timeout 600 python tools/checks/profile_pbm.py $k 4 2>&1 | grep "^solve" > gpurun_out/step2/dev_$k.txt
  VTS_NO_GRAPH=1 timeout 600 python tools/checks/profile_pbm.py $k 4 2>&1 | grep "^solve" > gpurun_out/step2/nograph_$k.txt
done
