#!/bin/bash
# repeated full C4 solves: device-resident Newton step vs host-orchestrated
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5pbm; mkdir -p $O
timeout 600 python tools/checks/profile_pbm.py C4 5 2>&1 | grep "^solve" > $O/dev_C4.txt
VTS_HOST_NEWTON=1 timeout 600 python tools/checks/profile_pbm.py C4 5 2>&1 | grep "^solve" > $O/host_C4.txt
timeout 600 python tools/checks/profile_pbm.py C1 5 2>&1 | grep "^solve" > $O/dev_C1.txt
paste $O/dev_C4.txt $O/host_C4.txt $O/dev_C1.txt
