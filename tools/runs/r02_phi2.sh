#!/bin/bash
# phi pass: kernel launch times fused vs split, and an ncu --set full capture of k_phi_tile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/phi2
timeout 200 python tools/checks/phi_ab.py fused > gpurun_out/phi2/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_phi|k_free_to_grid" --csv --log-file gpurun_out/phi2/launches_fused.csv python tools/checks/phi_ab.py fused > /dev/null 2>&1
VTS_PHI_SPLIT=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_phi|k_free_to_grid" --csv --log-file gpurun_out/phi2/launches_split.csv python tools/checks/phi_ab.py split > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_phi_tile -s 3 -c 1 -o gpurun_out/phi2/phi_tile python tools/checks/phi_ab.py fused > gpurun_out/phi2/ncu_full.log 2>&1
