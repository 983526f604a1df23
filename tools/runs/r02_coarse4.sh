#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/coarse4
timeout 600 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/coarse4/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/coarse4/pytest.log
for k in C1 C2; do timeout 300 python tools/checks/profile_pbm.py $k 3 2>&1 | head -4 > gpurun_out/coarse4/pbm_$k.txt; done
timeout 120 python tools/checks/quick_time.py c1 C1 > gpurun_out/coarse4/quick_c1.json 2>&1
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_BOT_PROBE -o gs_probe_bot gs_probe.cu -lcuda > ../../gpurun_out/coarse4/build.log 2>&1; cd ../..
VTS_DET_REPS=2 timeout 200 ./tools/probe/gs_probe_bot 3 16 > gpurun_out/coarse4/probe.txt 2>&1
