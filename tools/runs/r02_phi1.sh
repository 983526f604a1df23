#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/phi1
timeout 200 python tools/checks/phi_ab.py fused >> gpurun_out/phi1/times.jsonl 2>> gpurun_out/phi1/err.log
VTS_PHI_SPLIT=1 timeout 200 python tools/checks/phi_ab.py split >> gpurun_out/phi1/times.jsonl 2>> gpurun_out/phi1/err.log
python - >> gpurun_out/phi1/compare.txt 2>&1 <<'PY'
import numpy as np
a = np.load("/tmp/phi_fused.npz"); b = np.load("/tmp/phi_split.npz")
for k in a.files:
    print(k, "bitwise", np.array_equal(a[k], b[k]), "maxrel", float(np.abs(a[k] - b[k]).max() / max(np.abs(b[k]).max(), 1e-300)))
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_target.py tests/test_gpu_step.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/phi1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/phi1/compare.txt
timeout 300 python tools/checks/profile_pbm.py C4 3 2>&1 | grep "^solve" >> gpurun_out/phi1/compare.txt
