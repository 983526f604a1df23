#!/bin/bash
# DOC / minres contract / error-path tests, V-cycle diagnostics with saved vectors
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_doc.py -q -p no:cacheprovider > gpurun_out/pytest_doc.log 2>&1; echo "doc rc=$?" >> gpurun_out/status3.txt
timeout 600 python tools/checks/diag_vcycle_levels.py --small --save > gpurun_out/diag_small.log 2>&1; echo "diag rc=$?" >> gpurun_out/status3.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ip.py tests/test_gpu_properties.py -q -p no:cacheprovider > gpurun_out/pytest_regress.log 2>&1; echo "regress rc=$?" >> gpurun_out/status3.txt
