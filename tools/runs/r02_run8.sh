#!/bin/bash
# 3D hexahedral path: parity against the unmodified reference
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_hex.py -x -q -p no:cacheprovider > gpurun_out/pytest_hex.log 2>&1; echo "hex rc=$?" >> gpurun_out/status8.txt
