#!/bin/bash
# full GPU suite + smoke + bench after the RAP-order change
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke7.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status7.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status7.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench rc=$?" >> gpurun_out/status7.txt
