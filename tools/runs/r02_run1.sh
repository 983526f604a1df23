#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 300 python bench.py --steps 2 --warmup 3 --no-pbm --no-cpu > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_phi_elem|k_phi_node|k_phi_finish|k_mr_" -c 14 -o gpurun_out/prof_phi_mr python bench.py --steps 2 --warmup 3 --no-pbm --no-cpu > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/status.txt
