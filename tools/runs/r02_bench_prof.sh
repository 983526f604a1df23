#!/bin/bash
# round-2 bench line + profiles: launch list of a short bench, ncu --set full of the finest
# descent pair (gs_probe), of k_phi_tile and of the MINRES vector kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/r02/smi.txt
timeout 900 python bench.py > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-pbm --no-cpu > gpurun_out/r02/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-pbm --no-cpu > gpurun_out/r02/ncu_launch.log 2>&1
(cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o gs_probe gs_probe.cu -lcuda > ../../gpurun_out/r02/probe_build.log 2>&1)
timeout 120 ./tools/probe/gs_probe 9 > gpurun_out/r02/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gs_pair --launch-skip 10 --launch-count 1 -o gpurun_out/r02/pair_fine ./tools/probe/gs_probe 9 > gpurun_out/r02/ncu_pair.log 2>&1
timeout 200 python tools/checks/phi_ab.py fused > gpurun_out/r02/phi_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_phi_tile -s 3 -c 1 -o gpurun_out/r02/phi_tile python tools/checks/phi_ab.py fused > gpurun_out/r02/ncu_phi.log 2>&1
timeout 200 python tools/checks/quick_time.py q > gpurun_out/r02/quick_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mr_update|k_mr_lanczos|k_mr_givens|k_newton_apply" -s 40 -c 4 -o gpurun_out/r02/minres_vec python tools/checks/quick_time.py q > gpurun_out/r02/ncu_mr.log 2>&1
echo done > gpurun_out/r02/done.txt
