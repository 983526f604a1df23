#!/bin/bash
# end-of-round profiles: launch list of a short bench, ncu --set full of the finest descent pair (gs_probe)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5prof; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/smi.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-pbm --no-cpu > $O/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-pbm --no-cpu > $O/ncu_launch.log 2>&1
(cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o gs_probe gs_probe.cu -lcuda > ../../$O/probe_build.log 2>&1)
VTS_DET_REPS=2 timeout 120 ./tools/probe/gs_probe 9 > $O/probe_plain.log 2>&1 && \
VTS_DET_REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_pair --launch-skip 10 --launch-count 1 -o $O/pair_fine ./tools/probe/gs_probe 9 > $O/ncu_pair.log 2>&1
ls -la $O; tail -3 $O/ncu_pair.log
