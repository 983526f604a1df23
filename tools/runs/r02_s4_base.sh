#!/bin/bash
# session-4 restart: full GPU suite, smoke, bench on the restored tree
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/s4base
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s4base/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4base/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4base/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s4base/bench.json 2> gpurun_out/s4base/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s4base/bench_ref.json 2> gpurun_out/s4base/bench_ref.err
tail -3 gpurun_out/s4base/pytest.log; cat gpurun_out/s4base/smoke.log | tail -2; head -c 600 gpurun_out/s4base/bench.json
