#!/bin/bash
# full GPU suite, smoke, bench and the reference arm on the current tree
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5full; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
tail -3 $O/pytest.log; tail -2 $O/smoke.log; head -c 500 $O/bench.json
