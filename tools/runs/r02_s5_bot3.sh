#!/bin/bash
# fused bottom: first half-stencil prefetched by a bulk copy before the PDL wait
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5bot3; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label $KEY >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  KEY=C3 run prev VTS_LIB=$PWD/_ab/lib_prev.so
  KEY=C3 run new A=1
done
KEY=C1 run prevC1 VTS_LIB=$PWD/_ab/lib_prev.so
KEY=C1 run newC1 A=1
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5bot3/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py -x -q -p no:cacheprovider 2>&1 | tail -3
