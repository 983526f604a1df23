#!/bin/bash
# the level above the fused bottom: residual/restriction rows behind its pair vs separate launches
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5low; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label $KEY >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  KEY=C3 run sep VTS_NO_LOW_OVERLAP=1
  KEY=C3 run low A=1
done
KEY=C2 run sepC2 VTS_NO_LOW_OVERLAP=1
KEY=C2 run lowC2 A=1
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5low/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
tail -2 $O/err.log
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_properties.py -x -q -p no:cacheprovider 2>&1 | tail -3
