#!/bin/bash
# overlap only levels with at least N node rows (the coarsest overlapped levels may be faster level by level)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5minny; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
run base A=1
run d66 VTS_DOVL_MIN_NY=66
run d130 VTS_DOVL_MIN_NY=130
run a34 VTS_AOVL_MIN_NY=34
run a66 VTS_AOVL_MIN_NY=66
run d66a34 VTS_DOVL_MIN_NY=66 VTS_AOVL_MIN_NY=34
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5minny/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
tail -2 $O/err.log
