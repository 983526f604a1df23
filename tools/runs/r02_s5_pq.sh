#!/bin/bash
# prolongation items by ticket vs round robin (prev = the commit before)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5pq; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2 3; do
  run prev VTS_LIB=$PWD/_ab/lib_prev.so
  run pq A=1
  run pq12 VTS_OVL_BLOCKS=12,12,6,2
  run pq20 VTS_OVL_WORKERS=24 VTS_OVL_DIV=3
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5pq/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
tail -3 $O/err.log
