#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5queue2; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2 3; do
  run prev VTS_LIB=$PWD/_ab/lib_prev.so
  run static VTS_LIB=$PWD/_ab/lib_static.so
  run queue A=1
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5queue2/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {sum(x['its_per_s'] for x in v)/len(v):7.1f}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
