#!/bin/bash
# residual/restriction items by ticket in readiness order vs static round robin; block counts
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5queue; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run static VTS_LIB=$PWD/_ab/lib_static.so
  run queue A=1
  run q40 VTS_DOVL_BLOCKS=40,30,16,10
  run q32 VTS_DOVL_BLOCKS=32,24,14,8
  run q24 VTS_DOVL_BLOCKS=24,18,10,6
  run q32b VTS_DOVL_BLOCKS=32,36,20,12
  run q56 VTS_DOVL_BLOCKS=48,36,20,12 VTS_DOVL_WORKERS=64
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5queue/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {sum(x['its_per_s'] for x in v)/len(v):7.1f}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
tail -3 $O/err.log
