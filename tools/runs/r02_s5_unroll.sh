#!/bin/bash
# unroll factor of the fused bottom's wavefront loop (instruction-cache misses of its three instantiations against loop overhead)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5unroll; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run u4 A=1
  for v in u1 u2; do run $v VTS_LIB=$PWD/_ab/lib_$v.so; done
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5unroll/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:6s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f} xsum {v[0]['xsum']!r}")
PY
