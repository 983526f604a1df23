#!/bin/bash
# the pair's polling loader warps (x box, builder inputs) off the compute warp's sub-partition (warps 8, 12 -> 11, 15)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5warps; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run base A=1
  for v in w1115 w11 w15; do run $v VTS_LIB=$PWD/_ab/lib_$v.so; done
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5warps/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:6s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f} desc {v[0]['pair_desc_ms']:.4f} asc {v[0]['pair_asc_ms']:.4f} xsum {v[0]['xsum']!r}")
PY
