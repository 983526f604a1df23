#!/bin/bash
# cluster caps and block counts again on top of the ticket queues
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5cs4; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run base A=1
  run d7_5 VTS_PAIR_CS_DESC=0,5
  run d8_6 VTS_PAIR_CS_DESC=6
  run a8_6 VTS_PAIR_CS_ASC=6
  run rr40 VTS_DOVL_BLOCKS=40,30,16,10
  run rr56 VTS_DOVL_WORKERS=64
  run pdiv3 VTS_OVL_DIV=3 VTS_OVL_WORKERS=24
  run pdiv6 VTS_OVL_DIV=6
  run p12 VTS_OVL_WORKERS=12
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5cs4/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}")
PY
