#!/bin/bash
# finest descent pair: cluster sizes 9 / 7 / 6 / 5 (GPC packing beside the coarser pair's clusters of 9)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5cs3; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run base A=1
  run d8_9 VTS_PAIR_CS_DESC=9
  run d8_7 VTS_PAIR_CS_DESC=7
  run d8_6 VTS_PAIR_CS_DESC=6
  run d8_5 VTS_PAIR_CS_DESC=5
  run d8_6a9 VTS_PAIR_CS_DESC=6 VTS_PAIR_CS_ASC=9
  run d8_6a7_6 VTS_PAIR_CS_DESC=6 VTS_PAIR_CS_ASC=0,6
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5cs3/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {sum(x['its_per_s'] for x in v)/len(v):7.1f}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
