#!/bin/bash
# cluster-size caps again, now that a band's CTA leaves when its band is done (no closing cluster barrier)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5cs2; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run base A=1
  run d8_6 VTS_PAIR_CS_DESC=6
  run d8_4 VTS_PAIR_CS_DESC=4
  run a8_6 VTS_PAIR_CS_ASC=6
  run d6a6 VTS_PAIR_CS_DESC=6 VTS_PAIR_CS_ASC=6
  run d87_6 VTS_PAIR_CS_DESC=6,6
  run il VTS_PAIR_INTERLEAVE=1
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5cs2/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {sum(x['its_per_s'] for x in v)/len(v):7.1f}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
