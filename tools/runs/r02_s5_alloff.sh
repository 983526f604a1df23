#!/bin/bash
# the build with every switch of the round's last session off (the code of the session's start, through the new
# switches) against the default build: same bits, and the sum of the session's gains
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5alloff; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label $KEY >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
KEY=C3 run alloff VTS_LIB=$PWD/_ab/lib_alloff.so
KEY=C3 run default A=1
KEY=C2 run alloffC2 VTS_LIB=$PWD/_ab/lib_alloff.so
KEY=C2 run defaultC2 A=1
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5alloff/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
