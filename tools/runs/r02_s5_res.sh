#!/bin/bash
# descent residency: fewer residual blocks with small clusters for the coarser pairs (does early residency of level 7 pay?)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5res; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
run base A=1
run b32c5 VTS_DOVL_BLOCKS=32,24,14,8 VTS_PAIR_CS_DESC=0,5,5
run b32c3 VTS_DOVL_BLOCKS=32,24,14,8 VTS_PAIR_CS_DESC=0,3,3
run b40c5 VTS_DOVL_BLOCKS=40,24,14,8 VTS_PAIR_CS_DESC=0,5
run b24c5 VTS_DOVL_BLOCKS=24,18,10,6 VTS_PAIR_CS_DESC=0,5,5
run b48c5r12 VTS_DOVL_BLOCKS=48,12,8,6 VTS_PAIR_CS_DESC=0,5
run b36c7 VTS_DOVL_BLOCKS=36,24,14,8 VTS_PAIR_CS_DESC=0,7
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5res/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}")
PY
