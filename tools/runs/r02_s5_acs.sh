#!/bin/bash
# ascent cluster caps again after the ramp got shorter (the finest ascent pair is resident ~76 us after the ascent starts)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5acs; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
run base A=1
run a8_6 VTS_PAIR_CS_ASC=6
run a8_4 VTS_PAIR_CS_ASC=4
run a8_3 VTS_PAIR_CS_ASC=3
run a8_6il VTS_PAIR_CS_ASC=6 VTS_PAIR_INTERLEAVE=1
run a8_4il VTS_PAIR_CS_ASC=4 VTS_PAIR_INTERLEAVE=1
run a87_6 VTS_PAIR_CS_ASC=6,6
run a87_4il VTS_PAIR_CS_ASC=4,4 VTS_PAIR_INTERLEAVE=1
run il VTS_PAIR_INTERLEAVE=1
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5acs/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}")
PY
