#!/bin/bash
# prolongation block counts (each holds an SM the finest ascent pair's second sweep waits for)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5pblocks; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
run base A=1
run p12_12_8_2 VTS_OVL_BLOCKS=12,12,8,2
run p10_10_6_2 VTS_OVL_BLOCKS=10,10,6,2
run p16_12_8_2 VTS_OVL_BLOCKS=16,12,8,2
run p12_16_8_2 VTS_OVL_BLOCKS=12,16,8,2
run p8_8_6_2 VTS_OVL_BLOCKS=8,8,6,2
run p16_16_6_2 VTS_OVL_BLOCKS=16,16,6,2
run p20_16_8_2 VTS_OVL_BLOCKS=20,16,8,2
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5pblocks/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}")
PY
