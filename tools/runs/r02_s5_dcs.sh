#!/bin/bash
# descent: small clusters for the coarser pairs only (do they become resident earlier beside the finest pair?)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5dcs; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run base A=1
  run d7_5 VTS_PAIR_CS_DESC=0,5
  run d7_3 VTS_PAIR_CS_DESC=0,3
  run d76_5 VTS_PAIR_CS_DESC=0,5,5
  run d8_6 VTS_PAIR_CS_DESC=6
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5dcs/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {sum(x['its_per_s'] for x in v)/len(v):7.1f}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}  xsum {v[0]['xsum']!r}")
PY
cd tools/probe && timeout 300 nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DVTS_TIMELINE -DVTS_GS_PROBE -o gs_probe_tl gs_probe.cu -lcuda > ../../$O/build.log 2>&1; cd ../..
VTS_DET_REPS=2 VTS_PAIR_CS_DESC=0,5 timeout 200 ./tools/probe/gs_probe_tl 9 2>&1 | grep -A 12 "timeline rep 1" > $O/tl_d7_5.txt; cat $O/tl_d7_5.txt
