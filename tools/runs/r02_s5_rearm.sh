#!/bin/bash
# above-ring re-arm by the loader warp instead of the compute warp
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5rearm; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 120 python tools/checks/quick_time.py $label $KEY >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
KEY=C1 run newC1 A=1
KEY=C1 run prevC1 VTS_LIB=$PWD/_ab/lib_prev.so
KEY=C2 run newC2 A=1
KEY=C2 run prevC2 VTS_LIB=$PWD/_ab/lib_prev.so
for r in 1 2; do
  KEY=C3 run prev VTS_LIB=$PWD/_ab/lib_prev.so
  KEY=C3 run new A=1
done
cat $O/status.txt | tr '\n' ' '; echo
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5rearm/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:10s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f} sweep {v[0]['fine_sweep_ms']:.4f} desc {v[0]['pair_desc_ms']:.4f} asc {v[0]['pair_asc_ms']:.4f} xsum {v[0]['xsum']!r}")
PY
tail -3 $O/err.log
