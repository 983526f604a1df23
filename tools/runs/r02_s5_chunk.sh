#!/bin/bash
# prolongation chunk width under the ticket queue (32 / 48 / 64 columns), each at several placements
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5chunk; mkdir -p $O; rm -f $O/times.jsonl
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for v in base chunk32 chunk48; do
  for n in 0 1 7; do
    if [ $v = base ]; then L="A=1"; else L="VTS_LIB=$PWD/_ab/lib_$v.so"; fi
    if [ $n = 0 ]; then run ${v}_p0 $L; else run ${v}_p$n VTS_ARENA_PAD=$n $L; fi
  done
done
run chunk32_div8 VTS_LIB=$PWD/_ab/lib_chunk32.so VTS_OVL_DIV=8
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5chunk/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:14s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}")
PY
tail -3 $O/err.log
