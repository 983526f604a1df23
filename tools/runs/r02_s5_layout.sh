#!/bin/bash
# sensitivity of the V-cycle to the placement of the level arrays (n x 256 bytes of padding before each level)
cd $GRAFT_REPO_ROOT; O=gpurun_out/s5layout; mkdir -p $O
run() { local label=$1; shift; env "$@" timeout 150 python tools/checks/quick_time.py $label >> $O/times.jsonl 2>> $O/err.log; echo "$label rc=$?" >> $O/status.txt; }
for r in 1 2; do
  run pad0 A=1
  for n in 1 2 3 4 7 8 16 64 1024; do run pad$n VTS_ARENA_PAD=$n; done
done
python - <<'PY'
import json,collections
d=collections.defaultdict(list)
for l in open('gpurun_out/s5layout/times.jsonl'):
    j=json.loads(l); d[j['label']].append(j)
for k,v in d.items():
    print(f"{k:12s} its/s {' '.join('%.1f'%x['its_per_s'] for x in v)}  vcycle {sum(x['vcycle_ms'] for x in v)/len(v):.4f}")
PY
