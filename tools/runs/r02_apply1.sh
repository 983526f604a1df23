#!/bin/bash
# Newton-apply variants: bitwise comparison and cold/warm timing on C3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/apply
for v in tile 8x2 8x1 16x1 32x1 8x2b4; do
  if [ $v = tile ]; then export VTS_APPLY_KERNEL=tile; else unset VTS_APPLY_KERNEL; export VTS_APPLY_WK=$v; fi
  timeout 300 python tools/checks/apply_ab.py $v gpurun_out/apply >> gpurun_out/apply/times.jsonl 2>> gpurun_out/apply/err.log
done
unset VTS_APPLY_KERNEL VTS_APPLY_WK
for c in C1 C2; do
  VTS_APPLY_KERNEL=tile timeout 300 python tools/checks/apply_ab.py tile_$c gpurun_out/apply $c >> gpurun_out/apply/times.jsonl 2>> gpurun_out/apply/err.log
  timeout 300 python tools/checks/apply_ab.py rows_$c gpurun_out/apply $c >> gpurun_out/apply/times.jsonl 2>> gpurun_out/apply/err.log
done
python - <<'PY' >> gpurun_out/apply/compare.txt 2>&1
import numpy as np, glob
ref = np.load("/tmp/apply_tile.npz")
for f in sorted(glob.glob("/tmp/apply_*.npz")):
    if "_C" in f: continue
    d = np.load(f)
    print(f, "y maxdiff", np.abs(d["y"] - ref["y"]).max() / np.abs(ref["y"]).max(),
          "y bitwise(core)", np.array_equal(d["y"][:-1], ref["y"][:-1]), "ya", d["y"][-1], ref["y"][-1],
          "x maxdiff", np.abs(d["x"] - ref["x"]).max() / np.abs(ref["x"]).max())
for c in ("C1", "C2"):
    a = np.load(f"/tmp/apply_tile_{c}.npz"); b = np.load(f"/tmp/apply_rows_{c}.npz")
    print(c, "y maxdiff", np.abs(a["y"] - b["y"]).max() / np.abs(a["y"]).max(), "core bitwise", np.array_equal(a["y"][:-1], b["y"][:-1]))
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_target.py -x -q -p no:cacheprovider > gpurun_out/apply/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/apply/compare.txt
