"""Run the same PBM solve several times and report any run-to-run difference.

Usage: python tools/checks/repeat_pbm.py [config] [reps]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1904_06556_b200 as vts  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ref = None
for r in range(reps):
    trace = {}
    try:
        rep = vts.solve_pbm(vts.build_config(key), trace=trace)
        err = None
    except Exception as e:  # keep going: report where the run left the reference trajectory
        rep, err = None, e
    sig = list(zip(trace.get("kappa", []), trace.get("slope", [])))
    if ref is None:
        ref = sig
        print("run 0:", len(sig), "trace entries", "error" if err else "ok", flush=True)
        continue
    first = next((i for i, (a, b) in enumerate(zip(ref, sig)) if a != b), None)
    if first is None and len(sig) == len(ref) and err is None:
        continue
    print(f"run {r}: error={err!r} entries={len(sig)} first difference at entry {first}", flush=True)
    if first is not None:
        print("   ref:", ref[first])
        print("   got:", sig[first])
print("done", flush=True)
