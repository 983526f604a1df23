"""Write the raw-page subset (launch, time, dram bytes, stall samples) of an ncu report as 3-row CSV.

python tools/checks/ncu_subset.py report.ncu-rep out.csv
"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units, vals = rows[0], rows[1], rows[2]
keep = [i for i, k in enumerate(head)
        if k.startswith(("dram__bytes_read.sum", "dram__bytes_write.sum", "launch__", "smsp__pcsamp_warps_issue"))
        or k in ("gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__inst_executed.sum",
                 "TPC.TriageCompute.sm__cycles_active.avg")]
with open(sys.argv[2], "w", newline="") as fh:
    w = csv.writer(fh)
    for r in (head, units, vals):
        w.writerow([r[i] for i in keep])
