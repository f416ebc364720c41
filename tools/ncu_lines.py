"""Per-source-line instruction and stall-sample shares of one kernel from an
.ncu-rep captured with --import-source on (ncu --page source --print-source cuda,sass).
usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, agg, ti, ts = None, [], 0, 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name", ""):
        continue
    try:
        ins, smp = int(r[7]), int(r[4])
    except ValueError:
        continue
    agg.append((cur, int(r[0]), r[1].strip()[:88], smp, ins))
    ti += ins
    ts += smp
print("instructions", ti, "samples", ts)
for key, name in ((4, "instructions"), (3, "stall samples")):
    print("--- by", name)
    for a in sorted(agg, key=lambda x: -x[key])[:top]:
        print(f"{a[0]}:{a[1]:4d} inst {a[4] / ti * 100:5.1f}% smp {a[3] / ts * 100:5.1f}%  {a[2]}")
