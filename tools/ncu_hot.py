"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report:
   python tools/ncu_hot.py rep.ncu-rep <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{sys.argv[2]}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((float(r[ci["Warp Stall Sampling (All Samples)"]]), int(r[ci["Instructions Executed"]] or 0),
                     r[ci["Source"]].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
print(f"total samples {tot:.0f}, instructions {sum(d[1] for d in data)}")
for v, n, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {n:9d}  {s}")
