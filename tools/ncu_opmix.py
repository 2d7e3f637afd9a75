"""Executed-instruction mix (by SASS opcode) of one kernel: python tools/ncu_opmix.py rep kernel-regex"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{sys.argv[2]}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
seen = set()
for r in rows[2:]:
    if len(r) < len(hdr) or r[ci["Address"]] in seen:
        continue
    seen.add(r[ci["Address"]])
    op = r[ci["Source"]].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    v = r[ci["Instructions Executed"]]
    if not v.isdigit():
        continue
    mix[o.split(".")[0]] += int(v)
tot = sum(mix.values())
for o, c in mix.most_common(25):
    print(f"{o:12s} {c:12d} {100 * c / tot:5.1f}%")
print("total", tot)
