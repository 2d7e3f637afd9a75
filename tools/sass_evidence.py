"""Opcode evidence of tcgen05 / TMEM / TMA in the built objects (profiles/r2_sass_evidence.txt)."""
import collections
import re
import subprocess
import sys

OPS = re.compile(r"\b(UTC[A-Z]*MMA|LDTM[.A-Z0-9]*|UTMALDG[.A-Z0-9]*|UTMASTG[.A-Z0-9]*|UBLKCP[.A-Z0-9]*|SYNCS[.A-Z0-9]*|"
                 r"UTCBAR[.A-Z0-9]*|DFMA|HMMA)\b")
for obj in sys.argv[1:]:
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, counts = None, collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()[:90]
            continue
        for op in OPS.findall(line):
            counts[fn][op] += 1
    print(f"== {obj}")
    for f, c in counts.items():
        print(f"  {f}\n     " + ", ".join(f"{k} x{v}" for k, v in sorted(c.items())))
