"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu report, by
joining the report's SASS page with nvdisasm line info of the local build object:
   python tools/ncu_lines.py rep.ncu-rep <kernel-regex> <object.o> <mangled-fn-prefix> <source.cu> [top]"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile

rep, kre, obj, fn, srcf = sys.argv[1:6]
top = int(sys.argv[6]) if len(sys.argv) > 6 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
sass = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        sass.append((int(r[ci["Instructions Executed"]] or 0), float(r[ci["Warp Stall Sampling (All Samples)"]] or 0),
                     r[ci["Source"]].strip()))
    except ValueError:
        pass
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", __import__("os").path.abspath(obj)], cwd=d, capture_output=True)
    import glob
    cub = glob.glob(d + "/*.cubin")[0]
    dis = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if l.startswith(".text." + fn)][0]
cur, instrs = None, []
for l in dis[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r"line (\d+)", l)
    if "//## File" in l and m:
        cur = int(m.group(1))
        continue
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m2:
        instrs.append((cur, m2.group(2).strip()))
sass = sass[:len(instrs)]
mism = sum(1 for a, b in zip(instrs, sass) if a[1].split()[0] != b[2].split()[0])
agg = collections.defaultdict(lambda: [0, 0.0])
for (ln, _), (n, st, _) in zip(instrs, sass):
    agg[ln][0] += n
    agg[ln][1] += st
tot = sum(v[0] for v in agg.values()) or 1
tst = sum(v[1] for v in agg.values()) or 1
src = open(srcf).read().split("\n")
print(f"instructions {tot}, stall samples {tst:.0f}, sass rows {len(instrs)}, opcode mismatches {mism}")
for ln, (n, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    s = src[ln - 1].strip()[:100] if ln and ln <= len(src) else "?"
    print(f"{100 * n / tot:5.1f}% {100 * st / tst:5.1f}%  {ln}: {s}")
