"""Instructions executed per CUDA source line (file:line) of one kernel from an
ncu report: python tools/ncu_lines.py <report> <kernel regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
agg = collections.Counter()
src = {}
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    ie = hdr.index("Instructions Executed")
    if r[ie].strip().isdigit() and int(r[ie]):
        key = f"{fname}:{r[0]}"
        agg[key] += int(r[ie])
        src[key] = r[1].strip()[:80]
tot = sum(agg.values())
for k, n in agg.most_common(top):
    print(f"{n / tot * 100:5.1f}%  {k:22s} {src[k]}")
