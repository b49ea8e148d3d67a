"""Opcode mix (warp instructions executed) of one kernel from an ncu report's
SASS source page.  Usage: python tools/sass_mix.py <report> <kernel regex> [npix]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
npix = float(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}", "--launch-skip", str(int(sys.argv[4]) if len(sys.argv) > 4 else 0), "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hdr]
si, ie = h.index("Source"), h.index("Instructions Executed")
mix, tot = collections.Counter(), 0
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    if not r[ie].isdigit():
        continue
    n = int(r[ie])
    mix[o.split(".")[0]] += n
    tot += n
print(f"total warp instructions {tot:.4g}" + (f"  per px {32 * tot / npix:.2f}" if npix else ""))
for o, n in mix.most_common(int(__import__("os").environ.get("TOP", "30"))):
    print(f"  {o:12s} {n / tot * 100:6.2f}%" + (f"  {32 * n / npix:6.2f}/px" if npix else ""))
