#!/bin/bash
# A/B of the recolor kernels: current libspcn.so vs tools/_ab/libspcn_head.so.
# Quick device timings, then an ncu launch list (kernel durations) of each.
for lib in "" tools/_ab/libspcn_head.so; do
  echo "== lib ${lib:-current}"
  SPCN_LIB_PATH=$lib python tools/quick_xform_bench.py --iters 10 2>&1 | grep -E "^(fast|exact|MISMATCH)"
  tag=$(basename ${lib:-current} .so)
  SPCN_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab_${tag}.csv python tools/quick_xform_bench.py --iters 2 > /dev/null 2>&1
  python - gpurun_out/ab_${tag}.csv <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
agg = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    agg[d["Kernel Name"][:70]].append(float(d["Metric Value"]) / (1000 if d["Metric Unit"] in ("ns", "nsecond") else 1))
for k, v in agg.items():
    print(f"{len(v):4d} x  mean {sum(v)/len(v):9.1f} us  max {max(v):9.1f}  {k}")
PY
done
