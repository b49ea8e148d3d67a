#!/bin/bash
# ncu launch list of the batch workload, summarised per kernel.  Usage: tools/batch_launches.sh <tag> [batch]
tag=$1; b=${2:-1024}
bash tools/launch_list.sh $tag --workload batch --batch $b --steps 1 --warmup 3 > /dev/null
tail -1 gpurun_out/${tag}_plain.log | cut -c 1-200
python - gpurun_out/${tag}_launches.csv <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]
agg = collections.defaultdict(list)
for r in rows[h + 1:]:
    if len(r) != len(hd):
        continue
    d = dict(zip(hd, r))
    v = float(d["Metric Value"])
    u = d["Metric Unit"]
    v = v / 1000 if u in ("ns", "nsecond") else (v * 1000 if u in ("ms", "msecond") else v)
    agg[d["Kernel Name"][:60]].append(v)
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:10]:
    print(f"{len(v):4d} x mean {sum(v)/len(v):10.1f} us  tot {sum(v):10.1f}  {k}")
PY
