#!/bin/bash
# ncu launch list (per-kernel device time) of a short bench run.  Usage: tools/launch_list.sh <tag> [bench args]
tag=$1; shift
python bench.py --no-e2e --no-cpu --no-global-line "$@" > gpurun_out/${tag}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --no-e2e --no-cpu --no-global-line "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo "rc=$?"
