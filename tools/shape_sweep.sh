#!/bin/bash
# Sweep the compiled recolor-kernel shapes (quick device-resident timing),
# plus the identity (copy) ceiling of each shape's memory path.
for s in ${@:-16x16x2x1 16x32x2x1 8x16x2x2 12x32x2x1 20x16x2x1 16x32x1x1}; do
  echo "== shape $s"; SPCN_XFORM_SHAPE=$s python tools/quick_xform_bench.py --mpx 400 2>&1 | grep -v strict
  echo "-- identity"; SPCN_XFORM_IDENTITY=1 SPCN_XFORM_SHAPE=$s python tools/quick_xform_bench.py --mpx 400 2>&1 | grep "^fast"
done
