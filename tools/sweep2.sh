for s in ${@:-16x16x2x1x3 16x24x2x1x3 16x32x2x1x2 20x24x2x1x2}; do
  echo "== shape $s"; SPCN_XFORM_SHAPE=$s python tools/quick_xform_bench.py --mpx 400 --iters 10 2>&1 | grep -E "^(fast|exact\+cal|MISMATCH)"
done
