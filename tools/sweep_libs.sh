#!/bin/bash
# Sweep tuning builds (scratch/libbdeg_*.so) x item factors x S.
for lib in paper_1501_02237_b200/libbdeg.so scratch/libbdeg_mb3.so scratch/libbdeg_mb4.so; do
  for f in ${FACTORS:-0.25 1}; do
    echo "== lib $lib factor $f"
    BDEG_LIB=$lib BDEG_ITEM_FACTOR=$f python tools/sweep_inner.py ${WLS:-c5,w25,w26} ${SS:-3,4,5,6} | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['wl'], 'S', d['S'], 'ms %.2f' % d['kernel_ms'], 'rate %.3g' % d['rate'], d['degree'])"
  done
done
