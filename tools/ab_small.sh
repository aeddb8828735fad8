#!/bin/bash
# On the GPU box: config-3 TTV kernel time (bench secondary, L2 flushed) per variants/*.so.
cd "$(dirname "$0")/.."
cp paper_2510_01495_b200/libtk_b200.so /tmp/tk_keep.so
for v in variants/*.so; do
  cp "$v" paper_2510_01495_b200/libtk_b200.so
  timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
r = bench.secondary_measurements(0, 20)
print('$(basename $v .so)', round(r['cfg3_ttv']['kernel_ms'] * 1e3, 2), 'us cfg3', round(r['cfg4_ttv_dense']['kernel_ms'], 4), 'ms cfg4')
" 2>/dev/null
done
cp /tmp/tk_keep.so paper_2510_01495_b200/libtk_b200.so
