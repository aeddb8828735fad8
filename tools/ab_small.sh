#!/bin/bash
# On the GPU box: config-3 TTV kernel time (L2 flushed, tools/time_cfg3.py) per variants/*.so.
cd "$(dirname "$0")/.."
cp paper_2510_01495_b200/libtk_b200.so /tmp/tk_keep.so
for v in variants/*.so; do
  cp "$v" paper_2510_01495_b200/libtk_b200.so
  echo "$(basename $v .so): $(timeout 300 python tools/time_cfg3.py 2>&1 | tail -1)"
done
cp /tmp/tk_keep.so paper_2510_01495_b200/libtk_b200.so
