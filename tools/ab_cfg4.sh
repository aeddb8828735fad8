#!/bin/bash
# On the GPU box: time config 4 once per variants/*.so (see tools/variants.sh).
cd "$(dirname "$0")/.."
cp paper_2510_01495_b200/libtk_b200.so /tmp/tk_keep.so
for v in variants/*.so; do
  cp "$v" paper_2510_01495_b200/libtk_b200.so
  timeout 120 python tools/time_cfg4.py "$(basename $v .so)" 2>&1 | tail -1
done
cp /tmp/tk_keep.so paper_2510_01495_b200/libtk_b200.so
