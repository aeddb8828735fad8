#!/bin/bash
# On the GPU box: MTTKRP (config-4 tensor, mode 0) kernel time per variants/*.so for ranks "$@".
cd "$(dirname "$0")/.."
cp paper_2510_01495_b200/libtk_b200.so /tmp/tk_keep.so
for v in variants/*.so; do
  cp "$v" paper_2510_01495_b200/libtk_b200.so
  echo "== $(basename $v .so)"; timeout 300 python tools/time_mttkrp.py "$@" 2>/dev/null
done
cp /tmp/tk_keep.so paper_2510_01495_b200/libtk_b200.so
