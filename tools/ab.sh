#!/bin/bash
# On the GPU box: run the cfg5 bench once per variants/*.so (see tools/variants.sh); prints name, step ms, kernel ms.
cd "$(dirname "$0")/.."
cp paper_2510_01495_b200/libtk_b200.so /tmp/tk_keep.so
for v in variants/*.so; do
  cp "$v" paper_2510_01495_b200/libtk_b200.so
  for i in 1 2; do
    out=$(timeout 120 python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e --no-cpu "$@" 2>/tmp/ab_err.txt)
    if [ -z "$out" ]; then echo "$(basename $v .so) FAILED: $(tail -2 /tmp/ab_err.txt | tr '\n' ' ')"; continue; fi
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v .so)', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))"
  done
done
cp /tmp/tk_keep.so paper_2510_01495_b200/libtk_b200.so
