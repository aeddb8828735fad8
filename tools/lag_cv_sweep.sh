#!/bin/bash
# On the GPU box: config-5 step / kernel ms vs TK_TILE_LAG_RT (and TK_TILE_CARVEOUT if set).
cd "$(dirname "$0")/.."
for lag in ${LAGS:-768 1024 1280 1536}; do
  for i in 1 2; do
    out=$(TK_TILE_LAG_RT=$lag timeout 120 python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e --no-cpu 2>/tmp/err.txt)
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lag=$lag', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))" || tail -2 /tmp/err.txt
  done
done
