#!/bin/bash
# On the GPU box: config-3 TTV kernel time per run-time lag.
cd "$(dirname "$0")/.."
for lag in 1024 512 256 128 64 32 16; do TK_TILE_LAG_RT=$lag python tools/time_cfg3.py 2>&1 | tail -1; done
