#!/bin/bash
# On the GPU box: the evidence bundle for profiles/ (bench line, launch list, one full ncu capture).
#   tools/profile_round.sh <tag>
set -u
tag=${1:-r01}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-secondary --no-e2e --no-cpu > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ttv_tile -s 1 -c 1 -f \
  -o gpurun_out/${tag}_tile python tools/prof_ttv.py --what cfg5 --nnz 400000000 --iters 2 > gpurun_out/${tag}_ncu_full.log 2>&1
echo "full capture rc=$?"
# the middle-mode path (config 5, k = 1): per-kernel times of one call (ncu launch list, six calls averaged)
bash tools/launches_mid.sh > gpurun_out/${tag}_launches_mid.txt 2>&1
echo "mid launch list rc=$?"
