#!/bin/bash
# On the GPU box: ncu launch list (gpu__time_duration) of one middle-mode call sequence at config 5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TK_MID_ONLY=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_mid.csv -k regex:'mid_|lead_offsets|scan_|compact' python tools/time_mode1.py ${1:-400000000} > gpurun_out/launches_mid.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open('gpurun_out/launches_mid.csv') if l.startswith('"')))
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split('(')[0][:60]; v = float(r[vi].replace(',', ''))
    if r[ui] == 'ns': v /= 1000.0
    agg.setdefault(name, []).append(v)
tot = 0
for k, v in agg.items():
    per = sum(v) / 6; tot += per
    print(f"{per:10.1f} us/call  n={len(v):3d}  {k}")
print(f"{tot:10.1f} us/call total")
PY
