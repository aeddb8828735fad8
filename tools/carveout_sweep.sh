cd /root/repo
for cv in ${CVS:-100 86 72 100 86}; do
  out=$(TK_TILE_CARVEOUT=$cv timeout 120 python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e --no-cpu 2>/tmp/err.txt); grep "tk tile" /tmp/err.txt
  echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv=$cv', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))" || tail -3 /tmp/err.txt
done
