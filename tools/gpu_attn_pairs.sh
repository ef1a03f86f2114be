# decode attention: one CTA pair per head (cluster of 2, DSMEM merge) vs the row split -- parity + timing
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for p in 1 0; do
  FSVD_MK_ATTN_PAIRS=$p timeout 600 python bench.py --steps 5 --warmup 3 --no-c5 2>/dev/null | tail -1 > gpurun_out/bap.json
  python -c "import json; d=json.load(open('gpurun_out/bap.json')); print('pairs=$p', round(d['ms_per_step']/256, 4), 'ms/token', round(d['roofline']['frac'],4))"
done
FSVD_MK_ATTN_PAIRS=1 timeout 300 python tools/trace_decode.py --ctx 640 2>&1 | grep -E "L16\.|attention phase" | head -12
