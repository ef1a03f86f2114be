# env-only sweeps on the final build: L2 prefetch distance around the default, qkvB pair tile width
for D in 5 4 6 7; do
  FSVD_MK_L2_AHEAD=$D timeout 600 python bench.py --steps 3 --warmup 3 --no-c5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/es.json
  python -c "import json; d=json.load(open('gpurun_out/es.json')); print('l2_ahead=$D', round(d['decode_ms_per_token'],4), 'ms/token')"
done
for e in "" "192,1,1,2" "224,1,1,2" "160,1,1,2"; do
  FSVD_GEMM_E2=$e python tools/pf_trace.py --label "qkvB=$e" 2>&1 | grep "prefill 512"
done
