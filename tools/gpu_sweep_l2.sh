# decode megakernel: L2 prefetch distance (chunks beyond the ring) sweep
for D in 3 5 8 11; do
  FSVD_MK_L2_AHEAD=$D timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$D.log 2>&1
  python -c "import json,sys; j=json.loads(open('gpurun_out/sweep_$D.log').read().strip().splitlines()[-1]); print('D=$D', round(j['decode_ms_per_token'],4), round(j['roofline']['frac'],4))"
done
