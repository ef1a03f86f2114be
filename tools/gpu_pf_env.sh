for E in "X=1" "FSVD_GEMM_SPLITS=1" "FSVD_GEMM_BMT=1" "FSVD_GEMM_BMT=1 FSVD_GEMM_SPLITS=1" "FSVD_GEMM_BN=128 FSVD_GEMM_BMT=1"; do
  env $E timeout 300 python bench.py --steps 3 --warmup 3 --gen 8 --no-cpu-baseline > gpurun_out/pfenv.log 2>&1
  python -c "import json; j=json.loads(open('gpurun_out/pfenv.log').read().strip().splitlines()[-1]); print('$E', 'prefill ms', round(j['prefill_ms'],2), 'TF', round(j['prefill_tflops'],1))"
done
