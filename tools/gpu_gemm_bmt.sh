nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
for shp in "512 3696 4096" "512 4096 1280" "512 1792 11008" "512 4096 4096" "2048 4096 4096" "8192 8192 8192"; do
  echo -n "auto  "; timeout 60 /tmp/gemm_bench $shp 20 2>&1 | tail -1
  echo -n "BMT=2 "; FSVD_GEMM_BMT=2 timeout 60 /tmp/gemm_bench $shp 20 2>&1 | tail -1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('decode', round(j['decode_ms_per_token'],4), round(j['roofline']['frac'],4), 'prefill', j['prefill_ms'], j['prefill_tflops'])"
