nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
for shp in "512 3696 4096" "512 4096 1280" "512 1792 11008" "512 4096 4096" "2048 4096 4096" "8192 8192 8192" "8 4096 4096" "8 11008 1792"; do
  timeout 60 /tmp/gemm_bench $shp 20 2>&1 | tail -1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --gen 8 --no-cpu-baseline > gpurun_out/pfenv.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/pfenv.log').read().strip().splitlines()[-1]); print('prefill ms', round(j['prefill_ms'],2), 'TF', round(j['prefill_tflops'],1))"
FSVD_GEMM_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm|splitk|attn|rmsnorm" --csv --log-file gpurun_out/pf_auto.csv python tools/prefill_once.py > gpurun_out/pf_auto.log 2>&1
