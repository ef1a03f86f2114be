timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -3
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
timeout 300 /tmp/gemm_sweep 8 1 > gpurun_out/sweep8s.log 2>&1; grep auto gpurun_out/sweep8s.log
timeout 300 /tmp/gemm_sweep 16 1 > gpurun_out/sweep16s.log 2>&1; grep auto gpurun_out/sweep16s.log
for c in c3 c5; do
timeout 600 python bench.py --config $c --steps 1 --warmup 3 --gen 64 --no-cpu-baseline > gpurun_out/pf_$c.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/pf_$c.log').read().strip().splitlines()[-1]); print('$c decode', round(j['decode_ms_per_token'],3), 'frac', round(j['roofline']['frac'],3))"
done
