nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bench_stream.cu -o /tmp/bs && timeout 120 /tmp/bs > gpurun_out/bench_stream.log 2>&1
timeout 300 python tools/trace_decode.py > gpurun_out/trace.log 2>&1
