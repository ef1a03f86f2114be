timeout 900 python -m pytest tests/test_gpu_loader.py -x -q -s > gpurun_out/loader.log 2>&1; echo "loader rc=$?"; grep -E "streaming load|passed|failed|Error|error" gpurun_out/loader.log | tail -15
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "failed_session or reference" > gpurun_out/leak.log 2>&1; echo "leak rc=$?"; tail -3 gpurun_out/leak.log
