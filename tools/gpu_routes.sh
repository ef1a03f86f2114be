timeout 600 python -m pytest tests/test_gpu_routes.py tests/test_cli.py -x -q -m gpu > gpurun_out/routes.log 2>&1; echo "rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/routes.log | tail -15
