timeout 900 python -m pytest tests/test_gpu_regime.py -x -q -s > gpurun_out/regime.log 2>&1; echo "regime rc=$?"; grep -E "rel err|passed|failed|Error" gpurun_out/regime.log | tail -12
