FSVD_GEMM_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pf_list.csv python tools/prefill_once.py > gpurun_out/pf_list.log 2>&1
python tools/pf_summary.py gpurun_out/pf_list.csv 2>&1 | tail -30
grep -c "" gpurun_out/pf_list.log; head -40 gpurun_out/pf_list.log
