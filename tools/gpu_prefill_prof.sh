for mode in auto bmt1 old; do
  case $mode in auto) E="";; bmt1) E="FSVD_GEMM_BMT=1";; old) E="FSVD_GEMM_BMT=1 FSVD_GEMM_BN=128";; esac
  env $E FSVD_GEMM_LOG=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|splitk|attn|rmsnorm" --csv --log-file gpurun_out/pf_$mode.csv python tools/prefill_once.py > gpurun_out/pf_$mode.log 2>&1
done
