# dual (up/gate + SiLU) GEMM tile width, in-situ prefill
for e in "" "128,1,1,1" "192,1,1,1" "224,1,1,1" "256,1,1,1" "96,1,1,1"; do
  FSVD_GEMM_E3=$e python tools/pf_trace.py --label "dual=$e" 2>&1 | grep -E "prefill 512"
  FSVD_GEMM_E3=$e python tools/pf_trace.py --label "dual=$e" 2>&1 | grep -E "gemm_tc_kernel<[0-9]+, true" | head -1
done
