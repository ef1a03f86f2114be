# residual-add (oB, dB) and dual (upgateB) tile variants with CTA pairs, in-situ prefill time
python tools/pf_trace.py --label "default" 2>&1 | grep "prefill 512"
for e in "256,1,1,2" "128,1,1,2" "192,1,1,2" "256,1,2,2,1" "128,1,2,1,1"; do
  FSVD_GEMM_E1=$e python tools/pf_trace.py --label "addf32=$e" 2>&1 | grep "prefill 512"
done
for e in "128,1,1,2" "192,1,1,2" "256,1,1,2" "224,1,1,2" "160,1,1,2"; do
  FSVD_GEMM_E3=$e python tools/pf_trace.py --label "dual=$e" 2>&1 | grep "prefill 512"
done
