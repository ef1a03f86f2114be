python tools/pf_trace.py --label tc_attn 2>&1 | grep -v -i warn | head -14
FSVD_ATTN_MMA=1 python tools/pf_trace.py --label mma_attn 2>&1 | grep "prefill 512"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
