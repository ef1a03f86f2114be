# in-situ (CUPTI) per-kernel prefill timings
python tools/pf_trace.py --label default 2>&1 | grep -v -i warn
FSVD_NO_PDL=1 python tools/pf_trace.py --label nopdl 2>&1 | grep -v -i warn
