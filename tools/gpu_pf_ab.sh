# prefill A/B: CTA-pair cluster split-K on/off (in-situ CUPTI + event timing), then the GPU test suite
python tools/pf_trace.py --label pair 2>&1 | grep -v -i warn | head -40
FSVD_NO_PAIR=1 python tools/pf_trace.py --label nopair 2>&1 | grep -v -i warn | head -3
python tools/pf_trace.py --label pair2 2>&1 | grep -v -i warn | head -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
