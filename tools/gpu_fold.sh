# RMSNorm fold: prefill A/B (FSVD_NO_NORM_FOLD=1 on the same build), GPU tests, C3 bench line
for round in 1 2; do
  python tools/pf_trace.py --label fold 2>&1 | grep "prefill 512"
  FSVD_NO_NORM_FOLD=1 python tools/pf_trace.py --label nofold 2>&1 | grep "prefill 512"
done
python tools/pf_trace.py --label fold 2>&1 | grep -v -i warn | sed -n 3,12p
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
