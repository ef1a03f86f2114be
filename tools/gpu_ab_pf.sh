# same-box A/B of two builds (prefill trace), then GPU tests on the second
for round in 1 2; do for v in "$@"; do
  cp ab/$v.so paper_2605_08314_b200/libfsvd_b200.so
  python tools/pf_trace.py --label $v 2>&1 | grep "prefill 512"
done; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
