# round-2 final evidence refresh at the final code: tests, smoke, C2 bench + reference arm, C4 line,
# the ncu launch list of the bench command and the ncu decode-step capture
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -2 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/final/bench.log 2>&1; tail -1 gpurun_out/final/bench.log | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref.log 2>&1; tail -1 gpurun_out/final/ref.log | cut -c1-200
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 1 --warmup 3 --gen 8 --no-cpu-baseline --no-c5 > gpurun_out/final/ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/final/prof_step32 python tools/mk_profile_run.py 32 > gpurun_out/final/ncu_step.log 2>&1; echo "ncu full rc=$?"
for c in c3 c5; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 > gpurun_out/final/bench_$c.log 2>&1; tail -1 gpurun_out/final/bench_$c.log | cut -c1-120; done
timeout 1500 python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/final/bench_c4.log 2>&1; tail -1 gpurun_out/final/bench_c4.log | cut -c1-120
