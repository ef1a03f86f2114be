# one ncu --set full capture of a full 32-layer decode step (megakernel, full-step plan)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_step32 python tools/mk_profile_run.py 32 > gpurun_out/ncu_step.log 2>&1
tail -3 gpurun_out/ncu_step.log
