# one ncu --set full capture of the decode megakernel (4-layer 7B-width model, full-step plan)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_decode python tools/mk_profile_run.py 4 > gpurun_out/ncu_decode.log 2>&1
tail -5 gpurun_out/ncu_decode.log
