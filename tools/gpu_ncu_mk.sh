# ncu on the decode megakernel (a profiler replay launches it without the cluster attribute: the
# attention takes the row split there -- the bytes are the same)
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,launch__cluster_dim_x
timeout 600 ncu --metrics $M --clock-control none -k regex:decode_mk -s 2 -c 1 python tools/mk_profile_run.py 32 > gpurun_out/ncu_mk_kernel.log 2>&1; echo "kernel replay rc=$?"; tail -14 gpurun_out/ncu_mk_kernel.log
