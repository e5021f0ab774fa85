# ncu launch list of one config-3 bench step (kernels launched round by round: CBFS_BATCHED_HOSTLOOP=1),
# application replay (no device-memory save/restore of the ~150 GB working set)
CBFS_BATCHED_HOSTLOOP=1 timeout 2400 ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3400 --csv --log-file gpurun_out/r2f_c3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-clocks > gpurun_out/r2f_c3_ncu_list.log 2>&1; echo "ncu list rc $?"
grep -v "^==" gpurun_out/r2f_c3_launches.csv | wc -l
tail -n 3 gpurun_out/r2f_c3_ncu_list.log | cut -c1-300
