# L2 / DRAM throughput of a sequence of config-3 k_pull launches (first, second, third dense round of
# mid-selection batches): is the first dense round bound by DRAM, L2 throughput or latency?
mkdir -p gpurun_out
CBFS_BATCHED_HOSTLOOP=1 timeout 1500 ncu --replay-mode application --clock-control none -k regex:k_pull --launch-skip 90 -c 12 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.per_cycle_active \
  --csv --log-file gpurun_out/r2_pull_l2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-clocks > gpurun_out/r2_pull_l2.log 2>&1
echo "ncu rc $?"
