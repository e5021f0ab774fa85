# ncu --set full (with source) of a mid-selection FIRST dense round of the config-3 pull (launch 91 of k_pull)
mkdir -p gpurun_out
CBFS_BATCHED_HOSTLOOP=1 timeout 1500 ncu --replay-mode application --set full --import-source on --clock-control none \
  -k regex:k_pull --launch-skip 90 -c 1 -f -o gpurun_out/r2_pull_r1 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-clocks \
  > gpurun_out/r2_pull_r1.log 2>&1
echo "ncu rc $?"
ncu -i gpurun_out/r2_pull_r1.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_pull_r1_sass.csv 2>/dev/null; echo "src rc $?"
ncu -i gpurun_out/r2_pull_r1.ncu-rep --page source --csv > gpurun_out/r2_pull_r1_src.csv 2>/dev/null; echo "src2 rc $?"
