mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distributed.py -q -x > gpurun_out/dist.log 2>&1; echo "dist rc $?"; tail -1 gpurun_out/dist.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pll_bfs|k_pll_query|k_pll_sort" --launch-skip 600 --launch-count 3 -o gpurun_out/pll_full -f python tools/pll_probe.py c2_rmat20 64 2048 > gpurun_out/ncu_pll.log 2>&1; echo "ncu pll rc $?"
ls -la gpurun_out/ | tail -5
