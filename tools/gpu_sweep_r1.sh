mkdir -p gpurun_out
timeout 300 python bench.py --concurrency 1 --no-e2e --no-cpu > gpurun_out/bench_c1.log 2>&1
timeout 600 python tests/run_config.py c4_grid --check 8 --profile > gpurun_out/c4.log 2>&1
timeout 900 python tests/run_config.py c5_knn --check 4 --profile > gpurun_out/c5.log 2>&1
timeout 1200 python tests/run_config.py c3_rmat24 --check 2 --profile > gpurun_out/c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/ncu_launch.log 2>&1
tail -c 1500 gpurun_out/bench_c1.log; tail -c 1500 gpurun_out/c4.log; tail -c 1500 gpurun_out/c5.log; tail -c 2000 gpurun_out/c3.log
