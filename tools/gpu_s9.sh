mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-400
timeout 600 python bench.py --concurrency 8 --no-e2e --no-cpu > gpurun_out/bench_c2_conc8.log 2>&1; tail -1 gpurun_out/bench_c2_conc8.log | cut -c1-300
timeout 600 python bench.py --alpha 30 --no-e2e --no-cpu > gpurun_out/bench_c2_a30.log 2>&1; tail -1 gpurun_out/bench_c2_a30.log | cut -c1-300
timeout 900 python bench.py --config c4_grid --steps 1 --warmup 1 --e2e-steps 1 --e2e-warmup 0 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-300
