timeout 1200 python bench.py --config c3_rmat24 --steps 1 --warmup 1 --e2e-steps 1 --e2e-warmup 0 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo "c3 rc $?"
timeout 900 python bench.py --config c4_grid --steps 2 --warmup 1 --e2e-steps 1 --e2e-warmup 0 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc $?"
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "c2 rc $?"
for f in c3 c4 c2; do tail -1 gpurun_out/bench_$f.log | cut -c1-300; done
