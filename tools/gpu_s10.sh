(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log)
tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --config c5_knn --steps 1 --warmup 1 --e2e-steps 1 --e2e-warmup 0 --no-cpu > gpurun_out/bench_c5.log 2>&1; echo "c5 rc $?"
tail -1 gpurun_out/bench_c5.log | cut -c1-600
