mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log)
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tests/run_config.py c4_grid --check 8 --profile > gpurun_out/c4.log 2>&1
tail -c 1500 gpurun_out/c4.log
timeout 900 python tests/run_config.py c5_knn --check 4 --profile > gpurun_out/c5.log 2>&1
tail -c 1500 gpurun_out/c5.log
