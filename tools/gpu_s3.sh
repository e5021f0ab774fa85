mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log)
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tests/run_config.py c4_grid --clusters 64 --conc 1 --profile > gpurun_out/c4_64.log 2>&1
tail -c 600 gpurun_out/c4_64.log
timeout 600 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 6000 --launch-count 3 -f -o gpurun_out/sp_c4 python tests/run_config.py c4_grid --clusters 64 --conc 1 > gpurun_out/ncu_sp_c4.log 2>&1
tail -3 gpurun_out/ncu_sp_c4.log
