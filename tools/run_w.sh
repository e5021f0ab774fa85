mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/wide.log 2>&1; echo "wide rc $?"; tail -30 gpurun_out/wide.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ado.py -q -x > gpurun_out/w_par.log 2>&1; echo "par rc $?"; tail -2 gpurun_out/w_par.log
