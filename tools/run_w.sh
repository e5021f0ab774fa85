mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/wide.log 2>&1; echo "wide rc $?"; tail -3 gpurun_out/wide.log
timeout 600 python tools/wide_probe.py c2_rmat20 1,2,4,8 > gpurun_out/wide_probe.log 2>&1; echo "probe rc $?"; cat gpurun_out/wide_probe.log | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "select" > gpurun_out/w_sel.log 2>&1; echo "sel rc $?"; tail -1 gpurun_out/w_sel.log
