mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pll.py -q -x > gpurun_out/pll.log 2>&1; echo "pll rc $?"; tail -3 gpurun_out/pll.log
timeout 300 python tools/pll_probe.py c1_er 16 1024 > gpurun_out/pll_probe.log 2>&1; echo "c1 rc $?"
timeout 900 python tools/pll_probe.py c2_rmat20 64 2048 >> gpurun_out/pll_probe.log 2>&1; echo "c2 rc $?"
cat gpurun_out/pll_probe.log | tail -6
