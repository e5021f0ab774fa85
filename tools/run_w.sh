mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pll.py -q -x > gpurun_out/pll.log 2>&1; echo "pll rc $?"; tail -2 gpurun_out/pll.log
for i in 1 2; do timeout 300 python tools/pll_probe.py c2_rmat20 64 2048 > gpurun_out/pll_p$i.log 2>&1; tail -1 gpurun_out/pll_p$i.log | cut -c 150-400; done
timeout 300 python tools/pll_probe.py c1_er 16 1024 > gpurun_out/pll_c1.log 2>&1; tail -1 gpurun_out/pll_c1.log | cut -c 150-400
