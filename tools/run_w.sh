mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pll.py -q -x > gpurun_out/pll.log 2>&1; echo "pll rc $?"; tail -1 gpurun_out/pll.log
for c in 296 1000; do CBFS_PLL_CTAS=$c timeout 300 python tools/pll_probe.py c2_rmat20 64 2048 > gpurun_out/pll_1024_$c.log 2>&1; echo -n "ctas $c "; tail -1 gpurun_out/pll_1024_$c.log | cut -c 190-330; done
timeout 300 python tools/pll_probe.py c2_rmat20 64 2048 > gpurun_out/pll_def.log 2>&1; echo -n "default "; tail -1 gpurun_out/pll_def.log
timeout 300 python tools/pll_probe.py c1_er 16 1024 > gpurun_out/pll_c1.log 2>&1; echo -n "c1 "; tail -1 gpurun_out/pll_c1.log
