mkdir -p gpurun_out
LANES_TOTAL=256 timeout 1200 python tools/wide_probe.py c5_knn 1,2,4 > gpurun_out/wp_c5.log 2>&1; tail -3 gpurun_out/wp_c5.log
