mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distributed.py -q -x > gpurun_out/dist.log 2>&1; echo "dist rc $?"; tail -1 gpurun_out/dist.log
timeout 900 python tools/query_probe.py > gpurun_out/qprobe.log 2>&1; echo "qprobe rc $?"; tail -8 gpurun_out/qprobe.log
