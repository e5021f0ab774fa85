mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_pll.py tests/test_gpu_ado.py -q -x -p no:randomly > gpurun_out/rep$i.log 2>&1; echo "rep $i rc $?"; tail -1 gpurun_out/rep$i.log; done
