mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ado.py tests/test_gpu_distributed.py -q -x > gpurun_out/w_ado.log 2>&1; echo "ado rc $?"; tail -3 gpurun_out/w_ado.log
WS=0,64,32,16,8 timeout 900 python tools/eval_distortion.py c2_rmat20 100000 1024 > gpurun_out/w_dist_c2.log 2>&1; echo "dist rc $?"
WS=0,64,8 timeout 900 python tools/eval_distortion.py c5_knn 3000 1024 > gpurun_out/w_dist_c5.log 2>&1; echo "dist5 rc $?"
WS=0,64,8 timeout 900 python tools/eval_distortion.py c4_grid 2000 1024 > gpurun_out/w_dist_c4.log 2>&1; echo "dist4 rc $?"
cut -c1-200 gpurun_out/w_dist_c*.log
