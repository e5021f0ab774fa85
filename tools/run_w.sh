mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -q -x -k "query or stream" > gpurun_out/q.log 2>&1; echo "q rc $?"; tail -1 gpurun_out/q.log
for xp in cm CBFS_QUERY_VMAJOR; do for Q in 10000000; do env $xp=1 timeout 900 python bench.py --config c5_knn --clusters 512 --mode query --queries $Q --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/xq_$xp$Q.log 2>&1; echo -n "$xp Q=$Q: "; tail -1 gpurun_out/xq_$xp$Q.log | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['ms_per_step'], r['config'].get('phase_ms_rank0'))"; done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k c5 > gpurun_out/q5.log 2>&1; echo "c5 rc $?"; tail -1 gpurun_out/q5.log
