mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(round(r['ms_per_step'],2), r['config']['phase_ms_rank0'], round(r['roofline']['frac'],3), {k:v['event_ms_per_step'] for k,v in r['roofline']['per_kernel'].items()})"; }
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_skip$i.log 2>&1; echo -n "skip: "; summ gpurun_out/b_skip$i.log; done
CBFS_LIB_PATH=build_var/noskip/libcbfs.so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_noskip.log 2>&1; echo -n "noskip: "; summ gpurun_out/b_noskip.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/par.log 2>&1; echo "par rc $?"; tail -1 gpurun_out/par.log
