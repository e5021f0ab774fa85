mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(round(r['ms_per_step'],2), r['config']['phase_ms_rank0'], round(r['roofline']['frac'],3), {k:v['event_ms_per_step'] for k,v in r['roofline']['per_kernel'].items()})"; }
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_base$i.log 2>&1; echo -n "base: "; summ gpurun_out/b_base$i.log; 
for v in ff1 ff2; do CBFS_LIB_PATH=build_var/$v/libcbfs.so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$v.log 2>&1; echo -n "$v: "; summ gpurun_out/b_$v.log; done; done
CBFS_LIB_PATH=build_var/ff1/libcbfs.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random or config1" > gpurun_out/par_ff.log 2>&1; echo "par ff1 rc $?"; tail -1 gpurun_out/par_ff.log
