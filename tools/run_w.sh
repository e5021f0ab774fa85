mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_ado.py tests/test_gpu_distributed.py -q -x > gpurun_out/init.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/init.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b_init$i.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/b_init$i.log | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['value'], r['ms_per_step'], r['roofline']['frac'], r['e2e']['value'], r.get('phases_ms'))"; done
