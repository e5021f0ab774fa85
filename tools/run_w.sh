mkdir -p gpurun_out
timeout 1500 python bench.py --config c5_knn --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_c5_new.log 2>&1; echo "rc $?"; tail -1 gpurun_out/bench_c5_new.log | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['value'], r['ms_per_step'], r['roofline']['frac'], r['config'].get('phase_ms_rank0'), r['clocks'])"
