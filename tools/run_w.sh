mkdir -p gpurun_out
for m in query stats; do timeout 900 python bench.py --config c5_knn --clusters 512 --mode $m --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/c5_$m.log 2>&1; echo "$m rc $?"; tail -1 gpurun_out/c5_$m.log | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['ms_per_step'], r['config'].get('phase_ms_rank0'))"; done
