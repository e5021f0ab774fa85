timeout 900 python bench.py --config c4_grid --steps 2 --warmup 1 --e2e-steps 1 --e2e-warmup 0 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc $?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc $?"
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "c2 rc $?"
for f in c4 c2; do python -c "
import json;j=json.loads(open('gpurun_out/bench_$f.log').read().strip().splitlines()[-1]);print('$f', j['value'], j['ms_per_step'], j['config']['phase_ms_rank0'], round(j['roofline']['frac'],3), j['e2e']['value'] if j['e2e'] else None, j['cpu_baseline']['value'] if j['cpu_baseline'] else None)"; done
