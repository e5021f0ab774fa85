# config 3: concurrent batches 1 / 2 (default) / 3
for c in 1 0 3; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --concurrency $c > gpurun_out/r2_conc_$c.log 2>&1
tail -n 1 gpurun_out/r2_conc_$c.log | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('conc $c', round(j['value']/1e12,2), round(j['config']['cbfs_ms_per_step'],1), {a:(b['event_ms_per_step']) for a,b in j['roofline']['per_kernel'].items()})"
done
