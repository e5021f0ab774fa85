for r in 1 2; do
CBFS_TRACE=1 timeout 900 python bench.py --config c4_grid --steps 2 --no-cpu --no-e2e > gpurun_out/r2_c4full_$r.log 2>&1
tail -n 1 gpurun_out/r2_c4full_$r.log | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('c4', round(j['value']/1e9,1), j['config']['phase_ms_rank0'], {a:(b['event_ms_per_step'],b['launches_per_step']) for a,b in j['roofline']['per_kernel'].items()})"
grep "cbfs trace" gpurun_out/r2_c4full_$r.log | tail -4
done
