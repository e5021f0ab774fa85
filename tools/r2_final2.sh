# final re-check after the late changes: full GPU suite, smoke, default bench, config-4 bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2f2_pytest.log 2>&1; echo "pytest rc $?"; tail -n 13 gpurun_out/r2f2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2f2_smoke.log 2>&1; echo "smoke rc $?"
timeout 1200 python bench.py > gpurun_out/r2f2_bench_c3.log 2>&1; echo "bench rc $?"
timeout 900 python bench.py --config c4_grid --steps 2 > gpurun_out/r2f2_bench_c4.log 2>&1; echo "c4 rc $?"
for f in gpurun_out/r2f2_bench_c3.log gpurun_out/r2f2_bench_c4.log; do tail -n 1 $f | python -c "
import json,sys; j=json.loads(sys.stdin.read()); c=j['config']; print(c['workload'], round(j['value']/1e12,3), 'T', round(j['ms_per_step'],1), c['phase_ms_rank0'], j.get('parity'), j['roofline']['frac'], j['roofline']['traffic'], (j.get('e2e') or {}).get('value'), j.get('clocks'))"; done
