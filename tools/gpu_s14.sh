python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_ado.py -m gpu -x -q > gpurun_out/p14.log 2>&1; tail -1 gpurun_out/p14.log
python tests/run_config.py c4_grid --clusters 128 --conc 2 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('c4 none', j['cbfs_s'])"
python tests/run_config.py c4_grid --clusters 128 --conc 2 --relabel 8 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('c4 locality', j['cbfs_s'])"
timeout 1200 python bench.py --config c5_knn --steps 1 --warmup 1 --e2e-steps 1 --e2e-warmup 0 --no-cpu > gpurun_out/bench_c5.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/bench_c5.log').read().strip().splitlines()[-1]);print('c5', j['value']/1e9, j['ms_per_step'], j['config']['phase_ms_rank0'], j['roofline']['frac'])"
