set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py tests/test_gpu_golden.py tests/test_gpu_wide.py -x -q -k "not c3 and not c5" > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/r2_pytest.log
timeout 600 python bench.py --config c2_rmat20 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_c2.log 2>&1; echo "c2 rc $?"; python -c "
import json;j=json.loads(open('gpurun_out/r2_bench_c2.log').read().splitlines()[-1]); print('c2', j['value']/1e12, j['ms_per_step'], j['config']['cbfs_ms_per_step'], j['gpu_launches'], {k:(v['event_ms_per_step'],v['launches_per_step']) for k,v in j['roofline']['per_kernel'].items()})"
timeout 300 python tests/run_config.py c3_rmat24 --clusters 256 --profile > gpurun_out/r2_c3_dev.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_c3_dev.log').read().splitlines()[-1]); print('c3dev', round(j['cbfs_s'],3), {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items() if v['launches']})"
