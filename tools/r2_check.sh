set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
run() { tag=$1; shift; timeout 300 env "$@" python tests/run_config.py c3_rmat24 --clusters 256 --profile > gpurun_out/r2_v_$tag.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_v_$tag.log').read().splitlines()[-1]); print('$tag', round(j['cbfs_s'],3), {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items() if v['launches']})"; }
run hint64 X=1
run nohint CBFS_LIB_PATH=build_var/nohint/libcbfs.so
run hint32 CBFS_PULL_HUB_MB=32
run hint96 CBFS_PULL_HUB_MB=96
run hint0 CBFS_PULL_HUB_MB=0
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r2_bench_c3.log 2>&1; echo "bench rc $?"; python -c "
import json;j=json.loads(open('gpurun_out/r2_bench_c3.log').read().splitlines()[-1]); print('c3', j['value']/1e12, j['ms_per_step'], j['config']['cbfs_ms_per_step'], j['parity'], {k:(v['event_ms_per_step'],v['launches_per_step']) for k,v in j['roofline']['per_kernel'].items()})"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py tests/test_gpu_golden.py -x -q -k "not c3 and not c5" > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2_pytest.log
