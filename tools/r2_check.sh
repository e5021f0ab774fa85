set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
timeout 600 python tools/sanitize_cases.py > gpurun_out/r2_cases_plain.log 2>&1; echo "plain cases rc $?"; tail -2 gpurun_out/r2_cases_plain.log
CBFS_LIB_PATH=build_var/checks/libcbfs.so timeout 600 python tools/sanitize_cases.py > gpurun_out/r2_checks_cases.log 2>&1; echo "checks rc $?"; tail -2 gpurun_out/r2_checks_cases.log
CBFS_TRACE=1 timeout 900 python bench.py --config c4_grid --clusters 64 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_bench_c4_64.log 2>&1; grep "cbfs trace" gpurun_out/r2_bench_c4_64.log; python -c "
import json;j=json.loads(open('gpurun_out/r2_bench_c4_64.log').read().splitlines()[-1]); print('c4digest64', j['config']['cbfs_ms_per_step'], {k:(v['event_ms_per_step'],v['launches_per_step']) for k,v in j['roofline']['per_kernel'].items()})"
run() { tag=$1; cfg=$2; shift; shift; timeout 600 env "$@" python tests/run_config.py $cfg --clusters 128 --profile > gpurun_out/r2_sv_$tag.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_sv_$tag.log').read().splitlines()[-1]); print('$tag', round(j['cbfs_s'],3), {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items() if v['launches']})"; }
for v in base spm4 spm4i2 spm2i8 spg16; do
  if [ $v = base ]; then L=X=1; else L=CBFS_LIB_PATH=build_var/$v/libcbfs.so; fi
  run c4_$v c4_grid $L
  run c5_$v c5_knn $L
done
