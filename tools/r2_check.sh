set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "compact or diameter or random" > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2_pytest.log
run() { tag=$1; shift; timeout 300 env "$@" python tests/run_config.py c3_rmat24 --clusters 256 --profile > gpurun_out/r2_v_$tag.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_v_$tag.log').read().splitlines()[-1]); print('$tag', round(j['cbfs_s'],3), {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items() if v['launches']})"; }
run cl X=1
run nocl CBFS_PULL_CL=0
run cl_conc1 CBFS_PULL_CL=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_pull|k_fold" -c 8 --csv --log-file gpurun_out/r2_ncu_cl.csv python tests/run_config.py c3_rmat24 --clusters 64 > /dev/null 2>&1; echo ncu $?
