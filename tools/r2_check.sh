set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random or diameter or c1_full or hint or edge" > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2_pytest.log
run() { tag=$1; shift; timeout 300 env "$@" python tests/run_config.py c3_rmat24 --clusters 2304 --first 2048 --profile > gpurun_out/r2_sm_$tag.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_sm_$tag.log').read().splitlines()[-1]); print('$tag', round(j['cbfs_s'],3), {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items() if v['launches']})"; }
run smask X=1
run sm6 CBFS_LIB_PATH=build_var/sm6/libcbfs.so
run smlp4 CBFS_LIB_PATH=build_var/smlp4/libcbfs.so
timeout 300 python tests/run_config.py c3_rmat24 --clusters 256 --profile > gpurun_out/r2_sm_first.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_sm_first.log').read().splitlines()[-1]); print('first256', round(j['cbfs_s'],3), {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items() if v['launches']})"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_pull|k_fold" --csv --log-file gpurun_out/r2_c3_mid_smask.csv env CBFS_BATCHED_HOSTLOOP=1 python tests/run_config.py c3_rmat24 --clusters 2112 --first 2048 > /dev/null 2>&1; echo "ncu $?"
