# A/B of sparse-engine variants on configs 4 and 5 (128 clusters each), after the sparse parity tests
set -e
python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py -x -q -m gpu -k "random or sparse or diameter or edge or c1_full" 2>&1 | tail -2
python -m pytest tests/test_gpu_golden.py -x -q -m gpu -k "c4" 2>&1 | tail -2
for cfg in c5_knn c4_grid; do
for n in dyn0:build_var/dyn0 new:paper_2410_17226_b200 dynm4:build_var/dynm4 dynm2:build_var/dynm2 new2:paper_2410_17226_b200 dyn0b:build_var/dyn0; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 600 python tests/run_config.py $cfg --clusters 256 --reps 2 > gpurun_out/r2_sd_${cfg}_$k.log 2>&1
  echo $cfg $k $(python -c "
import json,sys
l=[x for x in open('gpurun_out/r2_sd_${cfg}_$k.log') if x.startswith('{')]
print([round(json.loads(x)['cbfs_s'],4) for x in l])")
done; done
