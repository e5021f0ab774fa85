# sparse engine after a change: parity (both push shapes), goldens of configs 4 and 5, timings at 256 clusters
set -e
python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py tests/test_gpu_wide.py -x -q -m gpu 2>&1 | tail -2
python -m pytest tests/test_gpu_golden.py -x -q -m gpu -k "c4 or c5" 2>&1 | tail -2
for cfg in c5_knn c4_grid; do
for n in dyn0:build_var/dyn0 new:paper_2410_17226_b200; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 600 python tests/run_config.py $cfg --clusters 256 --reps 2 > gpurun_out/r2_sc_${cfg}_$k.log 2>&1
  echo $cfg $k $(python -c "
import json,sys
l=[x for x in open('gpurun_out/r2_sc_${cfg}_$k.log') if x.startswith('{')]
print([round(json.loads(x)['cbfs_s'],4) for x in l])")
done; done
