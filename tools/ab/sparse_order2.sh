# ordered-frontier threshold sweep (CBFS_SP_BM_MIN) on configs 5 and 4
for cfg in c5_knn c4_grid; do
for bm in 1 100000 600000 2500000 0; do
  CBFS_SP_BM_MIN=$bm timeout 600 python tests/run_config.py $cfg --clusters 256 --reps 2 > gpurun_out/r2_sb_${cfg}_$bm.log 2>&1
  echo $cfg $bm $(python -c "
import json,sys
l=[x for x in open('gpurun_out/r2_sb_${cfg}_$bm.log') if x.startswith('{')]
print([round(json.loads(x)['cbfs_s'],4) for x in l])")
done; done
