# A/B of sparse-engine occupancy / ILP variants (128-256 clusters)
for cfg in c5_knn c4_grid; do
for n in new:paper_2410_17226_b200 dynm4:build_var/dynm4 dynm5:build_var/dynm5 dynm6:build_var/dynm6 dynm4e1:build_var/dynm4e1 dynm4i2:build_var/dynm4i2 dynm3i8:build_var/dynm3i8 dynm4b:build_var/dynm4; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 600 python tests/run_config.py $cfg --clusters 256 --reps 2 > gpurun_out/r2_sd_${cfg}_$k.log 2>&1
  echo $cfg $k $(python -c "
import json,sys
l=[x for x in open('gpurun_out/r2_sd_${cfg}_$k.log') if x.startswith('{')]
print([round(json.loads(x)['cbfs_s'],4) for x in l])")
done; done
