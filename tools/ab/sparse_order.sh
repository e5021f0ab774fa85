# ordered (bitmap-compacted) frontiers in the sparse engine: parity, goldens, timings vs the committed code
set -eo pipefail
python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py tests/test_gpu_wide.py -x -q -m gpu 2>&1 | tail -2
CBFS_SP_BM_MIN=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py -x -q -m gpu 2>&1 | tail -2
python -m pytest tests/test_gpu_golden.py -x -q -m gpu -k "c4 or c5" 2>&1 | tail -2
for cfg in c5_knn c4_grid; do
for n in head:build_var/head new:paper_2410_17226_b200 head2:build_var/head new2:paper_2410_17226_b200; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 600 python tests/run_config.py $cfg --clusters 256 --reps 2 > gpurun_out/r2_so_${cfg}_$k.log 2>&1
  echo $cfg $k $(python -c "
import json,sys
l=[x for x in open('gpurun_out/r2_so_${cfg}_$k.log') if x.startswith('{')]
print([round(json.loads(x)['cbfs_s'],4) for x in l])")
done; done
timeout 900 python bench.py --config c5_knn --clusters 1024 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_c5_1024b.log 2>&1; echo rc $?
python - << 'PY'
import json
l=[x for x in open("gpurun_out/r2_c5_1024b.log") if x.startswith("{")][-1]
j=json.loads(l); c=j["config"]
print(round(j["value"]/1e9,1), "G", round(j["ms_per_step"],1), c.get("phase_ms_rank0"), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in j["roofline"]["per_kernel"].items()})
PY
