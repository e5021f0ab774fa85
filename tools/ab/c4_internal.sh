# config 4 (locality relabel): sparse-engine staging by internal vs original id, digest-mode bench
set -eo pipefail
python -m pytest tests/test_gpu_consume.py -x -q -m gpu 2>&1 | tail -1
for n in orig:build_var/dint0 int:paper_2410_17226_b200 orig2:build_var/dint0 int2:paper_2410_17226_b200; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 900 python bench.py --config c4_grid --clusters 128 --steps 2 --warmup 1 --no-cpu --no-e2e --relabel locality > gpurun_out/r2_c4i_$k.log 2>&1
  python - $k << 'PY'
import json,sys
r=sys.argv[1]
l=[x for x in open(f"gpurun_out/r2_c4i_{r}.log") if x.startswith("{")][-1]
j=json.loads(l); c=j["config"]
print(r, round(j["value"]/1e9,1), "G", round(c["cbfs_ms_per_step"],1), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in j["roofline"]["per_kernel"].items()}, [k for k in c if 'gold' in k])
PY
done
