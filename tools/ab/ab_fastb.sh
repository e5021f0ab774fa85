# pull pass-B row-id / policy rewrite: parity, then config-3 bench A/B
set -e
python -m pytest tests/test_gpu_parity.py tests/test_gpu_consume.py -x -q -m gpu 2>&1 | tail -2
python -m pytest tests/test_gpu_golden.py -x -q -m gpu -k "c2 or c3" 2>&1 | tail -2
for n in fb0:build_var/fb0 new:paper_2410_17226_b200 fb0b:build_var/fb0 new2:paper_2410_17226_b200; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_ab_$k.log 2>&1
  python - $k << 'PY'
import json,sys
k=sys.argv[1]
l=[x for x in open(f"gpurun_out/r2_ab_{k}.log") if x.startswith("{")][-1]
j=json.loads(l); pk=j["roofline"]["per_kernel"]
print(k, round(j["value"]/1e12,2), round(j["config"]["cbfs_ms_per_step"],1), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in pk.items()})
PY
done
