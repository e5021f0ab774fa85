# digest consumer: skip the subset loads of unreached staging entries (CBFS_DG_SKIP) — parity, then A/B on config 3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_consume.py tests/test_gpu_golden.py -x -q -m gpu 2>&1 | tail -2
for n in skip:paper_2410_17226_b200 noskip:build_var/noskip skip2:paper_2410_17226_b200 noskip2:build_var/noskip; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_ab_$k.log 2>&1
  python - $k << 'PY'
import json,sys
k=sys.argv[1]
l=[x for x in open(f"gpurun_out/r2_ab_{k}.log") if x.startswith("{")][-1]
j=json.loads(l); pk=j["roofline"]["per_kernel"]
print(k, round(j["value"]/1e12,2), round(j["config"]["cbfs_ms_per_step"],1), j.get("parity"), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in pk.items()})
PY
done
