# config 4 under the locality relabel vs none: stats-only C-BFS and the digest-mode bench (outputs consumed)
for r in 0 8; do
  timeout 600 python tests/run_config.py c4_grid --clusters 256 --reps 2 --relabel $r > gpurun_out/r2_c4r_$r.log 2>&1
  echo relabel $r $(python -c "
import json
l=[x for x in open('gpurun_out/r2_c4r_$r.log') if x.startswith('{')]
print([round(json.loads(x)['cbfs_s'],4) for x in l])")
done
for r in none locality; do
  timeout 900 python bench.py --config c4_grid --clusters 128 --steps 2 --warmup 1 --no-cpu --no-e2e --relabel $r > gpurun_out/r2_c4b_$r.log 2>&1
  python - $r << 'PY'
import json,sys
r=sys.argv[1]
l=[x for x in open(f"gpurun_out/r2_c4b_{r}.log") if x.startswith("{")][-1]
j=json.loads(l); c=j["config"]
print(r, round(j["value"]/1e9,1), "G", round(c["cbfs_ms_per_step"],1), c.get("golden"), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in j["roofline"]["per_kernel"].items()})
PY
done
