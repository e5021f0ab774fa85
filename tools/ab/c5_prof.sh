# config 5 after the sparse-engine change: bench on 1,024 clusters (query mode), ncu of one large push round
timeout 900 python bench.py --config c5_knn --clusters 1024 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r2_c5_1024.log 2>&1; echo rc $?
python - << 'PY'
import json
l=[x for x in open("gpurun_out/r2_c5_1024.log") if x.startswith("{")][-1]
j=json.loads(l); c=j["config"]
print(round(j["value"]/1e9,1), "G", round(j["ms_per_step"],1), c.get("phase_ms_rank0"), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in j["roofline"]["per_kernel"].items()})
PY
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sp_push --launch-skip 150 -c 1 -f -o gpurun_out/r2_c5_sppush python tests/run_config.py c5_knn --clusters 64 > gpurun_out/r2_c5_ncu.log 2>&1; echo rc $?
tail -3 gpurun_out/r2_c5_ncu.log
