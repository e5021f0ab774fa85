mkdir -p gpurun_out
timeout 900 python tests/run_config.py c3_rmat24 --clusters 256 --profile > gpurun_out/c3p.log 2>&1; tail -1 gpurun_out/c3p.log | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print(r['cbfs_s'], r['source_edges_per_s']/1e12); print(json.dumps(r['kernels']))"
