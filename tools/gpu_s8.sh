mkdir -p gpurun_out
timeout 600 python tests/run_config.py c4_grid --check 8 --profile > gpurun_out/c4.log 2>&1
python -c "import json;j=json.loads(open('gpurun_out/c4.log').read().strip().splitlines()[-1]);print('c4', j['cbfs_s'], j['source_edges_per_s']/1e9, j['stats_match'], j['vectors_match'], j['kernels']['sparse'])"
timeout 900 python tests/run_config.py c5_knn --check 4 --profile > gpurun_out/c5.log 2>&1
python -c "import json;j=json.loads(open('gpurun_out/c5.log').read().strip().splitlines()[-1]);print('c5', j['cbfs_s'], j['source_edges_per_s']/1e9, j['stats_match'], j['vectors_match'], j['kernels']['sparse'], j['sumF_mean'])"
