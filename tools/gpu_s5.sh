mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log)
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tests/run_config.py c4_grid --clusters 64 --conc 1 --profile > gpurun_out/c4_64.log 2>&1
python -c "import json;j=json.loads(open('gpurun_out/c4_64.log').read().strip().splitlines()[-1]);print('c4/64', j['cbfs_s'], j['source_edges_per_s']/1e9)"
timeout 300 python tests/run_config.py c5_knn --clusters 64 --conc 1 --profile > gpurun_out/c5_64.log 2>&1
python -c "import json;j=json.loads(open('gpurun_out/c5_64.log').read().strip().splitlines()[-1]);print('c5/64', j['cbfs_s'], j['source_edges_per_s']/1e9)"
timeout 600 python tests/run_config.py c4_grid --check 4 > gpurun_out/c4.log 2>&1
python -c "import json;j=json.loads(open('gpurun_out/c4.log').read().strip().splitlines()[-1]);print('c4', j['cbfs_s'], j['source_edges_per_s']/1e9, j['stats_match'], j['vectors_match'])"
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 9000 --launch-count 3 -f -o gpurun_out/sp2_c4 python tests/run_config.py c4_grid --clusters 64 --conc 1 > gpurun_out/ncu_sp_c4.log 2>&1
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 450 --launch-count 3 -f -o gpurun_out/sp2_c5 python tests/run_config.py c5_knn --clusters 64 --conc 1 > gpurun_out/ncu_sp_c5.log 2>&1
