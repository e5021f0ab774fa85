mkdir -p gpurun_out
(timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log)
tail -3 gpurun_out/pytest_gpu.log
for cfg in c4_grid c5_knn; do for conc in 1 2 4; do
timeout 300 python tests/run_config.py $cfg --clusters 256 --conc $conc > gpurun_out/${cfg}_256_$conc.log 2>&1
python -c "import json;j=json.loads(open('gpurun_out/${cfg}_256_$conc.log').read().strip().splitlines()[-1]);print('$cfg 256 conc $conc', j['cbfs_s'], j['source_edges_per_s']/1e9)"
done; done
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 9000 --launch-count 3 -f -o gpurun_out/sp3_c4 python tests/run_config.py c4_grid --clusters 64 --conc 1 > gpurun_out/ncu_sp_c4.log 2>&1
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 450 --launch-count 3 -f -o gpurun_out/sp3_c5 python tests/run_config.py c5_knn --clusters 64 --conc 1 > gpurun_out/ncu_sp_c5.log 2>&1
