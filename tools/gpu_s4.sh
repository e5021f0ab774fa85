mkdir -p gpurun_out
CBFS_SPARSE_HOSTLOOP=1 timeout 300 python tests/run_config.py c4_grid --clusters 64 --conc 1 --profile > gpurun_out/c4_64_host.log 2>&1
tail -c 300 gpurun_out/c4_64_host.log
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 9000 --launch-count 3 -f -o gpurun_out/sp_c4 python tests/run_config.py c4_grid --clusters 64 --conc 1 > gpurun_out/ncu_sp_c4.log 2>&1
tail -3 gpurun_out/ncu_sp_c4.log
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on -k regex:k_sp_ --launch-skip 450 --launch-count 3 -f -o gpurun_out/sp_c5 python tests/run_config.py c5_knn --clusters 64 --conc 1 > gpurun_out/ncu_sp_c5.log 2>&1
tail -3 gpurun_out/ncu_sp_c5.log
