# one large config-4 push round under ncu --set full (final code: locality order, dynamic chunks)
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sp_push --launch-skip 3000 -c 1 -f -o gpurun_out/r2_c4_sppush2 python tests/run_config.py c4_grid --clusters 64 > gpurun_out/r2_c4_ncu2.log 2>&1; echo rc $?
tail -n 2 gpurun_out/r2_c4_ncu2.log | cut -c1-300
