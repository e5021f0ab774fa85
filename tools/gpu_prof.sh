mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/ncu_c2.log 2>&1; echo c2 $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pull|k_fold|k_push" --launch-count 9 -f -o gpurun_out/full_c2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/ncu_full_c2.log 2>&1; echo full $?
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sp_push --launch-skip 3000 --launch-count 2 -f -o gpurun_out/full_c4 python tests/run_config.py c4_grid --clusters 64 --conc 1 > gpurun_out/ncu_full_c4.log 2>&1; echo c4 $?
CBFS_SPARSE_HOSTLOOP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sp_push --launch-skip 150 --launch-count 2 -f -o gpurun_out/full_c5 python tests/run_config.py c5_knn --clusters 64 --conc 1 > gpurun_out/ncu_full_c5.log 2>&1; echo c5 $?
