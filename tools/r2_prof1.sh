set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
timeout 300 python tests/run_config.py c3_rmat24 --clusters 256 --profile > gpurun_out/r2_c3_256.log 2>&1; echo rc $?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r2_c3_64_launches.csv python tests/run_config.py c3_rmat24 --clusters 64 > gpurun_out/r2_c3_64_ncu.log 2>&1; echo rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pull -c 2 -f -o gpurun_out/r2_c3_pull python tests/run_config.py c3_rmat24 --clusters 64 > gpurun_out/r2_c3_pull_ncu.log 2>&1; echo rc $?
