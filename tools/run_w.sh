mkdir -p gpurun_out
CBFS_LIB_PATH=build_var/dbg/libcbfs.so timeout 600 python tools/pull_stats.py > gpurun_out/pstats.log 2>&1; tail -3 gpurun_out/pstats.log | cut -c1-400
