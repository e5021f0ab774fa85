mkdir -p gpurun_out
echo new; timeout 600 python tools/build_probe.py c3_rmat24 2 2>&1 | head -4
echo old; CBFS_LIB_PATH=build_var/old/libcbfs.so timeout 600 python tools/build_probe.py c3_rmat24 2 2>&1 | head -4
