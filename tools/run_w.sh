mkdir -p gpurun_out
run() { CBFS_LIB_PATH=$2 timeout 900 python bench.py --config $1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks $3 > gpurun_out/sp.log 2>&1; tail -1 gpurun_out/sp.log | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(round(r['ms_per_step'],1), r['config'].get('phase_ms_rank0')['cbfs'])"; }
for v in base mb4 ilp8 epl4 g12 ilp2mb4; do lib=build_var/$v/libcbfs.so; [ $v = base ] && lib=paper_2410_17226_b200/libcbfs.so; echo -n "$v c4: "; run c4_grid $lib ""; echo -n "$v c5/512: "; run c5_knn $lib "--clusters 512"; done
