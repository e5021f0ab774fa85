python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or random or c2_full" 2>&1 | tail -1
for v in default mlp12; do
  if [ $v = default ]; then unset CBFS_LIB_PATH; elif [ $v = old ]; then export CBFS_LIB_PATH=build_var/old_repo/paper_2410_17226_b200/libcbfs.so; else export CBFS_LIB_PATH=build_var/$v/libcbfs.so; fi
  for rep in 1 2; do
  python bench.py --no-e2e --no-cpu --engine 1 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v', round(j['ms_per_step'],2), j['config']['phase_ms_rank0'], round(j['roofline']['frac'],3))"
  done
done
