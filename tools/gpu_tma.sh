for v in tma tma16; do
  export CBFS_LIB_PATH=build_var/$v/libcbfs.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or random or diameter" > gpurun_out/tma_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/tma_$v.log)"
  for r in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v', round(j['ms_per_step'],2), j['config']['phase_ms_rank0'])"; done
done
unset CBFS_LIB_PATH
for r in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('default', round(j['ms_per_step'],2), j['config']['phase_ms_rank0'])"; done
