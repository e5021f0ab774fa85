python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for v in default minb3 minb2; do
  if [ $v = default ]; then unset CBFS_LIB_PATH; else export CBFS_LIB_PATH=build_var/$v/libcbfs.so; fi
  echo "== $v"; python tools/size_sweep.py 4096 | cut -c1-200
  python tests/run_config.py c5_knn --clusters 128 --conc 2 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('c5 128', j['cbfs_s'], j['source_edges_per_s']/1e9)"
done
