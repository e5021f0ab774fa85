for v in default e1c; do
  if [ $v = default ]; then unset CBFS_LIB_PATH; else export CBFS_LIB_PATH=build_var/$v/libcbfs.so; fi
  for c in 1 64; do
  python tests/run_config.py c4_grid --clusters $c --conc 1 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v c4 clusters $c', round(j['cbfs_s'],3), 'us/round', round(j['cbfs_s']/j['rounds_max']*1e6,1))"
  done
  python tests/run_config.py c5_knn --clusters 128 --conc 2 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v c5 128', j['cbfs_s'])"
done
