for v in default g3 g6 ilp8 ilp8m2 epl2 epl2ilp8 m4; do
  if [ $v = default ]; then unset CBFS_LIB_PATH; else export CBFS_LIB_PATH=build_var/$v/libcbfs.so; fi
  a=$(python tools/size_sweep.py 4096 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(j['s'],3), round(j['us_per_round'],1))")
  b=$(python tests/run_config.py c5_knn --clusters 128 --conc 2 | python -c "import json,sys;j=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(j['cbfs_s'],3))")
  echo "$v c4/64: $a  c5/128: $b"
done
