# ordered-frontier parity test, then the scaling probe for configs 4 and 5
set -o pipefail
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "ordered" 2>&1 | tail -1
timeout 900 python tools/shard_probe.py c4_grid 1 2 4 8 2>&1 | grep "N=" | tee gpurun_out/r2_shard_c4.log
timeout 1500 python tools/shard_probe.py c5_knn 1 4 8 2>&1 | grep "N=" | tee gpurun_out/r2_shard_c5.log
