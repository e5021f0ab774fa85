# oracle goldens on the GPU box's host cores (oracle only; the GPU is idle until the check at the end):
# config 3 beyond its first 512 sampled clusters, config 5 clusters from the top of the selection;
# the golden files are copied back into gpurun_out/ every minute; then the whole-config golden tests
mkdir -p gpurun_out
N=$(nproc); T3=$(( N * 3 / 4 )); T5=$(( N - T3 )); echo "cores $N: c3 $T3, c5 $T5"
(timeout ${GOLD_SECS:-3900} python tests/make_goldens.py c3_rmat24 --sample 4096 --threads $T3 > gpurun_out/gold_c3.log 2>&1) &
P3=$!
(timeout ${GOLD_SECS:-3900} python tests/make_goldens.py c5_knn --no-queries --range ${C5_RANGE:-6400:8192} --threads $T5 > gpurun_out/gold_c5.log 2>&1) &
P5=$!
while kill -0 $P3 2>/dev/null || kill -0 $P5 2>/dev/null; do
  sleep 60
  cp tests/golden/c3_rmat24.golden.txt gpurun_out/c3_box.golden.txt; cp tests/golden/c5_knn.golden.txt gpurun_out/c5_box.golden.txt
done
cp tests/golden/c3_rmat24.golden.txt gpurun_out/c3_box.golden.txt; cp tests/golden/c5_knn.golden.txt gpurun_out/c5_box.golden.txt
tail -n 2 gpurun_out/gold_c3.log gpurun_out/gold_c5.log
grep -vc "^#" tests/golden/c3_rmat24.golden.txt tests/golden/c5_knn.golden.txt
timeout 900 python -m pytest tests/test_gpu_golden.py -q -m gpu -k "c3_whole or c5_whole" 2>&1 | tail -3
