# config-5 golden lines on the GPU box's host cores (oracle only): clusters [4096, 8192) of the selection,
# stats + digests; the golden file is copied back into gpurun_out/ every minute
N=$(nproc); echo "cores $N"
(timeout ${GOLD_SECS:-5000} python tests/make_goldens.py c5_knn --no-queries --range ${GOLD_RANGE:-4096:8192} --threads $N > gpurun_out/gold_box.log 2>&1) &
P=$!
while kill -0 $P 2>/dev/null; do sleep 60; cp tests/golden/c5_knn.golden.txt gpurun_out/c5_box.golden.txt; done
cp tests/golden/c5_knn.golden.txt gpurun_out/c5_box.golden.txt
tail -n 3 gpurun_out/gold_box.log
