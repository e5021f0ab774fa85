mkdir -p gpurun_out
for cfg in c1_er:16 c2_rmat20:64; do name=${cfg%%:*}; r=${cfg##*:}
 for sched in "200 1000" "1 1"; do timeout 900 python tools/pll_probe.py $name $r 4096 $sched 100000 > gpurun_out/pll_seq.log 2>&1; echo -n "$name r=$r sched=$sched: "; tail -1 gpurun_out/pll_seq.log | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['labels_per_vertex'], r['max_labels'], r['batches'], r['ms_pbfs'])"; done; done
