# Round-2 measurement set: smoke, the default bench line (config 3) and the reference arm,
# bench lines of configs 2/4/5, the ncu launch list of one config-3 step and one ncu --set full k_pull capture.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2f_smoke.log
timeout 1200 python bench.py > gpurun_out/r2f_bench_c3.log 2>&1; echo "bench rc $?"
timeout 1200 python bench.py --impl reference > gpurun_out/r2f_ref_c3.log 2>&1; echo "reference rc $?"
timeout 900 python bench.py --config c2_rmat20 > gpurun_out/r2f_bench_c2.log 2>&1; echo "c2 rc $?"
timeout 900 python bench.py --config c4_grid --steps 2 > gpurun_out/r2f_bench_c4.log 2>&1; echo "c4 rc $?"
timeout 1500 python bench.py --config c5_knn --steps 1 --warmup 1 > gpurun_out/r2f_bench_c5.log 2>&1; echo "c5 rc $?"
CBFS_BATCHED_HOSTLOOP=1 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 3200 --csv --log-file gpurun_out/r2f_c3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-clocks > gpurun_out/r2f_c3_ncu_list.log 2>&1; echo "ncu list rc $?"
CBFS_BATCHED_HOSTLOOP=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_pull --launch-skip 97 -c 1 -f -o gpurun_out/r2f_c3_pull python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-clocks > gpurun_out/r2f_c3_ncu_full.log 2>&1; echo "ncu full rc $?"
for f in gpurun_out/r2f_bench_c3.log gpurun_out/r2f_ref_c3.log gpurun_out/r2f_bench_c2.log gpurun_out/r2f_bench_c4.log gpurun_out/r2f_bench_c5.log; do echo "== $f"; tail -n 1 $f | cut -c1-400; done
