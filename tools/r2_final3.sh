# final re-check after the pull chunk / pass-A changes: GPU suite, smoke, default bench, ncu launch list of one
# config-3 step and ncu --set full of a first dense round of the pull (kernel replay)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2f3_pytest.log 2>&1; echo "pytest rc $?"; tail -n 13 gpurun_out/r2f3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2f3_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2f3_smoke.log
timeout 1200 python bench.py > gpurun_out/r2f3_bench_c3.log 2>&1; echo "bench rc $?"; tail -n 1 gpurun_out/r2f3_bench_c3.log | cut -c1-400
CBFS_BATCHED_HOSTLOOP=1 timeout 1800 ncu --replay-mode application --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3400 --csv --log-file gpurun_out/r2f3_c3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-clocks > gpurun_out/r2f3_c3_ncu_list.log 2>&1; echo "ncu list rc $?"
python tools/launch_list.py gpurun_out/r2f3_c3_launches.csv > gpurun_out/r2f3_c3_launches.md 2>&1; head -20 gpurun_out/r2f3_c3_launches.md
CBFS_BATCHED_HOSTLOOP=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_pull --launch-skip 90 -c 1 -f -o gpurun_out/r2f3_c3_pull python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-clocks > gpurun_out/r2f3_c3_ncu_full.log 2>&1; echo "ncu full rc $?"
