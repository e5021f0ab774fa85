set -x
make -j8 all > gpurun_out/r2_make.log 2>&1 || { tail -30 gpurun_out/r2_make.log; exit 1; }
for rep in a b; do for cl in 1 0; do
CBFS_PULL_CL=$cl timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_ab_cl${cl}_$rep.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/r2_ab_cl${cl}_$rep.log').read().splitlines()[-1]); print('cl$cl$rep', round(j['value']/1e12,2), round(j['config']['cbfs_ms_per_step'],1), {k:(v['event_ms_per_step'],v['launches_per_step']) for k,v in j['roofline']['per_kernel'].items()})"
done; done
