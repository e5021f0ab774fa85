# runtime knobs on config 3 with the final library: hub-row L2 window (CBFS_PULL_HUB_MB), alpha, concurrency
mkdir -p gpurun_out
run() { k=$1; shift; env "$@" timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e $KARGS > gpurun_out/r2_kn_$k.log 2>&1
  python - $k << 'PY'
import json,sys
k=sys.argv[1]
l=[x for x in open(f"gpurun_out/r2_kn_{k}.log") if x.startswith("{")]
if not l: print(k,"FAILED"); sys.exit()
j=json.loads(l[-1]); pk=j["roofline"]["per_kernel"]
print(k, round(j["value"]/1e12,3), round(j["config"]["cbfs_ms_per_step"],1), (j.get("parity") or {}).get("match"), {a:b["event_ms_per_step"] for a,b in pk.items()})
PY
}
run base X=1
run hub32 CBFS_PULL_HUB_MB=32
run hub96 CBFS_PULL_HUB_MB=96
run hub128 CBFS_PULL_HUB_MB=128
KARGS="--alpha 50" run a50 X=1
KARGS="--alpha 200" run a200 X=1
KARGS="--concurrency 1" run conc1 X=1
run base2 X=1
