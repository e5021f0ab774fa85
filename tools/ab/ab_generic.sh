# ab_generic.sh "TESTS" name:libdir ... — parity tests with the default library, then config-3 bench A/B in the given order
mkdir -p gpurun_out
T="$1"; shift
if [ -n "$T" ]; then timeout 1200 python -m pytest $T -x -q -m gpu 2>&1 | tail -2; fi
for n in "$@"; do
  k=${n%%:*}; d=${n#*:}
  CBFS_LIB_PATH=$d/libcbfs.so timeout 600 python bench.py --steps ${AB_STEPS:-2} --warmup ${AB_WARM:-2} --no-cpu --no-e2e $AB_ARGS > gpurun_out/r2_ab_$k.log 2>&1
  python - $k << 'PY'
import json,sys
k=sys.argv[1]
try:
    l=[x for x in open(f"gpurun_out/r2_ab_{k}.log") if x.startswith("{")][-1]
except IndexError:
    print(k, "FAILED", open(f"gpurun_out/r2_ab_{k}.log").read()[-600:]); sys.exit()
j=json.loads(l); pk=j["roofline"]["per_kernel"]
print(k, round(j["value"]/1e12,3), round(j["config"]["cbfs_ms_per_step"],1), (j.get("parity") or {}).get("match"), {a:(b["event_ms_per_step"],b["launches_per_step"]) for a,b in pk.items()})
PY
done
