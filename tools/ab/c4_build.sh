# locality build: determinism across builds in one process and timings in the bench context
python - << 'PY'
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import cbfs_inputs as ci, paper_2410_17226_b200 as cb
el = ci.make_graph("c4_grid")
s = torch.from_numpy(el.src.view(np.int32)).cuda(); d = torch.from_numpy(el.dst.view(np.int32)).cuda()
st = torch.cuda.current_stream()
perms = []
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = cb.cbfs_graph_create(el.n, s, d, cb.CBFS_RELABEL_LOCALITY, 0, st)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    perms.append(cb.cbfs_graph_internal_order(h))
    print(f"build {1e3*t:.1f} ms, equal to first: {np.array_equal(perms[0], perms[-1])}", flush=True)
    if rep == 1:  # occupy memory like the bench's slot pool
        big = torch.empty((100 * 2**30,), dtype=torch.uint8, device="cuda")
    cb.cbfs_graph_destroy(h)
PY
for r in 1 2; do
timeout 900 python bench.py --config c4_grid --clusters 128 --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -n 1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print('c4', j['config']['phase_ms_rank0'])"
done
