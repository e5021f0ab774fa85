"""Time cbfs_graph_create for a config, alone and after a traversal (bench-like)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
name = sys.argv[1]
el = ci.make_graph(name); n = el.n
src_d = torch.from_numpy(el.src.view(np.int32)).cuda(); dst_d = torch.from_numpy(el.dst.view(np.int32)).cuda()
st = torch.cuda.current_stream()
def create():
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h = cb.cbfs_graph_create(n, src_d, dst_d, int(sys.argv[2]) if len(sys.argv) > 2 else 0, 0, st)
    e1.record(st); torch.cuda.synchronize()
    print(f"create: host {1000*(time.perf_counter()-t0):.1f} ms, events {e0.elapsed_time(e1):.1f} ms", flush=True)
    return h
for _ in range(3):
    cb.cbfs_graph_destroy(create())
h = create()
ss = torch.empty((64, 64), dtype=torch.int32, device="cuda"); sz = torch.empty((64,), dtype=torch.uint8, device="cuda")
cb.cbfs_select_clusters(h, 64, 64, 4, 1, 4, ss, sz, st)
stats = torch.zeros((64, 4), dtype=torch.int64, device="cuda")
cb.cbfs_run(h, ss, sz, 64, 4, 2, None, None, 5, stats)
cb.cbfs_graph_destroy(h)
for _ in range(2):
    cb.cbfs_graph_destroy(create())
print("--- second run with the slots already allocated")
h = create()
cb.cbfs_run(h, ss, sz, 64, 4, 2, None, None, 5, stats)
cb.cbfs_graph_destroy(h)
cb.cbfs_graph_destroy(create())
print("--- forced sparse engine (no probe)")
cb.cbfs_set_engine(cb.CBFS_ENGINE_SPARSE)
h = create()
cb.cbfs_run(h, ss, sz, 64, 4, 2, None, None, 5, stats)
cb.cbfs_graph_destroy(h)
cb.cbfs_graph_destroy(create())
