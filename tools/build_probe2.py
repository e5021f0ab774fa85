"""Slow graph build right after a traversal: is it time-dependent (background driver work)?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
el = ci.make_graph("c4_grid"); n = el.n
src_d = torch.from_numpy(el.src.view(np.int32)).cuda(); dst_d = torch.from_numpy(el.dst.view(np.int32)).cuda()
st = torch.cuda.current_stream()
def create(tag):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = cb.cbfs_graph_create(n, src_d, dst_d, 0, 0, st)
    torch.cuda.synchronize()
    print(f"{tag}: create {1000*(time.perf_counter()-t0):.1f} ms", flush=True)
    return h
ss = torch.empty((64, 64), dtype=torch.int32, device="cuda"); sz = torch.empty((64,), dtype=torch.uint8, device="cuda")
stats = torch.zeros((64, 4), dtype=torch.int64, device="cuda")
for sleep in (0.0, 0.0, 0.5, 2.0, 0.0):
    h = create("before run")
    cb.cbfs_select_clusters(h, 64, 64, 4, 1, 4, ss, sz, st)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cb.cbfs_run(h, ss, sz, 64, 4, 2, None, None, 5, stats)
    torch.cuda.synchronize(); print(f"  run {1000*(time.perf_counter()-t0):.0f} ms", flush=True)
    cb.cbfs_graph_destroy(h)
    time.sleep(sleep)
    cb.cbfs_graph_destroy(create(f"after run + sleep {sleep}"))
