"""Predicted scaling step time: one GPU doing rank (world-1)'s share of a
world x 1,024-cluster C2 step (graph build + overlapped selection + its
clusters' C-BFS) -- what every GPU of a world-rank run does, with no
inter-rank waiting in the data path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
el = ci.make_graph("c2_rmat20"); n = el.n; d = 2
src_d = torch.from_numpy(el.src.view(np.int32)).cuda(); dst_d = torch.from_numpy(el.dst.view(np.int32)).cuda()
st = torch.cuda.current_stream()
C = 1024
dist = torch.empty((n, C), dtype=torch.uint8, device="cuda"); masks = torch.empty((d + 1, n, C), dtype=torch.int64, device="cuda")
stats = torch.zeros((C, 4), dtype=torch.int64, device="cuda")
strong = (sys.argv[1] if len(sys.argv) > 1 else "strong") == "strong"
for world in (1, 2, 4, 8):
    r = C if strong else C * world
    src = torch.empty((r, 64), dtype=torch.int32, device="cuda"); sz = torch.empty((r,), dtype=torch.uint8, device="cuda")
    times = []
    for rep in range(4):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        e0.record(st)
        h = cb.cbfs_graph_create(n, src_d, dst_d, cb.CBFS_RELABEL_DEGREE, 0, st)
        e1.record(st)
        cb.cbfs_select_and_run_shard(h, r, 64, d, 0, 0, world, world - 1, src, sz, 1, dist, masks, d + 1, stats)
        e2.record(st)
        torch.cuda.synchronize()
        cb.cbfs_graph_destroy(h)
        if rep: times.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    b, s = np.mean(times, axis=0)
    Cr = len(range(world - 1, r, world))
    st_np = stats[:Cr].cpu().numpy()
    units = float((sz[world - 1::world][:Cr].cpu().numpy().astype(np.float64) * st_np[:, 3]).sum())
    print(f"{'strong' if strong else 'weak'} world {world}: build {b:.1f} ms, select+C-BFS {s:.1f} ms, "
          f"step {b + s:.1f} ms, rank units/s {units / ((b + s) / 1e3):.3e}", flush=True)
