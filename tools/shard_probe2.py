"""Traversal cost of rank (world-1)'s clusters vs the first 1,024 (C2), selection excluded."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
el = ci.make_graph("c2_rmat20"); n = el.n; d = 2
g = cb.Graph.from_edges(n, torch.from_numpy(el.src.view(np.int32)).cuda(), torch.from_numpy(el.dst.view(np.int32)).cuda(), relabel=True)
src, sz = g.select_clusters(8192, 64, d)
C = 1024
dist = torch.empty((n, C), dtype=torch.uint8, device="cuda"); masks = torch.empty((d + 1, n, C), dtype=torch.int64, device="cuda")
stats = torch.zeros((C, 4), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for world in (1, 2, 4, 8):
    s_r = src[world - 1::world][:C].contiguous(); z_r = sz[world - 1::world][:C].contiguous()
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); cb.cbfs_run(g.h, s_r, z_r, C, d, 1, dist, masks, d + 1, stats); e1.record(st)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    s = stats.cpu().numpy()
    units = float((z_r.cpu().numpy().astype(np.float64) * s[:, 3]).sum())
    print(f"world {world}: C-BFS {np.mean(ts[1:]):.1f} ms, mean k {z_r.float().mean().item():.1f}, rounds max {s[:,0].max()}, units/s {units/np.mean(ts[1:])*1e3:.3e}", flush=True)
