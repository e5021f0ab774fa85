"""Sparse engine: cost of writing the output vectors (C5, 128 clusters)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
cfg = ci.CONFIGS["c5_knn"]; el = ci.make_graph("c5_knn"); n = el.n; d = cfg["d"]
g = cb.Graph.from_edges(n, torch.from_numpy(el.src.view(np.int32)).cuda(), torch.from_numpy(el.dst.view(np.int32)).cuda())
src, sz = g.select_clusters(128, 64, d)
C = 128
stats = torch.zeros((C, 4), dtype=torch.int64, device="cuda")
for label, planes, want in (("stats", d + 1, False), ("dist+7 planes", d + 1, True), ("dist+6 planes", d, True), ("stats", d + 1, False)):
    dist = torch.empty((n, C), dtype=torch.int16, device="cuda") if want else None
    masks = torch.empty((planes, n, C), dtype=torch.int64, device="cuda") if want else None
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cb.cbfs_run(g.h, src, sz, C, d, 2, dist, masks, planes, stats)
    torch.cuda.synchronize()
    print(f"{label}: {time.perf_counter() - t0:.3f} s", flush=True)
    del dist, masks
