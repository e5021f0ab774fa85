"""Time the greedy selection alone (config 2, r clusters)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
el = ci.make_graph("c2_rmat20")
g = cb.Graph.from_edges(el.n, torch.from_numpy(el.src.view(np.int32)).cuda(), torch.from_numpy(el.dst.view(np.int32)).cuda(), relabel=True)
for r in (1024, 8192):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        src, sz = g.select_clusters(r, 64, 2)
        torch.cuda.synchronize()
        if rep: print(f"r={r}: {1000*(time.perf_counter()-t0):.1f} ms, {1e6*(time.perf_counter()-t0)/r:.2f} us/cluster", flush=True)
