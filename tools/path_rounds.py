"""Per-round fixed cost of the sparse engine: a path graph, one source (1 frontier entry per round)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_17226_b200 as cb
n = 60000
s = np.arange(n - 1, dtype=np.uint32); t = s + 1
g = cb.Graph.from_edges(n, s, t)
cb.cbfs_set_engine(cb.CBFS_ENGINE_SPARSE)
src = torch.full((1, 64), -1, dtype=torch.int32, device="cuda"); src[0, 0] = 0
sz = torch.ones((1,), dtype=torch.uint8, device="cuda")
for d in (1, 0):
    for rep in range(2):
        stats = torch.zeros((1, 4), dtype=torch.int64, device="cuda")
        torch.cuda.synchronize(); t0 = time.perf_counter()
        cb.cbfs_run(g.h, src, sz, 1, d, 2, None, None, d + 1, stats)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        r = int(stats[0, 0])
        print(f"d={d} rounds {r}: {dt * 1e6 / r:.2f} us per round", flush=True)
