"""Does a locality-preserving vertex order (BFS order from vertex 0, computed on
the host with scipy) speed up the sparse engine on the k-NN graph?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order, reverse_cuthill_mckee
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
el = ci.make_graph("c5_knn"); n = el.n
A = sp.coo_matrix((np.ones(len(el.src), np.int8), (el.src.astype(np.int64), el.dst.astype(np.int64))), shape=(n, n)).tocsr()
A = A + A.T
t0 = time.perf_counter()
order = breadth_first_order(A, 0, directed=False, return_predecessors=False)
print("bfs order", time.perf_counter() - t0, len(order), flush=True)
rest = np.setdiff1d(np.arange(n), order)
order = np.concatenate([order, rest])
newid = np.empty(n, np.uint32); newid[order] = np.arange(n, dtype=np.uint32)
variants = {"original": (el.src, el.dst), "bfs_order": (newid[el.src], newid[el.dst])}
for name, (s, t) in variants.items():
    g = cb.Graph.from_edges(n, torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(t.view(np.int32)).cuda())
    src, sz = g.select_clusters(128, 64, 6)
    stats = torch.zeros((128, 4), dtype=torch.int64, device="cuda")
    cb.cbfs_run(g.h, src, sz, 128, 6, 2, None, None, 7, stats)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cb.cbfs_run(g.h, src, sz, 128, 6, 2, None, None, 7, stats)
    torch.cuda.synchronize()
    st = stats.cpu().numpy()
    print(name, round(time.perf_counter() - t0, 3), "s", "sumE", st[:, 2].sum(), flush=True)
    g.close()
