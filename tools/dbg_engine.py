"""Debug helper: one grid case under each engine; prints which clusters mismatch the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import cbfs_inputs as ci
import oracle as orc
import paper_2410_17226_b200 as cb
from gpu_util import gpu_graph, run_clusters

el = ci.grid(200, 0.05, 0.001, 7)
d = 4
ref = orc.csr_from_edgelist(el)
src, sz = orc.select_clusters(ref, 100, 64, d)
om = orc.cluster_bfs_many(ref, src, sz, d, threads=8)
cb.cbfs_profile_enable(True)
for conc in (4, 1):
    cb.cbfs_set_concurrency(conc)
    for eng in (cb.CBFS_ENGINE_SPARSE, cb.CBFS_ENGINE_BATCHED, cb.CBFS_ENGINE_AUTO):
        g = gpu_graph(el)
        cb.cbfs_set_engine(eng)
        gd, gs, gst = run_clusters(g, src, sz, d)
        bad = [c for c in range(len(sz)) if not np.array_equal(gd[c], om["dist"][c])]
        print("conc", conc, "engine", eng, "bad clusters", bad[:10], len(bad), flush=True)
        g.close()
