"""Exact 2-hop oracle (PLL, NEXT-4) on a config's graph: r first-phase
clusters (the selection rule, d = 2), then batched pruned BFSs from the other
vertices; prints the paper's Table PLL columns (labels per vertex, index
size, C-BFS time, P-BFS time, total) and the query rate.

    python tools/pll_probe.py [config] [r] [cap] [first] [bmax] [queries]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402

a = sys.argv
name = a[1] if len(a) > 1 else "c2_rmat20"
r = int(a[2]) if len(a) > 2 else 64
cap = int(a[3]) if len(a) > 3 else 1024
first = int(a[4]) if len(a) > 4 else 200
bmax = int(a[5]) if len(a) > 5 else 1000
Q = int(a[6]) if len(a) > 6 else 1_000_000
cfg = ci.CONFIGS[name]
el = ci.make_graph(name)
dev = torch.device("cuda:0")
g = cb.Graph.from_edges(el.n, torch.from_numpy(el.src.view(np.int32)).to(dev),
                        torch.from_numpy(el.dst.view(np.int32)).to(dev), relabel=cfg.get("relabel", "none"))
src = torch.empty((max(r, 1), 64), dtype=torch.int32, device=dev)
sz = torch.empty((max(r, 1),), dtype=torch.uint8, device=dev)
got = cb.cbfs_select_clusters(g.h, r, 64, 2, cb.CBFS_ROOT_DEGREE, 0, src, sz) if r else 0
torch.cuda.synchronize()
t0 = time.perf_counter()
h = cb.cbfs_pll_build(g.h, src[:got].contiguous() if got else None, sz[:got].contiguous() if got else None, got, 2,
                      first, bmax, cap)
wall = time.perf_counter() - t0
info = cb.cbfs_pll_info(h)
n = g.n
s, t = ci.query_pairs(n, Q, seed=3, stream=4)
sd, td = torch.from_numpy(s.view(np.int32)).to(dev), torch.from_numpy(t.view(np.int32)).to(dev)
out = torch.empty((Q,), dtype=torch.int32, device=dev)
cb.cbfs_pll_query(h, sd, td, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cb.cbfs_pll_query(h, sd, td, out)
e1.record()
torch.cuda.synchronize()
qms = e0.elapsed_time(e1)
labels_phase2 = info["total_labels"]
cluster_bytes = got * (2 + 8 * 3) * n  # Delta u16 + d+1 subsets per vertex per cluster
index_bytes = labels_phase2 * 4 + cluster_bytes
print(json.dumps({"config": name, "n": n, "arcs": g.m, "r": got, "sources": int(sz[:got].sum().item()) if got else 0,
                  "labels_per_vertex": labels_phase2 / n, "max_labels": info["max_labels"],
                  "index_gb": index_bytes / 1e9, "roots": info["roots"], "batches": info["batches"],
                  "ms_cbfs": info["ms_cbfs"], "ms_pbfs": info["ms_pbfs"], "build_wall_s": wall,
                  "queries": Q, "query_ms": qms, "queries_per_s": Q / (qms / 1000.0),
                  "unreachable_frac": float((out == cb.CBFS_QUERY_UNREACHED).float().mean().item())}), flush=True)
cb.cbfs_pll_destroy(h)
g.close()
