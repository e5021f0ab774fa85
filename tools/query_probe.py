"""Time the label query kernel on config 5 (64 clusters, 10M queries), cold best and warm best."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
cfg = ci.CONFIGS["c5_knn"]; el = ci.make_graph("c5_knn"); n = el.n; d = cfg["d"]
g = cb.Graph.from_edges(n, torch.from_numpy(el.src.view(np.int32)).cuda(), torch.from_numpy(el.dst.view(np.int32)).cuda())
src, sz = g.select_clusters(128, 64, d)
s, t = ci.query_pairs(n, cfg["queries"], cfg["query_seed"])
sd = torch.from_numpy(s.view(np.int32)).cuda(); td = torch.from_numpy(t.view(np.int32)).cuda()
for planes in (d + 1, d):
    dist, masks, _ = g.run(src[:64].contiguous(), sz[:64].contiguous(), d, dist_bytes=2, planes=planes)
    dist2, masks2, _ = g.run(src[64:128].contiguous(), sz[64:128].contiguous(), d, dist_bytes=2, planes=planes)
    best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda")
    for label, (D, M, Z) in (("cold", (dist, masks, sz[:64])), ("warm", (dist2, masks2, sz[64:128])), ("again", (dist2, masks2, sz[64:128]))):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        cb.cbfs_query_distance(n, 64, d, planes, D, 2, M, Z.contiguous(), sd, td, best)
        torch.cuda.synchronize()
        print(f"planes {planes} {label}: {1000 * (time.perf_counter() - t0):.1f} ms", flush=True)
