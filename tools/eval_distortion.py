"""Distortion of the C-BFS landmark-label ADO.

    [TAUS=0,64] [WS=0,64,32,16,8] python tools/eval_distortion.py [config] [pairs] [budget_bytes] [d]

Index: the paper's memory budget per vertex (a record is
1 + d * w / 8 bytes, r = floor(budget / record) clusters of up to w
sources, in a label store of word size w), clusters selected by the
config's rule; pairs: uniformly random distinct mutually reachable ordered
pairs, exact distances by single-source C-BFS.  Prints one
JSON line per (w, tau).
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
from paper_2410_17226_b200 import ado  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat20"
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
budget = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
cfg = ci.CONFIGS[name]
d = int(sys.argv[4]) if len(sys.argv) > 4 else cfg["d"]
word_sizes = [int(x) for x in os.environ.get("WS", "64").split(",")]
el = ci.make_graph(name)
dev = torch.device("cuda:0")
g = cb.Graph.from_edges(el.n, torch.from_numpy(el.src.view(np.int32)).to(dev),
                        torch.from_numpy(el.dst.view(np.int32)).to(dev), relabel=cfg.get("relabel", "none"))
torch.cuda.synchronize()
t0 = time.perf_counter()
parts, have, stream = [], 0, 5
while have < pairs and stream < 40:  # candidate draws until enough distinct, mutually reachable pairs
    sc, tc = ci.query_pairs(el.n, int(1.2 * (pairs - have)) + 100, seed=11, stream=stream)
    parts.append(ado.sample_pairs(sc, tc, pairs - have, lambda a, b: ado.exact_distances(g, a, b)))
    have += len(parts[-1][0])
    stream += 1
s, t, dd = (np.concatenate([p[i] for p in parts]) for i in range(3))
t_exact = time.perf_counter() - t0
taus = [int(x) for x in os.environ.get("TAUS", "0").split(",")]
sd, td = torch.from_numpy(s.view(np.int32)).to(dev), torch.from_numpy(t.view(np.int32)).to(dev)
policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
for w in word_sizes:  # w = 0: plain landmarks (single vertices, d = 0, 1-byte records)
    dw = d if w else 0
    record = ado.record_bytes(w, dw)  # 1-byte Delta, as the paper counts
    r = budget // record
    for db in (1, 2):  # u8 Delta unless a distance exceeds 254 (R10), then u16
        try:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            idx = ado.LandmarkIndex(g, r, max(w, 1), dw, policy, cfg["root_seed"], word_bits=w, dist_bytes=db)
            torch.cuda.synchronize()
            t_index = time.perf_counter() - t0
            break
        except cb.CbfsError:
            if db == 2:
                raise
    for tau in taus:  # Appendix B: tau vertices visited per side by the bi-directional search (0 = index only)
        idx.query(sd, td, tau)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ans = idx.query(sd, td, tau)
        torch.cuda.synchronize()
        t_query = time.perf_counter() - t0
        res = ado.distortion(ans.cpu().numpy(), dd)
        res.update({"config": name, "budget_bytes_per_vertex": budget, "w": w, "record_bytes": record,
                    "dist_bytes": db, "clusters": idx.r, "landmarks": int(idx.sizes.sum().item()), "d": dw,
                    "tau": tau, "index_s": t_index, "query_s": t_query, "exact_s": t_exact,
                    "image_bytes_per_vertex": idx.image_bytes / el.n, "mean_delta": float(dd.mean())})
        print(json.dumps(res), flush=True)
    idx.close()
