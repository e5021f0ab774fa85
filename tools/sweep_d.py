"""C-BFS time vs the diameter bound d (the shape of the
paper's Table BFS_d, P:1337-1357 / P:1541-1584, where time grows with d).

    python tools/sweep_d.py [config] [clusters]

For d = 2..6: select `clusters` clusters with that d (members within
floor(d/2) hops), traverse them (stats only), print one JSON line
per d: cluster sizes, rounds, time per cluster, source-edges/s.
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

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat20"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = ci.CONFIGS[name]
el = ci.make_graph(name)
relabel = cb.Graph.relabel_flags(cfg.get("relabel", "none"))
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
h = cb.cbfs_graph_create(el.n, torch.from_numpy(el.src.view(np.int32)).to(dev),
                         torch.from_numpy(el.dst.view(np.int32)).to(dev),
                         relabel, 0, st)
policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
for d in range(2, 7):
    ss = torch.empty((C, 64), dtype=torch.int32, device=dev)
    sz = torch.empty((C,), dtype=torch.uint8, device=dev)
    got = cb.cbfs_select_clusters(h, C, 64, d, policy, cfg["root_seed"], ss, sz, st)
    stats = torch.zeros((got, 4), dtype=torch.int64, device=dev)
    cb.cbfs_run(h, ss[:got], sz[:got], got, d, 2, None, None, d + 1, stats)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    cb.cbfs_run(h, ss[:got], sz[:got], got, d, 2, None, None, d + 1, stats)
    e1.record(st)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1000.0
    s = stats.cpu().numpy().view(np.uint64)
    k = sz[:got].cpu().numpy().astype(np.float64)
    units = float((k * s[:, 3].astype(np.float64)).sum())
    print(json.dumps({"config": name, "d": d, "clusters": got, "k_mean": float(k.mean()), "rounds_max": int(s[:, 0].max()),
                      "sumF_per_cluster": float(s[:, 1].mean()), "seconds": t, "ms_per_cluster": 1000 * t / got,
                      "source_edges_per_s": units / t}), flush=True)
cb.cbfs_graph_destroy(h)
