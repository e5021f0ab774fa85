"""Throughput of clusters with k > 64 sources (cbfs_run_wide) on a config's
graph: for each words W, r = 1024 / W clusters of up to k = 64 W sources
(cbfs_select_clusters_wide, d from the config), full outputs, timed with CUDA
events after a warm-up; source-edges/s = sum_c |S_c| m_c / T (m_c = arcs of
the vertices the cluster reaches).  W = 1 is the bench's own workload shape.

    python tools/wide_probe.py [config] [W,W,...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat20"
Ws = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
cfg = ci.CONFIGS[name]
d = cfg["d"]
el = ci.make_graph(name)
dev = torch.device("cuda:0")
g = cb.Graph.from_edges(el.n, torch.from_numpy(el.src.view(np.int32)).to(dev),
                        torch.from_numpy(el.dst.view(np.int32)).to(dev), relabel=cfg.get("relabel", "none"))
n = g.n
total_lanes = int(os.environ.get("LANES_TOTAL", "1024"))
for W in Ws:
    r = total_lanes // W
    src = torch.empty((r, 64 * W), dtype=torch.int32, device=dev)
    sz = torch.empty((r,), dtype=torch.int16, device=dev)
    got = cb.cbfs_select_clusters_wide(g.h, r, 64 * W, d, cb.CBFS_ROOT_DEGREE, 0, W, src, sz)
    src, sz = src[:got].contiguous(), sz[:got].contiguous()
    db = 1 if cfg["kind"] in ("rmat", "er") else 2  # u8 Delta only where every distance fits (R10)
    dist = torch.empty((n, got), dtype=torch.uint8 if db == 1 else torch.int16, device=dev)
    masks = torch.empty((d + 1, n, got * W), dtype=torch.int64, device=dev)
    stats = torch.zeros((got * W, 4), dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times = []
    for it in range(4):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cb.cbfs_run_wide(g.h, src, sz, got, W, d, db, dist, masks, d + 1, stats)
        e1.record()
        torch.cuda.synchronize()
        if it:
            times.append(e0.elapsed_time(e1))
    T = float(np.median(times)) / 1000.0
    st = stats.cpu().numpy().view(np.uint64).reshape(got, W, 4)
    m_c = st[:, :, 3].max(axis=1).astype(np.float64)  # arcs reached (same component for every word)
    k = sz.cpu().numpy().view(np.uint16).astype(np.float64)
    units = float((k * m_c).sum())
    print(json.dumps({"config": name, "words": W, "clusters": got, "k_mean": float(k.mean()), "k_max": int(k.max()),
                      "sources": int(k.sum()), "d": d, "ms": T * 1000.0,
                      "source_edges_per_s": units / T, "lanes": got * W}), flush=True)
    del dist, masks, stats
    torch.cuda.empty_cache()
g.close()
