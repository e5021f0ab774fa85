"""Predicted strong-scaling curve: one GPU runs rank (N-1)'s share of an
N-GPU bench step (graph build + the whole deterministic selection + the
rank's round-robin clusters, r = N-1, 2N-1, ... ), exactly what every rank of
a `bench.py --gpus N` run does — the data path has no inter-rank exchange
(clusters are independent), so a rank's time is its own work.

    python tools/shard_probe.py [CONFIG] [N ...]

Prints per N: build / select / C-BFS phase times of the rank's share and the
predicted whole-job value (N x the rank's source-edges / its C-BFS phase, T
per SURVEY §8(d)) and the efficiency against N = 1 (rank N-1 holds the
smallest share of the degree-ordered round-robin, so the max over ranks is
within one batch of this)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_rmat24"
worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg = ci.CONFIGS[name]
el = ci.make_graph(name)
n, d = el.n, cfg["d"]
src_d = torch.from_numpy(el.src.view(np.int32)).cuda()
dst_d = torch.from_numpy(el.dst.view(np.int32)).cuda()
st = torch.cuda.current_stream()
C = cfg["clusters"]
flags = cb.Graph.relabel_flags(cfg.get("relabel", "none"))
policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
dist_bytes = 1 if cfg["kind"] in ("rmat", "er") else 2
src = torch.empty((C, 64), dtype=torch.int32, device="cuda")
sz = torch.empty((C,), dtype=torch.uint8, device="cuda")
base = None
for world in worlds:
    rank = world - 1
    Cr = len(range(rank, C, world))
    stats = torch.zeros((Cr, 4), dtype=torch.int64, device="cuda")
    dig = torch.zeros((Cr,), dtype=torch.int64, device="cuda")
    times = []
    for rep in range(2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        ev[0].record(st)
        h = cb.cbfs_graph_create(n, src_d, dst_d, flags, 0, st)
        ev[1].record(st)
        cb.cbfs_select_clusters(h, C, cfg["k"], d, policy, cfg["root_seed"], src, sz, st)
        ev[2].record(st)
        mine_src, mine_sz = src[rank::world].contiguous(), sz[rank::world].contiguous()
        cb.cbfs_run_digest(h, mine_src, mine_sz, Cr, d, dist_bytes, d + 1, dig, stats)
        ev[3].record(st)
        torch.cuda.synchronize()
        cb.cbfs_graph_destroy(h)
        if rep:
            times.append([ev[k].elapsed_time(ev[k + 1]) for k in range(3)])
    b, s, t = np.mean(times, axis=0)
    units = float((sz[rank::world].cpu().numpy().astype(np.float64) * stats.cpu().numpy()[:, 3]).sum())
    value = world * units / (t / 1e3)
    base = base or value
    print(f"{name} N={world}: rank {rank} has {Cr} clusters; build {b:.1f} ms, select {s:.1f} ms, C-BFS {t:.1f} ms; "
          f"predicted value {value:.3e} source-edges/s, efficiency {value / base / world:.3f}", flush=True)
