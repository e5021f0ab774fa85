"""Sparse-engine throughput vs graph size (grid configs, 64 clusters, d=4): TLB / L2 footprint probe."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
dev = torch.device("cuda:0")
cb.cbfs_set_concurrency(int(os.environ.get("CONC", "1")))
for side in [int(x) for x in sys.argv[1:]]:
    el = ci.grid(side, 0.05, 0.001, 4)
    src_d = torch.from_numpy(el.src.view(np.int32)).to(dev); dst_d = torch.from_numpy(el.dst.view(np.int32)).to(dev)
    st = torch.cuda.current_stream()
    h = cb.cbfs_graph_create(el.n, src_d, dst_d, 0, 0, st)
    C = 64
    ss = torch.empty((C, 64), dtype=torch.int32, device=dev); sz = torch.empty((C,), dtype=torch.uint8, device=dev)
    got = cb.cbfs_select_clusters(h, C, 64, 4, cb.CBFS_ROOT_RANDOM, 4, ss, sz, st)
    stats = torch.zeros((got, 4), dtype=torch.int64, device=dev)
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        cb.cbfs_run(h, ss[:got], sz[:got], got, 4, 2, None, None, 5, stats)
        e1.record(st); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1000
    s = stats.cpu().numpy().view(np.uint64)
    arcs = float(s[:, 2].astype(np.float64).sum()); ent = float(s[:, 1].astype(np.float64).sum())
    print(json.dumps({"side": side, "n": el.n, "state_GB": el.n * 64 * 32 / 1e9, "s": t, "rounds": int(s[:, 0].max()),
                      "arcs_per_s_G": arcs / t / 1e9, "entries_per_s_G": ent / t / 1e9,
                      "us_per_round": t / int(s[:, 0].max()) * 1e6}), flush=True)
    cb.cbfs_graph_destroy(h)
