"""Run one BASELINE.json config at full size on the GPU and (optionally) check
sampled clusters against the oracle.

    python tests/run_config.py c4_grid [--check 8] [--first-batch-outputs]

Prints one JSON line: timings of build / selection / C-BFS (outputs not
materialised for the whole config when they do not fit; stats always),
source-edges/s, and the parity verdict of the sampled clusters (full
distance vectors of the first batch of 64 clusters compared element by
element; round stats of every sampled cluster).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--check", type=int, default=0, help="number of sampled clusters checked against the oracle")
    ap.add_argument("--clusters", type=int, default=0, help="override the number of clusters")
    ap.add_argument("--relabel", type=int, default=-1)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--conc", type=int, default=0)
    ap.add_argument("--alpha", type=float, default=0.0)
    ap.add_argument("--first", type=int, default=0, help="traverse only clusters [first, clusters) of the selection")
    args = ap.parse_args()
    cfg = ci.CONFIGS[args.config]
    dev = torch.device("cuda:0")
    t0 = time.perf_counter()
    el = ci.make_graph(args.config)
    t_gen = time.perf_counter() - t0
    n = el.n
    relabel = cb.Graph.relabel_flags(cfg.get("relabel", "none")) if args.relabel < 0 else args.relabel
    src_d = torch.from_numpy(el.src.view(np.int32)).to(dev)
    dst_d = torch.from_numpy(el.dst.view(np.int32)).to(dev)
    C = args.clusters or cfg["clusters"]
    d, k = cfg["d"], cfg["k"]
    policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
    st = torch.cuda.current_stream()
    if args.conc:
        cb.cbfs_set_concurrency(args.conc)
    if args.alpha:
        cb.cbfs_set_direction_alpha(args.alpha)
    if args.profile:
        cb.cbfs_profile_enable(True)
    res = {"config": args.config, "n": n, "pairs": len(el.src), "gen_s": t_gen, "clusters": C, "d": d}
    for rep in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = cb.cbfs_graph_create(n, src_d, dst_d, relabel, 0, st)
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t0
        _, m, maxdeg = cb.cbfs_graph_info(h)
        ss = torch.empty((C, 64), dtype=torch.int32, device=dev)
        sz = torch.empty((C,), dtype=torch.uint8, device=dev)
        t0 = time.perf_counter()
        got = cb.cbfs_select_clusters(h, C, k, d, policy, cfg["root_seed"], ss, sz, st)
        torch.cuda.synchronize()
        t_sel = time.perf_counter() - t0
        f0 = min(args.first, got)
        stats = torch.zeros((got, 4), dtype=torch.int64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        cb.cbfs_run(h, ss[f0:got], sz[f0:got], got - f0, d, 2, None, None, d + 1, stats[f0:])  # stats only
        e1.record(st)
        torch.cuda.synchronize()
        t_run = e0.elapsed_time(e1) / 1000.0
        stn = stats[f0:].cpu().numpy().view(np.uint64)
        szn = sz[f0:got].cpu().numpy().astype(np.float64)
        units = float((szn * stn[:, 3].astype(np.float64)).sum())
        res.update({"m": m, "max_degree": maxdeg, "selected": got, "build_s": t_build, "select_s": t_sel,
                    "cbfs_s": t_run, "source_edges_per_s": units / t_run,
                    "rounds_max": int(stn[:, 0].max()), "rounds_mean": float(stn[:, 0].mean()),
                    "k_mean": float(szn.mean()), "sumF_mean": float(stn[:, 1].mean()),
                    "outputs": "stats only (full vectors would need %.0f GB)" % (n * got * (2 + 8 * (d + 1)) / 1e9)})
        if args.profile:
            res["kernels"] = cb.cbfs_profile_read(reset=True)
        if rep + 1 < args.reps:
            cb.cbfs_graph_destroy(h)
    if args.check:
        import oracle as orc
        t0 = time.perf_counter()
        g = orc.csr_from_edgelist(el)
        res["oracle_csr_s"] = time.perf_counter() - t0
        srcn = ss[:got].cpu().numpy().view(np.uint32)
        sample = sorted(set(np.linspace(0, got - 1, args.check).round().astype(int).tolist()))
        t0 = time.perf_counter()
        om = orc.cluster_bfs_many(g, srcn[sample], sz[:got].cpu().numpy()[sample], d,
                                  want_outputs=True)
        res["oracle_s"] = time.perf_counter() - t0
        stats_ok = bool(np.array_equal(stn[sample], om["stats"]))
        # full vectors of the sampled clusters through the GPU, compared element by element
        sel_src = ss[:got][torch.tensor(sample, device=dev)].contiguous()
        sel_sz = sz[:got][torch.tensor(sample, device=dev)].contiguous()
        Cs = len(sample)
        dist = torch.empty((n, Cs), dtype=torch.int16, device=dev)
        masks = torch.empty((d + 1, n, Cs), dtype=torch.int64, device=dev)
        st2 = torch.zeros((Cs, 4), dtype=torch.int64, device=dev)
        cb.cbfs_run(h, sel_src, sel_sz, Cs, d, 2, dist, masks, d + 1, st2)
        torch.cuda.synchronize()
        gd = dist.cpu().numpy().view(np.uint16).T
        vec_ok = bool(np.array_equal(gd, om["dist"]))
        for j in range(Cs):
            vec_ok &= bool(np.array_equal(masks[:, :, j].cpu().numpy().view(np.uint64), om["sub"][j]))
        res.update({"checked_clusters": sample, "stats_match": stats_ok, "vectors_match": vec_ok})
        # the oracle's selection too
        t0 = time.perf_counter()
        osrc, osz = orc.select_clusters(g, C, k, d, orc.ROOT_RANDOM if policy else orc.ROOT_DEGREE, cfg["root_seed"])
        res["oracle_select_s"] = time.perf_counter() - t0
        res["selection_match"] = bool(np.array_equal(osrc, srcn) and np.array_equal(osz, sz[:got].cpu().numpy()))
    cb.cbfs_graph_destroy(h)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
