#!/usr/bin/env python3
"""Write the oracle-generated golden files of the full-size parity tests.

    python tests/make_goldens.py CONFIG [--sample N] [--threads T] [--chunk K]

Calls only oracle/ (the CPU oracle) and cbfs_inputs/ (the seeded generators);
nothing here touches the CUDA product.  Output: tests/golden/CONFIG.golden.txt
(plus tests/golden/c5_knn.answers.npz for config 5), one line per cluster in
the oracle's Alg. 1 order of the selection (R12):

    cluster rounds sum_F sum_E m_reach digest [|F_0| E_0 |F_1| E_1 ...]

`digest` is oracle.digest_cluster of the cluster's full output vector (Delta
and the d+1 subsets).  The header records the graph (n, arcs), a
SHA-256 of the whole selection (sources padded with 0xFFFFFFFF + sizes) and
the cluster order.  Generation is resumable: clusters already in the file are
skipped, so a long run (config 3: ~52 s of oracle time per cluster per core)
can be extended later with a larger --sample.

Cluster order: config 3 (4,096 clusters, too many for the host) takes a
seeded sample — numpy PCG64(2410017226).permutation(4096), first N — others
take the clusters in selection order (all, or the first N with --sample).
Config 5 additionally runs the streaming query of
its 10M pairs over the clusters it covers, min-merged chunk by chunk
(checkpointed under tests/golden/.work/), and stores the answers' SHA-256,
their histogram and 100,000 sampled answers once every covered cluster is in
(`clusters` in the .npz: the streaming index over that selection prefix; the
oracle needs ~38 s per config-5 cluster per core with the 10M queries, so the
answers cover the first 1,024 of the 8,192 clusters).  The other config-5
clusters get stats + digest lines without the queries (`--no-queries`,
`--range A:B` to split the run over hosts; lines may arrive out of order).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
MAX_ROUNDS_RECORDED = 64  # per-round {|F_i|, E_i} kept for clusters with at most this many rounds
SAMPLE_SEED = 2410017226
N_SAMPLED_ANSWERS = 100_000


def selection_sha(src: np.ndarray, sz: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(src, dtype=np.uint32).tobytes())
    h.update(np.ascontiguousarray(sz, dtype=np.uint8).tobytes())
    return h.hexdigest()


def cluster_order(name: str, C: int, sample: int) -> list[int]:
    if name == "c3_rmat24":
        return [int(x) for x in np.random.Generator(np.random.PCG64(SAMPLE_SEED)).permutation(C)[:sample]]
    return list(range(C if not sample else min(sample, C)))


def read_done(path: str) -> dict[int, str]:
    done = {}
    if os.path.exists(path):
        for line in open(path):
            if line.startswith("#") or not line.strip():
                continue
            done[int(line.split()[0])] = line.rstrip("\n")
    return done


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--sample", type=int, default=0, help="clusters to compute (0 = all)")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--chunk", type=int, default=0, help="clusters per oracle call (default 2 x threads)")
    ap.add_argument("--range", default="", help="A:B — only clusters [A, B) of the order (split a long run)")
    ap.add_argument("--no-queries", action="store_true",
                    help="config 5: stats + digests only (clusters beyond the answers' prefix)")
    args = ap.parse_args()
    name = args.config
    cfg = ci.CONFIGS[name]
    d = cfg["d"]
    chunk = args.chunk or 2 * args.threads
    t0 = time.time()
    el = ci.make_graph(name)
    g = orc.csr_from_edgelist(el)
    print(f"[{name}] graph n={g.n} arcs={g.m} in {time.time() - t0:.0f}s", flush=True)
    policy = orc.ROOT_RANDOM if cfg["root"] == "random" else orc.ROOT_DEGREE
    src, sz = orc.select_clusters(g, cfg["clusters"], cfg["k"], d, policy, cfg["root_seed"])
    C = len(sz)
    sha = selection_sha(src, sz)
    order = cluster_order(name, C, args.sample)
    path = os.path.join(GOLDEN, f"{name}.golden.txt")
    done = read_done(path)
    header = {"config": name, "graph": el.name, "n": g.n, "arcs": g.m, "clusters": C, "d": d,
              "selection_sha256": sha, "sizes_sum": int(sz.astype(np.int64).sum()),
              "order": "PCG64(%d).permutation" % SAMPLE_SEED if name == "c3_rmat24" else "selection order",
              "generator": "tests/make_goldens.py (oracle/ only)"}
    if not os.path.exists(path):
        with open(path, "w") as f:
            f.write("# " + json.dumps(header) + "\n")
            f.write("# cluster rounds sum_F sum_E m_reach digest [|F_i| E_i per round, i = 0..rounds-1]\n")
    else:
        first = json.loads(open(path).readline()[2:])
        assert first["selection_sha256"] == sha, "golden file belongs to another selection"
    if args.range:
        lo_, hi_ = (int(x) for x in args.range.split(":"))
        order = order[lo_:hi_]
    todo = [c for c in order if c not in done]
    print(f"[{name}] {C} clusters, {len(done)} done, {len(todo)} to do", flush=True)
    if name == "c5_knn" and not args.no_queries:
        run_c5(g, src, sz, d, cfg, todo, path, args.threads, chunk, order)
        return
    for i in range(0, len(todo), chunk):
        part = todo[i:i + chunk]
        t1 = time.time()
        r = orc.cluster_bfs_many(g, src[part], sz[part], d, threads=args.threads, want_outputs=False,
                                 want_digest=True, max_rounds=MAX_ROUNDS_RECORDED)
        with open(path, "a") as f:
            for j, c in enumerate(part):
                st = r["stats"][j]
                line = f"{c} {st[0]} {st[1]} {st[2]} {st[3]} {r['digest'][j]}"
                R = int(st[0])
                if R <= MAX_ROUNDS_RECORDED:
                    line += " " + " ".join(f"{r['round_F'][j][q]} {r['round_E'][j][q]}" for q in range(R))
                f.write(line + "\n")
        print(f"[{name}] {i + len(part)}/{len(todo)} in {time.time() - t1:.0f}s", flush=True)


def run_c5(g, src, sz, d, cfg, todo, path, threads, chunk, todo_all):
    """Streaming query over the clusters in `todo` (checkpointed running min);
    the answers file is written once every cluster of `todo_all` is in."""
    work = os.path.join(GOLDEN, ".work")
    os.makedirs(work, exist_ok=True)
    best_path = os.path.join(work, "c5_best.npy")
    s, t = ci.query_pairs(g.n, cfg["queries"], cfg["query_seed"])
    best = np.load(best_path) if os.path.exists(best_path) else np.full(len(s), orc.INT32_MAX, np.int32)
    for i in range(0, len(todo), chunk):
        part = todo[i:i + chunk]
        t1 = time.time()
        ans, st, dg = orc.query_stream(g, src[part], sz[part], d, s, t, threads=threads, with_stats=True)
        np.minimum(best, ans, out=best)
        np.save(best_path + ".tmp.npy", best)
        os.replace(best_path + ".tmp.npy", best_path)  # checkpoint before the lines that claim it
        with open(path, "a") as f:
            for j, c in enumerate(part):
                f.write(f"{c} {st[j][0]} {st[j][1]} {st[j][2]} {st[j][3]} {dg[j]}\n")
        print(f"[c5_knn] {i + len(part)}/{len(todo)} in {time.time() - t1:.0f}s", flush=True)
    done = read_done(path)
    if all(c in done for c in todo_all):
        write_answers(best, len(s), len(todo_all))


def write_answers(best: np.ndarray, q: int, clusters: int):
    idx = np.random.Generator(np.random.PCG64(SAMPLE_SEED)).choice(q, N_SAMPLED_ANSWERS, replace=False)
    idx.sort()
    vals, counts = np.unique(best, return_counts=True)
    np.savez_compressed(os.path.join(GOLDEN, "c5_knn.answers.npz"), index=idx.astype(np.uint32),
                        answer=best[idx], sha256=np.array(hashlib.sha256(best.tobytes()).hexdigest()),
                        hist_values=vals, hist_counts=counts, clusters=np.array(clusters))
    print(f"[c5_knn] answers written: sha256 {hashlib.sha256(best.tobytes()).hexdigest()}", flush=True)


if __name__ == "__main__":
    main()
