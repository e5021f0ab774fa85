"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of libcbfs.so on config-1-sized inputs.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Covers: CSR build (+ degree / locality relabel, the latter's cooperative
kernel), selection, the sparse engine's ordered frontiers, the batched
engine in push / pull / auto, the sparse engine (fused fold+push, d >= 1, and
the separate fold, d = 0), wide clusters, the output digest consumer, the
per-round statistics, labels + query + streaming query, the Appendix B
search and the PLL build + query.  Prints one line per case; exits non-zero
on a library error (the sanitizer reports its own findings on stderr).
No oracle involved: this checks memory / race / sync hygiene, not values.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402

DEV = "cuda:0"


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    el = ci.make_graph("c1_er")
    grid = ci.grid(48, 0.05, 0.01, 4)
    g = cb.Graph.from_edges(el.n, el.src, el.dst, relabel=True)
    gl = cb.Graph.from_edges(el.n, el.src, el.dst, relabel="locality")
    gg = cb.Graph.from_edges(grid.n, grid.src, grid.dst)
    kn = ci.knn3d(3000, 10, seed=5)
    gk = cb.Graph.from_edges(kn.n, kn.src, kn.dst, relabel="locality")
    src, sz = g.select_clusters(8, 64, 2, cb.CBFS_ROOT_RANDOM, 1)
    C = len(sz)
    for direction, tag in ((cb.CBFS_DIR_PUSH, "push"), (cb.CBFS_DIR_PULL, "pull"), (cb.CBFS_DIR_AUTO, "auto")):
        cb.cbfs_set_engine(cb.CBFS_ENGINE_BATCHED)
        case(f"batched {tag}", lambda: g.run(src, sz, 2, dist_bytes=1, direction=direction))
    cb.cbfs_set_engine(cb.CBFS_ENGINE_SPARSE)
    gsrc, gsz = gg.select_clusters(20, 64, 4, cb.CBFS_ROOT_RANDOM, 4)
    case("sparse fused d=4", lambda: gg.run(gsrc, gsz, 4))
    one = torch.full_like(gsrc, -1)
    one[:, 0] = gsrc[:, 0]
    case("sparse d=0", lambda: gg.run(one, torch.ones_like(gsz), 0))
    dig4 = torch.zeros(len(gsz), dtype=torch.int64, device=DEV)
    case("sparse digest (cluster-major staging)", lambda: cb.cbfs_run_digest(gg.h, gsrc, gsz, len(gsz), 4, 2, 5, dig4))
    case("sparse locality graph", lambda: gl.run(*gl.select_clusters(8, 64, 2), 2))
    cb.cbfs_set_sparse_order(1)  # ordered frontiers (bitmap claims + compaction) on every round
    case("sparse ordered frontiers d=4", lambda: gg.run(gsrc, gsz, 4))
    case("sparse ordered frontiers d=0", lambda: gg.run(one, torch.ones_like(gsz), 0))
    case("sparse ordered frontiers, k-NN", lambda: gk.run(*gk.select_clusters(8, 64, 2), 2))
    cb.cbfs_set_sparse_order(-1)
    case("locality order (cooperative kernel), grid",
         lambda: cb.cbfs_graph_internal_order(cb.Graph.from_edges(grid.n, grid.src, grid.dst, relabel="locality").h))
    cb.cbfs_set_engine(cb.CBFS_ENGINE_AUTO)
    dig = torch.zeros(C, dtype=torch.int64, device=DEV)
    case("digest consumer", lambda: cb.cbfs_run_digest(g.h, src, sz, C, 2, 1, 3, dig))
    rounds = torch.zeros((C, 16, 2), dtype=torch.int64, device=DEV)
    case("round statistics", lambda: cb.cbfs_run_rounds(g.h, src, sz, C, 2, rounds, 16))
    wsrc = torch.full((4, 128), -1, dtype=torch.int32, device=DEV)
    wsz = torch.empty((4,), dtype=torch.int16, device=DEV)
    got = cb.cbfs_select_clusters_wide(g.h, 4, 100, 2, 0, 0, 2, wsrc, wsz)
    wd = torch.empty((g.n, got), dtype=torch.int16, device=DEV)
    wm = torch.empty((3, g.n, 2 * got), dtype=torch.int64, device=DEV)
    case("wide clusters", lambda: cb.cbfs_run_wide(g.h, wsrc[:got], wsz[:got], got, 2, 2, 2, wd, wm, 3))
    s, t = ci.query_pairs(g.n, 5000, seed=3)
    sd = torch.from_numpy(s.view(np.int32)).to(DEV)
    td = torch.from_numpy(t.view(np.int32)).to(DEV)
    best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device=DEV)
    lh = cb.cbfs_labels_build(g.h, src, sz, C, 2, 1, word_bits=64)
    case("labels + query", lambda: cb.cbfs_labels_query(lh, sd, td, best))
    cb.cbfs_labels_destroy(lh)
    case("streaming query", lambda: cb.cbfs_query_stream(g.h, src, sz, C, 2, sd, td, best))
    case("bidirectional search", lambda: cb.cbfs_query_bidir(g.h, sd, td, 64, best))
    ph = cb.cbfs_pll_build(g.h, src, sz, C, 2, 8, 32, 2048)
    out = torch.empty((len(s),), dtype=torch.int32, device=DEV)
    case("PLL build + query", lambda: cb.cbfs_pll_query(ph, sd, td, out))
    cb.cbfs_pll_destroy(ph)
    for h in (g, gl, gg):
        h.close()
    print("all cases ok", flush=True)


if __name__ == "__main__":
    main()
