"""Full-size parity for BASELINE.json configs 3-5 (config 2 is in
test_gpu_parity.py::test_c2_full_size_sampled), in the launch configuration
bench.py times: the whole config's selection on the GPU == the oracle's, all
clusters traversed in one cbfs_run (AUTO engine: batched for RMAT, sparse for
the grid and the k-NN graph), per-cluster round statistics of sampled
clusters == the oracle's, and the full distance vectors of sampled clusters
element by element.  Config 5 also checks the streaming label/query path on a
prefix of its clusters against the oracle's answers.  Bit-exact throughout."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402
from gpu_util import np_u32, np_u64  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _graph(name):
    cfg = ci.CONFIGS[name]
    el = ci.make_graph(name)
    relabel = cb.Graph.relabel_flags(cfg.get("relabel", "none"))
    src_d = torch.from_numpy(el.src.view(np.int32)).to(DEV)
    dst_d = torch.from_numpy(el.dst.view(np.int32)).to(DEV)
    g = cb.Graph(cb.cbfs_graph_create(el.n, src_d, dst_d, relabel, 0), 0)
    del src_d, dst_d
    return cfg, el, g


def _check_config(name, n_sample, clusters=None):
    cfg, el, g = _graph(name)
    ref = orc.csr_from_edgelist(el)
    assert g.m == ref.m
    C = clusters or cfg["clusters"]
    d, k = cfg["d"], cfg["k"]
    policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
    src_d, sz_d = g.select_clusters(C, k, d, policy, cfg["root_seed"])
    osrc, osz = orc.select_clusters(ref, C, k, d, orc.ROOT_RANDOM if policy else orc.ROOT_DEGREE, cfg["root_seed"])
    assert np.array_equal(np_u32(src_d), osrc) and np.array_equal(sz_d.cpu().numpy(), osz)
    got = len(osz)
    # every cluster in one call, statistics only (the full vectors of configs 3-5 do not fit HBM)
    stats = torch.zeros((got, 4), dtype=torch.int64, device=DEV)
    cb.cbfs_run(g.h, src_d, sz_d, got, d, 2, None, None, d + 1, stats)
    st = stats.cpu().numpy().view(np.uint64)
    sample = sorted(set(np.linspace(0, got - 1, n_sample).round().astype(int).tolist()))
    om = orc.cluster_bfs_many(ref, osrc[sample], osz[sample], d, want_outputs=True)
    assert np.array_equal(st[sample], om["stats"])
    # the sampled clusters' full vectors
    idx = torch.tensor(sample, device=DEV)
    Cs = len(sample)
    dist = torch.empty((g.n, Cs), dtype=torch.int16, device=DEV)
    masks = torch.empty((d + 1, g.n, Cs), dtype=torch.int64, device=DEV)
    cb.cbfs_run(g.h, src_d[idx].contiguous(), sz_d[idx].contiguous(), Cs, d, 2, dist, masks, d + 1, None)
    gd = dist.cpu().numpy().view(np.uint16)
    for j in range(Cs):
        assert np.array_equal(gd[:, j], om["dist"][j]), sample[j]
        assert np.array_equal(np_u64(masks[:, :, j].contiguous()), om["sub"][j]), sample[j]
    return cfg, el, g, ref, src_d, sz_d, osrc, osz


@pytest.mark.timeout(900)
def test_c3_full_size_sampled():
    g = _check_config("c3_rmat24", 2)[2]
    g.close()


@pytest.mark.timeout(600)
def test_c4_full_size_sampled():
    g = _check_config("c4_grid", 6)[2]
    g.close()


@pytest.mark.timeout(900)
def test_c5_prefix_sampled_and_queries():
    """Config 5 on its first 256 clusters (the full 8,192 take ~2.5 min: bench.py
    --config c5_knn), then the fused label build + query path (A10/A11) over the
    first 64 clusters against the oracle's streaming query, 200,000 pairs."""
    cfg, el, g, ref, src_d, sz_d, osrc, osz = _check_config("c5_knn", 4, clusters=256)
    d = cfg["d"]
    s, t = ci.query_pairs(g.n, cfg["queries"], cfg["query_seed"])
    s, t = s[:200_000].copy(), t[:200_000].copy()
    best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device=DEV)
    sd = torch.from_numpy(s.view(np.int32)).to(DEV)
    td = torch.from_numpy(t.view(np.int32)).to(DEV)
    cb.cbfs_query_stream(g.h, src_d[:64].contiguous(), sz_d[:64].contiguous(), 64, d, sd, td, best)
    expect = orc.query_stream(ref, osrc[:64], osz[:64], d, s, t)
    got = best.cpu().numpy()
    assert np.array_equal(got, expect)
    assert (expect < orc.INT32_MAX).sum() > 0
    g.close()


@pytest.mark.timeout(900)
def test_intact_grid_manhattan_full_size():
    """SURVEY §8(c) closed form at config 4's size: on the intact 4096² grid
    (no deletions, no diagonals; id = y·4096 + x, R21) the distance from a
    source is the Manhattan distance, so every Delta and every subset of
    every radius-2-ball cluster is known without an oracle.  64 clusters
    (random roots, d = 4) in one cbfs_run — ~8,000 rounds — checked element by
    element on the device, and their round counts = 1 + max distance."""
    side = 4096
    el = ci.grid(side, 0.0, 0.0, 4)
    g = cb.Graph(cb.cbfs_graph_create(el.n, torch.from_numpy(el.src.view(np.int32)).to(DEV),
                                      torch.from_numpy(el.dst.view(np.int32)).to(DEV), 0, 0), 0)
    assert g.m == 4 * side * (side - 1)
    d, C = 4, 64
    src = torch.empty((C, 64), dtype=torch.int32, device=DEV)
    sz = torch.empty((C,), dtype=torch.uint8, device=DEV)
    assert cb.cbfs_select_clusters(g.h, C, 64, d, cb.CBFS_ROOT_RANDOM, 4, src, sz) == C
    dist = torch.empty((g.n, C), dtype=torch.int16, device=DEV)
    masks = torch.empty((d + 1, g.n, C), dtype=torch.int64, device=DEV)
    stats = torch.zeros((C, 4), dtype=torch.int64, device=DEV)
    cb.cbfs_run(g.h, src, sz, C, d, 2, dist, masks, d + 1, stats)
    torch.cuda.synchronize()
    v = torch.arange(g.n, device=DEV, dtype=torch.int64)
    x, y = v % side, v // side
    st = stats.cpu().numpy()
    for c in range(C):
        k = int(sz[c])
        S = src[c, :k].to(torch.int64)
        D = (x[None, :] - (S % side)[:, None]).abs() + (y[None, :] - (S // side)[:, None]).abs()  # [k][n]
        delta = D.min(dim=0).values
        assert torch.equal(dist[:, c].to(torch.int64) & 0xFFFF, delta), c
        off = D - delta[None, :]
        assert int(off.max()) <= d  # a radius-2 ball has diameter <= 4
        bits = (torch.ones(k, dtype=torch.int64, device=DEV) << torch.arange(k, device=DEV))[:, None]
        for i in range(d + 1):
            expect = ((off == i).to(torch.int64) * bits).sum(dim=0)
            assert torch.equal(masks[i, :, c], expect), (c, i)
        assert int(st[c, 0]) == 1 + int(D.max()), c  # rounds executed = 1 + max distance
    g.close()
