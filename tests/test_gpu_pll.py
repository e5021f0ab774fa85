"""Exact 2-hop distance oracle: PLL with a C-BFS first
phase and batched pruned BFSs (reading R29) through
cbfs_pll_build / _export / _query, against the oracle's pll_build /
pll_query (pinned in test_oracle_pins.py by all-pairs BFS and a brute-force
label characterisation).  Bit-exact: every label list and every answer."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402
from gpu_util import gpu_graph, np_u32, to_dev_u8, to_dev_u32  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

GRAPHS = {
    "er": lambda: ci.erdos_renyi(1500, 5000, seed=71),
    "rmat": lambda: ci.rmat(10, 8, 0.57, 0.19, 0.19, seed=72),
    "grid": lambda: ci.grid(30, 0.05, 0.01, 73),
    "er_sparse": lambda: ci.erdos_renyi(2000, 1600, seed=74),  # many components
}


def build_both(el, C, k, first, bmax, cap, relabel):
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, C, k, 2) if C else (np.zeros((0, 64), np.uint32), np.zeros(0, np.uint8))
    oidx = orc.pll_build(ref, src, sz, 2, first=first, bmax=bmax, cap=cap)
    g = gpu_graph(el, relabel=relabel)
    h = cb.cbfs_pll_build(g.h, to_dev_u32(src) if len(sz) else None, to_dev_u8(sz) if len(sz) else None, len(sz), 2,
                          first, bmax, cap)
    return ref, g, h, oidx


@pytest.mark.parametrize("kind,C,k,first,bmax,relabel", [
    ("er", 0, 1, 1, 1, False), ("er", 4, 16, 4, 16, True), ("rmat", 16, 64, 200, 1000, True),
    ("rmat", 64, 64, 7, 50, False), ("grid", 8, 13, 5, 40, False), ("er_sparse", 3, 8, 16, 64, True),
    ("rmat", 0, 1, 200, 1000, False), ("rmat", 200, 64, 50, 400, True), ("er", 100, 8, 30, 90, False)])
def test_pll_labels_and_queries_match_oracle(kind, C, k, first, bmax, relabel):
    el = GRAPHS[kind]()
    cap = 512
    ref, g, h, oidx = build_both(el, C, k, first, bmax, cap, relabel)
    info = cb.cbfs_pll_info(h)
    assert info["total_labels"] == oidx["total"]
    counts = torch.empty((g.n,), dtype=torch.int32, device=DEV)
    entries = torch.empty((g.n, cap), dtype=torch.int32, device=DEV)
    cb.cbfs_pll_export(h, counts, entries)
    gc, ge = np_u32(counts), np_u32(entries)
    assert np.array_equal(gc, oidx["counts"])
    mask = np.arange(cap)[None, :] < gc[:, None]
    assert np.array_equal(np.where(mask, ge, 0), np.where(mask, oidx["entries"], 0))
    assert info["max_labels"] == int(gc.max())
    s, t = ci.query_pairs(g.n, 20000, seed=5, stream=9)
    s[:50] = t[:50]
    out = torch.empty((len(s),), dtype=torch.int32, device=DEV)
    cb.cbfs_pll_query(h, to_dev_u32(s), to_dev_u32(t), out)
    got = out.cpu().numpy()
    assert np.array_equal(got, orc.pll_query(oidx, s, t))
    for x in np.unique(s)[:30]:  # exact distances (the oracle is pinned; spot-check against BFS too)
        bfs = orc.plain_bfs(ref, int(x))
        sel = s == x
        assert np.array_equal(got[sel], np.where(bfs[t[sel]] == orc.INF32, orc.INT32_MAX, bfs[t[sel]]))
    cb.cbfs_pll_destroy(h)
    g.close()


def test_pll_c1_all_pairs_exact():
    """Config 1's graph (ER, n = 4,096): the index answers all 16.8M ordered
    pairs exactly (against 4,096 textbook BFSs)."""
    el = ci.make_graph("c1_er")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 16, 64, 2)
    g = gpu_graph(el)
    h = cb.cbfs_pll_build(g.h, to_dev_u32(src), to_dev_u8(sz), len(sz), 2, 200, 1000, 1024)
    n = g.n
    D = np.stack([orc.plain_bfs(ref, v) for v in range(n)]).astype(np.int64)
    D[D == orc.INF32] = orc.INT32_MAX
    s = torch.arange(n, device=DEV, dtype=torch.int32).repeat_interleave(n)
    t = torch.arange(n, device=DEV, dtype=torch.int32).repeat(n)
    out = torch.empty((n * n,), dtype=torch.int32, device=DEV)
    cb.cbfs_pll_query(h, s, t, out)
    assert np.array_equal(out.cpu().numpy().astype(np.int64), D.reshape(-1))
    cb.cbfs_pll_destroy(h)
    g.close()


def test_pll_errors():
    el = GRAPHS["grid"]()
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el)
    with pytest.raises(cb.CbfsError):  # a grid's labels do not fit 3 entries
        cb.cbfs_pll_build(g.h, None, None, 0, 2, 200, 1000, 3)
    src, sz = orc.select_clusters(ref, 65, 13, 2)
    with pytest.raises(cb.CbfsError):  # a root's cluster labels must fit shared memory (checked before any read)
        cb.cbfs_pll_build(g.h, to_dev_u32(src), to_dev_u8(sz), 800, 31, 200, 1000, 256)
    h = cb.cbfs_pll_build(g.h, to_dev_u32(src[:4]), to_dev_u8(sz[:4]), 4, 2, 200, 1000, g.n)
    bad = torch.tensor([g.n], dtype=torch.int32, device=DEV)
    out = torch.empty((1,), dtype=torch.int32, device=DEV)
    with pytest.raises(cb.CbfsError):
        cb.cbfs_pll_query(h, bad, bad, out)
    cb.cbfs_pll_destroy(h)
    g.close()


def test_pll_cap_overflow_across_batches():
    """Lists that overflow cap in an early batch are reported (EOVERFLOW) and
    the later batches of the same build, which read the batch-start lengths,
    stay inside the lists (config 1's graph, 8 random-root clusters, batches
    of 8..32 roots, cap 16 and 256); the device stays usable afterwards."""
    el = ci.make_graph("c1_er")
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=True)
    src, sz = orc.select_clusters(ref, 8, 64, 2, orc.ROOT_RANDOM, 1)
    for cap in (16, 256):
        try:
            h = cb.cbfs_pll_build(g.h, to_dev_u32(src), to_dev_u8(sz), len(sz), 2, 8, 32, cap)
            cb.cbfs_pll_destroy(h)
        except cb.CbfsError as e:
            assert e.code == cb.CBFS_EOVERFLOW, e
    h = cb.cbfs_pll_build(g.h, to_dev_u32(src), to_dev_u8(sz), len(sz), 2, 8, 32, g.n)
    s, t = ci.query_pairs(g.n, 2000, seed=5)
    out = torch.empty((len(s),), dtype=torch.int32, device=DEV)
    cb.cbfs_pll_query(h, torch.from_numpy(s.view(np.int32)).to(DEV), torch.from_numpy(t.view(np.int32)).to(DEV), out)
    D = np.array([orc.plain_bfs(ref, int(x))[int(y)] for x, y in zip(s[:200], t[:200])], np.int64)
    got = out.cpu().numpy()[:200].astype(np.int64)
    D[D == orc.INF32] = orc.INT32_MAX
    assert np.array_equal(got, D)
    cb.cbfs_pll_destroy(h)
    g.close()


def test_pll_edgeless_and_tiny():
    """Degenerate inputs (R26): an edgeless graph labels every vertex with
    itself only (answers 0 on the diagonal, INT32_MAX elsewhere); a single
    edge; both equal the oracle."""
    for n, pairs in ((100, []), (2, [(0, 1)]), (5, [(1, 2), (2, 3)])):
        src = np.array([p[0] for p in pairs], np.uint32)
        dst = np.array([p[1] for p in pairs], np.uint32)
        ref = orc.csr_from_edges(n, src, dst)
        oidx = orc.pll_build(ref, np.zeros((0, 64), np.uint32), np.zeros(0, np.uint8), 2, first=2, bmax=4, cap=8)
        g = cb.Graph.from_edges(n, src, dst)
        h = cb.cbfs_pll_build(g.h, None, None, 0, 2, 2, 4, 8)
        counts = torch.empty((n,), dtype=torch.int32, device=DEV)
        entries = torch.empty((n, 8), dtype=torch.int32, device=DEV)
        cb.cbfs_pll_export(h, counts, entries)
        assert np.array_equal(np_u32(counts), oidx["counts"])
        s = np.repeat(np.arange(n), n).astype(np.uint32); t = np.tile(np.arange(n), n).astype(np.uint32)
        out = torch.empty((n * n,), dtype=torch.int32, device=DEV)
        cb.cbfs_pll_query(h, to_dev_u32(s), to_dev_u32(t), out)
        assert np.array_equal(out.cpu().numpy(), orc.pll_query(oidx, s, t))
        if not pairs:
            assert (np_u32(counts) == 1).all()
            assert (out.cpu().numpy().reshape(n, n) == np.where(np.eye(n, dtype=bool), 0, orc.INT32_MAX)).all()
        cb.cbfs_pll_destroy(h)
        g.close()


@pytest.mark.timeout(600)
def test_pll_c2_full_size_exact_sampled():
    """Config 2's graph at full size (RMAT-20, r = 64 clusters, the paper's
    batch schedule): the index is an exact distance oracle — 40 sampled
    sources × 5,000 targets each against textbook BFS (the oracle PLL is too
    slow at this size; its labels are pinned on smaller graphs above)."""
    el = ci.make_graph("c2_rmat20")
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=True)
    src = torch.empty((64, 64), dtype=torch.int32, device=DEV)
    sz = torch.empty((64,), dtype=torch.uint8, device=DEV)
    got = cb.cbfs_select_clusters(g.h, 64, 64, 2, cb.CBFS_ROOT_DEGREE, 0, src, sz)
    h = cb.cbfs_pll_build(g.h, src[:got].contiguous(), sz[:got].contiguous(), got, 2, 200, 1000, 2048)
    info = cb.cbfs_pll_info(h)
    assert info["roots"] == g.n - int(sz[:got].sum()) and info["total_labels"] > 0
    rng = np.random.default_rng(5)
    deg = ref.degrees()
    cand = np.flatnonzero(deg > 0)
    sources = np.concatenate([rng.choice(cand, 36, replace=False), np.argsort(-deg.astype(np.int64))[:4]])
    for x in sources:
        bfs = orc.plain_bfs(ref, int(x))
        tt = rng.integers(0, g.n, 5000).astype(np.uint32)
        ss = np.full(len(tt), x, np.uint32)
        out = torch.empty((len(tt),), dtype=torch.int32, device=DEV)
        cb.cbfs_pll_query(h, to_dev_u32(ss), to_dev_u32(tt), out)
        expect = np.where(bfs[tt] == orc.INF32, orc.INT32_MAX, bfs[tt]).astype(np.int64)
        assert np.array_equal(out.cpu().numpy().astype(np.int64), expect), int(x)
    cb.cbfs_pll_destroy(h)
    g.close()
