"""NEXT-3: the landmark-label ADO's distortion computed through
the C-ABI (paper_2410_17226_b200/ado.py) equals the oracle's on the same
pairs: exact distances (single-source C-BFS vs textbook BFS), answers (GPU
query vs oracle query), epsilon; and the one-sided error holds."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
from gpu_util import gpu_graph  # noqa: E402
from paper_2410_17226_b200 import ado  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,d", [("rmat", 2), ("grid", 4)])
def test_distortion_matches_oracle(kind, d):
    el = ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=21) if kind == "rmat" else ci.grid(60, 0.05, 0.01, 21)
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=(kind == "rmat"))
    r = 1024 // (1 + d * 8)
    idx = ado.LandmarkIndex(g, r, 64, d)
    osrc, osz = orc.select_clusters(ref, r, 64, d)
    assert idx.r == len(osz)
    sc, tc = ci.query_pairs(el.n, 4000, seed=3, stream=5)
    s, t, dd = ado.sample_pairs(sc, tc, 3000, lambda a, b: ado.exact_distances(g, a, b))
    # exact distances against the textbook BFS
    for src in np.unique(s)[:40]:
        ref_d = orc.plain_bfs(ref, int(src))
        sel = s == src
        assert np.array_equal(dd[sel], ref_d[t[sel]])
    # the sample is the first 3000 distinct, mutually reachable candidates
    keep = sc != tc
    reach = np.array([orc.plain_bfs(ref, int(a))[b] != orc.INF32 for a, b in zip(sc[keep], tc[keep])])
    assert len(s) == min(3000, int(reach.sum())) and len(s) > 0
    assert np.array_equal(s, sc[keep][reach][:len(s)]) and np.array_equal(t, tc[keep][reach][:len(s)])
    ans = idx.query(torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(t.view(np.int32)).cuda()).cpu().numpy()
    expect = orc.query_stream(ref, osrc, osz, d, s, t)
    assert np.array_equal(ans, expect)
    res = ado.distortion(ans, dd)
    assert res["one_sided"] and res["covered"] > 0 and res["epsilon_pct"] >= 0.0
    psi = expect[expect < orc.INT32_MAX] / dd[expect < orc.INT32_MAX].astype(np.float64)
    assert res["epsilon_pct"] == pytest.approx(100.0 * (psi.mean() - 1.0), abs=0, rel=1e-12)
    g.close()


# ------------------------------------------------------------------ NEXT-2: bidirectional refinement
@pytest.mark.parametrize("kind,relabel", [("rmat", True), ("rmat", False), ("grid", False)])
def test_bidir_refine_parity(kind, relabel):
    """cbfs_query_bidir == the oracle's Appendix B search (reading R27) for
    several tau, and after the landmark query it gives min(index, search)."""
    import paper_2410_17226_b200 as cb
    el = ci.rmat(11, 8, 0.57, 0.19, 0.19, seed=31) if kind == "rmat" else ci.grid(50, 0.05, 0.01, 31)
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=relabel)
    s, t = ci.query_pairs(el.n, 3000, seed=8, stream=6)
    s[:20] = t[:20]  # u = v
    sd = torch.from_numpy(s.view(np.int32)).cuda()
    td = torch.from_numpy(t.view(np.int32)).cuda()
    for tau in (0, 1, 2, 5, 64, 1024):
        best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda")
        cb.cbfs_query_bidir(g.h, sd, td, tau, best)
        assert np.array_equal(best.cpu().numpy(), orc.bidir_refine(ref, s, t, tau)), tau
    # combined query: landmark labels, then the refinement min-merged
    idx = ado.LandmarkIndex(g, 12, 64, 2)
    osrc, osz = orc.select_clusters(ref, 12, 64, 2)
    best = idx.query(sd, td)
    cb.cbfs_query_bidir(g.h, sd, td, 32, best)
    expect = np.minimum(orc.query_stream(ref, osrc, osz, 2, s, t), orc.bidir_refine(ref, s, t, 32))
    assert np.array_equal(best.cpu().numpy(), expect)
    with pytest.raises(cb.CbfsError):
        cb.cbfs_query_bidir(g.h, sd, td, cb.CBFS_BIDIR_MAX_TAU + 1, best)
    g.close()


# ------------------------------------------------------------------ word size w (Tables 4/8)
@pytest.mark.parametrize("kind,d", [("rmat", 2), ("grid", 4)])
@pytest.mark.parametrize("w", [0, 8, 16, 32, 64])
def test_word_size_store_matches_oracle(kind, d, w):
    """A store of word size w under a t = 256 bytes-per-vertex budget: the
    cluster count and record size follow the paper's arithmetic (the oracle's
    pinned record_bytes), the image has exactly that many record bytes, and
    its answers equal the oracle's streaming query over the same k <= w
    clusters; an exported packed image answers identically after import.
    w = 0 is plain landmark labeling (k = 1, d = 0, 1-byte records)."""
    import paper_2410_17226_b200 as cb
    if w == 0:
        d = 0
    el = ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=51) if kind == "rmat" else ci.grid(60, 0.05, 0.01, 51)
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=(kind == "rmat"))
    assert ado.record_bytes(w, d) == orc.record_bytes(w, d)
    r = ado.clusters_for_budget(256, w, d)
    assert r == orc.budget_to_clusters(256, w, d)
    k = max(w, 1)
    idx = ado.LandmarkIndex(g, r, k, d, word_bits=w, dist_bytes=1)
    osrc, osz = orc.select_clusters(ref, r, k, d)
    assert idx.r == len(osz) and int(osz.max()) <= k
    info = cb.cbfs_labels_info(idx.labels)
    assert info["word_bits"] == w
    pad16 = lambda x: (x + 15) // 16 * 16  # noqa: E731
    assert info["image_bytes"] - 64 - pad16(idx.r) == pad16(g.n * idx.r) + g.n * idx.r * d * w // 8
    assert g.n * idx.r * ado.record_bytes(w, d) <= g.n * 256
    s, t = ci.query_pairs(el.n, 20000, seed=13, stream=7)
    sd, td = torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(t.view(np.int32)).cuda()
    expect = orc.query_stream(ref, osrc, osz, d, s, t)
    assert np.array_equal(idx.query(sd, td).cpu().numpy(), expect)
    img = torch.empty(info["image_bytes"], dtype=torch.uint8, device="cuda")
    cb.cbfs_labels_export(idx.labels, img)
    h2 = cb.cbfs_labels_import(g.h, img)
    best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda")
    cb.cbfs_labels_query(h2, sd, td, best)
    assert np.array_equal(best.cpu().numpy(), expect)
    cb.cbfs_labels_destroy(h2)
    idx.close()
    g.close()


def test_word_size_rejects_wide_clusters():
    import paper_2410_17226_b200 as cb
    el = ci.rmat(10, 8, 0.57, 0.19, 0.19, seed=52)
    g = gpu_graph(el, relabel=True)
    src = torch.empty((4, 64), dtype=torch.int32, device="cuda")
    sz = torch.empty((4,), dtype=torch.uint8, device="cuda")
    got = cb.cbfs_select_clusters(g.h, 4, 64, 2, cb.CBFS_ROOT_DEGREE, 0, src, sz)
    assert int(sz[:got].max()) > 16
    with pytest.raises(cb.CbfsError):
        cb.cbfs_labels_build(g.h, src, sz, got, 2, 2, word_bits=16)
    with pytest.raises(cb.CbfsError):
        cb.cbfs_labels_build(g.h, src, sz, got, 2, 2, word_bits=12)
    with pytest.raises(cb.CbfsError):  # plain landmarks need d = 0 and single sources
        cb.cbfs_labels_build(g.h, src, sz, got, 0, 2, word_bits=0)
    h = cb.cbfs_labels_build(g.h, src, sz, got, 2, 2, word_bits=64)
    assert cb.cbfs_labels_info(h)["word_bits"] == 64
    cb.cbfs_labels_destroy(h)
    g.close()
