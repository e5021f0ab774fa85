"""Clusters of more than 64 sources (the paper's general
k: P:448) through cbfs_run_wide / cbfs_decode_wide /
cbfs_query_distance_wide, against the oracle's written-out definition
(brute_cluster_wide, query_brute; pinned in test_oracle_pins.py).
Bit-exact: every Delta and every word of every subset plane."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402
from gpu_util import gpu_graph, np_u16, np_u64, to_dev_u32  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def wide_clusters(g: orc.CSR, C: int, W: int, d: int, rng, min_k: int = 1):
    """C clusters of diameter <= d (root + members within floor(d/2) hops,
    by degree desc then id asc, R12's order), sizes drawn in [min_k, 64 W];
    roots are distinct high-degree vertices.  Returns (sources [C][64 W],
    sizes uint16 [C], member lists)."""
    deg = g.degrees()
    roots = np.argsort(-deg.astype(np.int64), kind="stable")[:C]
    src = np.full((C, 64 * W), orc.PAD, np.uint32)
    sz = np.zeros(C, np.uint16)
    lists = []
    for c, r in enumerate(roots):
        D = orc.plain_bfs(g, int(r))
        cand = np.flatnonzero((D >= 1) & (D <= d // 2))
        cand = cand[np.lexsort((cand, -deg[cand].astype(np.int64)))]
        k = int(rng.integers(min_k, 64 * W + 1))
        S = np.concatenate([[r], cand[:k - 1]]).astype(np.uint32)
        src[c, :len(S)] = S
        sz[c] = len(S)
        lists.append(S)
    return src, sz, lists


def run_wide(g, src, sz, W, d, planes=None, dist_bytes=2, direction=cb.CBFS_DIR_AUTO, stats=False):
    C = len(sz)
    planes = d + 1 if planes is None else planes
    dist = torch.empty((g.n, C), dtype=torch.int16 if dist_bytes == 2 else torch.uint8, device=DEV)
    masks = torch.empty((planes, g.n, C * W), dtype=torch.int64, device=DEV)
    st = torch.zeros((C * W, 4), dtype=torch.int64, device=DEV) if stats else None
    cb.cbfs_run_wide(g.h, to_dev_u32(src), torch.from_numpy(sz.view(np.int16)).to(DEV), C, W, d, dist_bytes, dist,
                     masks, planes, st, direction)
    return dist, masks, st


def check_against_oracle(ref, lists, dist, masks, W, d, planes):
    dh = dist.cpu().numpy()
    if dh.dtype == np.int16:
        dh = dh.view(np.uint16)
    else:  # u8 Delta, 0xFF = unreachable
        dh = dh.astype(np.uint16)
        dh[dh == 0xFF] = orc.INF16
    mh = np_u64(masks)
    for c, S in enumerate(lists):
        od, osub, over = orc.brute_cluster_wide(ref, S, d)
        assert not over
        assert np.array_equal(dh[:, c], od), c
        Wc = osub.shape[2]
        got = mh[:, :, c * W:(c + 1) * W]
        assert np.array_equal(got[:, :, :Wc], osub[:planes]), c
        assert not got[:, :, Wc:].any(), c  # words past the cluster's size stay empty


GRAPHS = {
    "rmat": lambda: ci.rmat(11, 16, 0.57, 0.19, 0.19, seed=61),
    "er": lambda: ci.erdos_renyi(3000, 30000, seed=62),
    "grid": lambda: ci.grid(40, 0.05, 0.01, 63),
}


@pytest.mark.parametrize("kind,d,W,C", [("rmat", 2, 2, 37), ("rmat", 2, 4, 20), ("rmat", 4, 8, 9), ("er", 4, 4, 18),
                                        ("er", 4, 8, 10), ("grid", 6, 2, 40), ("rmat", 2, 1, 70)])
@pytest.mark.parametrize("relabel", [False, True])
def test_run_wide_matches_definition(kind, d, W, C, relabel):
    el = GRAPHS[kind]()
    ref = orc.csr_from_edgelist(el)
    rng = np.random.default_rng(1000 + W * 7 + d)
    src, sz, lists = wide_clusters(ref, C, W, d, rng)
    g = gpu_graph(el, relabel=relabel)
    dist, masks, _ = run_wide(g, src, sz, W, d)
    torch.cuda.synchronize()
    check_against_oracle(ref, lists, dist, masks, W, d, d + 1)
    g.close()


@pytest.mark.parametrize("direction", [cb.CBFS_DIR_PUSH, cb.CBFS_DIR_PULL])
def test_run_wide_directions_and_u8(direction):
    el = GRAPHS["rmat"]()
    ref = orc.csr_from_edgelist(el)
    src, sz, lists = wide_clusters(ref, 24, 4, 2, np.random.default_rng(5), min_k=65)
    g = gpu_graph(el, relabel=True)
    dist, masks, st = run_wide(g, src, sz, 4, 2, dist_bytes=1, direction=direction, stats=True)
    check_against_oracle(ref, lists, dist, masks, 4, 2, 3)
    # each 64-source word's statistics are those of Alg. 1 on that word alone
    sth = st.cpu().numpy().view(np.uint64)
    for c in (0, 7, 23):
        for w in range(4):
            S = lists[c][64 * w:64 * (w + 1)]
            if len(S):
                assert np.array_equal(sth[c * 4 + w], orc.cluster_bfs(ref, S, 2).stats), (c, w)
            else:
                assert not sth[c * 4 + w].any()
    g.close()


@pytest.mark.parametrize("kind,d,W", [("rmat", 2, 4), ("grid", 4, 2), ("er", 4, 8)])
def test_wide_labels_decode_and_query(kind, d, W):
    """planes = d label records (R14, S_v[d] rebuilt word by word), decode
    of every source == its BFS, and the query == the brute-force landmark
    query over the clusters' sources."""
    el = GRAPHS[kind]()
    ref = orc.csr_from_edgelist(el)
    src, sz, lists = wide_clusters(ref, 12, W, d, np.random.default_rng(9))
    g = gpu_graph(el, relabel=(kind == "rmat"))
    for planes in (d, d + 1):
        dist, masks, _ = run_wide(g, src, sz, W, d, planes=planes)
        check_against_oracle(ref, lists, dist, masks, W, d, planes)
        for c in (0, 5, 11):
            k = int(sz[c])
            out = torch.empty((k, g.n), dtype=torch.int16, device=DEV)
            cb.cbfs_decode_wide(g.n, len(sz), W, d, planes, dist, 2, masks, c, k, out)
            oh = np_u16(out)
            for j in (0, k // 3, k - 1):
                bfs = orc.plain_bfs(ref, int(lists[c][j]))
                assert np.array_equal(oh[j], np.where(bfs == orc.INF32, 0xFFFF, bfs).astype(np.uint16)), (c, j)
        s, t = ci.query_pairs(g.n, 5000, seed=17, stream=3)
        best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device=DEV)
        cb.cbfs_query_distance_wide(g.n, len(sz), W, d, planes, dist, 2, masks,
                                    torch.from_numpy(sz.view(np.int16)).to(DEV), to_dev_u32(s), to_dev_u32(t), best)
        assert np.array_equal(best.cpu().numpy(), orc.query_brute(ref, lists, s, t))
    g.close()


@pytest.mark.parametrize("engine", ["batched", "sparse"])
def test_run_wide_each_engine(engine):
    """Both engines (forced) give the definition's output for wide clusters,
    on a low- and a high-diameter graph."""
    eng = cb.CBFS_ENGINE_BATCHED if engine == "batched" else cb.CBFS_ENGINE_SPARSE
    cb.cbfs_set_engine(eng)
    try:
        for kind, d, W in (("rmat", 2, 4), ("grid", 4, 2), ("er", 4, 8)):
            el = GRAPHS[kind]()
            ref = orc.csr_from_edgelist(el)
            src, sz, lists = wide_clusters(ref, 20, W, d, np.random.default_rng(77 + W))
            g = gpu_graph(el, relabel=(kind == "rmat"))
            for dist_bytes in (1, 2):
                dist, masks, _ = run_wide(g, src, sz, W, d, dist_bytes=dist_bytes)
                check_against_oracle(ref, lists, dist, masks, W, d, d + 1)
            g.close()
    finally:
        cb.cbfs_set_engine(cb.CBFS_ENGINE_AUTO)


def test_wide_errors_and_empty():
    el = GRAPHS["rmat"]()
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el)
    src, sz, lists = wide_clusters(ref, 3, 2, 2, np.random.default_rng(3), min_k=70)
    with pytest.raises(cb.CbfsError):  # words must be 1, 2, 4 or 8
        run_wide(g, src.reshape(3, 128), sz, 3, 2)
    bad = sz.copy(); bad[1] = 0
    with pytest.raises(cb.CbfsError):
        run_wide(g, src, bad, 2, 2)
    bad = sz.copy(); bad[2] = 129
    with pytest.raises(cb.CbfsError):
        run_wide(g, src, bad, 2, 2)
    dup = src.copy(); dup[0, 64] = dup[0, 3]  # the same source in two words (R2; sizes >= 70)
    with pytest.raises(cb.CbfsError):
        run_wide(g, dup, sz, 2, 2)
    oor = src.copy(); oor[1, 65] = g.n
    with pytest.raises(cb.CbfsError):
        run_wide(g, oor, sz, 2, 2)
    # zero clusters is a no-op; a valid call after the errors still matches
    cb.cbfs_run_wide(g.h, to_dev_u32(src), torch.from_numpy(sz.view(np.int16)).to(DEV), 0, 2, 2, 2, None, None, 3,
                     None)
    dist, masks, _ = run_wide(g, src, sz, 2, 2)
    check_against_oracle(ref, lists, dist, masks, 2, 2, 3)
    g.close()


@pytest.mark.timeout(600)
def test_wide_c2_full_size_sampled():
    """Config 2's graph (RMAT-20) at full size: 64 hub clusters of up to 256
    sources (d = 2) in one call; two sampled clusters word for word."""
    el = ci.make_graph("c2_rmat20")
    ref = orc.csr_from_edgelist(el)
    src, sz, lists = wide_clusters(ref, 64, 4, 2, np.random.default_rng(11), min_k=200)
    g = gpu_graph(el, relabel=True)
    dist, masks, _ = run_wide(g, src, sz, 4, 2, planes=3)
    torch.cuda.synchronize()
    dh, mh = np_u16(dist), np_u64(masks)
    for c in (0, 63):
        od, osub, over = orc.brute_cluster_wide(ref, lists[c], 2)
        assert not over
        assert np.array_equal(dh[:, c], od)
        assert np.array_equal(mh[:, :, c * 4:c * 4 + osub.shape[2]], osub)
    g.close()


@pytest.mark.parametrize("kind,d,W,k,relabel,policy", [("rmat", 2, 4, 256, True, 0), ("rmat", 2, 2, 100, False, 0),
                                                       ("er", 4, 8, 512, True, 0), ("grid", 4, 2, 70, False, 1),
                                                       ("rmat", 2, 8, 300, True, 1)])
def test_select_wide_matches_oracle_and_runs(kind, d, W, k, relabel, policy):
    """cbfs_select_clusters_wide == the oracle's selection (R12, general k),
    and the selected clusters through cbfs_run_wide == the definition."""
    el = GRAPHS[kind]()
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=relabel)
    r = 40
    src = torch.empty((r, 64 * W), dtype=torch.int32, device=DEV)
    sz = torch.empty((r,), dtype=torch.int16, device=DEV)
    got = cb.cbfs_select_clusters_wide(g.h, r, k, d, policy, 5, W, src, sz)
    osrc, osz = orc.select_clusters_wide(ref, r, k, d, W, policy, seed=5)
    assert got == len(osz)
    assert np.array_equal(src[:got].cpu().numpy().view(np.uint32), osrc)
    assert np.array_equal(sz[:got].cpu().numpy().view(np.uint16), osz)
    assert int(osz.max()) > 64 or W == 2 or policy == 1
    lists = [osrc[c, :osz[c]] for c in range(got)]
    dist, masks, _ = run_wide(g, osrc, osz, W, d)
    check_against_oracle(ref, lists[:12], dist, masks, W, d, d + 1)
    g.close()
