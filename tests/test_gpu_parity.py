"""GPU parity: the CUDA path through the C-ABI against the CPU oracle, element
by element, bit-exact (integer/bitwise path: BASELINE.json north_star asks
for bit-exact distances, masks, labels and answers)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci
import oracle as orc
import paper_2410_17226_b200 as cb
from gpu_util import gpu_graph, np_u16, np_u32, np_u64, run_clusters, to_dev_u32, to_dev_u8

pytestmark = pytest.mark.gpu

ENGINES = [cb.CBFS_ENGINE_BATCHED, cb.CBFS_ENGINE_SPARSE]


@pytest.fixture(params=ENGINES, ids=["batched", "sparse"])
def engine(request):
    """Run the test under each traversal engine (identical outputs, R8/R25)."""
    cb.cbfs_set_engine(request.param)
    yield request.param
    cb.cbfs_set_engine(cb.CBFS_ENGINE_AUTO)


@pytest.fixture(autouse=True)
def _reset_engine():
    yield
    cb.cbfs_set_engine(cb.CBFS_ENGINE_AUTO)


def each_mode():
    """(engine, direction) pairs: batched push / pull / auto and the sparse engine."""
    return [(cb.CBFS_ENGINE_BATCHED, cb.CBFS_DIR_AUTO), (cb.CBFS_ENGINE_BATCHED, cb.CBFS_DIR_PUSH),
            (cb.CBFS_ENGINE_BATCHED, cb.CBFS_DIR_PULL), (cb.CBFS_ENGINE_SPARSE, cb.CBFS_DIR_AUTO),
            (cb.CBFS_ENGINE_AUTO, cb.CBFS_DIR_AUTO)]


def random_el(seed, n, kind):
    rng = np.random.default_rng(seed)
    if kind == "er":
        m = int(rng.integers(n, 5 * n))
        s = rng.integers(0, n, m).astype(np.uint32); t = rng.integers(0, n, m).astype(np.uint32)
    elif kind == "rmat":
        scale = max(4, int(np.log2(n)))
        return ci.rmat(scale, 8, 0.57, 0.19, 0.19, seed=seed)
    elif kind == "path":
        s = np.arange(n - 1, dtype=np.uint32); t = s + 1
    else:  # grid
        side = int(np.sqrt(n))
        return ci.grid(side, 0.05, 0.01, seed)
    return ci.EdgeList(n, s, t)


def ball_clusters(g: orc.CSR, rng, C, d, kmax):
    """C clusters of random roots plus random vertices within floor(d/2) hops."""
    src = np.full((C, 64), orc.PAD, np.uint32)
    sz = np.zeros(C, np.uint8)
    h = d // 2
    for c in range(C):
        root = int(rng.integers(0, g.n))
        dist = orc.plain_bfs(g, root)
        cand = np.flatnonzero((dist >= 1) & (dist <= h))
        rng.shuffle(cand)
        S = [root] + cand[:kmax - 1].tolist()
        src[c, :len(S)] = S
        sz[c] = len(S)
    return src, sz


# ------------------------------------------------------------------ A0 CSR build
@pytest.mark.parametrize("relabel", [False, True, "locality"])
@pytest.mark.parametrize("case", ["c1", "er", "rmat", "grid", "empty"])
def test_csr_build_parity(case, relabel):
    if case == "c1":
        el = ci.make_graph("c1_er")
    elif case == "empty":
        el = ci.EdgeList(7, np.array([3, 3], np.uint32), np.array([3, 3], np.uint32))
    else:
        el = random_el(5, 3000, case)
    g = gpu_graph(el, relabel=relabel)
    ref = orc.csr_from_edgelist(el)
    off, cols = g.export_csr()
    assert g.n == ref.n and g.m == ref.m
    assert np.array_equal(off, ref.off) and np.array_equal(cols, ref.cols)
    assert g.max_degree == (int(ref.degrees().max()) if ref.n else 0)


def _locality_order_ref(ref):
    """The documented CBFS_RELABEL_LOCALITY order (include/cbfs.h), written out:
    BFS from the highest-degree vertex (ties: smallest id); level L+1 sorted by
    (smallest position of a parent in level L, id); unreached vertices
    appended in id order.  Internal position -> original id."""
    n = ref.n
    deg = np.diff(ref.off.astype(np.int64))
    root = int(np.lexsort((np.arange(n), -deg))[0])
    pos = np.full(n, -1, np.int64)
    order = [root]
    pos[root] = 0
    lo, hi = 0, 1
    while hi > lo:
        key = {}
        for p in range(lo, hi):
            u = order[p]
            for v in ref.cols[ref.off[u]:ref.off[u + 1]]:
                v = int(v)
                if pos[v] < 0 and v not in key:
                    key[v] = p
        nxt = sorted(key, key=lambda v: (key[v], v))
        for v in nxt:
            pos[v] = len(order)
            order.append(v)
        lo, hi = hi, len(order)
    order += [v for v in range(n) if pos[v] < 0]
    return np.array(order, np.uint32)


@pytest.mark.parametrize("case", ["grid", "er", "path", "rmat", "two", "knn"])
def test_locality_order_definition(case):
    """The locality relabel (one cooperative kernel over all BFS levels) gives
    exactly the documented order — several components, hubs and long paths
    (thousands of levels) included."""
    if case == "two":  # two components + isolated vertices
        a = random_el(11, 900, "grid")
        s_ = np.concatenate([a.src, a.src + a.n]).astype(np.uint32)
        t_ = np.concatenate([a.dst, a.dst + a.n]).astype(np.uint32)
        el = ci.EdgeList(2 * a.n + 5, s_, t_)
    elif case == "path":
        el = random_el(12, 4000, "path")
    elif case == "knn":
        el = ci.knn3d(20000, 10, seed=14)
    else:
        el = random_el(13, 2500, case)
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel="locality")
    assert np.array_equal(cb.cbfs_graph_internal_order(g.h), _locality_order_ref(ref))
    off, cols = g.export_csr()
    assert np.array_equal(off, ref.off) and np.array_equal(cols, ref.cols)
    g0 = gpu_graph(el, relabel=False)
    assert np.array_equal(cb.cbfs_graph_internal_order(g0.h), np.arange(el.n, dtype=np.uint32))


def test_csr_build_from_device_and_csr_input():
    el = random_el(9, 2000, "er")
    ref = orc.csr_from_edgelist(el)
    g = cb.Graph.from_edges(el.n, to_dev_u32(el.src), to_dev_u32(el.dst))
    off, cols = g.export_csr()
    assert np.array_equal(off, ref.off) and np.array_equal(cols, ref.cols)
    g2 = cb.Graph.from_csr(ref.n, ref.off, ref.cols, relabel=True)
    off2, cols2 = g2.export_csr()
    assert np.array_equal(off2, ref.off) and np.array_equal(cols2, ref.cols)


def test_csr_build_rejects_bad_ids():
    with pytest.raises(cb.CbfsError) as e:
        cb.Graph.from_edges(4, np.array([0, 9], np.uint32), np.array([1, 2], np.uint32))
    assert e.value.code == cb.CBFS_EINVAL


# ------------------------------------------------------------------ A1 selection
@pytest.mark.parametrize("relabel", [False, True, "locality"])
@pytest.mark.parametrize("policy,d,k", [(0, 2, 64), (1, 2, 64), (0, 4, 13), (1, 4, 64), (0, 6, 64), (0, 3, 5),
                                        (0, 0, 1), (1, 1, 64)])
def test_selection_parity(policy, d, k, relabel):
    el = random_el(21, 4000, "rmat")
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=relabel)
    r = 200
    src, sz = g.select_clusters(r, k, d, policy, seed=77)
    osrc, osz = orc.select_clusters(ref, r, k, d, policy, seed=77)
    assert np.array_equal(sz.cpu().numpy(), osz)
    assert np.array_equal(np_u32(src), osrc)


def test_selection_runs_out():
    el = ci.EdgeList(10, np.array([0, 2, 4], np.uint32), np.array([1, 3, 5], np.uint32))
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el)
    for policy in (0, 1):
        src, sz = g.select_clusters(50, 64, 2, policy, seed=3)
        osrc, osz = orc.select_clusters(ref, 50, 64, 2, policy, seed=3)
        assert len(osz) == 3 and np.array_equal(sz.cpu().numpy(), osz) and np.array_equal(np_u32(src), osrc)


def test_selection_c1_and_c2_full_size():
    for name, policy, seed in (("c1_er", 1, 1), ("c2_rmat20", 0, 0)):
        cfg = ci.CONFIGS[name]
        el = ci.make_graph(name)
        ref = orc.csr_from_edgelist(el)
        g = gpu_graph(el, relabel=(name != "c1_er"))
        src, sz = g.select_clusters(cfg["clusters"], cfg["k"], cfg["d"], policy, seed=seed)
        osrc, osz = orc.select_clusters(ref, cfg["clusters"], cfg["k"], cfg["d"], policy, seed=seed)
        assert np.array_equal(sz.cpu().numpy(), osz), name
        assert np.array_equal(np_u32(src), osrc), name


# ------------------------------------------------------------------ A2-A8 C-BFS
def compare_many(g, ref, src, sz, d, **kw):
    gd, gs, gst = run_clusters(g, src, sz, d, **kw)
    om = orc.cluster_bfs_many(ref, src, sz, d, threads=8)
    planes = gs.shape[1]
    assert np.array_equal(gd, om["dist"])
    assert np.array_equal(gs, om["sub"][:, :planes, :])
    assert np.array_equal(gst, om["stats"])
    return gd, gs, gst


@pytest.mark.parametrize("direction", [cb.CBFS_DIR_AUTO, cb.CBFS_DIR_PUSH, cb.CBFS_DIR_PULL])
@pytest.mark.parametrize("relabel", [False, True])
def test_c1_full_parity(direction, relabel, engine):
    cfg = ci.CONFIGS["c1_er"]
    el = ci.make_graph("c1_er")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, cfg["clusters"], cfg["k"], cfg["d"], orc.ROOT_RANDOM, seed=cfg["root_seed"])
    g = gpu_graph(el, relabel=relabel)
    gd, gs, _ = compare_many(g, ref, src, sz, cfg["d"], direction=direction, dist_bytes=1)
    # and against the definition: 64 x 8 independent BFS runs (BASELINE.json config 1)
    for c in range(len(sz)):
        bd, bs, over = orc.brute_cluster(ref, src[c, :sz[c]], cfg["d"])
        assert not over and np.array_equal(gd[c], bd) and np.array_equal(gs[c], bs)


@pytest.mark.parametrize("seed", range(16))
def test_random_graphs_parity(seed):
    rng = np.random.default_rng(4000 + seed)
    kind = ["er", "rmat", "grid", "path"][seed % 4]
    n = int(rng.integers(300, 3000))
    el = random_el(seed, n, kind)
    ref = orc.csr_from_edgelist(el)
    d = [0, 1, 2, 3, 4, 6][seed % 6]
    C = [1, 5, 31, 32, 33, 70][seed % 6]  # ragged batches
    src, sz = ball_clusters(ref, rng, C, d, [1, 7, 64][seed % 3] if d else 1)
    g = gpu_graph(el, relabel=[False, True, "locality"][seed % 3])
    for eng, direction in each_mode():
        cb.cbfs_set_engine(eng)
        compare_many(g, ref, src, sz, d, direction=direction)


@pytest.mark.parametrize("seed", range(4))
def test_pull_hint_threshold_parity(seed):
    """The pull's L2-hint threshold (cbfs_set_pull_hub_rows) changes only cache
    policies: outputs equal the oracle's for 0, 8 and all rows as hubs."""
    rng = np.random.default_rng(4100 + seed)
    el = random_el(seed + 7, int(rng.integers(500, 3000)), ["er", "rmat"][seed % 2])
    ref = orc.csr_from_edgelist(el)
    src, sz = ball_clusters(ref, rng, 40, 2, 64)
    g = gpu_graph(el, relabel=True)
    cb.cbfs_set_engine(cb.CBFS_ENGINE_BATCHED)
    try:
        for hub in (0, 8, 1 << 30):
            cb.cbfs_set_pull_hub_rows(hub)
            compare_many(g, ref, src, sz, 2, direction=cb.CBFS_DIR_PULL)
    finally:
        cb.cbfs_set_pull_hub_rows(131072)


@pytest.mark.parametrize("seed", range(6))
def test_sparse_ordered_frontier_parity(seed):
    """The sparse engine's ordered frontiers (claims through the bitmap, F_{i+1}
    compacted in (cluster, vertex) order) change only the order of frontier
    entries: outputs equal the oracle's with the bitmap used on every round
    (threshold 1), on every round of >= 64 entries, and never — on low- and
    high-degree graphs (both push shapes), d = 0 (separate fold) included."""
    rng = np.random.default_rng(5200 + seed)
    kind = ["er", "rmat", "grid", "path", "er", "grid"][seed]
    el = random_el(seed + 300, int(rng.integers(800, 3000)), kind)
    ref = orc.csr_from_edgelist(el)
    d = [0, 1, 2, 3, 4, 6][seed]
    src, sz = ball_clusters(ref, rng, [5, 33, 64, 70, 40, 64][seed], d, [1, 7, 64][seed % 3] if d else 1)
    g = gpu_graph(el, relabel=[False, True, "locality"][seed % 3])
    cb.cbfs_set_engine(cb.CBFS_ENGINE_SPARSE)
    try:
        for thr in (1, 64, 0):
            cb.cbfs_set_sparse_order(thr)
            compare_many(g, ref, src, sz, d)
    finally:
        cb.cbfs_set_sparse_order(-1)
        cb.cbfs_set_engine(cb.CBFS_ENGINE_AUTO)
    with pytest.raises(cb.CbfsError):
        cb.cbfs_set_sparse_order(-2)


@pytest.mark.parametrize("seed", range(6))
def test_diameter_exceeds_d_parity(seed):
    """R9: clusters whose diameter exceeds d still give Alg. 1's output exactly,
    in every direction mode."""
    rng = np.random.default_rng(5000 + seed)
    el = random_el(seed + 50, 1500, ["er", "rmat", "grid"][seed % 3])
    ref = orc.csr_from_edgelist(el)
    C = 40
    src = np.full((C, 64), orc.PAD, np.uint32)
    sz = np.zeros(C, np.uint8)
    for c in range(C):
        k = int(rng.integers(1, 65))
        S = rng.choice(el.n, size=k, replace=False)
        src[c, :k] = S; sz[c] = k
    d = [1, 2, 3][seed % 3]
    g = gpu_graph(el, relabel=[False, True, "locality"][seed % 3])
    for eng, direction in each_mode():
        cb.cbfs_set_engine(eng)
        compare_many(g, ref, src, sz, d, direction=direction)


def test_label_planes_and_u8_dist(engine):
    el = random_el(77, 2500, "rmat")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 40, 64, 2)
    g = gpu_graph(el, relabel=True)
    compare_many(g, ref, src, sz, 2, planes=2, dist_bytes=1)


def test_edge_cases(engine):
    # isolated source; graph without edges; single-vertex cluster on a path with d=0 (plain BFS)
    el = ci.EdgeList(6, np.array([1, 2], np.uint32), np.array([2, 3], np.uint32))
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el)
    src = np.full((3, 64), orc.PAD, np.uint32); sz = np.array([1, 2, 1], np.uint8)
    src[0, 0] = 0; src[1, :2] = [1, 3]; src[2, 0] = 5
    compare_many(g, ref, src, sz, 2)
    g0 = gpu_graph(ci.EdgeList(5, np.array([], np.uint32), np.array([], np.uint32)))
    ref0 = orc.csr_from_edges(5, np.array([], np.uint32), np.array([], np.uint32))
    src0 = np.full((1, 64), orc.PAD, np.uint32); src0[0, :3] = [0, 2, 4]
    compare_many(g0, ref0, src0, np.array([3], np.uint8), 0)
    # zero clusters: nothing to do, no error
    cb.cbfs_run(g.h, to_dev_u32(src), to_dev_u8(sz), 0, 2, 2, None, None, 3)


def test_invalid_sources_rejected(engine):
    el = random_el(3, 500, "er")
    g = gpu_graph(el)
    for S, k in (([1, 1], 2), ([600], 1), ([0], 0)):
        src = np.full((1, 64), orc.PAD, np.uint32); src[0, :len(S)] = S
        with pytest.raises(cb.CbfsError) as e:
            g.run(to_dev_u32(src), to_dev_u8(np.array([k], np.uint8)), 2)
        assert e.value.code == cb.CBFS_EINVAL
    # the workspace stays usable after an error
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 3, 64, 2)
    compare_many(g, ref, src, sz, 2)


def test_overflow_u8(engine):
    n = 600
    el = random_el(0, n, "path")
    g = gpu_graph(el)
    src = np.full((1, 64), orc.PAD, np.uint32); src[0, 0] = 0
    with pytest.raises(cb.CbfsError) as e:
        g.run(to_dev_u32(src), to_dev_u8(np.array([1], np.uint8)), 0, dist_bytes=1)
    assert e.value.code == cb.CBFS_EOVERFLOW
    ref = orc.csr_from_edgelist(el)
    compare_many(g, ref, src, np.array([1], np.uint8), 0)  # u16 is fine


@pytest.mark.parametrize("staging", [False, True])
def test_run_host_equals_device(engine, staging, monkeypatch):
    """cbfs_run_host: device-resident output + one DMA, and (forced) per-batch staging."""
    if staging:
        monkeypatch.setenv("CBFS_HOST_STAGING", "1")
    el = random_el(8, 3000, "rmat")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 45, 64, 2)
    g = gpu_graph(el, relabel=True)
    C, n, d = len(sz), g.n, 2
    hd = np.empty((n, C), np.uint16); hm = np.empty((d + 1, n, C), np.uint64); hs = np.zeros((C, 4), np.uint64)
    cb.cbfs_run_host(g.h, np.ascontiguousarray(src), np.ascontiguousarray(sz), C, d, 2, hd, hm, d + 1, hs)
    om = orc.cluster_bfs_many(ref, src, sz, d)
    assert np.array_equal(hd.T, om["dist"]) and np.array_equal(hm.transpose(2, 0, 1), om["sub"])
    assert np.array_equal(hs, om["stats"])


# ------------------------------------------------------------------ A9 decode
def test_decode_parity():
    el = random_el(12, 2000, "er")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 5, 64, 2)
    g = gpu_graph(el, relabel=True)
    for planes in (3, 2):
        dist, masks, _ = g.run(to_dev_u32(src), to_dev_u8(sz), 2, planes=planes)
        for c in range(len(sz)):
            k = int(sz[c])
            out = torch.empty((k, g.n), dtype=torch.int16, device="cuda:0")
            cb.cbfs_decode(g.n, len(sz), 2, planes, dist, 2, masks, c, k, out)
            got = np_u16(out).astype(np.int64)
            for j in range(k):
                ref_d = orc.plain_bfs(ref, int(src[c, j])).astype(np.int64)
                ref_d[ref_d == orc.INF32] = 0xFFFF
                assert np.array_equal(got[j], ref_d)


# ------------------------------------------------------------------ A10/A11 labels and queries
@pytest.mark.parametrize("d,planes,dist_bytes", [(2, 2, 1), (2, 3, 2), (4, 4, 2), (6, 6, 2)])
def test_query_parity(d, planes, dist_bytes, engine):
    el = random_el(31 + d, 3000, "rmat" if d == 2 else "grid")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 70, 64, d)
    g = gpu_graph(el, relabel=(d == 2))
    C = len(sz)
    dist, masks, _ = g.run(to_dev_u32(src), to_dev_u8(sz), d, dist_bytes=dist_bytes, planes=planes)
    q = 20000
    s, t = ci.query_pairs(g.n, q, seed=7)
    s[:50] = src[0, 0]; t[:50] = src[0, 0]  # u = v = landmark -> 0
    best = torch.full((q,), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda:0")
    cb.cbfs_query_distance(g.n, C, d, planes, dist, dist_bytes, masks, to_dev_u8(sz), to_dev_u32(s), to_dev_u32(t),
                           best)
    om = orc.cluster_bfs_many(ref, src, sz, d)
    expect = orc.query(om["dist"], om["sub"], s, t)
    assert np.array_equal(best.cpu().numpy(), expect)
    assert np.all(expect[:50] == 0)
    # streaming build+query gives the same answers without a resident store
    best2 = torch.full((q,), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda:0")
    cb.cbfs_query_stream(g.h, to_dev_u32(src), to_dev_u8(sz), C, d, to_dev_u32(s), to_dev_u32(t), best2)
    assert np.array_equal(best2.cpu().numpy(), expect)


def test_query_bad_ids():
    el = random_el(3, 500, "er")
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 2, 8, 2)
    g = gpu_graph(el)
    dist, masks, _ = g.run(to_dev_u32(src), to_dev_u8(sz), 2)
    best = torch.full((1,), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda:0")
    with pytest.raises(cb.CbfsError):
        cb.cbfs_query_distance(g.n, len(sz), 2, 3, dist, 2, masks, to_dev_u8(sz), to_dev_u32(np.array([0], np.uint32)),
                               to_dev_u32(np.array([999], np.uint32)), best)


# ------------------------------------------------------------------ full size (config 2, as bench.py runs it)
def test_c2_full_size_sampled():
    """BASELINE.json config 2 at full size in the bench launch configuration:
    GPU selection == oracle selection, all 1024 clusters traversed in one
    cbfs_run, per-cluster round stats of every cluster == oracle, and 40
    sampled clusters compared element by element."""
    cfg = ci.CONFIGS["c2_rmat20"]
    el = ci.make_graph("c2_rmat20")
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=True)
    src_d, sz_d = g.select_clusters(cfg["clusters"], cfg["k"], cfg["d"], cb.CBFS_ROOT_DEGREE, 0)
    src, sz = np_u32(src_d), sz_d.cpu().numpy()
    osrc, osz = orc.select_clusters(ref, cfg["clusters"], cfg["k"], cfg["d"])
    assert np.array_equal(src, osrc) and np.array_equal(sz, osz)
    C, d = len(sz), cfg["d"]
    dist = torch.empty((g.n, C), dtype=torch.uint8, device="cuda:0")
    masks = torch.empty((d + 1, g.n, C), dtype=torch.int64, device="cuda:0")
    stats = torch.zeros((C, 4), dtype=torch.int64, device="cuda:0")
    cb.cbfs_run(g.h, src_d, sz_d, C, d, 1, dist, masks, d + 1, stats)
    torch.cuda.synchronize()
    st = stats.cpu().numpy().view(np.uint64)
    sample = sorted(set([0, 1, 31, 32, 33, 500, 767, C - 1] + list(np.random.default_rng(0).choice(C, 32, False))))
    om = orc.cluster_bfs_many(ref, src[sample], sz[sample], d)
    for j, c in enumerate(sample):
        gd = dist[:, c].cpu().numpy().astype(np.uint16)
        gd[gd == 0xFF] = 0xFFFF
        assert np.array_equal(gd, om["dist"][j]), c
        assert np.array_equal(np_u64(masks[:, :, c].contiguous()), om["sub"][j]), c
        assert np.array_equal(st[c], om["stats"][j]), c
    allst = orc.cluster_bfs_many(ref, src, sz, d, want_outputs=False)["stats"]
    assert np.array_equal(st, allst)


@pytest.mark.parametrize("policy,r", [(0, 150), (1, 70), (0, 5000)])
def test_select_and_run_equals_separate_calls(policy, r, engine):
    """A1 overlapped with A2-A8 (cbfs_select_and_run) == cbfs_select_clusters + cbfs_run == oracle."""
    el = random_el(91, 5000, "rmat")
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=True)
    d = 2
    src = torch.empty((r, 64), dtype=torch.int32, device="cuda:0")
    sz = torch.empty((r,), dtype=torch.uint8, device="cuda:0")
    dist = torch.empty((g.n, r), dtype=torch.uint8, device="cuda:0")
    masks = torch.empty((d + 1, g.n, r), dtype=torch.int64, device="cuda:0")
    stats = torch.zeros((r, 4), dtype=torch.int64, device="cuda:0")
    got = cb.cbfs_select_and_run(g.h, r, 64, d, policy, 5, src, sz, 1, dist, masks, d + 1, stats)
    osrc, osz = orc.select_clusters(ref, r, 64, d, policy, seed=5)
    assert got == len(osz) and got <= r
    assert np.array_equal(np_u32(src[:got]), osrc) and np.array_equal(sz[:got].cpu().numpy(), osz)
    om = orc.cluster_bfs_many(ref, osrc, osz, d)
    gd = dist.cpu().numpy().astype(np.uint16)
    gd[gd == 0xFF] = 0xFFFF
    assert np.array_equal(gd.T[:got], om["dist"])
    assert np.array_equal(np_u64(masks).transpose(2, 0, 1)[:got], om["sub"])
    assert np.array_equal(stats.cpu().numpy().view(np.uint64)[:got], om["stats"])
    if got < r:  # columns past the selected clusters stay unreached
        assert np.all(gd.T[got:] == 0xFFFF) and not np.any(np_u64(masks).transpose(2, 0, 1)[got:])


# ------------------------------------------------------------------ engines
def test_auto_engine_choice_and_equivalence():
    """AUTO picks SPARSE on a high-diameter grid and BATCHED on an RMAT graph;
    every engine gives the oracle's output on both (R8/R25)."""
    for el, d in ((ci.grid(200, 0.05, 0.001, 7), 4), (ci.rmat(13, 16, 0.57, 0.19, 0.19, seed=7), 2)):
        ref = orc.csr_from_edgelist(el)
        src, sz = orc.select_clusters(ref, 100, 64, d)
        g = gpu_graph(el)
        for eng in (cb.CBFS_ENGINE_AUTO, cb.CBFS_ENGINE_BATCHED, cb.CBFS_ENGINE_SPARSE):
            cb.cbfs_set_engine(eng)
            cb.cbfs_profile_enable(True)
            cb.cbfs_profile_read(reset=True)
            try:
                compare_many(g, ref, src, sz, d)
            except AssertionError as e:
                gd, gs, gst = run_clusters(g, src, sz, d)
                om = orc.cluster_bfs_many(ref, src, sz, d, threads=8)
                bad = [c for c in range(len(sz)) if not np.array_equal(gd[c], om["dist"][c])]
                raise AssertionError(f"{el.name} engine {eng}: {cb.cbfs_profile_read()} bad(rerun) {bad} "
                                     f"stats {gst[60:70].tolist()} vs {om['stats'][60:70].tolist()}") from e
            prof = cb.cbfs_profile_read(reset=True)
            cb.cbfs_profile_enable(False)
            used_sparse = prof["sparse"]["launches"] > 0
            if eng == cb.CBFS_ENGINE_AUTO:
                assert used_sparse == (d == 4), (el.name, prof)
            else:
                assert used_sparse == (eng == cb.CBFS_ENGINE_SPARSE)


def test_sparse_engine_round_cap_and_recovery():
    """A path longer than 65534 rounds: EOVERFLOW from the device-side loop;
    the workspace is usable afterwards."""
    n = 70000
    el = random_el(0, n, "path")
    g = gpu_graph(el)
    cb.cbfs_set_engine(cb.CBFS_ENGINE_SPARSE)
    src = np.full((1, 64), orc.PAD, np.uint32); src[0, 0] = 0
    with pytest.raises(cb.CbfsError) as e:
        g.run(to_dev_u32(src), to_dev_u8(np.array([1], np.uint8)), 0)
    assert e.value.code == cb.CBFS_EOVERFLOW
    el2 = random_el(5, 2000, "grid")
    ref2 = orc.csr_from_edgelist(el2)
    src2, sz2 = orc.select_clusters(ref2, 20, 64, 2)
    compare_many(gpu_graph(el2), ref2, src2, sz2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_select_and_run_shard_round_robin(world, engine):
    """cbfs_select_and_run_shard: rank r's outputs are exactly the oracle's for
    clusters r, r + world, ... of the full selection."""
    el = random_el(93, 4000, "rmat")
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=True)
    d, r = 2, 200
    osrc, osz = orc.select_clusters(ref, r, 64, d, 0, seed=0)
    om = orc.cluster_bfs_many(ref, osrc, osz, d)
    for rank in range(world):
        Cr = (r - rank + world - 1) // world
        src = torch.empty((r, 64), dtype=torch.int32, device="cuda:0")
        sz = torch.empty((r,), dtype=torch.uint8, device="cuda:0")
        dist = torch.empty((g.n, Cr), dtype=torch.uint8, device="cuda:0")
        masks = torch.empty((d + 1, g.n, Cr), dtype=torch.int64, device="cuda:0")
        stats = torch.zeros((Cr, 4), dtype=torch.int64, device="cuda:0")
        got = cb.cbfs_select_and_run_shard(g.h, r, 64, d, 0, 0, world, rank, src, sz, 1, dist, masks, d + 1, stats)
        assert got == len(osz) == r
        assert np.array_equal(np_u32(src), osrc)
        idx = np.arange(rank, r, world)
        gd = dist.cpu().numpy().astype(np.uint16)
        gd[gd == 0xFF] = 0xFFFF
        assert np.array_equal(gd.T, om["dist"][idx])
        assert np.array_equal(np_u64(masks).transpose(2, 0, 1), om["sub"][idx])
        assert np.array_equal(stats.cpu().numpy().view(np.uint64), om["stats"][idx])
