"""Pins for the CPU oracle (`-m "not gpu"`).

Every check here fixes the oracle against something other than itself:
scipy's BFS (a library routine) encoded through the definition P:630-639,
closed forms, values the paper prints (tests/golden/), hand-worked cases and
invariants stated by the paper.  A plausible mistake in Alg. 1 (a dropped
fold, a wrong cap sign, seeding per the literal P:707-708 instead of R1, an
off-by-one offset) fails at least one of them.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

import cbfs_inputs as ci
import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ helpers
def scipy_dist(g: orc.CSR, S) -> np.ndarray:
    """[k][n] hop distances via scipy (BFS on unit weights); inf -> -1."""
    A = sp.csr_matrix((np.ones(g.m), g.cols.astype(np.int64), g.off.astype(np.int64)), shape=(g.n, g.n))
    D = shortest_path(A, method="D", unweighted=True, directed=False, indices=np.asarray(S, dtype=np.int64))
    D = np.atleast_2d(D)
    out = np.where(np.isinf(D), -1, D).astype(np.int64)
    return out


def encode_definition(D: np.ndarray, d: int):
    """Cluster distance vector from a [k][n] distance matrix."""
    k, n = D.shape
    dist = np.full(n, orc.INF16, np.uint16)
    sub = np.zeros((d + 1, n), np.uint64)
    for v in range(n):
        col = D[:, v]
        reach = col >= 0
        if not reach.any():
            continue
        mn = int(col[reach].min())
        dist[v] = mn
        for j in range(k):
            if col[j] >= 0:
                i = int(col[j]) - mn
                assert i <= d, "cluster diameter exceeds d"
                sub[i, v] |= np.uint64(1 << j)
    return dist, sub


def graph_from_pairs(n, pairs) -> orc.CSR:
    pairs = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
    return orc.csr_from_edges(n, pairs[:, 0], pairs[:, 1])


def ball_cluster(g: orc.CSR, root: int, h: int, k: int, rng) -> list:
    """root + up to k-1 random vertices within h hops: diameter <= 2h."""
    D = scipy_dist(g, [root])[0]
    cand = [v for v in np.flatnonzero((D >= 1) & (D <= h)).tolist()]
    rng.shuffle(cand)
    return [root] + cand[:k - 1]


def random_graph(rng, n, kind):
    if kind == "er":
        m = int(rng.integers(n, 4 * n))
        s = rng.integers(0, n, m); t = rng.integers(0, n, m)
    else:  # preferential-attachment-like: new vertex links to existing ones by degree
        s, t = [], []
        deg = np.ones(n)
        for v in range(1, n):
            for _ in range(int(rng.integers(1, 4))):
                p = deg[:v] / deg[:v].sum()
                u = int(rng.choice(v, p=p))
                s.append(v); t.append(u); deg[u] += 1; deg[v] += 1
        s, t = np.array(s), np.array(t)
    return orc.csr_from_edges(n, s.astype(np.uint32), t.astype(np.uint32))


# ------------------------------------------------------------------ CSR build
def test_csr_matches_scipy():
    el = ci.erdos_renyi(500, 3000, seed=11)
    g = orc.csr_from_edgelist(el)
    A = sp.coo_matrix((np.ones(len(el.src)), (el.src.astype(np.int64), el.dst.astype(np.int64))), shape=(500, 500))
    A = ((A + A.T) > 0).astype(np.int8).tolil()
    A.setdiag(0)
    A = A.tocsr(); A.eliminate_zeros(); A.sort_indices()
    assert np.array_equal(g.off.astype(np.int64), A.indptr.astype(np.int64))
    assert np.array_equal(g.cols.astype(np.int64), A.indices.astype(np.int64))
    # symmetric, no self loops, strictly ascending rows
    for v in range(g.n):
        row = g.cols[g.off[v]:g.off[v + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0) and v not in row


@pytest.mark.parametrize("seed", range(3))
def test_csr_c_builder_matches_scipy(seed):
    """The C normaliser used for large edge lists (or_csr_build) gives scipy's
    symmetrised, self-loop-free, deduplicated sorted CSR (and numpy's)."""
    n = [300, 1000, 5000][seed]
    rng = np.random.default_rng(100 + seed)
    P = 6 * n
    s = rng.integers(0, n, P).astype(np.uint32); t = rng.integers(0, n, P).astype(np.uint32)
    s[:50] = t[:50]  # self loops
    s[50:60] = s[60:70]; t[50:60] = t[60:70]  # duplicates
    g = orc.csr_from_edges_c(n, s, t, threads=3)
    A = sp.coo_matrix((np.ones(P), (s.astype(np.int64), t.astype(np.int64))), shape=(n, n))
    A = ((A + A.T) > 0).astype(np.int8).tolil()
    A.setdiag(0)
    A = A.tocsr(); A.eliminate_zeros(); A.sort_indices()
    assert np.array_equal(g.off.astype(np.int64), A.indptr.astype(np.int64))
    assert np.array_equal(g.cols.astype(np.int64), A.indices.astype(np.int64))
    g2 = orc.csr_from_edges(n, s, t)
    assert np.array_equal(g.off, g2.off) and np.array_equal(g.cols, g2.cols)
    with pytest.raises(ValueError):
        orc.csr_from_edges_c(3, np.array([0], np.uint32), np.array([3], np.uint32))


def test_csr_empty_and_isolated():
    g = orc.csr_from_edges(5, np.array([], np.uint32), np.array([], np.uint32))
    assert g.m == 0 and g.off.tolist() == [0] * 6
    g = orc.csr_from_edges(3, np.array([1, 1], np.uint32), np.array([1, 1], np.uint32))  # self loops only
    assert g.m == 0


# ------------------------------------------------------------------ plain BFS
def test_plain_bfs_path_and_scipy():
    g = graph_from_pairs(3, [0, 1, 1, 2])
    assert orc.plain_bfs(g, 0).tolist() == [0, 1, 2]  # SPEC plain_bfs example
    g = random_graph(np.random.default_rng(1), 300, "er")
    d = orc.plain_bfs(g, 7).astype(np.int64)
    d[d == orc.INF32] = -1
    assert np.array_equal(d, scipy_dist(g, [7])[0])


# ------------------------------------------------------------------ Alg. 1 vs definition
@pytest.mark.parametrize("seed", range(40))
def test_alg1_equals_definition_random(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(20, 160))
    g = random_graph(rng, n, "er" if seed % 2 else "pa")
    d = [0, 1, 2, 3, 4, 6][seed % 6]
    k = [1, 7, 64][seed % 3] if d > 0 else 1
    root = int(rng.integers(0, n))
    S = ball_cluster(g, root, d // 2, k, rng)
    res = orc.cluster_bfs(g, S, d)
    dist, sub = encode_definition(scipy_dist(g, S), d)
    assert np.array_equal(res.dist, dist)
    assert np.array_equal(res.sub, sub)
    # the oracle's own brute force agrees too
    bd, bs, over = orc.brute_cluster(g, S, d)
    assert not over and np.array_equal(bd, dist) and np.array_equal(bs, sub)


@pytest.mark.parametrize("seed", range(12))
def test_alg1_invariants(seed):
    """Rounds = 1 + max delta (<= D + d + 1); |F_i| = #{v: some delta(s,v)=i};
    E_i = sum of their degrees; each vertex in <= d+1 frontiers."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(50, 200))
    g = random_graph(rng, n, "er")
    d = [1, 2, 3, 4][seed % 4]
    S = ball_cluster(g, int(rng.integers(0, n)), d // 2, 64, rng)
    res = orc.cluster_bfs(g, S, d)
    D = scipy_dist(g, S)
    maxd = int(D.max())
    assert int(res.stats[0]) == 1 + maxd
    deg = g.degrees().astype(np.int64)
    appear = np.zeros(n, np.int64)
    for i in range(maxd + 1):
        Fi = np.flatnonzero((D == i).any(axis=0))
        assert int(res.round_F[i]) == len(Fi)
        assert int(res.round_E[i]) == int(deg[Fi].sum())
        appear[Fi] += 1
    assert appear.max() <= d + 1
    assert int(res.stats[1]) == int(appear.sum())
    reached = (D >= 0).any(axis=0)
    assert int(res.stats[3]) == int(deg[reached].sum())


def test_k1_d0_is_plain_bfs():
    g = random_graph(np.random.default_rng(5), 400, "er")
    res = orc.cluster_bfs(g, [17], 0)
    ref = scipy_dist(g, [17])[0]
    assert np.array_equal(np.where(res.dist == orc.INF16, -1, res.dist.astype(np.int64)), ref)
    assert np.array_equal(res.sub[0], np.where(ref >= 0, 1, 0).astype(np.uint64))


# ------------------------------------------------------------------ closed forms
def test_path_closed_form():
    n = 40
    g = graph_from_pairs(n, [x for i in range(n - 1) for x in (i, i + 1)])
    S = [10, 11, 12]  # diameter 2
    res = orc.cluster_bfs(g, S, 2)
    for v in range(n):
        ds = [abs(v - s) for s in S]
        mn = min(ds)
        assert res.dist[v] == mn
        for i in range(3):
            assert int(res.sub[i, v]) == sum(1 << j for j, x in enumerate(ds) if x - mn == i)


def test_cycle_closed_form():
    n = 31
    g = graph_from_pairs(n, [x for i in range(n) for x in (i, (i + 1) % n)])
    S = [0, 1, 30, 2]  # within 2 hops of each other... 30-2 distance 3 -> d=3
    res = orc.cluster_bfs(g, S, 3)
    for v in range(n):
        ds = [min(abs(v - s), n - abs(v - s)) for s in S]
        mn = min(ds)
        assert res.dist[v] == mn
        for i in range(4):
            assert int(res.sub[i, v]) == sum(1 << j for j, x in enumerate(ds) if x - mn == i)


def test_star_closed_form():
    """K_{1,L}, S = centre + 63 leaves (SURVEY §8(c) closed forms)."""
    L = 100
    g = graph_from_pairs(L + 1, [x for i in range(1, L + 1) for x in (0, i)])
    S = [0] + list(range(1, 64))
    res = orc.cluster_bfs(g, S, 2)
    leaves = sum(1 << j for j in range(1, 64))
    assert res.dist[0] == 0 and res.sub[0, 0] == 1 and res.sub[1, 0] == leaves and res.sub[2, 0] == 0
    for j in range(1, 64):  # member leaf
        assert res.dist[j] == 0 and res.sub[0, j] == 1 << j and res.sub[1, j] == 1
        assert res.sub[2, j] == leaves & ~(1 << j)
    for v in range(64, L + 1):  # other leaf
        assert res.dist[v] == 1 and res.sub[0, v] == 1 and res.sub[1, v] == leaves and res.sub[2, v] == 0


def test_complete_graph_closed_form():
    n = 12
    g = graph_from_pairs(n, [x for i in range(n) for j in range(i + 1, n) for x in (i, j)])
    S = [3, 5, 7]
    res = orc.cluster_bfs(g, S, 1)
    for v in range(n):
        if v in S:
            assert res.dist[v] == 0 and res.sub[0, v] == 1 << S.index(v) and res.sub[1, v] == 7 & ~(1 << S.index(v))
        else:
            assert res.dist[v] == 1 and res.sub[0, v] == 7 and res.sub[1, v] == 0
    assert int(res.stats[0]) == 2


def test_intact_grid_manhattan():
    side = 24
    pairs = []
    for y in range(side):
        for x in range(side):
            v = y * side + x
            if x + 1 < side: pairs += [v, v + 1]
            if y + 1 < side: pairs += [v, v + side]
    g = graph_from_pairs(side * side, pairs)
    cx, cy = 9, 13
    S = [(cy + dy) * side + cx + dx for dy in range(-2, 3) for dx in range(-2, 3) if abs(dx) + abs(dy) <= 2]
    S.remove(cy * side + cx); S = [cy * side + cx] + S  # radius-2 ball, 13 sources, diameter 4
    assert len(S) == 13
    res = orc.cluster_bfs(g, S, 4)
    for v in range(side * side):
        x, y = v % side, v // side
        ds = [abs(x - s % side) + abs(y - s // side) for s in S]
        mn = min(ds)
        assert res.dist[v] == mn
        for i in range(5):
            assert int(res.sub[i, v]) == sum(1 << j for j, t in enumerate(ds) if t - mn == i)


# ------------------------------------------------------------------ readings
def test_R1_seeding_gives_source_subset0():
    """R1: the literal init S_seen[s]={s} would leave S_s[0] empty;
    the oracle seeds S_next so that Delta_s = 0 and S_s[0] = {s}."""
    g = graph_from_pairs(4, [0, 1, 1, 2, 2, 3])
    res = orc.cluster_bfs(g, [1, 2], 1)
    assert res.dist[1] == 0 and res.sub[0, 1] == 0b01 and res.sub[1, 1] == 0b10
    assert res.dist[2] == 0 and res.sub[0, 2] == 0b10 and res.sub[1, 2] == 0b01


def test_R9_hand_worked_diameter_exceeds_d():
    """Path 0-1-2, S=[0,2] (diameter 2), d=1: worked by hand through Alg. 1.
    Round 0 folds the sources, pushes both into vertex 1; round 1 folds vertex 1
    (Delta=1, S[0]={0,2}); its pushes back to 0 and 2 are blocked by the cap
    i - Delta < d (1 - 0 < 1 is false).  So vertex 0 never learns source 2."""
    g = graph_from_pairs(3, [0, 1, 1, 2])
    res = orc.cluster_bfs(g, [0, 2], 1)
    assert res.dist.tolist() == [0, 1, 0]
    assert res.sub[:, 0].tolist() == [0b01, 0] and res.sub[:, 1].tolist() == [0b11, 0]
    assert res.sub[:, 2].tolist() == [0b10, 0]
    assert int(res.stats[0]) == 2


def test_fig2_values():
    lines = [l.split() for l in open(os.path.join(GOLD, "fig2.txt")) if l.strip() and not l.startswith("#")]
    kv = {l[0]: l[1:] for l in lines}
    pairs = [int(x) for e in kv["edges"] for x in e.split("-")]
    g = graph_from_pairs(6, pairs)
    S = [int(x) for x in kv["sources"]]
    d = int(kv["d"][0])
    res = orc.cluster_bfs(g, S, d)
    v = int(kv["vertex"][0])
    assert res.dist[v] == int(kv["vertex"][2])
    assert res.sub[1, v] == int(kv["vertex"][4], 16)  # {A,C}
    # decode: delta(A,F) = delta(C,F) = Delta_F + 1 = 2
    for j in (0, 2):
        assert res.sub[1, v] >> j & 1 and res.dist[v] + 1 == 2


def test_invalid_clusters_rejected():
    g = graph_from_pairs(3, [0, 1, 1, 2])
    for S in ([], [0, 0], [5]):
        with pytest.raises(ValueError):
            orc.cluster_bfs(g, S, 2)
    g70 = graph_from_pairs(70, [x for i in range(69) for x in (i, i + 1)])
    with pytest.raises(ValueError):
        orc.cluster_bfs(g70, list(range(65)), 2)  # k > 64 (single-word bit-subsets)


def test_isolated_source():
    g = orc.csr_from_edges(4, np.array([1], np.uint32), np.array([2], np.uint32))
    res = orc.cluster_bfs(g, [0], 2)
    assert res.dist.tolist() == [0, orc.INF16, orc.INF16, orc.INF16]
    assert res.sub[0].tolist() == [1, 0, 0, 0] and int(res.stats[0]) == 1


def test_many_equals_single():
    el = ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=5)
    g = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(g, 6, 64, 2)
    out = orc.cluster_bfs_many(g, src, sz, 2, threads=3)
    for c in range(len(sz)):
        r = orc.cluster_bfs(g, src[c, :sz[c]], 2)
        assert np.array_equal(out["dist"][c], r.dist) and np.array_equal(out["sub"][c], r.sub)
        assert np.array_equal(out["stats"][c], r.stats)
        assert int(out["hash"][c]) == orc.hash_cluster(r.dist, r.sub)


# ------------------------------------------------------------------ selection
def test_select_star_k1_70():
    """SPEC select_clusters example: K_{1,70}, k=64, d=2 -> centre + its 63 lowest-id leaves."""
    centre = 35
    leaves = [v for v in range(71) if v != centre]
    g = graph_from_pairs(71, [x for v in leaves for x in (centre, v)])
    src, sz = orc.select_clusters(g, 1, 64, 2)
    assert sz.tolist() == [64]
    assert src[0, 0] == centre and src[0, 1:].tolist() == leaves[:63]


@pytest.mark.parametrize("seed", range(10))
def test_select_greedy_properties(seed):
    """Brute-force greedy restated over scipy hop distances: each root is the
    best unmarked non-isolated vertex by (deg desc, id asc) (or the random
    draw), members are the best k-1 unmarked vertices of the floor(d/2)-ball,
    clusters are disjoint and have diameter <= d."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(30, 120))
    g = random_graph(rng, n, "pa" if seed % 2 else "er")
    d = [2, 4, 6, 3, 2][seed % 5]
    k = [5, 64, 9][seed % 3]
    policy = seed % 2
    src, sz = orc.select_clusters(g, 6, k, d, policy, seed=seed)
    deg = g.degrees().astype(np.int64)
    marked = np.zeros(n, bool)
    key = lambda v: (-deg[v], v)
    t_draw = 0
    for c in range(len(sz)):
        S = src[c, :sz[c]].tolist()
        root = S[0]
        if policy == 0:
            best = min((v for v in range(n) if not marked[v] and deg[v] > 0), key=key)
            assert root == best
        else:
            while True:
                v = ci.bounded(ci.rand(seed, 1, t_draw), n); t_draw += 1
                if not marked[v] and deg[v] > 0:
                    break
            assert root == v
        D = scipy_dist(g, [root])[0]
        cand = sorted((v for v in range(n) if 1 <= D[v] <= d // 2 and not marked[v]), key=key)
        assert S[1:] == cand[:k - 1]
        marked[S] = True
        DS = scipy_dist(g, S)
        assert DS[:, S].max() <= d and (DS[:, S] >= 0).all()
        assert all(s != orc.PAD for s in S) and np.all(src[c, sz[c]:] == orc.PAD)
    if len(sz) < 6:  # stopped early: nothing unmarked and non-isolated left
        assert not any(not marked[v] and deg[v] > 0 for v in range(n))


# ------------------------------------------------------------------ budget
def test_budget_paper_numbers():
    rows = [l.split() for l in open(os.path.join(GOLD, "budget.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 4
    for t, w, d, rb, r, *_ in rows:
        assert orc.record_bytes(int(w), int(d)) == int(rb)
        assert orc.budget_to_clusters(int(t), int(w), int(d)) == int(r)
    # w=64 selects 60*64 = 3840 landmarks, w=8 selects 341*8 = 2728
    assert orc.budget_to_clusters(1024, 64, 2) * 64 == 3840 and orc.budget_to_clusters(1024, 8, 2) * 8 == 2728
    assert orc.budget_to_clusters(10, 64, 2) == -1


# ------------------------------------------------------------------ queries
@pytest.mark.parametrize("seed", range(8))
def test_query_pins(seed):
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(40, 150))
    g = random_graph(rng, n, "er" if seed % 2 else "pa")
    d = [2, 4, 2, 6][seed % 4]
    src, sz = orc.select_clusters(g, 4, 16, d, seed % 2, seed=seed)
    C = len(sz)
    many = orc.cluster_bfs_many(g, src, sz, d, threads=2)
    q = 300
    s = rng.integers(0, n, q).astype(np.uint32); t = rng.integers(0, n, q).astype(np.uint32)
    ans = orc.query(many["dist"], many["sub"], s, t)
    # per-cluster brute force min_j delta(u,s_j) + delta(s_j,v) from scipy distances
    Dall = [scipy_dist(g, src[c, :sz[c]]) for c in range(C)]
    truth = scipy_dist(g, np.arange(n))
    for j in range(q):
        u, v = int(s[j]), int(t[j])
        best = orc.INT32_MAX
        for c in range(C):
            D = Dall[c]
            vals = [D[x, u] + D[x, v] for x in range(D.shape[0]) if D[x, u] >= 0 and D[x, v] >= 0]
            if vals:
                best = min(best, int(min(vals)))
        assert ans[j] == best
        if best != orc.INT32_MAX:
            assert best >= truth[u, v] >= 0  # one-sided error
    # exact when a landmark lies on a shortest path: query(u, s_j) = delta(u, s_j)
    for c in range(C):
        for x in src[c, :sz[c]]:
            us = rng.integers(0, n, 20).astype(np.uint32)
            a = orc.query(many["dist"], many["sub"], us, np.full(20, x, np.uint32))
            for u, val in zip(us, a):
                if truth[u, x] >= 0:
                    assert val == truth[u, x]
            assert orc.query(many["dist"], many["sub"], np.array([x], np.uint32), np.array([x], np.uint32))[0] == 0
    # adding clusters never increases an answer (monotone)
    a1 = orc.query(many["dist"][:1], many["sub"][:1], s, t)
    assert np.all(ans <= a1)
    # stream mode == resident mode
    assert np.array_equal(orc.query_stream(g, src, sz, d, s, t, threads=2), ans)


def test_query_empty_index_unreachable():
    g = graph_from_pairs(4, [0, 1, 2, 3])
    src = np.full((1, 64), orc.PAD, np.uint32); src[0, 0] = 0
    many = orc.cluster_bfs_many(g, src, np.array([1], np.uint8), 2)
    a = orc.query(many["dist"], many["sub"], np.array([0, 2], np.uint32), np.array([1, 3], np.uint32))
    assert a.tolist() == [1, orc.INT32_MAX]
    a = orc.query(many["dist"][:0], many["sub"][:0], np.array([0], np.uint32), np.array([1], np.uint32))
    assert a.tolist() == [orc.INT32_MAX]


# ------------------------------------------------------------------ NEXT-2 bidirectional refinement
def test_bidir_refine_pins():
    """Appendix B, reading R27: tau >= n gives the exact distance
    (scipy BFS); tau = 0 gives nothing; tau = 1 only meets at u = v; the
    answer never undercuts delta and never grows with tau; hand-worked path."""
    rng = np.random.default_rng(5)
    g = random_graph(rng, 300, "er")
    D = scipy_dist(g, np.arange(g.n))
    s = rng.integers(0, g.n, 400).astype(np.uint32)
    t = rng.integers(0, g.n, 400).astype(np.uint32)
    exact = orc.bidir_refine(g, s, t, g.n)
    ref = D[s.astype(int), t.astype(int)].astype(np.float64)
    ref[ref < 0] = np.inf
    reach = np.isfinite(ref)
    assert reach.any() and np.array_equal(exact[reach], ref[reach].astype(np.int32))
    assert np.all(exact[~reach] == orc.INT32_MAX)
    assert np.all(orc.bidir_refine(g, s, t, 0) == orc.INT32_MAX)
    one = orc.bidir_refine(g, s, t, 1)
    assert np.all(one[s == t] == 0) and np.all(one[s != t] == orc.INT32_MAX)
    prev = None
    for tau in (2, 4, 16, 64, 300):
        cur = orc.bidir_refine(g, s, t, tau)
        fin = cur < orc.INT32_MAX
        assert np.all(cur[fin] >= ref[fin])  # one-sided
        if prev is not None:
            assert np.all(cur <= prev)  # more search never hurts
        prev = cur
    # path 0-1-2-...-9: BFS from 0 visits 0,1,2,.. ; from 9 visits 9,8,...
    p = orc.csr_from_edges(10, np.arange(9, dtype=np.uint32), np.arange(1, 10, dtype=np.uint32))
    a = np.array([0], np.uint32); b = np.array([9], np.uint32)
    assert orc.bidir_refine(p, a, b, 5)[0] == orc.INT32_MAX  # {0..4} and {5..9} are disjoint
    assert orc.bidir_refine(p, a, b, 6)[0] == 9               # they meet at 4 and 5


# ------------------------------------------------------------------ clusters of k > 64 (NEXT-1)
def _wide_from_definition(D: np.ndarray, d: int):
    """The definition P:630-636 from a scipy [k][n] matrix, one word per 64 sources."""
    k, n = D.shape
    W = (k + 63) // 64
    dist = np.full(n, orc.INF16, np.uint16)
    sub = np.zeros((d + 1, n, W), np.uint64)
    for v in range(n):
        col = D[:, v]
        if not (col >= 0).any():
            continue
        mn = int(col[col >= 0].min())
        dist[v] = mn
        for j in np.flatnonzero(col >= 0):
            sub[int(col[j]) - mn, v, j // 64] |= np.uint64(1 << (int(j) % 64))
    return dist, sub


@pytest.mark.parametrize("seed", range(4))
def test_wide_definition_matches_scipy_and_alg1(seed):
    """brute_cluster_wide == the definition over scipy distances for k up to
    300, and == Alg. 1 (the C oracle, pinned above) word for word when
    k <= 64."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(400, 700))
    g = random_graph(rng, n, "er" if seed % 2 else "pa")
    root = int(np.argmax(g.degrees()))
    for h in range(2, 8):  # the smallest ball radius that holds more than 64 sources
        S = ball_cluster(g, root, h, 300, rng)
        if len(S) > 64:
            break
    assert len(S) > 64
    d = 2 * h
    dist, sub, over = orc.brute_cluster_wide(g, S, d)
    assert not over
    rd, rs = _wide_from_definition(scipy_dist(g, S), d)
    assert np.array_equal(dist, rd) and np.array_equal(sub, rs)
    small = S[:40]
    dist, sub, _ = orc.brute_cluster_wide(g, small, d)
    res = orc.cluster_bfs(g, small, d)
    assert sub.shape[2] == 1
    assert np.array_equal(dist, res.dist) and np.array_equal(sub[:, :, 0], res.sub)


def test_wide_star_closed_form():
    """K_{1,L} with S = centre + 199 leaves (4 words): centre Delta 0,
    S[0] = {c}, S[1] = the member leaves; a member leaf: S[0] = itself,
    S[1] = {c}, S[2] = the other members; any other leaf: Delta 1,
    S[0] = {c}, S[1] = the members (SURVEY §8(c) closed forms at k > 64)."""
    L, k = 260, 200
    g = graph_from_pairs(L + 1, [x for i in range(1, L + 1) for x in (0, i)])
    S = list(range(k))
    dist, sub, over = orc.brute_cluster_wide(g, S, 2)
    assert not over and sub.shape == (3, L + 1, 4)

    def words(bits):
        w = [0, 0, 0, 0]
        for j in bits:
            w[j // 64] |= 1 << (j % 64)
        return [np.uint64(x) for x in w]
    members = range(1, k)
    assert dist[0] == 0 and list(sub[0, 0]) == words([0]) and list(sub[1, 0]) == words(members)
    for j in (1, 63, 64, 130, 199):
        assert dist[j] == 0 and list(sub[0, j]) == words([j]) and list(sub[1, j]) == words([0])
        assert list(sub[2, j]) == words([x for x in members if x != j])
    for v in (200, 260):
        assert dist[v] == 1 and list(sub[0, v]) == words([0]) and list(sub[1, v]) == words(members)
        assert not sub[2, v].any()


def test_wide_query_brute_pins():
    """query_brute == the C R15 scan (orc.query over Alg. 1 labels, pinned in
    test_query_pins) on k <= 64 clusters of diameter <= d, and on a path it
    is min_j |u - s_j| + |s_j - v| (closed form) for a cluster of 150."""
    rng = np.random.default_rng(77)
    g = random_graph(rng, 300, "pa")
    d = 4
    src, sz = orc.select_clusters(g, 5, 30, d)
    many = orc.cluster_bfs_many(g, src, sz, d, threads=2)
    s = rng.integers(0, g.n, 400).astype(np.uint32); t = rng.integers(0, g.n, 400).astype(np.uint32)
    clusters = [src[c, :sz[c]] for c in range(len(sz))]
    assert np.array_equal(orc.query_brute(g, clusters, s, t), orc.query(many["dist"], many["sub"], s, t))
    n = 500
    g = graph_from_pairs(n, [x for i in range(n - 1) for x in (i, i + 1)])
    S = np.arange(200, 350)
    s = rng.integers(0, n, 300); t = rng.integers(0, n, 300)
    got = orc.query_brute(g, [S], s, t)
    expect = [min(abs(int(u) - int(x)) + abs(int(x) - int(v)) for x in S) for u, v in zip(s, t)]
    assert np.array_equal(got, np.array(expect, np.int32))


def test_select_wide_pins():
    """Selection with k > 64 (R12, general k): equals the k <= 64
    rule (pinned above) when k <= 64; on K_{1,300} with k = 200 the first
    cluster is the centre + the 199 lowest-id leaves (all leaves tie on
    degree), the next roots are the remaining leaves in id order; clusters
    are disjoint and within floor(d/2) hops of their root."""
    rng = np.random.default_rng(31)
    g = random_graph(rng, 400, "pa")
    a_src, a_sz = orc.select_clusters(g, 9, 40, 2)
    b_src, b_sz = orc.select_clusters_wide(g, 9, 40, 2, 2)
    assert np.array_equal(a_sz, b_sz) and np.array_equal(a_src, b_src[:, :64]) and (b_src[:, 64:] == orc.PAD).all()
    L = 300
    star = graph_from_pairs(L + 1, [x for i in range(1, L + 1) for x in (0, i)])
    src, sz = orc.select_clusters_wide(star, 3, 200, 2, 4)
    assert list(sz) == [200, 1, 1]
    assert list(src[0, :200]) == list(range(200)) and (src[0, 200:] == orc.PAD).all()
    assert src[1, 0] == 200 and src[2, 0] == 201
    src, sz = orc.select_clusters_wide(g, 6, 150, 4, 4)
    seen = set()
    for c in range(len(sz)):
        S = src[c, :sz[c]].tolist()
        assert not (set(S) & seen)
        seen |= set(S)
        D = scipy_dist(g, [S[0]])[0]
        assert all(0 <= D[x] <= 2 for x in S)
        degs = g.degrees()[S[1:]].astype(np.int64)
        assert all((degs[i] > degs[i + 1]) or (degs[i] == degs[i + 1] and S[1 + i] < S[2 + i])
                   for i in range(len(degs) - 1))


# ------------------------------------------------------------------ exact 2-hop oracle (PLL, NEXT-4)
def _pll_order(g):
    deg = g.degrees().astype(np.int64)
    return np.lexsort((np.arange(g.n), -deg))  # degree desc, id asc


def _batches(nroots, first, bmax):
    out, r0, b = [], 0, min(first, bmax)
    while r0 < nroots:
        out.append((r0, min(r0 + b, nroots)))
        r0 += b
        b = min(bmax, b * 3 // 2)
    return out


@pytest.mark.parametrize("seed", range(6))
def test_pll_exact_and_label_characterisation(seed):
    """PLL (R29): every pair's answer is the BFS distance, and the label set
    is exactly {(h, delta(h, v)) : h a phase-2 root reaching v, no vertex
    visible to h's batch (cluster sources and roots of earlier batches) on a
    shortest h-v path} — computed by brute force from all-pairs distances.
    With no clusters and batches of one this is sequential PLL's canonical
    labeling."""
    rng = np.random.default_rng(1300 + seed)
    n = int(rng.integers(60, 130))
    g = random_graph(rng, n, "er" if seed % 2 else "pa")
    C = [0, 3, 2, 0, 5, 1][seed]
    first, bmax = [(1, 1), (4, 16), (3, 7), (5, 30), (2, 9), (200, 1000)][seed]
    src, sz = orc.select_clusters(g, C, 16, 2) if C else (np.zeros((0, 64), np.uint32), np.zeros(0, np.uint8))
    idx = orc.pll_build(g, src, sz, 2, first=first, bmax=bmax, cap=n)
    D = scipy_dist(g, np.arange(n))  # -1 = unreachable
    s = np.repeat(np.arange(n), n).astype(np.uint32); t = np.tile(np.arange(n), n).astype(np.uint32)
    truth = np.where(D < 0, orc.INT32_MAX, D).reshape(-1)
    assert np.array_equal(orc.pll_query(idx, s, t), truth)
    order = _pll_order(g)
    pos = np.empty(n, np.int64); pos[order] = np.arange(n)
    covered = set(src[c, j] for c in range(len(sz)) for j in range(sz[c]))
    roots = [int(v) for v in order if v not in covered]
    visible = np.zeros(n, bool); visible[list(covered)] = True
    expect = {v: [] for v in range(n)}
    for r0, r1 in _batches(len(roots), first, bmax):
        vis_idx = np.flatnonzero(visible)
        for h in roots[r0:r1]:
            for v in range(n):
                if D[h, v] < 0:
                    continue
                on_path = [(D[h, w] >= 0 and D[w, v] >= 0 and D[h, w] + D[w, v] == D[h, v]) for w in vis_idx]
                if not any(on_path):
                    expect[v].append((int(pos[h]) << 8) | int(D[h, v]))
        visible[roots[r0:r1]] = True
    for v in range(n):
        assert list(idx["entries"][v, :idx["counts"][v]]) == sorted(expect[v]), v


def test_pll_cap_overflow_and_isolated():
    g = graph_from_pairs(6, [0, 1, 1, 2])  # vertices 3..5 isolated
    idx = orc.pll_build(g, np.zeros((0, 64), np.uint32), np.zeros(0, np.uint8), 2, first=1, bmax=1, cap=4)
    for v in (3, 4, 5):  # an isolated vertex's only label is itself
        assert idx["counts"][v] == 1 and idx["entries"][v, 0] & 255 == 0
    a = orc.pll_query(idx, np.array([0, 3, 3], np.uint32), np.array([2, 3, 4], np.uint32))
    assert list(a) == [2, 0, orc.INT32_MAX]
    path = graph_from_pairs(40, [x for i in range(39) for x in (i, i + 1)])
    with pytest.raises(OverflowError):
        orc.pll_build(path, np.zeros((0, 64), np.uint32), np.zeros(0, np.uint8), 2, first=40, bmax=40, cap=3)
