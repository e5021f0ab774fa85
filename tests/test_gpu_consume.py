"""GPU parity of the output consumers and the per-round statistics, through
the C-ABI, against the oracle (bit-exact): cbfs_run_digest (full outputs
staged per batch and reduced to one digest per cluster), cbfs_digest_store
(the same digest over cbfs_run's store) and cbfs_run_rounds (|F_i|, E_i of
every round), on random graphs in every engine / direction, with
ragged batches and d < diameter cases; plus the per-round invariants of
SURVEY §8(c) checked on the GPU's own records (at most d+1 frontier
appearances per vertex; rounds = 1 + max source distance)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402
from gpu_util import gpu_graph, np_u64, to_dev_u32, to_dev_u8  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
MODES = [(cb.CBFS_ENGINE_BATCHED, cb.CBFS_DIR_AUTO), (cb.CBFS_ENGINE_BATCHED, cb.CBFS_DIR_PUSH),
         (cb.CBFS_ENGINE_BATCHED, cb.CBFS_DIR_PULL), (cb.CBFS_ENGINE_SPARSE, cb.CBFS_DIR_AUTO)]


@pytest.fixture(autouse=True)
def _reset_engine():
    yield
    cb.cbfs_set_engine(cb.CBFS_ENGINE_AUTO)


def graphs():
    yield "er", ci.erdos_renyi(3000, 9000, seed=11), 2
    yield "rmat", ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=12), 2
    yield "grid", ci.grid(60, 0.05, 0.01, 13), 4
    yield "knn", ci.knn3d(4000, 6, seed=14), 3


@pytest.mark.parametrize("case", range(4))
def test_run_digest_and_rounds_match_oracle(case):
    name, el, d = list(graphs())[case]
    ref = orc.csr_from_edgelist(el)
    C = 70  # a full batch of 64 and a ragged one
    src, sz = orc.select_clusters(ref, C, 64, d)
    C = len(sz)
    R = 96
    om = orc.cluster_bfs_many(ref, src, sz, d, want_outputs=False, want_digest=True, max_rounds=R)
    g = gpu_graph(el, relabel=(name == "rmat"))
    sd, zd = to_dev_u32(src), to_dev_u8(sz)
    for eng, direction in MODES:
        cb.cbfs_set_engine(eng)
        dig = torch.zeros(C, dtype=torch.int64, device=DEV)
        stats = torch.zeros((C, 4), dtype=torch.int64, device=DEV)
        cb.cbfs_run_digest(g.h, sd, zd, C, d, 2, d + 1, dig, stats, direction)
        assert np.array_equal(np_u64(dig), om["digest"]), (name, eng, direction)
        assert np.array_equal(np_u64(stats), om["stats"]), (name, eng, direction)
        rounds = torch.zeros((C, R, 2), dtype=torch.int64, device=DEV)
        cb.cbfs_run_rounds(g.h, sd, zd, C, d, rounds, R, None, direction)
        r = np_u64(rounds)
        assert np.array_equal(r[:, :, 0], om["round_F"].astype(np.uint64)), (name, eng, direction)
        assert np.array_equal(r[:, :, 1], om["round_E"]), (name, eng, direction)
    g.close()


@pytest.mark.parametrize("dist_bytes", [1, 2])
def test_digest_store_equals_oracle_and_run_digest(dist_bytes):
    """cbfs_digest_store over cbfs_run's [n][C] store == the oracle's digest of
    each cluster == cbfs_run_digest (u8 and u16 Delta: the digest uses the
    16-bit value)."""
    el = ci.rmat(11, 8, 0.57, 0.19, 0.19, seed=21)
    ref = orc.csr_from_edgelist(el)
    d = 2
    src, sz = orc.select_clusters(ref, 131, 64, d)
    C = len(sz)
    om = orc.cluster_bfs_many(ref, src, sz, d)
    expect = np.array([orc.digest_cluster(om["dist"][c], om["sub"][c]) for c in range(C)], np.uint64)
    g = gpu_graph(el, relabel=True)
    sd, zd = to_dev_u32(src), to_dev_u8(sz)
    dist = torch.empty((g.n, C), dtype=torch.uint8 if dist_bytes == 1 else torch.int16, device=DEV)
    masks = torch.empty((d + 1, g.n, C), dtype=torch.int64, device=DEV)
    cb.cbfs_run(g.h, sd, zd, C, d, dist_bytes, dist, masks, d + 1)
    dig = torch.zeros(C, dtype=torch.int64, device=DEV)
    cb.cbfs_digest_store(g.n, C, d + 1, dist, dist_bytes, masks, dig)
    assert np.array_equal(np_u64(dig), expect)
    dig2 = torch.zeros(C, dtype=torch.int64, device=DEV)
    cb.cbfs_run_digest(g.h, sd, zd, C, d, dist_bytes, d + 1, dig2)
    assert np.array_equal(np_u64(dig2), expect)
    # label-record planes (d): the digest covers the stored planes only
    masks2 = torch.empty((d, g.n, C), dtype=torch.int64, device=DEV)
    cb.cbfs_run(g.h, sd, zd, C, d, dist_bytes, dist, masks2, d)
    cb.cbfs_digest_store(g.n, C, d, dist, dist_bytes, masks2, dig)
    expect_d = np.array([orc.digest_cluster(om["dist"][c], om["sub"][c][:d]) for c in range(C)], np.uint64)
    assert np.array_equal(np_u64(dig), expect_d)
    g.close()


def test_digest_detects_a_single_flip():
    """The digest of a store changes when any one entry changes (Delta or a
    subset word), and columns are independent."""
    el = ci.erdos_renyi(500, 1500, seed=5)
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 3, 64, 2)
    g = gpu_graph(el)
    dist, masks, _ = g.run(to_dev_u32(src), to_dev_u8(sz), 2)
    C = len(sz)
    base = torch.zeros(C, dtype=torch.int64, device=DEV)
    cb.cbfs_digest_store(g.n, C, 3, dist, 2, masks, base)
    rng = np.random.default_rng(0)
    for _ in range(20):
        v, c, p = int(rng.integers(g.n)), int(rng.integers(C)), int(rng.integers(4))
        m2, d2 = masks.clone(), dist.clone()
        if p == 3:
            d2[v, c] ^= 1
        else:
            m2[p, v, c] ^= 1 << int(rng.integers(63))
        out = torch.zeros(C, dtype=torch.int64, device=DEV)
        cb.cbfs_digest_store(g.n, C, 3, d2, 2, m2, out)
        diff = np.flatnonzero(np_u64(out) != np_u64(base))
        assert diff.tolist() == [c]
    g.close()


@pytest.mark.parametrize("eng", [cb.CBFS_ENGINE_BATCHED, cb.CBFS_ENGINE_SPARSE])
def test_round_invariants_on_gpu_records(eng):
    """SURVEY §8(c) invariants on the GPU's per-round records of clusters with
    diameter <= d: sum of |F_i| <= (d+1) * reached vertices (R6),
    rounds = 1 + max source distance (from plain BFS), and each |F_i|
    = #{v : some source at distance exactly i} (closed form)."""
    cb.cbfs_set_engine(eng)
    el = ci.erdos_renyi(2000, 5000, seed=31)
    ref = orc.csr_from_edgelist(el)
    d = 2
    src, sz = orc.select_clusters(ref, 20, 64, d)
    C = len(sz)
    g = gpu_graph(el)
    R = 64
    rounds = torch.zeros((C, R, 2), dtype=torch.int64, device=DEV)
    stats = torch.zeros((C, 4), dtype=torch.int64, device=DEV)
    cb.cbfs_run_rounds(g.h, to_dev_u32(src), to_dev_u8(sz), C, d, rounds, R, stats)
    r, st = np_u64(rounds), np_u64(stats)
    for c in range(C):
        S = src[c, :sz[c]]
        D = np.stack([orc.plain_bfs(ref, int(x)) for x in S]).astype(np.int64)
        D[D == orc.INF32] = -1
        reach = (D >= 0).any(axis=0)
        maxd = int(D.max())
        assert int(st[c, 0]) == 1 + maxd
        assert r[c, :, 0].sum() <= (d + 1) * reach.sum()
        for i in range(1 + maxd):
            assert int(r[c, i, 0]) == int(((D == i).any(axis=0)).sum()), (c, i)
        assert not r[c, 1 + maxd:].any()
    g.close()
