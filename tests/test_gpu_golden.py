"""Whole-config parity at BASELINE.json's full sizes against oracle-generated
golden files (tests/golden/CONFIG.golden.txt, written by
tests/make_goldens.py, which calls only oracle/): for every cluster in the
golden file its round statistics, its per-round {|F_i|, E_i} and the digest
of its full output vector (Delta + d+1 subsets; digest definition
in include/cbfs.h cbfs_digest_store), and the SHA-256 of the whole
selection.  The GPU runs every cluster of the config in the launch path the
bench times (config 2: cbfs_select_and_run_shard with the full [n][C] store;
config 3: cbfs_run_digest).  Config 5: the streaming label build + the
10M queries over the selection prefix its golden covers — round statistics
of every covered cluster and every answer against the oracle's (SHA-256 of
all 10M answers + 100,000 stored answers)."""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402
from gpu_util import np_u32, np_u64  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(autouse=True)
def _release_workspace():
    yield
    cb.cbfs_release_workspace(0)  # full-size configs leave multi-GB slot caches behind


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.golden.txt")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/make_goldens.py {name})")
    lines = open(path).read().splitlines()
    header = json.loads(lines[0][2:])
    rows = {}
    for line in lines[1:]:
        if line.startswith("#") or not line.strip():
            continue
        f = [int(x) for x in line.split()]
        c, R = f[0], f[1]
        rounds = np.array(f[6:], np.uint64).reshape(-1, 2) if len(f) > 6 else None
        assert rounds is None or len(rounds) == R
        rows[c] = dict(stats=np.array(f[1:5], np.uint64), digest=np.uint64(f[5]), rounds=rounds)
    return header, rows


def selection_sha(src, sz):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(np_u32(src)).tobytes())
    h.update(np.ascontiguousarray(sz.cpu().numpy().astype(np.uint8)).tobytes())
    return h.hexdigest()


def build(name):
    cfg = ci.CONFIGS[name]
    el = ci.make_graph(name)
    relabel = cb.Graph.relabel_flags(cfg.get("relabel", "none"))
    src_d = torch.from_numpy(el.src.view(np.int32)).to(DEV)
    dst_d = torch.from_numpy(el.dst.view(np.int32)).to(DEV)
    g = cb.Graph(cb.cbfs_graph_create(el.n, src_d, dst_d, relabel, 0), 0)
    del src_d, dst_d
    return cfg, el, g


def select(g, cfg, header):
    policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
    src, sz = g.select_clusters(cfg["clusters"], cfg["k"], cfg["d"], policy, cfg["root_seed"])
    assert len(sz) == header["clusters"]
    assert selection_sha(src, sz) == header["selection_sha256"], "GPU selection != oracle selection"
    return src, sz


def check_rounds(g, src, sz, d, rows, idx):
    """cbfs_run_rounds over the clusters `idx` against the golden per-round records."""
    idx = [c for c in idx if rows[c]["rounds"] is not None]
    if not idx:
        return
    R = max(int(rows[c]["stats"][0]) for c in idx)
    t = torch.tensor(idx, device=DEV)
    rounds = torch.zeros((len(idx), R, 2), dtype=torch.int64, device=DEV)
    cb.cbfs_run_rounds(g.h, src[t].contiguous(), sz[t].contiguous(), len(idx), d, rounds, R)
    r = np_u64(rounds)
    for j, c in enumerate(idx):
        Rc = int(rows[c]["stats"][0])
        assert np.array_equal(r[j, :Rc], rows[c]["rounds"]), c
        assert not r[j, Rc:].any(), c


def check_digest_config(name, timeout_note=""):
    header, rows = load_golden(name)
    cfg, el, g = build(name)
    assert (g.n, g.m) == (header["n"], header["arcs"])
    src, sz = select(g, cfg, header)
    C, d = len(sz), cfg["d"]
    dist_bytes = 1 if cfg["kind"] in ("rmat", "er") else 2
    dig = torch.zeros(C, dtype=torch.int64, device=DEV)
    stats = torch.zeros((C, 4), dtype=torch.int64, device=DEV)
    cb.cbfs_run_digest(g.h, src, sz, C, d, dist_bytes, d + 1, dig, stats)
    dg, st = np_u64(dig), np_u64(stats)
    for c, row in rows.items():
        assert np.array_equal(st[c], row["stats"]), c
        assert dg[c] == row["digest"], c
    check_rounds(g, src, sz, d, rows, sorted(rows)[:256])
    g.close()
    return len(rows), C


@pytest.mark.timeout(600)
def test_c1_whole_config_golden():
    got, C = check_digest_config("c1_er")
    assert got == C


@pytest.mark.timeout(900)
def test_c2_whole_config_golden_bench_path():
    """Config 2 in bench.py's launch path: cbfs_select_and_run_shard writing the
    full [n][1024] store (u8 Delta + 3 planes), then every column's digest and
    every cluster's stats against the golden (all 1,024 clusters)."""
    header, rows = load_golden("c2_rmat20")
    cfg, el, g = build("c2_rmat20")
    C, d = cfg["clusters"], cfg["d"]
    src = torch.empty((C, 64), dtype=torch.int32, device=DEV)
    sz = torch.empty((C,), dtype=torch.uint8, device=DEV)
    dist = torch.empty((g.n, C), dtype=torch.uint8, device=DEV)
    masks = torch.empty((d + 1, g.n, C), dtype=torch.int64, device=DEV)
    stats = torch.zeros((C, 4), dtype=torch.int64, device=DEV)
    got = cb.cbfs_select_and_run_shard(g.h, C, cfg["k"], d, cb.CBFS_ROOT_DEGREE, cfg["root_seed"], 1, 0, src, sz, 1,
                                       dist, masks, d + 1, stats)
    assert got == header["clusters"] == C
    assert selection_sha(src, sz) == header["selection_sha256"]
    dig = torch.zeros(C, dtype=torch.int64, device=DEV)
    cb.cbfs_digest_store(g.n, C, d + 1, dist, 1, masks, dig)
    dg, st = np_u64(dig), np_u64(stats)
    assert len(rows) == C
    for c, row in rows.items():
        assert np.array_equal(st[c], row["stats"]), c
        assert dg[c] == row["digest"], c
    del dist, masks
    check_rounds(g, src, sz, d, rows, list(range(0, C, 4)))
    g.close()


@pytest.mark.timeout(900)
def test_c3_whole_config_golden():
    """Config 3 (RMAT-24, 4,096 clusters): all clusters through cbfs_run_digest
    (every batch's full vectors written and consumed in HBM); the golden holds
    the oracle's seeded sample (the oracle needs ~52 s per cluster per core)."""
    got, C = check_digest_config("c3_rmat24")
    assert got >= 256 and C == 4096


@pytest.mark.timeout(900)
def test_c4_whole_config_golden():
    got, C = check_digest_config("c4_grid")
    assert got == C == 512


@pytest.mark.timeout(900)
def test_c5_whole_config_golden_digests():
    """Config 5: every cluster of the selection through cbfs_run_digest (the
    sparse engine with ordered frontiers, full vectors staged and consumed) —
    stats and full-vector digest of every cluster the golden holds (the query
    prefix plus the clusters generated with --no-queries)."""
    got, C = check_digest_config("c5_knn")
    assert got >= 1024 and C == 8192


@pytest.mark.timeout(1800)
def test_c5_full_size_golden_queries():
    """Config 5 at full size (10M-point k-NN graph, d = 6): the whole
    selection (SHA-256 of all 8,192 clusters), then the streaming label build
    + all 10M queries (bench.py's query path, cbfs_query_stream) over the
    clusters the golden covers (a selection prefix: the oracle needs ~38 s per
    config-5 cluster per core) — every answer (SHA-256 of the 10M-vector and
    100,000 stored answers) and every covered cluster's round statistics —
    and the full-vector digests of the first 256 clusters."""
    header, rows = load_golden("c5_knn")
    ans_path = os.path.join(GOLDEN, "c5_knn.answers.npz")
    if not os.path.exists(ans_path):
        pytest.skip("config 5 golden incomplete")
    ans = np.load(ans_path)
    Cq = int(ans["clusters"])
    assert all(c in rows for c in range(Cq))
    cfg, el, g = build("c5_knn")
    src, sz = select(g, cfg, header)
    d = cfg["d"]
    s, t = ci.query_pairs(g.n, cfg["queries"], cfg["query_seed"])
    best = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device=DEV)
    stats = torch.zeros((Cq, 4), dtype=torch.int64, device=DEV)
    cb.cbfs_query_stream(g.h, src[:Cq].contiguous(), sz[:Cq].contiguous(), Cq, d,
                         torch.from_numpy(s.view(np.int32)).to(DEV), torch.from_numpy(t.view(np.int32)).to(DEV), best,
                         stats)
    b = best.cpu().numpy()
    assert np.array_equal(b[ans["index"]], ans["answer"])
    assert hashlib.sha256(b.tobytes()).hexdigest() == str(ans["sha256"])
    st = np_u64(stats)
    for c in range(Cq):
        assert np.array_equal(st[c], rows[c]["stats"]), c
    first = list(range(256))
    t_idx = torch.tensor(first, device=DEV)
    dig = torch.zeros(len(first), dtype=torch.int64, device=DEV)
    cb.cbfs_run_digest(g.h, src[t_idx].contiguous(), sz[t_idx].contiguous(), len(first), d, 2, d + 1, dig)
    dg = np_u64(dig)
    for j, c in enumerate(first):
        assert dg[j] == rows[c]["digest"], c
    g.close()
