"""CPU oracle for the C-BFS hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  It shares no code with the
CUDA product (paper_2410_17226_b200/); its only common dependency is the
input generator module ``cbfs_inputs`` (random numbers, no method arithmetic).

Layers (each cites PAPER.md lines; readings R1..R26 are in DESIGN.md §2):
  * csr_from_edges  — graph normalisation (R17): symmetrise, drop
    self loops, sort + dedup, CSR.  numpy ``unique`` is the sort/dedup step.
  * plain_bfs / brute_cluster — single-source BFS and the
    definition of the cluster distance vector, in C;
    brute_cluster_wide / query_brute — the same definition and the landmark
    query for clusters of any size k (multi-word subsets, NEXT-1), numpy
    over plain_bfs.
  * cluster_bfs / cluster_bfs_many — Alg. 1, sequential C.
  * select_clusters — P:1061-1069 with R12, sequential C.
  * query / query_stream — P:1013-1021, P:1074-1086 with R14-R16, C.
  * budget_to_clusters — P:1445-1447.
Pins live in tests/test_oracle_*.py.  Parity of every function here is pinned
(no "parity unpinned" entries); see DESIGN.md §5.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

import cbfs_inputs

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

INF16 = 0xFFFF
INF32 = 0xFFFFFFFF
INT32_MAX = 2**31 - 1
PAD = 0xFFFFFFFF


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", src, "-o", _LIB_PATH])
    return _LIB_PATH


def _P(t):
    return ctypes.POINTER(t)


_RANDFN = ctypes.CFUNCTYPE(ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64)
_rand_cb = None


def lib():
    global _lib, _rand_cb
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u32p, u64p, u16p, u8p, i32p = _P(ctypes.c_uint32), _P(ctypes.c_uint64), _P(ctypes.c_uint16), \
            _P(ctypes.c_uint8), _P(ctypes.c_int32)
        L.or_plain_bfs.argtypes = [ctypes.c_uint32, u64p, u32p, ctypes.c_uint32, u32p]
        L.or_brute_cluster.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, ctypes.c_uint32, ctypes.c_uint32, u16p, u64p]
        L.or_cluster_bfs.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, ctypes.c_uint32, ctypes.c_uint32, u16p, u64p,
                                     u64p, u32p, u64p, ctypes.c_uint32]
        L.or_cluster_bfs_many.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, u8p, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_int, u16p, u64p, u64p, u64p]
        L.or_cluster_bfs_many_ex.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, u8p, ctypes.c_uint32,
                                             ctypes.c_uint32, ctypes.c_int, u16p, u64p, u64p, u64p, u64p, u32p, u64p,
                                             ctypes.c_uint32]
        L.or_digest_cluster.restype = ctypes.c_uint64
        L.or_digest_cluster.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u16p, u64p]
        L.or_query_stream_ex.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, u8p, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_uint64, u32p, u32p, ctypes.c_int, i32p, u64p, u64p]
        L.or_hash_cluster.restype = ctypes.c_uint64
        L.or_hash_cluster.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u16p, u64p]
        L.or_select_clusters.restype = ctypes.c_int64
        L.or_select_clusters.argtypes = [ctypes.c_uint32, u64p, u32p, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, _RANDFN, u32p, u8p]
        L.or_select_clusters_wide.restype = ctypes.c_int64
        L.or_select_clusters_wide.argtypes = [ctypes.c_uint32, u64p, u32p, ctypes.c_uint32, ctypes.c_uint32,
                                              ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, _RANDFN,
                                              ctypes.c_uint32, u32p, u16p]
        L.or_pll_build.restype = ctypes.c_int64
        L.or_pll_build.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, u8p, ctypes.c_uint32, ctypes.c_uint32, u16p,
                                   u64p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p]
        L.or_pll_query.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u16p, u64p, ctypes.c_uint32,
                                   u32p, u32p, ctypes.c_uint64, u32p, u32p, i32p]
        L.or_query.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, u16p, u64p, ctypes.c_uint64, u32p,
                               u32p, i32p]
        L.or_query_stream.argtypes = [ctypes.c_uint32, u64p, u32p, u32p, u8p, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_uint64, u32p, u32p, ctypes.c_int, i32p]
        L.or_bidir_refine.argtypes = [ctypes.c_uint32, u64p, u32p, ctypes.c_uint64, u32p, u32p, ctypes.c_uint32, i32p]
        L.or_csr_build.restype = ctypes.c_int64
        L.or_csr_build.argtypes = [ctypes.c_uint32, ctypes.c_uint64, u32p, u32p, ctypes.c_int, u32p, u64p]
        L.or_record_bytes.restype = ctypes.c_int64
        L.or_record_bytes.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        L.or_budget_to_clusters.restype = ctypes.c_int64
        L.or_budget_to_clusters.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        # the shared counter-based generator (cbfs_inputs) for random roots
        _rand_cb = _RANDFN(lambda s, st, i: cbfs_inputs.lib().cg_rand(s, st, i))
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    assert a.flags.c_contiguous, "array must be C-contiguous"
    return a.ctypes.data_as(_P(ct))


def default_threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


# ---------------------------------------------------------------- graph
@dataclass
class CSR:
    """Symmetric, sorted, deduplicated CSR without self loops."""
    n: int
    off: np.ndarray   # uint64 [n+1]
    cols: np.ndarray  # uint32 [m]

    @property
    def m(self) -> int:
        return int(self.off[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.off).astype(np.uint32)


def csr_from_edges(n: int, src: np.ndarray, dst: np.ndarray) -> CSR:
    """Normalise an undirected edge list (SPEC load_edge_list semantics, R17):
    every pair {u,v} with u != v becomes arcs u->v and v->u; duplicates
    removed; neighbour lists ascending.  m = number of arcs."""
    src = np.asarray(src, dtype=np.uint64)
    dst = np.asarray(dst, dtype=np.uint64)
    if src.size and max(int(src.max()), int(dst.max())) >= n:
        raise ValueError("vertex id out of range")
    keep = src != dst
    s, d = src[keep], dst[keep]
    keys = np.unique(np.concatenate([(s << np.uint64(32)) | d, (d << np.uint64(32)) | s]))
    rows = (keys >> np.uint64(32)).astype(np.int64)
    cols = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    counts = np.bincount(rows, minlength=n).astype(np.uint64)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(counts, out=off[1:])
    return CSR(n, off, np.ascontiguousarray(cols))


def csr_from_edges_c(n: int, src: np.ndarray, dst: np.ndarray, threads: int | None = None) -> CSR:
    """Same normalisation in C (oracle.c or_csr_build: per-row sort + dedup),
    for edge lists too large for numpy's unique (config 3: 537M pairs)."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    work = np.empty(max(1, 2 * len(src)), np.uint32)
    off = np.zeros(n + 1, np.uint64)
    m = lib().or_csr_build(n, len(src), _p(src, ctypes.c_uint32), _p(dst, ctypes.c_uint32),
                           threads or default_threads(), _p(work, ctypes.c_uint32), _p(off, ctypes.c_uint64))
    if m < 0:
        raise ValueError("vertex id out of range")
    cols = work[:m].copy() if m < len(work) // 2 else work[:m]
    return CSR(n, off, cols)


def csr_from_edgelist(el) -> CSR:
    if len(el.src) > (8 << 20):
        return csr_from_edges_c(el.n, el.src, el.dst)
    return csr_from_edges(el.n, el.src, el.dst)


# ---------------------------------------------------------------- BFS
def plain_bfs(g: CSR, s: int) -> np.ndarray:
    dist = np.empty(g.n, np.uint32)
    rc = lib().or_plain_bfs(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32), s,
                            _p(dist, ctypes.c_uint32))
    if rc:
        raise ValueError("bad source")
    return dist


@dataclass
class ClusterResult:
    dist: np.ndarray   # uint16 [n], INF16 = unreachable
    sub: np.ndarray    # uint64 [d+1][n]
    stats: np.ndarray  # uint64 [4]: rounds, sumF, sumE, sum_{reached} deg
    round_F: np.ndarray | None = None
    round_E: np.ndarray | None = None


def _sources(S) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(S, dtype=np.uint32))


def brute_cluster(g: CSR, S, d: int):
    """Definition P:630-639 via k queue BFS runs.  Returns (dist, sub, over)
    where over=True means some source lies more than d beyond Delta_v."""
    S = _sources(S)
    dist = np.empty(g.n, np.uint16)
    sub = np.empty((d + 1, g.n), np.uint64)
    rc = lib().or_brute_cluster(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32),
                                _p(S, ctypes.c_uint32), len(S), d, _p(dist, ctypes.c_uint16),
                                _p(sub, ctypes.c_uint64))
    if rc < 0:
        raise ValueError("invalid cluster")
    return dist, sub, bool(rc)


def brute_cluster_wide(g: CSR, S, d: int):
    """The definition P:630-639 for a cluster of any size k (the paper's
    general k), written out: Delta_v =
    min_j delta(s_j, v) and S_v[i] = {j : delta(s_j, v) = Delta_v + i},
    i = 0..d, each subset W = ceil(k / 64) words with bit j of the cluster in
    bit j % 64 of word j // 64 (R11).  delta from k queue BFS runs.
    Returns (dist uint16 [n] (INF16 = unreachable), sub uint64 [d+1][n][W],
    over) where over means some source lies more than d beyond Delta_v."""
    S = _sources(S)
    k = len(S)
    W = (k + 63) // 64
    D = np.stack([plain_bfs(g, int(x)) for x in S]).astype(np.int64)
    reach = D != INF32
    Delta = np.where(reach, D, INF32).min(axis=0)
    sub = np.zeros((d + 1, g.n, W), np.uint64)
    over = False
    for j in range(k):
        off = D[j] - Delta
        over |= bool((reach[j] & (off > d)).any())
        for i in range(d + 1):
            sel = reach[j] & (off == i)
            sub[i, sel, j // 64] |= np.uint64(1 << (j % 64))
    dist = np.where(Delta == INF32, INF16, Delta).astype(np.uint16)
    return dist, sub, over


def query_brute(g: CSR, clusters, s, t) -> np.ndarray:
    """Landmark query with each cluster's sources as its landmarks
    (R16): min over clusters and sources s_j of delta(u, s_j) +
    delta(s_j, v), INT32_MAX when no source reaches both ends; clusters of
    any size.  For clusters of diameter <= d this is the value of the
    (d+1)^2 subset scan (R15)."""
    s = np.asarray(s, dtype=np.int64)
    t = np.asarray(t, dtype=np.int64)
    big = np.int64(1) << 40
    best = np.full(len(s), big, np.int64)
    for S in clusters:
        for x in _sources(S):
            D = plain_bfs(g, int(x)).astype(np.int64)
            D[D == INF32] = big
            best = np.minimum(best, D[s] + D[t])
    return np.where(best >= big, INT32_MAX, best).astype(np.int32)


def cluster_bfs(g: CSR, S, d: int, max_rounds: int = 1 << 16) -> ClusterResult:
    """Alg. 1, sequential."""
    S = _sources(S)
    dist = np.empty(g.n, np.uint16)
    sub = np.empty((d + 1, g.n), np.uint64)
    stats = np.zeros(4, np.uint64)
    rF = np.zeros(max_rounds, np.uint32)
    rE = np.zeros(max_rounds, np.uint64)
    rc = lib().or_cluster_bfs(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32), _p(S, ctypes.c_uint32),
                              len(S), d, _p(dist, ctypes.c_uint16), _p(sub, ctypes.c_uint64),
                              _p(stats, ctypes.c_uint64), _p(rF, ctypes.c_uint32), _p(rE, ctypes.c_uint64),
                              max_rounds)
    if rc:
        raise ValueError("invalid cluster (k=0, k>64, duplicate or out-of-range source)")
    R = int(stats[0])
    return ClusterResult(dist, sub, stats, rF[:min(R, max_rounds)].copy(), rE[:min(R, max_rounds)].copy())


def cluster_bfs_many(g: CSR, sources: np.ndarray, sizes: np.ndarray, d: int, threads: int | None = None,
                     want_outputs: bool = True, want_digest: bool = False, max_rounds: int = 0):
    """Alg. 1 per cluster, clusters over host threads.  sources [C][64] uint32,
    sizes [C] uint8.  Returns dict(dist [C][n], sub [C][d+1][n], stats [C][4],
    hash [C]); with want_digest also digest [C] (digest_cluster of each
    output), with max_rounds > 0 also round_F [C][max_rounds] (|F_i|) and
    round_E [C][max_rounds] (E_i), zero past the cluster's last round."""
    sources = np.ascontiguousarray(sources, dtype=np.uint32)
    sizes = np.ascontiguousarray(sizes, dtype=np.uint8)
    C = sources.shape[0]
    assert sources.shape == (C, 64) and sizes.shape == (C,)
    stats = np.zeros((C, 4), np.uint64)
    h = np.zeros(C, np.uint64)
    dg = np.zeros(C, np.uint64) if want_digest else None
    rF = np.zeros((C, max_rounds), np.uint32) if max_rounds else None
    rE = np.zeros((C, max_rounds), np.uint64) if max_rounds else None
    dist = np.empty((C, g.n), np.uint16) if want_outputs else None
    sub = np.empty((C, d + 1, g.n), np.uint64) if want_outputs else None
    rc = lib().or_cluster_bfs_many_ex(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32),
                                      _p(sources, ctypes.c_uint32), _p(sizes, ctypes.c_uint8), C, d,
                                      threads or default_threads(),
                                      _p(dist, ctypes.c_uint16) if want_outputs else None,
                                      _p(sub, ctypes.c_uint64) if want_outputs else None,
                                      _p(stats, ctypes.c_uint64), _p(h, ctypes.c_uint64),
                                      _p(dg, ctypes.c_uint64) if want_digest else None,
                                      _p(rF, ctypes.c_uint32) if max_rounds else None,
                                      _p(rE, ctypes.c_uint64) if max_rounds else None, max_rounds)
    if rc:
        raise ValueError("invalid cluster in batch")
    out = dict(dist=dist, sub=sub, stats=stats, hash=h)
    if want_digest:
        out["digest"] = dg
    if max_rounds:
        out["round_F"], out["round_E"] = rF, rE
    return out


def digest_cluster(dist: np.ndarray, sub: np.ndarray) -> int:
    """Order-independent digest of one cluster's output (oracle.c
    or_digest_cluster): sum over v of a SplitMix64 chain over (v and Delta_v,
    then S_v[0..planes-1]), mod 2^64.  dist uint16 [n], sub uint64 [planes][n]."""
    dist = np.ascontiguousarray(dist, dtype=np.uint16)
    sub = np.ascontiguousarray(sub, dtype=np.uint64)
    return int(lib().or_digest_cluster(dist.shape[0], sub.shape[0], _p(dist, ctypes.c_uint16),
                                       _p(sub, ctypes.c_uint64)))


def hash_cluster(dist: np.ndarray, sub: np.ndarray) -> int:
    d = sub.shape[0] - 1
    dist = np.ascontiguousarray(dist, dtype=np.uint16)
    sub = np.ascontiguousarray(sub, dtype=np.uint64)
    return int(lib().or_hash_cluster(dist.shape[0], d, _p(dist, ctypes.c_uint16), _p(sub, ctypes.c_uint64)))


# ---------------------------------------------------------------- selection
ROOT_DEGREE, ROOT_RANDOM = 0, 1


def select_clusters(g: CSR, r: int, k: int, d: int, policy: int = ROOT_DEGREE, seed: int = 0):
    """P:1061-1069 with R12.  Returns (sources [r'][64] uint32 padded with
    0xFFFFFFFF, sizes [r'] uint8)."""
    lib()
    out = np.full((max(r, 1), 64), PAD, np.uint32)
    sizes = np.zeros(max(r, 1), np.uint8)
    got = lib().or_select_clusters(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32), r, k, d, policy,
                                   seed, _rand_cb, _p(out, ctypes.c_uint32), _p(sizes, ctypes.c_uint8))
    if got < 0:
        raise ValueError("bad selection arguments")
    return out[:got].copy(), sizes[:got].copy()


def select_clusters_wide(g: CSR, r: int, k: int, d: int, words: int, policy: int = ROOT_DEGREE, seed: int = 0):
    """The same rule (R12) for clusters of up to k <= 64 * words
    sources (the paper's general k).  Returns (sources [r'][64 words]
    uint32 padded with 0xFFFFFFFF, sizes [r'] uint16)."""
    out = np.full((max(r, 1), 64 * words), PAD, np.uint32)
    sizes = np.zeros(max(r, 1), np.uint16)
    got = lib().or_select_clusters_wide(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32), r, k, d,
                                        policy, seed, _rand_cb, words, _p(out, ctypes.c_uint32),
                                        _p(sizes, ctypes.c_uint16))
    if got < 0:
        raise ValueError("bad selection arguments")
    return out[:got].copy(), sizes[:got].copy()


# ---------------------------------------------------------------- queries
def query(dist: np.ndarray, sub: np.ndarray, s: np.ndarray, t: np.ndarray) -> np.ndarray:
    """dist [C][n] uint16, sub [C][d+1][n] uint64 (cluster-major labels)."""
    dist = np.ascontiguousarray(dist, dtype=np.uint16)
    sub = np.ascontiguousarray(sub, dtype=np.uint64)
    C, n = dist.shape
    d = sub.shape[1] - 1
    s = np.ascontiguousarray(s, dtype=np.uint32)
    t = np.ascontiguousarray(t, dtype=np.uint32)
    out = np.empty(len(s), np.int32)
    rc = lib().or_query(n, d, C, _p(dist, ctypes.c_uint16), _p(sub, ctypes.c_uint64), len(s),
                        _p(s, ctypes.c_uint32), _p(t, ctypes.c_uint32), _p(out, ctypes.c_int32))
    if rc:
        raise ValueError("query vertex out of range")
    return out


def query_stream(g: CSR, sources, sizes, d: int, s, t, threads: int | None = None, with_stats: bool = False):
    """Streaming index build + query (Alg. 2 with C-BFS, then
    P:1013-1021).  Returns the answers int32 [q]; with_stats also returns
    (answers, stats [C][4], digest [C]) of every cluster's Alg. 1 run."""
    sources = np.ascontiguousarray(sources, dtype=np.uint32)
    sizes = np.ascontiguousarray(sizes, dtype=np.uint8)
    s = np.ascontiguousarray(s, dtype=np.uint32)
    t = np.ascontiguousarray(t, dtype=np.uint32)
    out = np.empty(len(s), np.int32)
    C = sources.shape[0]
    stats = np.zeros((C, 4), np.uint64) if with_stats else None
    dg = np.zeros(C, np.uint64) if with_stats else None
    rc = lib().or_query_stream_ex(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32),
                                  _p(sources, ctypes.c_uint32), _p(sizes, ctypes.c_uint8), C, d, len(s),
                                  _p(s, ctypes.c_uint32), _p(t, ctypes.c_uint32), threads or default_threads(),
                                  _p(out, ctypes.c_int32), _p(stats, ctypes.c_uint64) if with_stats else None,
                                  _p(dg, ctypes.c_uint64) if with_stats else None)
    if rc:
        raise ValueError("bad stream query")
    return (out, stats, dg) if with_stats else out


def bidir_refine(g: CSR, s, t, tau: int) -> np.ndarray:
    """Appendix B with reading R27: tau vertices visited from
    each side in BFS order over the sorted CSR, min over common vertices of
    dist_s + dist_t; INT32_MAX when disjoint."""
    s = np.ascontiguousarray(s, dtype=np.uint32)
    t = np.ascontiguousarray(t, dtype=np.uint32)
    out = np.empty(len(s), np.int32)
    rc = lib().or_bidir_refine(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32), len(s),
                               _p(s, ctypes.c_uint32), _p(t, ctypes.c_uint32), tau, _p(out, ctypes.c_int32))
    if rc:
        raise ValueError("query vertex out of range")
    return out


def record_bytes(w: int, d: int) -> int:
    return int(lib().or_record_bytes(w, d))


def budget_to_clusters(t: int, w: int, d: int) -> int:
    return int(lib().or_budget_to_clusters(t, w, d))


# ---------------------------------------------------------------- exact 2-hop oracle (PLL, NEXT-4)
def pll_build(g: CSR, sources, sizes, d: int, first: int = 200, bmax: int = 1000, cap: int = 256,
              threads: int | None = None) -> dict:
    """PLL with a C-BFS first phase, reading R29: the given
    clusters' labels (Alg. 1) for every vertex, then pruned BFSs from the
    uncovered vertices in (degree desc, id asc) order, batches first,
    floor(3/2 b), ... up to bmax, each batch pruned against the index as of
    its start.  Returns dict(counts [n], entries [n][cap] (pos << 8 | dist,
    ascending), cdist [C][n], csub [C][d+1][n], total, d, cap)."""
    sources = np.ascontiguousarray(sources, dtype=np.uint32).reshape(-1, 64)
    sizes = np.ascontiguousarray(sizes, dtype=np.uint8)
    C = len(sizes)
    if C:
        many = cluster_bfs_many(g, sources, sizes, d, threads=threads)
        cdist, csub = many["dist"], many["sub"]
    else:
        cdist = np.zeros((0, g.n), np.uint16)
        csub = np.zeros((0, d + 1, g.n), np.uint64)
    counts = np.zeros(max(g.n, 1), np.uint32)
    entries = np.zeros((max(g.n, 1), cap), np.uint32)
    total = lib().or_pll_build(g.n, _p(g.off, ctypes.c_uint64), _p(g.cols, ctypes.c_uint32),
                               _p(sources, ctypes.c_uint32), _p(sizes, ctypes.c_uint8), C, d,
                               _p(np.ascontiguousarray(cdist), ctypes.c_uint16),
                               _p(np.ascontiguousarray(csub), ctypes.c_uint64), first, bmax, cap,
                               _p(counts, ctypes.c_uint32), _p(entries, ctypes.c_uint32))
    if total == -2:
        raise OverflowError("a label list exceeds cap")
    if total < 0:
        raise ValueError(f"pll_build failed ({total})")
    return dict(counts=counts[:g.n], entries=entries[:g.n], cdist=cdist, csub=csub, total=int(total), d=d, cap=cap,
                n=g.n)


def pll_query(idx: dict, s, t) -> np.ndarray:
    """Exact distance by the 2-hop cover: min of the cluster
    labels' value (R15 scan) and min over common hubs; INT32_MAX unreachable."""
    s = np.ascontiguousarray(s, dtype=np.uint32)
    t = np.ascontiguousarray(t, dtype=np.uint32)
    out = np.empty(len(s), np.int32)
    C = idx["cdist"].shape[0]
    rc = lib().or_pll_query(idx["n"], C, idx["d"], _p(np.ascontiguousarray(idx["cdist"]), ctypes.c_uint16),
                            _p(np.ascontiguousarray(idx["csub"]), ctypes.c_uint64), idx["cap"],
                            _p(np.ascontiguousarray(idx["counts"]), ctypes.c_uint32),
                            _p(np.ascontiguousarray(idx["entries"]), ctypes.c_uint32), len(s),
                            _p(s, ctypes.c_uint32), _p(t, ctypes.c_uint32), _p(out, ctypes.c_int32))
    if rc:
        raise ValueError("query vertex out of range")
    return out
