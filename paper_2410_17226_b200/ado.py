"""Approximate distance oracle (ADO) on C-BFS landmark labels, and its
distortion.

PAPER.md §4.2: landmark labeling answers query(u, v) = min over
landmarks h of delta(u, h) + delta(h, v); with clusters of landmarks the
per-cluster value is Delta_u + Delta_v + min{i + j : S_u[i] & S_v[j] != 0}
(P:1074-1086).  The error is one-sided (query >= delta) and the distortion is
psi = query / delta, reported as epsilon = mean(psi) - 1 over
sampled pairs (100,000 pairs, 10,000 on the largest graphs).

Everything here drives the C-ABI (argument marshalling only): the index is
`cbfs_select_clusters` + `cbfs_labels_build_w` (R14 records in a store of
word size w), the answers come from `cbfs_labels_query`, and the
exact distances of the sampled pairs
from C-BFS itself: a cluster of one source with d = 0 is a plain BFS
(R3), so each batch of 64 single-source "clusters" yields the true
distances from 64 sampled sources at once.
"""
from __future__ import annotations

import numpy as np
import torch

from . import (CBFS_QUERY_UNREACHED, CBFS_ROOT_DEGREE, cbfs_budget_clusters, cbfs_labels_build, cbfs_labels_destroy,
               cbfs_labels_info, cbfs_labels_query, cbfs_query_bidir, cbfs_record_bytes, cbfs_run,
               cbfs_select_clusters)

UNREACHED16 = 0xFFFF


def record_bytes(word_bits: int, d: int, dist_bytes: int = 1) -> int:
    """Bytes of one (cluster, vertex) record (cbfs_record_bytes)."""
    return cbfs_record_bytes(word_bits, d, dist_bytes)


def clusters_for_budget(t_bytes: int, word_bits: int, d: int, dist_bytes: int = 1) -> int:
    """Clusters whose records fit t bytes per vertex (cbfs_budget_clusters)."""
    return cbfs_budget_clusters(t_bytes, word_bits, d, dist_bytes)


class LandmarkIndex:
    """Labels of r clusters (k <= w sources, diameter bound d) in a label
    store of word size w = word_bits (cbfs_labels_build_w): per vertex and
    cluster Delta (dist_bytes) + S_v[0..d-1] in w-bit words (R14)."""

    def __init__(self, graph, r: int, k: int = 64, d: int = 2, root_policy: int = CBFS_ROOT_DEGREE, seed: int = 0,
                 word_bits: int = 64, dist_bytes: int = 2):
        """word_bits = 0: plain landmark labeling (k = 1, d = 0: r single
        vertices by the same selection rule, 1-2 byte records)."""
        if not 1 <= k <= max(word_bits, 1) or (word_bits == 0 and d != 0):
            raise ValueError("cluster size k must be 1..word_bits (plain landmarks: k = 1, d = 0)")
        dev = f"cuda:{graph.device}"
        src = torch.empty((max(r, 1), 64), dtype=torch.int32, device=dev)
        sz = torch.empty((max(r, 1),), dtype=torch.uint8, device=dev)
        got = cbfs_select_clusters(graph.h, r, k, d, root_policy, seed, src, sz) if r else 0
        self.graph, self.d, self.r, self.word_bits, self.dist_bytes = graph, d, got, word_bits, dist_bytes
        self.sources, self.sizes = src[:got].contiguous(), sz[:got].contiguous()
        self.labels = cbfs_labels_build(graph.h, self.sources, self.sizes, got, d, dist_bytes,
                                        word_bits=word_bits) if got else None

    @property
    def image_bytes(self) -> int:
        return cbfs_labels_info(self.labels)["image_bytes"] if self.labels else 0

    def query(self, s: torch.Tensor, t: torch.Tensor, tau: int = 0) -> torch.Tensor:
        """int32 answers, CBFS_QUERY_UNREACHED where no cluster reaches both
        ends; tau > 0 adds the Appendix B bi-directional search:
        the answer is the minimum of the index's and the search's."""
        best = torch.full((int(s.shape[0]),), CBFS_QUERY_UNREACHED, dtype=torch.int32, device=s.device)
        if self.labels:
            cbfs_labels_query(self.labels, s, t, best)
        if tau:
            cbfs_query_bidir(self.graph.h, s, t, tau, best)
        return best

    def close(self):
        if self.labels:
            cbfs_labels_destroy(self.labels)
            self.labels = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def exact_distances(graph, s: np.ndarray, t: np.ndarray) -> np.ndarray:
    """delta(s[q], t[q]) for every pair (uint32, 0xFFFF = unreachable), from
    single-source C-BFS runs (k = 1, d = 0 is a plain BFS), 64 distinct
    sources per batch."""
    dev = f"cuda:{graph.device}"
    s = np.asarray(s, dtype=np.uint32)
    t = np.asarray(t, dtype=np.uint32)
    out = np.empty(len(s), np.uint32)
    uniq, inv = np.unique(s, return_inverse=True)
    dist = torch.empty((graph.n, 64), dtype=torch.int16, device=dev)
    td = torch.from_numpy(t.astype(np.int64)).to(dev)
    for b0 in range(0, len(uniq), 64):
        blk = uniq[b0:b0 + 64]
        C = len(blk)
        src = torch.full((C, 64), -1, dtype=torch.int32, device=dev)
        src[:, 0] = torch.from_numpy(blk.view(np.int32)).to(dev)
        sz = torch.ones((C,), dtype=torch.uint8, device=dev)
        dd = dist[:, :C].contiguous() if C < 64 else dist
        cbfs_run(graph.h, src, sz, C, 0, 2, dd, None, 1, None)
        sel = np.nonzero((inv >= b0) & (inv < b0 + C))[0]
        col = torch.from_numpy((inv[sel] - b0).astype(np.int64)).to(dev)
        vals = dd[td[torch.from_numpy(sel).to(dev)], col]
        out[sel] = vals.cpu().numpy().view(np.uint16).astype(np.uint32)
    return out


def sample_pairs(s_cand: np.ndarray, t_cand: np.ndarray, count: int, exact_fn):
    """The first `count` candidate pairs (drawn uniformly by the caller) that
    are distinct and mutually reachable.  Returns (s, t, delta)."""
    s = np.asarray(s_cand, dtype=np.uint32)
    t = np.asarray(t_cand, dtype=np.uint32)
    keep = s != t
    s, t = s[keep], t[keep]
    dd = exact_fn(s, t)
    ok = dd != UNREACHED16
    return s[ok][:count], t[ok][:count], dd[ok][:count]


def distortion(answers: np.ndarray, exact: np.ndarray) -> dict:
    """epsilon = mean(query / delta) - 1 over the pairs the index covers
    (P:1031-1034); coverage = share of pairs with a finite answer."""
    answers = np.asarray(answers, dtype=np.int64)
    exact = np.asarray(exact, dtype=np.int64)
    cov = answers < CBFS_QUERY_UNREACHED
    if not cov.any():
        return {"pairs": int(len(exact)), "covered": 0, "epsilon_pct": None, "max_psi": None, "exact_hits": 0.0,
                "one_sided": True}
    psi = answers[cov] / exact[cov]
    return {"pairs": int(len(exact)), "covered": int(cov.sum()), "epsilon_pct": float(100.0 * (psi.mean() - 1.0)),
            "max_psi": float(psi.max()), "exact_hits": float((answers[cov] == exact[cov]).mean()),
            "one_sided": bool((answers[cov] >= exact[cov]).all())}
