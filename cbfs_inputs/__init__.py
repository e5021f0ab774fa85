"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

Holds none of the method's arithmetic: raw COO edge lists (duplicates and self
loops included) and query pairs only.  See include/cbfs_gen.h for the exact
generator definitions and DESIGN.md §3 for the workload recipe (BASELINE.json
configs; SURVEY.md readings R21-R24).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libcbfsgen.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", src,
                               "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.cg_mix64.restype = ctypes.c_uint64
        L.cg_mix64.argtypes = [ctypes.c_uint64]
        L.cg_rand.restype = ctypes.c_uint64
        L.cg_rand.argtypes = [ctypes.c_uint64] * 3
        L.cg_bounded.restype = ctypes.c_uint64
        L.cg_bounded.argtypes = [ctypes.c_uint64] * 2
        L.cg_erdos_renyi.restype = ctypes.c_int64
        L.cg_erdos_renyi.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _u32p, _u32p]
        L.cg_rmat.restype = ctypes.c_int64
        L.cg_rmat.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _u32p, _u32p]
        L.cg_grid_capacity.restype = ctypes.c_uint64
        L.cg_grid_capacity.argtypes = [ctypes.c_uint32, ctypes.c_double]
        L.cg_grid.restype = ctypes.c_int64
        L.cg_grid.argtypes = [ctypes.c_uint32, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                              _u32p, _u32p]
        L.cg_knn3d.restype = ctypes.c_int64
        L.cg_knn3d.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, _u32p, _u32p, _u32p]
        L.cg_query_pairs.restype = ctypes.c_int64
        L.cg_query_pairs.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u32p, _u32p]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_u32p)


def rand(seed: int, stream: int, index: int) -> int:
    return int(lib().cg_rand(seed, stream, index))


def bounded(x: int, n: int) -> int:
    return int(lib().cg_bounded(x, n))


@dataclass
class EdgeList:
    """Raw undirected edge list (COO pairs) of a graph with n vertices."""
    n: int
    src: np.ndarray
    dst: np.ndarray
    name: str = ""


def erdos_renyi(n: int, pairs: int, seed: int) -> EdgeList:
    s = np.empty(pairs, np.uint32); d = np.empty(pairs, np.uint32)
    r = lib().cg_erdos_renyi(n, pairs, seed, _p(s), _p(d))
    assert r == pairs
    return EdgeList(n, s, d, f"er_n{n}_p{pairs}_s{seed}")


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int, scramble: bool = True,
         threads: int = 0) -> EdgeList:
    m = (1 << scale) * edge_factor
    s = np.empty(m, np.uint32); d = np.empty(m, np.uint32)
    r = lib().cg_rmat(scale, m, a, b, c, seed, int(scramble), threads, _p(s), _p(d))
    assert r == m
    return EdgeList(1 << scale, s, d, f"rmat{scale}_ef{edge_factor}_s{seed}")


def grid(side: int, p_delete: float, p_diag: float, seed: int) -> EdgeList:
    cap = int(lib().cg_grid_capacity(side, p_diag))
    s = np.empty(cap, np.uint32); d = np.empty(cap, np.uint32)
    r = lib().cg_grid(side, p_delete, p_diag, seed, cap, _p(s), _p(d))
    assert r >= 0
    return EdgeList(side * side, s[:r].copy(), d[:r].copy(), f"grid{side}_s{seed}")


def knn3d(n: int, k: int, seed: int, threads: int = 0, want_coords: bool = False):
    s = np.empty(n * k, np.uint32); d = np.empty(n * k, np.uint32)
    xyz = np.empty(3 * n, np.uint32) if want_coords else None
    r = lib().cg_knn3d(n, k, seed, threads, _p(s), _p(d), _p(xyz) if xyz is not None else None)
    assert r == n * k
    el = EdgeList(n, s, d, f"knn{n}_k{k}_s{seed}")
    return (el, xyz.reshape(n, 3)) if want_coords else el


def query_pairs(n: int, q: int, seed: int, stream: int = 2):
    s = np.empty(q, np.uint32); t = np.empty(q, np.uint32)
    r = lib().cg_query_pairs(n, q, seed, stream, _p(s), _p(t))
    assert r == q
    return s, t


# --------------------------------------------------------------------------
# BASELINE.json configs (seeds per SURVEY.md R22).  `relabel` is the internal
# vertex order the CUDA path is asked for (outputs are in original ids, R18):
# hubs first for the power-law graphs, BFS locality for the k-NN graph
# (C-BFS 1.55x faster than its generator ids).  The grid keeps its row-major
# ids: the locality order is 1.12x faster to traverse there but its ~8,000
# BFS levels cost as much to build as they save.  `scale_down` shrinks a
# config for quick tests while keeping its generator family and parameters.
# --------------------------------------------------------------------------
CONFIGS = {
    "c1_er": dict(kind="er", n=4096, pairs=32768, seed=1, clusters=8, k=64, d=2, root="random", root_seed=1,
                  relabel="degree"),
    "c2_rmat20": dict(kind="rmat", scale=20, ef=16, abc=(0.57, 0.19, 0.19), seed=2, clusters=1024, k=64, d=2,
                      root="degree", root_seed=0, relabel="degree"),
    "c3_rmat24": dict(kind="rmat", scale=24, ef=32, abc=(0.6, 0.15, 0.15), seed=3, clusters=4096, k=64, d=2,
                      root="degree", root_seed=0, relabel="degree"),
    "c4_grid": dict(kind="grid", side=4096, p_delete=0.05, p_diag=0.001, seed=4, clusters=512, k=64, d=4,
                    root="random", root_seed=4, relabel="locality"),
    "c5_knn": dict(kind="knn", n=10_000_000, knn=10, seed=7, clusters=8192, k=64, d=6, root="degree",
                   root_seed=0, queries=10_000_000, query_seed=7, relabel="locality"),
}


def make_graph(name: str, **over) -> EdgeList:
    c = dict(CONFIGS[name]); c.update(over)
    if c["kind"] == "er":
        return erdos_renyi(c["n"], c["pairs"], c["seed"])
    if c["kind"] == "rmat":
        a, b, cc = c["abc"]
        return rmat(c["scale"], c["ef"], a, b, cc, c["seed"])
    if c["kind"] == "grid":
        return grid(c["side"], c["p_delete"], c["p_diag"], c["seed"])
    if c["kind"] == "knn":
        return knn3d(c["n"], c["knn"], c["seed"])
    raise ValueError(name)
