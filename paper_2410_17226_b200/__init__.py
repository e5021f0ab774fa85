"""paper_2410_17226_b200 — thin Python binding of libcbfs.so (include/cbfs.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels (sm_100a).  Functions keep the C-ABI names; device buffers are
torch CUDA tensors (PyTorch is used for device memory and streams only),
host buffers are numpy arrays.  There is no CPU fallback: importing this
package without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CBFS_LIB_PATH") or os.path.join(_HERE, "libcbfs.so")  # override: experiments only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or `make`); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ constants (include/cbfs.h)
CBFS_OK, CBFS_EINVAL, CBFS_ENOMEM, CBFS_ECUDA, CBFS_EOVERFLOW, CBFS_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
CBFS_MAX_K, CBFS_MAX_D, CBFS_MAX_N = 64, 31, (1 << 26) - 1
CBFS_PAD = 0xFFFFFFFF
CBFS_UNREACHED_U16, CBFS_UNREACHED_U8 = 0xFFFF, 0xFF
CBFS_QUERY_UNREACHED = 0x7FFFFFFF
CBFS_BIDIR_MAX_TAU = 1024
CBFS_RELABEL_DEGREE, CBFS_INPUT_DEVICE, CBFS_RELABEL_LOCALITY = 2, 4, 8
CBFS_ROOT_DEGREE, CBFS_ROOT_RANDOM = 0, 1
CBFS_DIR_AUTO, CBFS_DIR_PUSH, CBFS_DIR_PULL = 0, 1, 2
CBFS_ENGINE_AUTO, CBFS_ENGINE_BATCHED, CBFS_ENGINE_SPARSE = 0, 1, 2

_vp, _u32, _u64, _i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("cbfs_graph_create", [_u32, _vp, _vp, _u64, _u32, _i32, _vp, ctypes.POINTER(_vp)])
_sig("cbfs_graph_create_csr", [_u32, _vp, _vp, _u64, _u32, _i32, _vp, ctypes.POINTER(_vp)])
_sig("cbfs_graph_info", [_vp, ctypes.POINTER(_u32), ctypes.POINTER(_u64), ctypes.POINTER(_u32)])
_sig("cbfs_graph_export_csr", [_vp, _vp, _vp])
_sig("cbfs_graph_internal_order", [_vp, _vp])
_sig("cbfs_graph_destroy", [_vp])
_sig("cbfs_select_clusters", [_vp, _u32, _u32, _u32, _u32, _u64, _vp, _vp, ctypes.POINTER(_u32), _vp])
_sig("cbfs_select_clusters_wide", [_vp, _u32, _u32, _u32, _u32, _u64, _u32, _vp, _vp, ctypes.POINTER(_u32), _vp])
_sig("cbfs_run", [_vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _u32, _vp, _u32, _vp])
_sig("cbfs_select_and_run", [_vp, _u32, _u32, _u32, _u32, _u64, _vp, _vp, ctypes.POINTER(_u32), _u32, _vp, _vp,
                              _u32, _vp, _u32, _vp])
_sig("cbfs_select_and_run_shard", [_vp, _u32, _u32, _u32, _u32, _u64, _u32, _u32, _vp, _vp, ctypes.POINTER(_u32), _u32,
                                    _vp, _vp, _u32, _vp, _u32, _vp])
_sig("cbfs_run_digest", [_vp, _vp, _vp, _u32, _u32, _u32, _u32, _vp, _vp, _u32, _vp])
_sig("cbfs_run_rounds", [_vp, _vp, _vp, _u32, _u32, _vp, _u32, _vp, _u32, _vp])
_sig("cbfs_digest_store", [_u32, _u32, _u32, _vp, _u32, _vp, _vp, _vp])
_sig("cbfs_run_host", [_vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _u32, _vp, _u32, _vp])
_sig("cbfs_run_wide", [_vp, _vp, _vp, _u32, _u32, _u32, _u32, _vp, _vp, _u32, _vp, _u32, _vp])
_sig("cbfs_decode_wide", [_u32, _u32, _u32, _u32, _u32, _vp, _u32, _vp, _u32, _u32, _vp, _vp])
_sig("cbfs_query_distance_wide", [_u32, _u32, _u32, _u32, _u32, _vp, _u32, _vp, _vp, _vp, _vp, _u64, _vp, _vp])
_sig("cbfs_decode", [_u32, _u32, _u32, _u32, _vp, _u32, _vp, _u32, _u32, _vp, _vp])
_sig("cbfs_query_distance", [_u32, _u32, _u32, _u32, _vp, _u32, _vp, _vp, _vp, _vp, _u64, _vp, _vp])
_sig("cbfs_query_stream", [_vp, _vp, _vp, _u32, _u32, _vp, _vp, _u64, _vp, _vp, _vp])
_sig("cbfs_query_bidir", [_vp, _vp, _vp, _u64, _u32, _vp, _vp])
_sig("cbfs_pll_build", [_vp, _vp, _vp, _u32, _u32, _u32, _u32, _u32, ctypes.POINTER(_vp), _vp])
_sig("cbfs_pll_info", [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u32), ctypes.POINTER(_u32), ctypes.POINTER(_u32),
                       ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)])
_sig("cbfs_pll_export", [_vp, _vp, _vp, _vp])
_sig("cbfs_pll_query", [_vp, _vp, _vp, _u64, _vp, _vp])
_sig("cbfs_pll_destroy", [_vp])
_sig("cbfs_labels_build", [_vp, _vp, _vp, _u32, _u32, _u32, ctypes.POINTER(_vp), _vp])
_sig("cbfs_labels_build_w", [_vp, _vp, _vp, _u32, _u32, _u32, _u32, ctypes.POINTER(_vp), _vp])
_sig("cbfs_labels_word_bits", [_vp, ctypes.POINTER(_u32)])
_sig("cbfs_labels_info", [_vp, ctypes.POINTER(_u32), ctypes.POINTER(_u32), ctypes.POINTER(_u32), ctypes.POINTER(_u32),
                          ctypes.POINTER(_u64)])
_sig("cbfs_labels_export", [_vp, _vp, _u64])
_sig("cbfs_labels_import", [_vp, _vp, _u64, ctypes.POINTER(_vp)])
_sig("cbfs_labels_query", [_vp, _vp, _vp, _u64, _vp, _vp])
_sig("cbfs_labels_destroy", [_vp])
_sig("cbfs_record_bytes", [_u32, _u32, _u32, ctypes.POINTER(_u64)])
_sig("cbfs_budget_clusters", [_u64, _u32, _u32, _u32, ctypes.POINTER(_u64)])
_sig("cbfs_set_direction_alpha", [ctypes.c_double])
_sig("cbfs_set_concurrency", [_i32])
_sig("cbfs_set_pull_hub_rows", [_u32])
_sig("cbfs_set_sparse_order", [ctypes.c_int64])
_sig("cbfs_release_workspace", [_i32])
_sig("cbfs_set_engine", [_i32])
_sig("cbfs_profile_enable", [_i32])
_sig("cbfs_profile_read", [_vp, _vp, _vp, _vp, _vp, _vp, _i32])
_sig("cbfs_graph_nonisolated", [_vp, ctypes.POINTER(_u32)])
_sig("cbfs_launch_count", [_i32], _u64)
_sig("cbfs_last_error", [], ctypes.c_char_p)
_sig("cbfs_version", [], ctypes.c_char_p)


class CbfsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"cbfs error {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != CBFS_OK:
        raise CbfsError(rc, _lib.cbfs_last_error().decode())


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data
    assert x.is_contiguous()
    return x.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return stream if isinstance(stream, int) else stream.cuda_stream


def _is_device(x) -> bool:
    return not isinstance(x, np.ndarray) and getattr(x, "is_cuda", False)


# ------------------------------------------------------------------ C-ABI mirrors
def cbfs_graph_create(n, src, dst, flags=0, device=0, stream=None):
    h = _vp()
    dev = _is_device(src)
    if dev:
        flags |= CBFS_INPUT_DEVICE
    _check(_lib.cbfs_graph_create(n, _ptr(src), _ptr(dst), len(src), flags, device, _stream(stream), ctypes.byref(h)))
    return h


def cbfs_graph_create_csr(n, offsets, cols, flags=0, device=0, stream=None):
    h = _vp()
    if _is_device(offsets):
        flags |= CBFS_INPUT_DEVICE
    _check(_lib.cbfs_graph_create_csr(n, _ptr(offsets), _ptr(cols), len(cols), flags, device, _stream(stream),
                                      ctypes.byref(h)))
    return h


def cbfs_graph_info(h):
    n, m, md = _u32(), _u64(), _u32()
    _check(_lib.cbfs_graph_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(md)))
    return n.value, m.value, md.value


def cbfs_graph_export_csr(h):
    n, m, _ = cbfs_graph_info(h)
    off = np.empty(n + 1, np.uint64)
    cols = np.empty(max(m, 1), np.uint32)
    _check(_lib.cbfs_graph_export_csr(h, _ptr(off), _ptr(cols)))
    return off, cols[:m]


def cbfs_graph_internal_order(h):
    n, _, _ = cbfs_graph_info(h)
    perm = np.empty(max(n, 1), np.uint32)
    _check(_lib.cbfs_graph_internal_order(h, _ptr(perm)))
    return perm[:n]


def cbfs_graph_destroy(h):
    _check(_lib.cbfs_graph_destroy(h))


def cbfs_select_clusters(h, r, k, d, root_policy, seed, out_sources, out_sizes, stream=None) -> int:
    got = _u32()
    _check(_lib.cbfs_select_clusters(h, r, k, d, root_policy, seed, _ptr(out_sources), _ptr(out_sizes),
                                     ctypes.byref(got), _stream(stream)))
    return got.value


def cbfs_select_clusters_wide(h, r, k, d, root_policy, seed, words, out_sources, out_sizes, stream=None) -> int:
    """out_sources [r][64 * words] int32, out_sizes [r] int16 (uint16 values)."""
    got = _u32()
    _check(_lib.cbfs_select_clusters_wide(h, r, k, d, root_policy, seed, words, _ptr(out_sources), _ptr(out_sizes),
                                          ctypes.byref(got), _stream(stream)))
    return got.value


def cbfs_run(h, sources, sizes, n_clusters, d, dist_bytes, out_dist, out_masks, planes, out_stats=None,
             direction=CBFS_DIR_AUTO, stream=None):
    _check(_lib.cbfs_run(h, _ptr(sources), _ptr(sizes), n_clusters, d, dist_bytes, _ptr(out_dist), _ptr(out_masks),
                         planes, _ptr(out_stats), direction, _stream(stream)))


def cbfs_select_and_run(h, r, k, d, root_policy, seed, out_sources, out_sizes, dist_bytes, out_dist, out_masks,
                        planes, out_stats=None, direction=CBFS_DIR_AUTO, stream=None) -> int:
    got = _u32()
    _check(_lib.cbfs_select_and_run(h, r, k, d, root_policy, seed, _ptr(out_sources), _ptr(out_sizes),
                                    ctypes.byref(got), dist_bytes, _ptr(out_dist), _ptr(out_masks), planes,
                                    _ptr(out_stats), direction, _stream(stream)))
    return got.value


def cbfs_select_and_run_shard(h, r, k, d, root_policy, seed, world, rank, out_sources, out_sizes, dist_bytes, out_dist,
                              out_masks, planes, out_stats=None, direction=CBFS_DIR_AUTO, stream=None) -> int:
    got = _u32()
    _check(_lib.cbfs_select_and_run_shard(h, r, k, d, root_policy, seed, world, rank, _ptr(out_sources),
                                          _ptr(out_sizes), ctypes.byref(got), dist_bytes, _ptr(out_dist),
                                          _ptr(out_masks), planes, _ptr(out_stats), direction, _stream(stream)))
    return got.value


def cbfs_run_digest(h, sources, sizes, n_clusters, d, dist_bytes, planes, out_digest, out_stats=None,
                    direction=CBFS_DIR_AUTO, stream=None):
    """Full output vectors of every cluster written batch by batch to HBM staging and reduced to one 64-bit
    digest per cluster (out_digest [C] int64/uint64 device)."""
    _check(_lib.cbfs_run_digest(h, _ptr(sources), _ptr(sizes), n_clusters, d, dist_bytes, planes, _ptr(out_digest),
                                _ptr(out_stats), direction, _stream(stream)))


def cbfs_run_rounds(h, sources, sizes, n_clusters, d, out_rounds, max_rounds, out_stats=None,
                    direction=CBFS_DIR_AUTO, stream=None):
    """Per-round frontier statistics: out_rounds [C][max_rounds][2] {|F_i|, E_i} (device)."""
    _check(_lib.cbfs_run_rounds(h, _ptr(sources), _ptr(sizes), n_clusters, d, _ptr(out_rounds), max_rounds,
                                _ptr(out_stats), direction, _stream(stream)))


def cbfs_digest_store(n, C, planes, dist, dist_bytes, masks, out_digest, stream=None):
    """Digest of every column of a vertex-major store dist [n][C], masks [planes][n][C] (cbfs_run's layout)."""
    _check(_lib.cbfs_digest_store(n, C, planes, _ptr(dist), dist_bytes, _ptr(masks), _ptr(out_digest),
                                  _stream(stream)))


def cbfs_run_host(h, sources, sizes, n_clusters, d, dist_bytes, out_dist, out_masks, planes, out_stats=None,
                  direction=CBFS_DIR_AUTO, stream=None):
    _check(_lib.cbfs_run_host(h, _ptr(sources), _ptr(sizes), n_clusters, d, dist_bytes, _ptr(out_dist),
                              _ptr(out_masks), planes, _ptr(out_stats), direction, _stream(stream)))


def cbfs_run_wide(h, sources, sizes, n_clusters, words, d, dist_bytes, out_dist, out_masks, planes, out_stats=None,
                  direction=CBFS_DIR_AUTO, stream=None):
    """sources [C][64 * words] int32, sizes [C] int16/uint16 (k <= 64 * words);
    out_masks [planes][n][C * words] (word w of cluster c at column c * words + w)."""
    _check(_lib.cbfs_run_wide(h, _ptr(sources), _ptr(sizes), n_clusters, words, d, dist_bytes, _ptr(out_dist),
                              _ptr(out_masks), planes, _ptr(out_stats), direction, _stream(stream)))


def cbfs_decode_wide(n, C, words, d, planes, dist, dist_bytes, masks, c, k, out, stream=None):
    _check(_lib.cbfs_decode_wide(n, C, words, d, planes, _ptr(dist), dist_bytes, _ptr(masks), c, k, _ptr(out),
                                 _stream(stream)))


def cbfs_query_distance_wide(n, C, words, d, planes, dist, dist_bytes, masks, sizes, s, t, inout_best, stream=None):
    _check(_lib.cbfs_query_distance_wide(n, C, words, d, planes, _ptr(dist), dist_bytes, _ptr(masks), _ptr(sizes),
                                         _ptr(s), _ptr(t), len(s), _ptr(inout_best), _stream(stream)))


def cbfs_decode(n, C, d, planes, dist, dist_bytes, masks, c, k, out, stream=None):
    _check(_lib.cbfs_decode(n, C, d, planes, _ptr(dist), dist_bytes, _ptr(masks), c, k, _ptr(out), _stream(stream)))


def cbfs_query_distance(n, C, d, planes, dist, dist_bytes, masks, sizes, s, t, inout_best, stream=None):
    _check(_lib.cbfs_query_distance(n, C, d, planes, _ptr(dist), dist_bytes, _ptr(masks), _ptr(sizes), _ptr(s),
                                    _ptr(t), len(s), _ptr(inout_best), _stream(stream)))


def cbfs_query_stream(h, sources, sizes, n_clusters, d, s, t, inout_best, out_stats=None, stream=None):
    _check(_lib.cbfs_query_stream(h, _ptr(sources), _ptr(sizes), n_clusters, d, _ptr(s), _ptr(t), len(s),
                                  _ptr(inout_best), _ptr(out_stats), _stream(stream)))


def cbfs_query_bidir(h, s, t, tau, inout_best, stream=None):
    _check(_lib.cbfs_query_bidir(h, _ptr(s), _ptr(t), len(s), tau, _ptr(inout_best), _stream(stream)))


def cbfs_pll_build(g, sources, sizes, n_clusters, d, first=200, bmax=1000, cap=256, stream=None):
    h = _vp()
    _check(_lib.cbfs_pll_build(g, _ptr(sources), _ptr(sizes), n_clusters, d, first, bmax, cap, ctypes.byref(h),
                               _stream(stream)))
    return h


def cbfs_pll_info(ph):
    tot, mx, roots, nb = _u64(), _u32(), _u32(), _u32()
    m1, m2 = ctypes.c_float(), ctypes.c_float()
    _check(_lib.cbfs_pll_info(ph, ctypes.byref(tot), ctypes.byref(mx), ctypes.byref(roots), ctypes.byref(nb),
                              ctypes.byref(m1), ctypes.byref(m2)))
    return dict(total_labels=tot.value, max_labels=mx.value, roots=roots.value, batches=nb.value,
                ms_cbfs=m1.value, ms_pbfs=m2.value)


def cbfs_pll_export(ph, counts, entries, stream=None):
    _check(_lib.cbfs_pll_export(ph, _ptr(counts), _ptr(entries), _stream(stream)))


def cbfs_pll_query(ph, s, t, out, stream=None):
    _check(_lib.cbfs_pll_query(ph, _ptr(s), _ptr(t), len(s), _ptr(out), _stream(stream)))


def cbfs_pll_destroy(ph):
    _check(_lib.cbfs_pll_destroy(ph))


def cbfs_labels_build(g, sources, sizes, n_clusters, d, dist_bytes=2, stream=None, word_bits=64):
    h = _vp()
    if word_bits == 64:
        _check(_lib.cbfs_labels_build(g, _ptr(sources), _ptr(sizes), n_clusters, d, dist_bytes, ctypes.byref(h),
                                      _stream(stream)))
    else:
        _check(_lib.cbfs_labels_build_w(g, _ptr(sources), _ptr(sizes), n_clusters, d, dist_bytes, word_bits,
                                        ctypes.byref(h), _stream(stream)))
    return h


def cbfs_labels_info(lh):
    n, C, d, db, b, w = _u32(), _u32(), _u32(), _u32(), _u64(), _u32()
    _check(_lib.cbfs_labels_info(lh, ctypes.byref(n), ctypes.byref(C), ctypes.byref(d), ctypes.byref(db),
                                 ctypes.byref(b)))
    _check(_lib.cbfs_labels_word_bits(lh, ctypes.byref(w)))
    return dict(n=n.value, clusters=C.value, d=d.value, dist_bytes=db.value, image_bytes=b.value,
                word_bits=w.value)


def cbfs_labels_export(lh, buf):
    nbytes = buf.nbytes if isinstance(buf, np.ndarray) else buf.numel() * buf.element_size()
    _check(_lib.cbfs_labels_export(lh, _ptr(buf), nbytes))


def cbfs_labels_import(g, buf):
    h = _vp()
    nbytes = buf.nbytes if isinstance(buf, np.ndarray) else buf.numel() * buf.element_size()
    _check(_lib.cbfs_labels_import(g, _ptr(buf), nbytes, ctypes.byref(h)))
    return h


def cbfs_labels_query(lh, s, t, inout_best, stream=None):
    _check(_lib.cbfs_labels_query(lh, _ptr(s), _ptr(t), len(s), _ptr(inout_best), _stream(stream)))


def cbfs_labels_destroy(lh):
    _check(_lib.cbfs_labels_destroy(lh))


def cbfs_record_bytes(word_bits: int, d: int, dist_bytes: int = 1) -> int:
    out = _u64()
    _check(_lib.cbfs_record_bytes(word_bits, d, dist_bytes, ctypes.byref(out)))
    return out.value


def cbfs_budget_clusters(t_bytes: int, word_bits: int, d: int, dist_bytes: int = 1) -> int:
    out = _u64()
    _check(_lib.cbfs_budget_clusters(t_bytes, word_bits, d, dist_bytes, ctypes.byref(out)))
    return out.value


def cbfs_set_direction_alpha(alpha: float):
    _check(_lib.cbfs_set_direction_alpha(alpha))


def cbfs_release_workspace(device: int = 0):
    _check(_lib.cbfs_release_workspace(device))


def cbfs_set_pull_hub_rows(rows: int):
    _check(_lib.cbfs_set_pull_hub_rows(rows))


def cbfs_set_sparse_order(min_entries: int):
    _check(_lib.cbfs_set_sparse_order(min_entries))


def cbfs_set_concurrency(batches: int):
    _check(_lib.cbfs_set_concurrency(batches))


def cbfs_set_engine(engine: int):
    _check(_lib.cbfs_set_engine(engine))


def cbfs_profile_enable(on: bool = True):
    _check(_lib.cbfs_profile_enable(int(on)))


def cbfs_profile_read(reset: bool = False) -> dict:
    ms = np.zeros(5, np.float64)
    la, arcs, ent, ui, uo = (np.zeros(5, np.uint64) for _ in range(5))
    _check(_lib.cbfs_profile_read(_ptr(ms), _ptr(la), _ptr(arcs), _ptr(ent), _ptr(ui), _ptr(uo), int(reset)))
    return {name: dict(ms=float(ms[i]), launches=int(la[i]), arcs=int(arcs[i]), entries=int(ent[i]),
                       u_in=int(ui[i]), u_out=int(uo[i]))
            for i, name in enumerate(("fold", "push", "pull", "sparse", "consume"))}


def cbfs_graph_nonisolated(h) -> int:
    c = _u32()
    _check(_lib.cbfs_graph_nonisolated(h, ctypes.byref(c)))
    return c.value


def cbfs_launch_count(reset: bool = False) -> int:
    return int(_lib.cbfs_launch_count(int(reset)))


def cbfs_version() -> str:
    return _lib.cbfs_version().decode()


# ------------------------------------------------------------------ convenience wrapper
class Graph:
    """Owning wrapper of a cbfs_graph handle."""

    def __init__(self, handle, device=0):
        self.h = handle
        self.device = device
        self.n, self.m, self.max_degree = cbfs_graph_info(handle)

    @staticmethod
    def relabel_flags(relabel) -> int:
        """False / None -> 0; True / "degree" -> CBFS_RELABEL_DEGREE; "locality" -> CBFS_RELABEL_LOCALITY."""
        if relabel in (False, None, "none"):
            return 0
        if relabel in (True, "degree"):
            return CBFS_RELABEL_DEGREE
        if relabel == "locality":
            return CBFS_RELABEL_LOCALITY
        raise ValueError(f"unknown relabel {relabel!r}")

    @classmethod
    def from_edges(cls, n, src, dst, relabel=False, device=0, stream=None):
        return cls(cbfs_graph_create(n, src, dst, cls.relabel_flags(relabel), device, stream), device)

    @classmethod
    def from_csr(cls, n, offsets, cols, relabel=False, device=0, stream=None):
        return cls(cbfs_graph_create_csr(n, offsets, cols, cls.relabel_flags(relabel), device, stream), device)

    def export_csr(self):
        return cbfs_graph_export_csr(self.h)

    def select_clusters(self, r, k, d, root_policy=CBFS_ROOT_DEGREE, seed=0):
        import torch
        src = torch.empty((max(r, 1), 64), dtype=torch.int32, device=f"cuda:{self.device}")
        sz = torch.empty(max(r, 1), dtype=torch.uint8, device=f"cuda:{self.device}")
        got = cbfs_select_clusters(self.h, r, k, d, root_policy, seed, src, sz)
        return src[:got], sz[:got]

    def run(self, sources, sizes, d, dist_bytes=2, planes=None, want_dist=True, want_masks=True, want_stats=True,
            direction=CBFS_DIR_AUTO):
        """Device outputs: dist [n][C] (uint8/int16 bits), masks [planes][n][C] (int64 bits), stats [C][4]."""
        import torch
        C = int(sizes.shape[0])
        planes = d + 1 if planes is None else planes
        dev = f"cuda:{self.device}"
        dist = torch.empty((self.n, C), dtype=torch.uint8 if dist_bytes == 1 else torch.int16, device=dev) \
            if want_dist else None
        masks = torch.empty((planes, self.n, C), dtype=torch.int64, device=dev) if want_masks else None
        stats = torch.zeros((C, 4), dtype=torch.int64, device=dev) if want_stats else None
        cbfs_run(self.h, sources, sizes, C, d, dist_bytes, dist, masks, planes, stats, direction)
        return dist, masks, stats

    def close(self):
        if self.h:
            cbfs_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
