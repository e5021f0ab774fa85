"""Check the GPU locality order (CBFS_RELABEL_LOCALITY) of a config's graph against a
vectorised numpy statement of its definition (include/cbfs.h), and time the build.

    python tools/locality_check.py [CONFIG]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_knn"
el = ci.make_graph(name)
n = el.n
src_d = torch.from_numpy(el.src.view(np.int32)).cuda()
dst_d = torch.from_numpy(el.dst.view(np.int32)).cuda()
st = torch.cuda.current_stream()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = cb.cbfs_graph_create(n, src_d, dst_d, cb.CBFS_RELABEL_LOCALITY, 0, st)
    torch.cuda.synchronize()
    print(f"{name}: build with the locality order {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    if rep == 0:
        cb.cbfs_graph_destroy(h)
perm = cb.cbfs_graph_internal_order(h)
off, cols = cb.cbfs_graph_export_csr(h)
off = off.astype(np.int64)
t0 = time.perf_counter()
deg = np.diff(off)
root = int(np.lexsort((np.arange(n), -deg))[0])
pos = np.full(n, -1, np.int64)
order = np.empty(n, np.int64)
order[0] = root
pos[root] = 0
lo, hi, levels = 0, 1, 0
while hi > lo:
    par = order[lo:hi]
    d = deg[par]
    pp = np.repeat(np.arange(lo, hi), d)  # parent position per arc
    starts = off[par]
    idx = np.repeat(starts - np.concatenate(([0], np.cumsum(d)[:-1])), d) + np.arange(d.sum())
    v = cols[idx].astype(np.int64)
    m = pos[v] < 0
    v, pp = v[m], pp[m]
    key = np.full(n, np.iinfo(np.int64).max, np.int64)
    np.minimum.at(key, v, pp)
    ch = np.unique(v)
    ch = ch[np.lexsort((ch, key[ch]))]
    order[hi:hi + len(ch)] = ch
    pos[ch] = np.arange(hi, hi + len(ch))
    lo, hi = hi, hi + len(ch)
    levels += 1
rest = np.flatnonzero(pos < 0)
order[hi:] = rest
print(f"numpy reference: {levels} levels, {hi} reached, {len(rest)} appended, {time.perf_counter() - t0:.1f} s")
print("order equal:", bool(np.array_equal(order.astype(np.uint32), perm)))
