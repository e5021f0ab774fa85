"""Debug-build counters of the pull kernel per launch (build_var/dbg with -DCBFS_PULL_STATS)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
cfg = ci.CONFIGS["c2_rmat20"]; el = ci.make_graph("c2_rmat20")
dev = torch.device("cuda:0")
n, C, d = el.n, 64, 2
g = cb.Graph.from_edges(n, el.src, el.dst, relabel=True)
ss, sz = g.select_clusters(C, 64, d)
out = (ctypes.c_ulonglong * 8)()
cb._lib.cbfs_debug_read(out)
cb.cbfs_profile_enable(True); cb.cbfs_profile_read(reset=True)
g.run(ss, sz, d, dist_bytes=1)
cb._lib.cbfs_debug_read(out)
print("groups %d active_vertices %d list_entries %d group_arcs %d early_exits %d skipped_entries %d" % tuple(out[:6]))
print(cb.cbfs_profile_read())
