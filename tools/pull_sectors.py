"""Pull-round statistics of a -DCBFS_PULL_STATS build (tools/build_variant.sh
stats "-DCBFS_PULL_STATS"; CBFS_LIB_PATH=build_var/stats/libcbfs.so): per
round i, the S_seen rows the dense pull gathered, their non-zero 64-bit
words (clusters) and their set bits (sources), for the hub rows (the first
64 MiB of rows, evict_last) and the others.

    python tools/pull_sectors.py CONFIG [CLUSTERS] [FIRST]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import paper_2410_17226_b200 as cb  # noqa: E402

name = sys.argv[1]
C = int(sys.argv[2]) if len(sys.argv) > 2 else 64
F0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = ci.CONFIGS[name]
el = ci.make_graph(name)
src_d = torch.from_numpy(el.src.view(np.int32)).cuda()
dst_d = torch.from_numpy(el.dst.view(np.int32)).cuda()
g = cb.Graph(cb.cbfs_graph_create(el.n, src_d, dst_d, cb.Graph.relabel_flags(cfg.get("relabel", "none")), 0), 0)
del src_d, dst_d
src, sz = g.select_clusters(F0 + C, cfg["k"], cfg["d"])
src, sz = src[F0:].contiguous(), sz[F0:].contiguous()
cb._lib.cbfs_debug_read.argtypes = [ctypes.c_void_p]
buf = np.zeros(32, np.uint64)
cb._lib.cbfs_debug_read(buf.ctypes.data)
stats = torch.zeros((len(sz), 4), dtype=torch.int64, device="cuda")
cb.cbfs_run(g.h, src, sz, len(sz), cfg["d"], 2, None, None, cfg["d"] + 1, stats)
torch.cuda.synchronize()
cb._lib.cbfs_debug_read(buf.ctypes.data)
out = {}
for i in range(4):
    hr, hw, hb, orow, ow, ob = (int(x) for x in buf[8 * i:8 * i + 6])
    if hr + orow:
        out[i] = {"hub_rows": hr, "hub_words_per_row": hw / max(hr, 1), "hub_bits_per_row": hb / max(hr, 1),
                  "other_rows": orow, "other_words_per_row": ow / max(orow, 1),
                  "other_bits_per_row": ob / max(orow, 1)}
print(json.dumps({"config": name, "clusters": len(sz), "first": F0, "rounds": out}))
