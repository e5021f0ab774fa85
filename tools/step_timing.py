"""Quick experiment: time bench steps with/without the library's kernel profiling."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb

cfg = ci.CONFIGS["c2_rmat20"]
el = ci.make_graph("c2_rmat20")
dev = torch.device("cuda:0")
src = torch.from_numpy(el.src.view(np.int32)).to(dev); dst = torch.from_numpy(el.dst.view(np.int32)).to(dev)
n, C, d = el.n, cfg["clusters"], cfg["d"]
dist = torch.empty((n, C), dtype=torch.uint8, device=dev)
masks = torch.empty((d + 1, n, C), dtype=torch.int64, device=dev)
stats = torch.zeros((C, 4), dtype=torch.int64, device=dev)
ss = torch.empty((C, 64), dtype=torch.int32, device=dev); sz = torch.empty((C,), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()

def step(parts):
    t = {}
    t0 = time.perf_counter()
    h = cb.cbfs_graph_create(n, src, dst, cb.CBFS_RELABEL_DEGREE, 0, st)
    torch.cuda.synchronize(); t["build"] = time.perf_counter() - t0; t0 = time.perf_counter()
    cb.cbfs_select_clusters(h, C, 64, d, 0, 0, ss, sz, st)
    torch.cuda.synchronize(); t["select"] = time.perf_counter() - t0; t0 = time.perf_counter()
    cb.cbfs_run(h, ss, sz, C, d, 1, dist, masks, d + 1, stats, int(os.environ.get("DIR", "0")), st)
    torch.cuda.synchronize(); t["run"] = time.perf_counter() - t0; t0 = time.perf_counter()
    cb.cbfs_graph_destroy(h)
    torch.cuda.synchronize(); t["destroy"] = time.perf_counter() - t0
    return t

if os.environ.get("ALPHA"): cb.cbfs_set_direction_alpha(float(os.environ["ALPHA"]))
if os.environ.get("CONC"): cb.cbfs_set_concurrency(int(os.environ["CONC"]))
for it in range(3):
    step(None)
for prof in (False, True, False):
    cb.cbfs_profile_enable(prof); cb.cbfs_profile_read(reset=True)
    ts = [step(None) for _ in range(3)]
    print("prof" if prof else "noprof", {k: round(1000 * np.mean([t[k] for t in ts]), 2) for k in ts[0]},
          {k: round(v["ms"] / 3, 2) for k, v in cb.cbfs_profile_read().items()})
