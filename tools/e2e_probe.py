"""Time the pieces of bench.py's end-to-end C2 step (host buffers)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import cbfs_inputs as ci
import paper_2410_17226_b200 as cb
el = ci.make_graph("c2_rmat20"); n = el.n; C = 1024; d = 2
src_h = torch.from_numpy(el.src.view(np.int32)).pin_memory(); dst_h = torch.from_numpy(el.dst.view(np.int32)).pin_memory()
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
sel_src = torch.empty((C, 64), dtype=torch.int32, device=dev); sel_sz = torch.empty((C,), dtype=torch.uint8, device=dev)
hd = torch.empty((n, C), dtype=torch.uint8).pin_memory(); hm = torch.empty((d + 1, n, C), dtype=torch.int64).pin_memory()
hs = torch.zeros((C, 4), dtype=torch.int64).pin_memory(); hsrc = torch.empty((C, 64), dtype=torch.int32).pin_memory()
hsz = torch.empty((C,), dtype=torch.uint8).pin_memory()
for it in range(3):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    h = cb.cbfs_graph_create(n, src_h, dst_h, cb.CBFS_RELABEL_DEGREE, 0, st); torch.cuda.synchronize(); t.append(time.perf_counter())
    cb.cbfs_select_clusters(h, C, 64, d, 0, 0, sel_src, sel_sz, st); hsrc.copy_(sel_src); hsz.copy_(sel_sz); t.append(time.perf_counter())
    cb._check(cb._lib.cbfs_run_host(h, ctypes.c_void_p(hsrc.data_ptr()), ctypes.c_void_p(hsz.data_ptr()), C, d, 1,
                                    ctypes.c_void_p(hd.data_ptr()), ctypes.c_void_p(hm.data_ptr()), d + 1,
                                    ctypes.c_void_p(hs.data_ptr()), 0, ctypes.c_void_p(st.cuda_stream)))
    t.append(time.perf_counter())
    cb.cbfs_graph_destroy(h); torch.cuda.synchronize(); t.append(time.perf_counter())
    print("build %.1f select %.1f run_host %.1f destroy %.1f ms" % tuple(1000 * (t[i + 1] - t[i]) for i in range(4)),
          "free GB", torch.cuda.mem_get_info()[0] / 1e9, flush=True)
