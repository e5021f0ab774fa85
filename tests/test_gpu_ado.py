"""NEXT-3: the landmark-label ADO's distortion computed through
the C-ABI (paper_2410_17226_b200/ado.py) equals the oracle's on the same
pairs: exact distances (single-source C-BFS vs textbook BFS), answers (GPU
query vs oracle query), epsilon; and the one-sided error holds."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
from gpu_util import gpu_graph  # noqa: E402
from paper_2410_17226_b200 import ado  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,d", [("rmat", 2), ("grid", 4)])
def test_distortion_matches_oracle(kind, d):
    el = ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=21) if kind == "rmat" else ci.grid(60, 0.05, 0.01, 21)
    ref = orc.csr_from_edgelist(el)
    g = gpu_graph(el, relabel=(kind == "rmat"))
    r = 1024 // (1 + d * 8)
    idx = ado.LandmarkIndex(g, r, 64, d)
    osrc, osz = orc.select_clusters(ref, r, 64, d)
    assert idx.r == len(osz)
    sc, tc = ci.query_pairs(el.n, 4000, seed=3, stream=5)
    s, t, dd = ado.sample_pairs(sc, tc, 3000, lambda a, b: ado.exact_distances(g, a, b))
    # exact distances against the textbook BFS
    for src in np.unique(s)[:40]:
        ref_d = orc.plain_bfs(ref, int(src))
        sel = s == src
        assert np.array_equal(dd[sel], ref_d[t[sel]])
    # the sample is the first 3000 distinct, mutually reachable candidates
    keep = sc != tc
    reach = np.array([orc.plain_bfs(ref, int(a))[b] != orc.INF32 for a, b in zip(sc[keep], tc[keep])])
    assert len(s) == min(3000, int(reach.sum())) and len(s) > 0
    assert np.array_equal(s, sc[keep][reach][:len(s)]) and np.array_equal(t, tc[keep][reach][:len(s)])
    ans = idx.query(torch.from_numpy(s.view(np.int32)).cuda(), torch.from_numpy(t.view(np.int32)).cuda()).cpu().numpy()
    expect = orc.query_stream(ref, osrc, osz, d, s, t)
    assert np.array_equal(ans, expect)
    res = ado.distortion(ans, dd)
    assert res["one_sided"] and res["covered"] > 0 and res["epsilon_pct"] >= 0.0
    psi = expect[expect < orc.INT32_MAX] / dd[expect < orc.INT32_MAX].astype(np.float64)
    assert res["epsilon_pct"] == pytest.approx(100.0 * (psi.mean() - 1.0), abs=0, rel=1e-12)
    g.close()
