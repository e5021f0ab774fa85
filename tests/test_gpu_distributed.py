"""A12 on the GPU: the sharded label build + NCCL all-gather and
the streaming query + NCCL MIN all-reduce, through the C-ABI kernels, in a
world-size-1 NCCL group (one GPU per run box; the world-size-2 host logic is
covered with gloo in test_dist_cpu.py).  Bit-exact against the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import cbfs_inputs as ci  # noqa: E402
import oracle as orc  # noqa: E402
from gpu_util import gpu_graph, to_dev_u32, to_dev_u8  # noqa: E402
from paper_2410_17226_b200 import distributed as pd  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    yield None
    dist.destroy_process_group()


@pytest.mark.parametrize("d,dist_bytes", [(2, 1), (4, 2)])
def test_label_gather_and_query(nccl_group, d, dist_bytes):
    el = ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=41) if d == 2 else ci.grid(60, 0.05, 0.01, 41)
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 90, 64, d)
    g = gpu_graph(el, relabel=(d == 2))
    dist_t, masks, szp = pd.build_label_shard(g, to_dev_u32(src), to_dev_u8(sz), d, dist_bytes)
    assert masks.shape[0] == d  # label records keep S_v[0..d-1] (R14)
    stores = pd.gather_labels(dist_t, masks, szp)
    assert len(stores) == 1
    s, t = ci.query_pairs(g.n, 30000, seed=9)
    best = pd.query_gathered(stores, d, to_dev_u32(s), to_dev_u32(t), dist_bytes)
    expect = orc.query_stream(ref, src, sz, d, s, t)
    assert np.array_equal(best.cpu().numpy(), expect)
    g.close()


def test_query_stream_sharded(nccl_group):
    el = ci.grid(70, 0.05, 0.01, 43)
    ref = orc.csr_from_edgelist(el)
    d = 6
    src, sz = orc.select_clusters(ref, 75, 64, d)
    g = gpu_graph(el)
    s, t = ci.query_pairs(g.n, 20000, seed=10)
    best = pd.query_stream_sharded(g, to_dev_u32(src), to_dev_u8(sz), d, to_dev_u32(s), to_dev_u32(t))
    expect = orc.query_stream(ref, src, sz, d, s, t)
    assert np.array_equal(best.cpu().numpy(), expect)
    g.close()


@pytest.mark.parametrize("d,dist_bytes,w", [(2, 1, 64), (0, 2, 64), (6, 2, 64), (2, 1, 8), (4, 2, 16), (0, 1, 0)])
def test_label_images_gather_and_query(nccl_group, d, dist_bytes, w):
    """cbfs_labels_build_w -> export -> NCCL all_gather -> import -> query ==
    the oracle, for stores of word size w (0 = plain landmarks); host-buffer
    export/import round trip; bad images rejected."""
    import paper_2410_17226_b200 as cb
    el = ci.rmat(12, 8, 0.57, 0.19, 0.19, seed=44) if d <= 2 else ci.grid(50, 0.05, 0.01, 44)
    ref = orc.csr_from_edgelist(el)
    src, sz = orc.select_clusters(ref, 70, max(w, 1) if w < 64 else 64, max(d, 1) if d else 2)
    if d == 0:  # d = 0 labels: single-source clusters (plain BFS landmarks)
        src = src.copy(); src[:, 1:] = orc.PAD; sz = np.ones_like(sz)
    g = gpu_graph(el, relabel=(d == 2))
    h = pd.build_local_labels(g, to_dev_u32(src), to_dev_u8(sz), d, dist_bytes, word_bits=w)
    info = cb.cbfs_labels_info(h)
    assert info["clusters"] == len(sz) and info["d"] == d and info["n"] == g.n and info["word_bits"] == w
    handles = pd.gather_label_images(g, h)
    s, t = ci.query_pairs(g.n, 20000, seed=12)
    best = pd.query_label_handles(handles, to_dev_u32(s), to_dev_u32(t))
    expect = orc.query_stream(ref, src, sz, d, s, t)
    assert np.array_equal(best.cpu().numpy(), expect)
    by_index = pd.query_index_sharded(lambda a, b: pd.query_label_handles(handles, a, b), to_dev_u32(s), to_dev_u32(t))
    assert np.array_equal(by_index.cpu().numpy(), expect)
    img = np.zeros(info["image_bytes"], np.uint8)  # host round trip
    cb.cbfs_labels_export(h, img)
    h2 = cb.cbfs_labels_import(g.h, img)
    best2 = torch.full((len(s),), cb.CBFS_QUERY_UNREACHED, dtype=torch.int32, device="cuda:0")
    cb.cbfs_labels_query(h2, to_dev_u32(s), to_dev_u32(t), best2)
    assert np.array_equal(best2.cpu().numpy(), expect)
    bad = img.copy(); bad[0] ^= 0xFF
    with pytest.raises(cb.CbfsError):
        cb.cbfs_labels_import(g.h, bad)
    with pytest.raises(cb.CbfsError):
        cb.cbfs_labels_export(h, np.zeros(16, np.uint8))
    for x in handles + [h, h2]:
        cb.cbfs_labels_destroy(x)
    g.close()
