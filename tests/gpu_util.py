"""Helpers shared by the GPU parity tests (marshalling only)."""
import numpy as np
import torch

import paper_2410_17226_b200 as cb


def dev():
    return torch.device("cuda:0")


def to_dev_u32(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(dev())


def to_dev_u8(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).to(dev())


def np_u16(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def np_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def np_u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def gpu_graph(el, relabel=False):
    return cb.Graph.from_edges(el.n, np.ascontiguousarray(el.src), np.ascontiguousarray(el.dst), relabel=relabel)


def run_clusters(g: cb.Graph, sources: np.ndarray, sizes: np.ndarray, d: int, dist_bytes=2, planes=None,
                 direction=cb.CBFS_DIR_AUTO):
    """Returns host arrays in the oracle's cluster-major layout:
    dist [C][n] uint16 (u8 widened, 0xFF -> 0xFFFF), sub [C][planes][n] uint64, stats [C][4]."""
    src_d = to_dev_u32(sources)
    sz_d = to_dev_u8(sizes)
    dist, masks, stats = g.run(src_d, sz_d, d, dist_bytes=dist_bytes, planes=planes, direction=direction)
    torch.cuda.synchronize()
    if dist_bytes == 1:
        dh = dist.cpu().numpy().astype(np.uint16)
        dh[dh == 0xFF] = 0xFFFF
    else:
        dh = np_u16(dist)
    return np.ascontiguousarray(dh.T), np.ascontiguousarray(np_u64(masks).transpose(2, 0, 1)), \
        stats.cpu().numpy().view(np.uint64)
