"""Multi-process (world_size 2, gloo, CPU) checks of bench.py's N > 1 host
logic: weak-scaling shard layout, timing max / unit sum reductions, and the
reference arm under torchrun (rank 0 alone prints one JSON line)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx = bench.allreduce_max(float(10 + rank), world)
    sm = bench.allreduce_sum(float(1 + rank), world)
    total, first, mine = bench.shard(1024, world, rank)
    wtotal, wfirst, wmine = bench.shard(1024, world, rank, strong=False)
    bench.barrier(world)
    out.put((rank, mx, sm, total, first, mine, wtotal, wmine))
    dist.destroy_process_group()


def test_gloo_reductions_and_shards():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # round-robin: rank 1 owns clusters 1, 3, 5, ... of the config's 1,024 (strong) or of 2,048 (weak)
    assert res[0][1:] == (11.0, 3.0, 1024, 0, 512, 2048, 1024)
    assert res[1][1:] == (11.0, 3.0, 1024, 1, 512, 2048, 1024)


def test_reference_arm_under_torchrun():
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
           "2", "--steps", "1", "--warmup", "0", "--config", "c1_er", "--ref-sample", "4"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["unit"] == "source-edges/s" and j["value"] > 0
    assert j["cpu_baseline"]["kind"] == "oracle" and j["e2e"]["h2d_bytes_per_step"] == 0


# ---------------------------------------------------------------- A12
def _a12_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist

    import cbfs_inputs as ci
    import oracle as orc
    from paper_2410_17226_b200 import distributed as pd
    dist.init_process_group("gloo", rank=rank, world_size=world)
    el = ci.erdos_renyi(400, 900, seed=11)
    g = orc.csr_from_edgelist(el)
    d = 2
    src, sz = orc.select_clusters(g, 11, 64, d, orc.ROOT_DEGREE, 0)  # 11 clusters: ragged over 2 ranks
    C = len(sz)
    s, t = ci.query_pairs(g.n, 500, seed=5)
    # the rank's clusters (round-robin) -> its partial answers -> MIN all-reduce
    idx = pd.cluster_shard(C, world, rank).numpy()
    part = orc.query_stream(g, src[idx], sz[idx], d, s, t, threads=1) if len(idx) else \
        np.full(len(s), orc.INT32_MAX, np.int32)
    best = pd.min_reduce_answers(torch.from_numpy(part.copy()))
    # label shards padded to shard_width columns with unreachable clusters, all-gathered
    W = pd.shard_width(C, world)
    r = orc.cluster_bfs_many(g, src[idx], sz[idx], d, threads=1)
    dist_sh = np.full((W, g.n), 0xFFFF, np.uint16)
    sub_sh = np.zeros((W, d + 1, g.n), np.uint64)
    dist_sh[:len(idx)] = r["dist"]
    sub_sh[:len(idx)] = r["sub"]
    parts = pd.all_gather_shards([torch.from_numpy(dist_sh.view(np.int16)), torch.from_numpy(sub_sh.view(np.int64))])
    merged = np.full(len(s), orc.INT32_MAX, np.int32)
    for dp, mp_ in zip(*parts):
        merged = np.minimum(merged, orc.query(dp.numpy().view(np.uint16), mp_.numpy().view(np.uint64), s, t))
    full = orc.query_stream(g, src, sz, d, s, t, threads=1)

    def answer(sb, tb):  # every gathered shard, min-merged, for one block of queries
        a = np.full(len(sb), orc.INT32_MAX, np.int32)
        for dp, mp_ in zip(*parts):
            a = np.minimum(a, orc.query(dp.numpy().view(np.uint16), mp_.numpy().view(np.uint64), sb.numpy(),
                                        tb.numpy()))
        return torch.from_numpy(a)
    # queries sharded by index after the gather, answers all-gathered (501 = ragged over 2 ranks)
    s2, t2 = ci.query_pairs(g.n, 501, seed=6)
    by_index = pd.query_index_sharded(answer, torch.from_numpy(s2.astype(np.int64)),
                                      torch.from_numpy(t2.astype(np.int64)))
    ok_index = bool(np.array_equal(by_index.numpy(), orc.query_stream(g, src, sz, d, s2, t2, threads=1)))
    lo, hi, per = pd.query_block(501, world, rank)
    out.put((rank, idx.tolist(), bool(np.array_equal(best.numpy(), full)), bool(np.array_equal(merged, full)),
             int((full < orc.INT32_MAX).sum()), ok_index, (lo, hi, per)))
    dist.destroy_process_group()


def test_a12_shard_min_reduce_and_label_gather_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_a12_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == [0, 2, 4, 6, 8, 10] and res[1][1] == [1, 3, 5, 7, 9]
    assert res[0][6] == (0, 251, 251) and res[1][6] == (251, 501, 251)
    for _, _, ok_min, ok_gather, reached, ok_index, _ in res:
        assert ok_min and ok_gather and reached > 0 and ok_index


def test_cluster_shard_partition():
    from paper_2410_17226_b200 import distributed as pd
    for C in (0, 1, 7, 64, 1024, 1031):
        for R in (1, 2, 3, 8):
            parts = [pd.cluster_shard(C, R, r).tolist() for r in range(R)]
            assert sorted(sum(parts, [])) == list(range(C))
            assert max((len(p) for p in parts), default=0) <= pd.shard_width(C, R)
