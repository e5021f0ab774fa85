#!/usr/bin/env python3
"""bench.py — C-BFS source-edges/s on B200 (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3_rmat24]

Workload (N=1): BASELINE.json configs[2] — the largest configuration that
fits one GPU: RMAT scale 24, edge factor 32, a/b/c/d = .6/.15/.15/.1,
symmetrised (16.7M vertices, 1.01B arcs); 4,096 clusters of up to 64
sources (highest-degree root + its best neighbours, d = 2).
Every cluster's full distance vector (u8 Delta + 3 u64 bit-subset planes per
vertex) is written to HBM and consumed inside the step: 1.7 TB in total, so
each batch of 64 clusters writes its vectors into a staging store that a
digest kernel reads back and resets (cbfs_run_digest; the digests are what
the parity tests compare with the oracle).  Synthetic seeded input
(cbfs_inputs, seed 3).  Other configs: --config (c1/c2 write the whole
[n][C] store, c4 is consumed like c3, c5 runs the 10M-query streaming index).

One step = the whole hot path over the resident edge list: A0 CSR build
(symmetrise, dedup, relabel) -> A1 cluster selection -> A2-A9 C-BFS of
every cluster -> outputs written and consumed.  `value` = sum_c |S_c| * m_c
/ T, m_c = arcs whose tail is reachable from S_c, T = device time of the
C-BFS phase (A2-A11 incl. the output writes and their consumer) of the K
steps, CUDA events on the launching stream, max over ranks — SURVEY §8(d)'s
definition, which reports graph build and selection separately
(`config.phase_ms_rank0`; `config.value_incl_build_select` divides by the
whole step, which `ms_per_step` reports).

N>1 (torchrun, one rank per GPU, NCCL): strong scaling by default — the
config's clusters are split round-robin over the ranks (rank r owns
clusters r, r+N, ...), the graph is replicated, every rank
runs the deterministic selection; no data-path collective (clusters are
independent) except the MIN all-reduce of query answers in query
mode; the timing MAX and the unit totals are all-reduced.  `--scaling weak`
gives every rank C clusters of an N x C selection instead.

`--impl reference` times the CPU oracle (oracle/, sequential Alg. 1 per
cluster) on a bounded sample of the same workload: one cluster per step,
the steps spread over the host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import cbfs_inputs as ci  # noqa: E402

METRIC = "C-BFS source-edges/sec (GTEPS x sources)"
UNIT = "source-edges/s"
BYTES_PER_FRONTIER_ARC = 22     # 4 B column + 2 B Delta cap read + 16 B OR-update
BYTES_PER_FRONTIER_ENTRY = 40   # offsets, frontier id w/r, next read, seen RMW
BYTES_PER_ARC = 4                # batched pull: one u32 CSR column per arc per launch
BYTES_PER_VROW = 64 * 2 + 8      # batched pull: a vertex's Delta row (64 clusters) + its 64-bit "subset full" word
BYTES_PER_ROW = 64 * 8           # batched pull: one 64-cluster bit-subset row


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy peak)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 500):
        self.gpu = gpu_index
        self.period = period_ms
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ distributed plumbing
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def shard(n_clusters: int, world: int, rank: int, strong: bool = True):
    """Rank r owns clusters r, r + N, r + 2N, ... of the selection (SURVEY
    §8(e): round-robin balances the degree-ordered selection).  Strong scaling
    (default, SURVEY §8(e) "per-rank work is r/R clusters"): the config's
    selection is split over the N ranks; weak: an N x C selection, C per rank.
    Returns (selection size, rank's first cluster, rank's cluster count);
    the stride is N."""
    total = n_clusters if strong else n_clusters * world
    return total, rank, len(range(rank, total, world))


# ------------------------------------------------------------------ CPU oracle
_ORACLE = {}


def oracle_setup(cfg_name: str, el):
    """The oracle's own A0 (CSR) and A1 (selection) of the config, built once
    per process on the host (never from the CUDA path)."""
    if cfg_name not in _ORACLE:
        import oracle as orc
        cfg = ci.CONFIGS[cfg_name]
        t0 = time.perf_counter()
        g = orc.csr_from_edgelist(el)
        t_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        pol = orc.ROOT_RANDOM if cfg["root"] == "random" else orc.ROOT_DEGREE
        src, sz = orc.select_clusters(g, cfg["clusters"], cfg["k"], cfg["d"], pol, cfg["root_seed"])
        _ORACLE[cfg_name] = dict(g=g, src=src, sz=sz, build_s=t_build, select_s=time.perf_counter() - t0)
    return _ORACLE[cfg_name]


def oracle_steps(cfg_name: str, el, threads: int, steps: int, warmup: int):
    """The oracle as it stands on a bounded sample of the workload: one
    cluster per step (sequential Alg. 1), clusters evenly spaced
    over the selection, the warmup + steps steps spread over `threads` host
    threads (ctypes releases the GIL), each step timed on its own thread.
    Returns (value, per-step seconds of the timed steps, description)."""
    import oracle as orc
    cfg = ci.CONFIGS[cfg_name]
    O = oracle_setup(cfg_name, el)
    C = len(O["sz"])
    total = warmup + steps
    idx = np.linspace(0, C - 1, total).round().astype(int)
    res = [None] * total
    nxt = [0]
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                j = nxt[0]
                nxt[0] += 1
            if j >= total:
                return
            c = idx[j:j + 1]
            t0 = time.perf_counter()
            r = orc.cluster_bfs_many(O["g"], O["src"][c], O["sz"][c], cfg["d"], threads=1, want_outputs=False)
            dt = time.perf_counter() - t0
            res[j] = (float(O["sz"][c[0]]) * float(r["stats"][0, 3]), dt)

    T = max(1, min(threads, total))
    ths = [threading.Thread(target=worker) for _ in range(T)]
    t_wall = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    t_wall = time.perf_counter() - t_wall
    timed = res[warmup:]
    units = sum(u for u, _ in timed)
    secs = [s for _, s in timed]
    value = units / (sum(secs) / T) if secs else 0.0  # T threads each running one step at a time
    desc = (f"{steps} timed + {warmup} warm-up steps of one cluster each (clusters evenly spaced over the "
            f"{C}-cluster selection), sequential Alg. 1 per step, steps spread over {T} host threads "
            f"({t_wall:.1f}s wall); value = timed units / (sum of step times / {T}); the oracle's CSR build "
            f"({O['build_s']:.1f}s) and selection ({O['select_s']:.1f}s) run once, not in the rate")
    return value, secs, desc


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


# ------------------------------------------------------------------ reference arm
def run_reference(args, world, rank):
    if rank != 0:
        return
    cfg = ci.CONFIGS[args.config]
    el = ci.make_graph(args.config)
    cores, model = cpu_info()
    value, secs, desc = oracle_steps(args.config, el, cores, args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * float(np.mean(secs)) if secs else None,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": args.config, "graph": el.name, "n": el.n, "clusters": cfg["clusters"],
                       "k": cfg["k"], "d": cfg["d"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, args.steps + args.warmup),
                             "kind": "oracle", "sample": desc, "cpu": model},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
# How a config's outputs are consumed:
#   full   — every cluster's full distance vector (Delta + d+1 bit-subset
#            planes) is written to HBM-resident [n][C] output buffers (configs
#            1, 2);
#   digest — the whole store does not fit HBM (1.7 TB / 0.43 TB for configs 3
#            / 4): every batch writes its full vectors to an HBM staging store
#            that a digest kernel reads back and resets (cbfs_run_digest); the
#            per-cluster digests leave the library (stated in `config.outputs`);
#   query  — config 5: the labels of every batch are consumed by 10M distance
#            queries as soon as they are built (cbfs_query_stream, H3); with
#            N ranks the answers are MIN-all-reduced (NCCL, A12).
MODES = {"c1_er": "full", "c2_rmat20": "full", "c3_rmat24": "digest", "c4_grid": "digest", "c5_knn": "query"}
INT32_MAX = 2**31 - 1


def alg_bytes_model(prof, stats_np, n, m_h, n_ni, d, planes, dist_bytes, C, mode, queries):
    """Algorithmic HBM bytes of the step's C-BFS kernels in this design
    (the lower bound each kernel must move):
    batched pull, per launch: 4 B per CSR arc + 136 B per non-isolated vertex
    row (Delta row + "subset full" word) + 512 B per distinct frontier row
    read and per claimed row written; fold: 40 B per entry; push: 22 B per
    (cluster, arc) pair; sparse engine: SURVEY §8(d)'s
    22 B x sum_i E_i + 40 B x sum_i |F_i|; init: 10 B per (vertex, cluster)
    (S_seen + Delta); outputs: the full vectors written once; digest
    consumer: the staged vectors read once and reset once; query mode: 4 B
    per (query, cluster) Delta reads."""
    pull, fold, push, sp = prof["pull"], prof["fold"], prof["push"], prof["sparse"]
    parts = {}
    parts["pull"] = pull["launches"] * (BYTES_PER_ARC * m_h + BYTES_PER_VROW * n_ni) + \
        BYTES_PER_ROW * (pull["u_in"] + pull["u_out"])
    parts["fold"] = BYTES_PER_FRONTIER_ENTRY * fold["entries"]
    parts["push"] = BYTES_PER_FRONTIER_ARC * push["arcs"]
    if sp["launches"]:
        parts["sparse"] = BYTES_PER_FRONTIER_ARC * float(stats_np[:, 2].astype(np.float64).sum()) + \
            BYTES_PER_FRONTIER_ENTRY * float(stats_np[:, 1].astype(np.float64).sum())
    parts["init"] = 10.0 * n * C
    vec = float(n) * C * (dist_bytes + 8 * planes)
    if mode in ("full", "digest"):
        parts["outputs"] = vec
    if mode == "digest":
        parts["consume"] = 2.0 * vec
    if mode == "query":
        parts["queries"] = 4.0 * queries * C
    return parts


def sec8d_bytes(stats_np, n, d):
    """SURVEY §8(d)'s per-cluster byte model, summed over the step's clusters:
    22 B x sum_i E_i + 40 B x sum_i |F_i| + n (20 + 8 (d+1))."""
    st = stats_np.astype(np.float64)
    return float(22.0 * st[:, 2].sum() + 40.0 * st[:, 1].sum() + len(st) * n * (20.0 + 8.0 * (d + 1)))


def golden_check(cfg_name, digests, stats_np, first, world):
    """The step's digests and round statistics against tests/golden (oracle-
    generated, tests/make_goldens.py), when the golden file exists."""
    path = os.path.join(ROOT, "tests", "golden", f"{cfg_name}.golden.txt")
    if not os.path.exists(path) or digests is None:
        return None
    ok = True
    checked = 0
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        f = [int(x) for x in line.split()[:6]]
        c = f[0]
        if c % world != first:
            continue
        j = c // world
        if j >= len(digests):
            continue
        checked += 1
        ok &= int(digests[j]) == f[5] and [int(x) for x in stats_np[j]] == f[1:5]
    return {"golden": os.path.relpath(path, ROOT), "clusters_checked": checked, "match": bool(ok)}


def run_ours(args, world, rank, local):
    import torch

    import paper_2410_17226_b200 as cb
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    cfg = ci.CONFIGS[args.config]
    mode = args.mode or MODES[args.config]
    d, k = cfg["d"], cfg["k"]
    C_cfg = args.clusters or cfg["clusters"]
    strong = args.scaling == "strong"
    r_total, first, C = shard(C_cfg, world, rank, strong)  # C = this rank's clusters
    policy = cb.CBFS_ROOT_RANDOM if cfg["root"] == "random" else cb.CBFS_ROOT_DEGREE
    relabel = args.relabel or cfg.get("relabel", "none")
    rflags = cb.Graph.relabel_flags(relabel)
    dist_bytes = 1 if cfg["kind"] in ("rmat", "er") else 2
    planes = d + 1

    t0 = time.perf_counter()
    el = ci.make_graph(args.config)
    log(f"[rank {rank}] generated {el.name}: n={el.n} pairs={len(el.src)} in {time.perf_counter() - t0:.1f}s")
    src_h = torch.from_numpy(el.src.view(np.int32)).pin_memory()
    dst_h = torch.from_numpy(el.dst.view(np.int32)).pin_memory()
    src_d, dst_d = src_h.to(dev), dst_h.to(dev)
    n = el.n
    Q = 0
    dist_out = masks_out = best = qs_d = qt_d = digest = None
    if mode == "full":
        dist_out = torch.empty((n, C), dtype=torch.uint8 if dist_bytes == 1 else torch.int16, device=dev)
        masks_out = torch.empty((planes, n, C), dtype=torch.int64, device=dev)
    if mode == "digest":
        digest = torch.zeros((C,), dtype=torch.int64, device=dev)
    if mode == "query":
        Q = args.queries or cfg.get("queries", 0)
        qs, qt = ci.query_pairs(n, Q, cfg.get("query_seed", 7))
        qs_h = torch.from_numpy(qs.view(np.int32)).pin_memory()
        qt_h = torch.from_numpy(qt.view(np.int32)).pin_memory()
        qs_d, qt_d = qs_h.to(dev), qt_h.to(dev)
        best = torch.empty((Q,), dtype=torch.int32, device=dev)
    stats = torch.zeros((C, 4), dtype=torch.int64, device=dev)
    sel_src = torch.empty((r_total, 64), dtype=torch.int32, device=dev)
    sel_sz = torch.empty((r_total,), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream()
    if args.alpha:
        cb.cbfs_set_direction_alpha(args.alpha)
    if args.concurrency:
        cb.cbfs_set_concurrency(args.concurrency)
    if args.engine:
        cb.cbfs_set_engine(args.engine)
    overlap = mode == "full" and args.overlap_select

    phase_ms = {"build": 0.0, "select": 0.0, "cbfs": 0.0}

    def traverse(h):
        blk_src = sel_src[first::world].contiguous()  # this rank's clusters (round-robin)
        blk_sz = sel_sz[first::world].contiguous()
        if mode == "full":
            cb.cbfs_run(h, blk_src, blk_sz, C, d, dist_bytes, dist_out, masks_out, planes, stats, args.direction,
                        stream)
        elif mode == "digest":
            cb.cbfs_run_digest(h, blk_src, blk_sz, C, d, dist_bytes, planes, digest, stats, args.direction, stream)
        else:
            best.fill_(INT32_MAX)
            cb.cbfs_query_stream(h, blk_src, blk_sz, C, d, qs_d, qt_d, best, stats, stream)
            if world > 1:
                import torch.distributed as tdist
                tdist.all_reduce(best, op=tdist.ReduceOp.MIN)  # A12: answers MIN-all-reduced over ranks

    def step(timed_phases: bool):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        evs[0].record(stream)
        h = cb.cbfs_graph_create(n, src_d, dst_d, rflags, local, stream)
        evs[1].record(stream)
        if overlap:
            # A1 overlapped with A2-A8: traversal of batch b starts once its clusters are selected
            evs[2].record(stream)
            got = cb.cbfs_select_and_run_shard(h, r_total, k, d, policy, cfg["root_seed"], world, rank, sel_src,
                                               sel_sz, dist_bytes, dist_out, masks_out, planes, stats,
                                               args.direction, stream)
        else:
            got = cb.cbfs_select_clusters(h, r_total, k, d, policy, cfg["root_seed"], sel_src, sel_sz, stream)
            evs[2].record(stream)
            traverse(h)
        assert got == r_total, f"selection produced {got} < {r_total} clusters"
        evs[3].record(stream)
        cb.cbfs_graph_destroy(h)
        if timed_phases:
            torch.cuda.synchronize()
            phase_ms["build"] += evs[0].elapsed_time(evs[1])
            phase_ms["select"] += evs[1].elapsed_time(evs[2])
            phase_ms["cbfs"] += evs[2].elapsed_time(evs[3])

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()

    clocks = ClockSampler(local, args.clock_ms)
    if not args.no_clocks:
        clocks.start()
    cb.cbfs_launch_count(reset=True)
    cb.cbfs_profile_enable(True)
    cb.cbfs_profile_read(reset=True)
    total_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the timed region)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(True)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        total_ms += e0.elapsed_time(e1)
    launches = cb.cbfs_launch_count(reset=True)
    prof = cb.cbfs_profile_read(reset=True)
    cb.cbfs_profile_enable(False)
    clk = clocks.stop()
    phase_ms = {kk: v / args.steps for kk, v in phase_ms.items()}  # per timed step
    st = stats.cpu().numpy().view(np.uint64)
    sizes = sel_sz[first::world].cpu().numpy().astype(np.float64)
    units_step = float((sizes * st[:, 3].astype(np.float64)).sum())
    hh = cb.cbfs_graph_create(n, src_d, dst_d, 0, local, stream)
    n_h, m_h, maxdeg = cb.cbfs_graph_info(hh)
    n_ni = cb.cbfs_graph_nonisolated(hh)
    cb.cbfs_graph_destroy(hh)
    digests_np = digest.cpu().numpy().view(np.uint64) if digest is not None else None
    parity = golden_check(args.config, digests_np, st, first, world) if strong else None

    # T = device time of the C-BFS phase (A2-A11: init, traversal, output writes and their
    # consumer) over all clusters, max over ranks; graph build (A0) and selection (A1) are reported
    # separately (phase_ms) and in value_incl_build_select, which divides by the whole timed step.
    T_step = allreduce_max(total_ms, world) / 1000.0
    T = allreduce_max(phase_ms["cbfs"] * args.steps, world) / 1000.0
    units_all = allreduce_sum(units_step * args.steps, world)
    value = units_all / T

    # ---- roofline of the dominant kernel (its algorithmic bytes per step over its summed launch times,
    # CUDA events on the launching stream), the step-level figure of all traversal kernels, and SURVEY
    # §8(d)'s per-cluster byte model
    peak, peak_src = peaks()
    perstep = {kk: {f: (v / args.steps if f in ("ms", "launches", "arcs", "entries", "u_in", "u_out") else v)
                    for f, v in pk.items()} for kk, pk in prof.items()}
    parts = alg_bytes_model(perstep, st, n, m_h, n_ni, d, planes, dist_bytes, C, mode, Q)
    alg_step = float(sum(parts.values()))
    cbfs_s = phase_ms["cbfs"] / 1000.0
    ksum = sum(v["ms"] for v in perstep.values()) or 1e-9
    per_kernel = {kk: {"event_ms_per_step": round(v["ms"], 3), "launches_per_step": v["launches"],
                       "share_of_event_time": round(v["ms"] / ksum, 4)}
                  for kk, v in perstep.items() if v["launches"]}
    for kk, pk in per_kernel.items():
        if kk in parts and pk["event_ms_per_step"] > 0:
            pk["alg_bytes_per_step"] = float(parts[kk])
            pk["alg_gbs"] = round(parts[kk] / (pk["event_ms_per_step"] / 1000.0) / 1e9, 1)
    dom = max(per_kernel, key=lambda kk: per_kernel[kk]["event_ms_per_step"]) if per_kernel else None
    dom_name = {"fold": "k_fold", "push": "k_push", "pull": "k_pull", "sparse": "k_sp_push (sparse round loop)",
                "consume": "k_digest"}.get(dom, dom)
    achieved = per_kernel[dom].get("alg_gbs", 0.0) if dom else 0.0
    traffic = None
    ncu_json = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(ncu_json):
        try:
            tk = json.load(open(ncu_json)).get("dominant_kernel_traffic", {}).get(args.config)
            if tk and dom and tk.get("kernel") == dom_name.split()[0]:
                traffic = float(tk["dram_bytes_per_launch"])
        except Exception:
            traffic = None
    s8 = sec8d_bytes(st, n, d)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom_name,
                "achieved_note": ("the dominant kernel's algorithmic bytes (this design's lower bound, DESIGN.md §5) "
                                  "over its summed per-launch CUDA-event times; traffic = its ncu DRAM bytes per "
                                  "launch (profiles/)"),
                "alg_bytes_per_launch": (float(parts.get(dom, 0.0)) / per_kernel[dom]["launches_per_step"]
                                         if dom and per_kernel[dom]["launches_per_step"] else None),
                "step": {"alg_bytes": alg_step, "phase_s": cbfs_s,
                         "achieved": alg_step / cbfs_s / 1e9 if cbfs_s > 0 else 0.0,
                         "frac": (alg_step / cbfs_s / 1e9) / peak if cbfs_s > 0 else 0.0,
                         "parts": {kk: float(v) for kk, v in parts.items()},
                         "note": "all traversal + consumer kernels of the step over the C-BFS phase time"},
                "sec8d": {"bytes": s8, "achieved": s8 / cbfs_s / 1e9 if cbfs_s > 0 else 0.0,
                          "frac": (s8 / cbfs_s / 1e9) / peak if cbfs_s > 0 else 0.0,
                          "note": ("SURVEY §8(d) per-cluster model 22 sum E + 40 sum |F| + n (20 + 8 (d+1)), summed "
                                   "over clusters: a per-cluster traversal's bytes; batching 64 clusters shares one "
                                   "column read and one row gather per vertex, so this exceeds the bytes moved")},
                "model": alg_bytes_model.__doc__.split("\n\n")[0].strip().replace("\n    ", " "),
                "peak_source": peak_src, "per_kernel": per_kernel}

    # ---- end to end through the public API with host buffers (rank-local)
    e2e = None
    if not args.no_e2e:
        import ctypes
        e2e_ms = 0.0
        hs = torch.zeros((C, 4), dtype=torch.int64).pin_memory()
        hsrc = torch.empty((C, 64), dtype=torch.int32).pin_memory()
        hsz = torch.empty((C,), dtype=torch.uint8).pin_memory()
        hd = hm = hbest = hdig = None
        if mode == "full":
            hd = torch.empty((n, C), dtype=dist_out.dtype).pin_memory()
            hm = torch.empty((planes, n, C), dtype=torch.int64).pin_memory()
        if mode == "query":
            hbest = torch.empty((Q,), dtype=torch.int32).pin_memory()
        if mode == "digest":
            hdig = torch.empty((C,), dtype=torch.int64).pin_memory()
        for it in range(args.e2e_warmup + args.e2e_steps):
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h = cb.cbfs_graph_create(n, src_h, dst_h, rflags, local, stream)
            cb.cbfs_select_clusters(h, r_total, k, d, policy, cfg["root_seed"], sel_src, sel_sz, stream)
            if mode == "query":
                qs_d.copy_(qs_h, non_blocking=True)
                qt_d.copy_(qt_h, non_blocking=True)
                traverse(h)
                hbest.copy_(best)
            elif mode == "digest":
                traverse(h)
                hdig.copy_(digest)
                hs.copy_(stats)
            else:
                hsrc.copy_(sel_src[first::world])
                hsz.copy_(sel_sz[first::world])
                cb._check(cb._lib.cbfs_run_host(h, ctypes.c_void_p(hsrc.data_ptr()),
                                                ctypes.c_void_p(hsz.data_ptr()), C, d, dist_bytes,
                                                ctypes.c_void_p(hd.data_ptr()) if hd is not None else None,
                                                ctypes.c_void_p(hm.data_ptr()) if hm is not None else None, planes,
                                                ctypes.c_void_p(hs.data_ptr()), args.direction,
                                                ctypes.c_void_p(stream.cuda_stream)))
            cb.cbfs_graph_destroy(h)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if os.environ.get("CBFS_BENCH_DEBUG"):
                log(f"[e2e] iteration {it}: {1000 * dt:.1f} ms, device free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB")
            if it >= args.e2e_warmup:
                e2e_ms += 1000 * dt
        Te = allreduce_max(e2e_ms, world) / 1000.0
        units_e = allreduce_sum(units_step * args.e2e_steps, world)
        h2d = 2 * 4 * len(el.src) + (8 * Q if mode == "query" else 0) + (64 * 4 * C + C if mode == "full" else 0)
        d2h = (r_total * 65 * (mode == "full") + C * 32 +
               (hd.numel() * hd.element_size() + hm.numel() * 8 if mode == "full" else 0)
               + (4 * Q if mode == "query" else 0) + (8 * C if mode == "digest" else 0))
        e2e = {"value": units_e / Te, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": args.e2e_steps, "ms_per_step": 1000 * Te / args.e2e_steps,
               "timing": "host wall clock around the public C-ABI calls, max over ranks",
               "path": {"full": "cbfs_graph_create (host COO) + cbfs_select_clusters + cbfs_run_host (host outputs)",
                        "digest": "cbfs_graph_create (host COO) + cbfs_select_clusters + cbfs_run_digest + D2H of "
                                  "the digests and statistics",
                        "query": "cbfs_graph_create (host COO) + cbfs_select_clusters + H2D queries + "
                                 "cbfs_query_stream + D2H answers"}[mode]}

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores, model = cpu_info()
        nsteps = args.ref_sample or cores
        v, secs, desc = oracle_steps(args.config, el, cores, nsteps, 0)
        cpu = {"value": v, "unit": UNIT, "cores": min(cores, nsteps), "kind": "oracle", "sample": desc, "cpu": model}

    if rank == 0:
        K = args.steps
        vec_gb = n * C * (dist_bytes + 8 * planes) / 1e9
        outputs = {"full": f"full distance vectors written to HBM ({vec_gb:.1f} GB, [n][C] store)",
                   "digest": (f"full distance vectors of every cluster ({vec_gb:.0f} GB per step) written to HBM "
                              f"staging batch by batch and consumed by the digest kernel (cbfs_run_digest)"),
                   "query": f"labels of every batch consumed by {Q} distance queries (cbfs_query_stream)"}[mode]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": 1000 * T_step / K, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "u64", "data": "synthetic",
            "config": {"workload": args.config, "graph": el.name, "n": n, "arcs": m_h, "max_degree": maxdeg,
                       "clusters": r_total, "clusters_rank0": C, "k": k, "d": d, "dist_bytes": dist_bytes,
                       "relabel": relabel,
                       "mode": mode, "outputs": outputs, "queries": Q,
                       "parallelism": f"clusters round-robin over {world} rank(s), graph replicated",
                       "step": ("A0 CSR build + A1 selection + A2-A9 C-BFS of the rank's clusters"
                                + (" (A1 overlapped with A2-A8: cbfs_select_and_run_shard)" if overlap else "")
                                + (" + output digest" if mode == "digest" else "")
                                + (" + A10/A11 labels and queries" if mode == "query" else "")),
                       "l2": "flushed between timed steps (256 MiB write); inputs and outputs > L2",
                       "units_per_step_rank0": units_step,
                       "timing": ("value = sum_c |S_c| m_c / T with T the C-BFS phase (A2-A11 incl. output "
                                  "writes and their consumer; CUDA events, max over ranks), SURVEY §8(d); "
                                  "ms_per_step is the whole step incl. A0 build and A1 selection"),
                       "cbfs_ms_per_step": 1000 * T / K,
                       "value_incl_build_select": units_all / T_step,
                       "value_whole_graph_m": float(sizes.sum()) * m_h * args.steps * world / T,
                       "phase_ms_rank0": {kk: round(v, 3) for kk, v in phase_ms.items()},
                       "phase_note": ("with the overlap, 'select' is 0 and 'cbfs' covers A1+A2-A8" if overlap
                                      else "'cbfs' covers A2-A9 + the output consumer"),
                       "direction": ["auto", "push", "pull"][args.direction],
                       "engine": ["auto", "batched", "sparse"][args.engine],
                       "alpha": args.alpha or 100.0},
            "parity": parity,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3_rmat24")
    ap.add_argument("--direction", type=int, default=0)
    ap.add_argument("--alpha", type=float, default=0.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=0, help="cpu_baseline steps (default: one per host core)")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--overlap-select", action="store_true",
                    help="full mode: overlap A1 with A2-A8 (cbfs_select_and_run_shard); T then includes A1")
    ap.add_argument("--clock-ms", type=int, default=100)
    ap.add_argument("--concurrency", type=int, default=0, help="concurrent batches per GPU (0 = library default)")
    ap.add_argument("--engine", type=int, default=0, help="0 auto, 1 batched, 2 sparse (cbfs_set_engine)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's clusters split over the ranks; weak: C clusters per rank")
    ap.add_argument("--mode", default="", choices=["", "full", "digest", "query"], help="override the config's mode")
    ap.add_argument("--clusters", type=int, default=0, help="clusters per GPU (default: the config's)")
    ap.add_argument("--relabel", default="", choices=["", "none", "degree", "locality"],
                    help="override the config's internal vertex order (outputs are in original ids either way)")
    ap.add_argument("--queries", type=int, default=0, help="queries (query mode; default: the config's)")
    args = ap.parse_args()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
