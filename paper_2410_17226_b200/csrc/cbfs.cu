// cbfs.cu — the C-BFS engine (§8(a) rows A2-A8): Alg. 1 of PAPER.md
// with the direction-optimised EdgeMap, run for a
// batch of LANES = 64 clusters at once in lock-step rounds.
//
// B200 design:
//  * vertex-major state: for vertex v the 64 clusters of a batch own the 64
//    consecutive words seen[v*64 + c] / pend[v*64 + c] (u64 bit-subsets,
//    P:641-645) and dist[v*64 + c] (u16 Delta).  In the dense pull a
//    warp reads one neighbour's state for all 64 clusters as one coalesced
//    512-byte access (16 B per lane, lane l = clusters 2l and 2l+1), so the
//    random neighbour gathers move whole sectors and one load instruction
//    serves two clusters.
//  * S_next of Alg. 1 is kept as `pend` = S_next \ S_seen (the bits that
//    arrived this round and are not yet folded).  pend is zero outside the
//    pending entries; the first writer that turns a pend word non-zero owns
//    the claim (R4), so no separate r[] array is needed.
//  * a frontier is a list of packed (v*64 + c) entries; the pending list of
//    round i IS F_i.
//  * round i = fold kernel (vertex phase P:714-720) -> push kernel (sparse,
//    P:1758-1768, edge-balanced over the frontier's arcs, 64-bit atomicOr)
//    or pull kernel (dense).  Kernel boundaries are the
//    barriers that H9 requires between the two phases.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.cuh"

namespace cbfs {

static double g_alpha = 100.0;
constexpr uint32_t SCAN_BLOCKS = 592;    // the push's degree scan: blocks of the tile sums
// rows of S_seen the pull keeps in L2 with an evict_last hint (64 MiB of
// 512-byte rows; CBFS_PULL_HUB_MB overrides, for measurements)
static uint32_t g_hub_rows = [] {
  const char* e = getenv("CBFS_PULL_HUB_MB");
  const uint64_t mb = e ? (uint64_t)atoll(e) : 64;
  return (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, (mb << 20) / (LANES * 8));
}();
static int g_max_slots = 4;

// ---- optional per-kernel timing (cbfs_profile_*): CUDA events recorded on
// the launching stream around each fold / push / pull launch; read after the
// round's counters arrive, so no extra sync is added.  With concurrent
// batches a launch's time includes the time it shares the GPU.
struct Prof {
  bool on = false;
  double ms[PK_N] = {};
  uint64_t launches[PK_N] = {};
  uint64_t arcs[PK_N] = {};     // frontier (cluster, arc) pairs processed
  uint64_t entries[PK_N] = {};  // frontier entries processed
  uint64_t u_in[PK_N] = {};     // distinct frontier vertices |U_i|
  uint64_t u_out[PK_N] = {};    // distinct claimed vertices |U_{i+1}|
};
static Prof g_prof;
bool prof_on() { return g_prof.on; }
void prof_add(int kind, double ms, uint64_t launches, uint64_t entries) {
  g_prof.ms[kind] += ms;
  g_prof.launches[kind] += launches;
  g_prof.entries[kind] += entries;
}

// The slots are cached per device and reused by every graph handle
// (allocating and mapping a few GB per cbfs_run would cost tens of ms).  A
// traversal holds the device's lock for its duration.
constexpr int MAX_DEV = 64;
static DevSlots g_dev[MAX_DEV];
static std::mutex g_work_mu[MAX_DEV];

static void slot_free(Slot* w) {
  cudaFree(w->blk); cudaFree(w->listA); cudaFree(w->listB);
  cudaFree(w->ubits); cudaFree(w->bstats);
  cudaFree(w->scan_tmp);
  cudaFree(w->fullm);
  cudaFree(w->bs); cudaFreeHost(w->bs_h);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      if (w->b_exec[a][b]) cudaGraphExecDestroy(w->b_exec[a][b]);
      if (w->b_graph[a][b]) cudaGraphDestroy(w->b_graph[a][b]);
    }
  sparse_free(w);
  if (w->s) cudaStreamDestroy(w->s);
  if (w->ready) cudaEventDestroy(w->ready);
  delete w;
}

void work_free(Graph* g) { g->work = nullptr; }  // the cache outlives graphs

// One block per slot holds the per-cell state of either engine: the batched
// engine's seen [cap + 64] | pend [cap] | pre [cap + 1] (u64) | dist [cap]
// (u16), or the sparse engine's 32-byte cells (sparse.cu).
// The block is sized for the engine the call uses (-1: either).
static uint64_t blk_bytes(uint64_t cap, int engine) {
  const uint64_t batched = (cap + LANES) * 8 + cap * 8 + (cap + LANES) * 8 + cap * 2;
  if (engine == ENGINE_BATCHED) return batched;
  return std::max<uint64_t>(batched, cap * SPARSE_CELL_BYTES);
}

static uint64_t slot_bytes(uint64_t cap, int engine) {
  return blk_bytes(cap, engine) + cap * 4 * 2 + cap / 4 + cap / 8;
}

static int slot_alloc(Slot* w, uint64_t cap, uint64_t blk) {
  w->cap = cap;
  const uint64_t ubw = 2 * ((cap / LANES >> 5) + 1);
  CBFS_CUDA(cudaMalloc(&w->blk, blk));
  w->seen = reinterpret_cast<uint64_t*>(w->blk);  // [cap + LANES]: + all-zero row n
  w->pend = w->seen + cap + LANES;
  w->pre = w->pend + cap;
  w->dist = reinterpret_cast<uint16_t*>(w->pre + cap + LANES);  // 512-byte aligned rows
  CBFS_CUDA(cudaMalloc(&w->listA, cap * sizeof(uint32_t)));
  CBFS_CUDA(cudaMalloc(&w->listB, cap * sizeof(uint32_t)));
  CBFS_CUDA(cudaMalloc(&w->ubits, ubw * sizeof(uint32_t)));
  CBFS_CUDA(cudaMalloc(&w->bs, sizeof(BState)));
  CBFS_CUDA(cudaMallocHost(&w->bs_h, sizeof(BState)));
  CBFS_CUDA(cudaMemset(w->bs, 0, sizeof(BState)));
  CBFS_CUDA(cudaMalloc(&w->bstats, LANES * 4 * sizeof(uint64_t)));
  CBFS_CUDA(cudaMalloc(&w->fullm, (cap / LANES + 1) * sizeof(uint64_t)));
  CBFS_CUDA(cudaMemset(w->pend, 0, cap * sizeof(uint64_t)));  // zero-invariant from here on
  w->pend_clean_cells = cap;
  CBFS_CUDA(cudaMemset(w->ubits, 0, ubw * sizeof(uint32_t)));  // both bitmaps zero between batches
  CBFS_CUDA(cudaMalloc(&w->scan_tmp, SCAN_BLOCKS * sizeof(uint64_t)));
  CBFS_CUDA(cudaStreamCreateWithFlags(&w->s, cudaStreamNonBlocking));
  CBFS_CUDA(cudaEventCreateWithFlags(&w->ready, cudaEventDisableTiming));
  return sparse_alloc(w);
}

static void work_release(DevSlots& D) {
  for (Slot* w : D.slots) slot_free(w);
  D.slots.clear();
  D.cap = 0;
  D.blk = 0;
}

// Slots for graphs of n vertices and the given engine (-1: either).  As many
// concurrent batches as half the free memory allows (>= 1, <= the
// concurrency setting); a caller that stages `extra` bytes per slot next to
// it (output consumers) bounds the count by 90% of the free memory.
static int work_grow(DevSlots& D, uint32_t n, int engine, uint64_t extra) {
  const uint64_t cap = (uint64_t)(n ? n : 1) * LANES;
  const uint64_t blk = blk_bytes(cap, engine);
  if (D.cap >= cap && D.blk >= blk && !D.slots.empty()) return CBFS_OK;
  work_release(D);
  size_t fr = 0, tot = 0;
  CBFS_CUDA(cudaMemGetInfo(&fr, &tot));
  const uint64_t sb = slot_bytes(cap, engine);
  uint64_t P = std::min<uint64_t>((uint64_t)g_max_slots, std::max<uint64_t>(1, (fr / 2) / sb));
  if (extra) P = std::min<uint64_t>(P, std::max<uint64_t>(1, (uint64_t)(0.9 * fr) / (sb + extra)));
  D.cap = cap;
  D.blk = blk;
  for (uint64_t k = 0; k < P; ++k) {
    Slot* w = new Slot();
    w->idx = (int)k;  // its constant-memory BState mirror
    D.slots.push_back(w);
    int rc = slot_alloc(w, cap, blk);
    if (rc) return rc;
  }
  CBFS_CUDA(cudaDeviceSynchronize());
  return CBFS_OK;
}

WorkLease::WorkLease(Graph* g, int engine, uint64_t extra_per_slot) : g_(g) {
  if (g->device < 0 || g->device >= MAX_DEV) { rc = fail(CBFS_EUNSUPPORTED, "device ordinal >= 64"); return; }
  g_work_mu[g->device].lock();
  locked_ = true;
  rc = work_grow(g_dev[g->device], g->n, engine, extra_per_slot);
  if (rc == CBFS_OK) g->work = reinterpret_cast<struct Work*>(&g_dev[g->device]);
}

WorkLease::~WorkLease() {
  if (g_) g_->work = nullptr;
  if (locked_) g_work_mu[g_->device].unlock();
}

constexpr uint32_t LSHIFT = 6;  // log2(LANES)
static_assert((1u << LSHIFT) == LANES, "LANES must be 64");

// warp-aggregated append of `e` for lanes with `flag`
__device__ __forceinline__ void warp_append(bool flag, uint32_t e, uint32_t* __restrict__ list,
                                            unsigned long long* __restrict__ count) {
  unsigned mask = __ballot_sync(FULLW, flag);
  if (!mask) return;
  const uint32_t lane = lane_id();
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(count, (unsigned long long)__popc(mask));
  base = __shfl_sync(FULLW, base, leader);
  if (flag) list[base + __popc(mask & ((1u << lane) - 1))] = e;
}

// union-frontier bit of vertex v, one atomic per distinct word in the warp
// returns the number of bits this lane newly set (distinct vertices added)
__device__ __forceinline__ uint32_t warp_set_bit(bool flag, uint32_t v, uint32_t* __restrict__ bits) {
  const uint32_t word = flag ? (v >> 5) : 0xFFFFFFFFu;
  const unsigned grp = __match_any_sync(FULLW, word);
  const unsigned b = __reduce_or_sync(grp, flag ? (1u << (v & 31)) : 0u);
  if (flag && lane_id() == (uint32_t)(__ffs(grp) - 1)) return __popc(b & ~atomicOr(&bits[word], b));
  return 0;
}

// ------------------------------------------------------------------ stats
// Per-cluster statistics are counted where an entry is CLAIMED for the next
// frontier (so the fold stays a pure streaming kernel): bstats[c] =
// {rounds, sum_i |F_i|, sum_i E_i, sum of degrees of first visits}.
// With `rstats` (cbfs_run_rounds) the counts also go to the per-round record
// rstats[c][rounds - 1] = {|F_i|, E_i} of the round the claims belong to.
__device__ __forceinline__ void stats_flush(uint64_t* __restrict__ bstats, uint32_t c, unsigned long long aF,
                                            unsigned long long aE, unsigned long long aM, uint32_t rounds,
                                            uint64_t* __restrict__ rstats = nullptr, uint32_t R = 0) {
  if (!aF) return;
  atomicAdd((unsigned long long*)&bstats[c * 4 + 1], aF);
  atomicAdd((unsigned long long*)&bstats[c * 4 + 2], aE);
  if (aM) atomicAdd((unsigned long long*)&bstats[c * 4 + 3], aM);
  atomicMax((unsigned long long*)&bstats[c * 4 + 0], (unsigned long long)rounds);
  if (rstats && rounds - 1 < R) {
    uint64_t* r = rstats + ((uint64_t)c * R + rounds - 1) * 2;
    atomicAdd((unsigned long long*)&r[0], aF);
    atomicAdd((unsigned long long*)&r[1], aE);
  }
}

// The graph / batch / slot-array fields of each slot's BState are mirrored in
// constant memory (written on the slot's stream before its batch starts): the
// kernels read them as constant-bank operands instead of holding ~20 pointers
// in registers; the round state (counters, round, direction, profile) lives in
// the global BState the loop advances.
constexpr int BS_MAX = 8;  // slots per device (cbfs_set_concurrency <= 8); kernels are instantiated per slot so
                           // that the mirror's fields are direct constant-bank operands
__constant__ BState c_bs[BS_MAX];

// ------------------------------------------------------------------ init
// R1 seeding (S_next[s_j] = {s_j}; F_0 = S): pend[s_j, c] = bit j.
__device__ __forceinline__ void seed_body(const uint32_t* __restrict__ sources, const uint8_t* __restrict__ sizes,
                                          uint32_t nb, uint32_t n, const uint32_t* __restrict__ inv,
                                          const uint64_t* __restrict__ off, uint64_t* __restrict__ pend,
                                          uint32_t* __restrict__ list, uint32_t* __restrict__ ubits0,
                                          uint64_t* __restrict__ bstats, unsigned long long* __restrict__ ctr,
                                          unsigned long long* __restrict__ err, int allow_empty,
                                          uint64_t* __restrict__ rstats, uint32_t R) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // 64 threads per cluster
  const uint32_t c = t >> 6, j = t & 63;
  bool claim = false;
  uint32_t e = 0, x = 0;
  unsigned long long deg = 0;
  if (c < nb) {
    const uint32_t k = sizes[c];
    if ((k == 0 && !allow_empty) || k > 64) {
      if (j == 0) atomicOr(err, ERR_BAD_SIZE);
    } else if (j < k) {
      const uint32_t s = sources[(uint64_t)c * 64 + j];
      if (s >= n) {
        atomicOr(err, ERR_BAD_SOURCE);
      } else {
        x = inv ? inv[s] : s;
        e = (x << LSHIFT) + c;
        unsigned long long old = atomicOr((unsigned long long*)&pend[e], 1ULL << j);
        if (old != 0) {
          atomicOr(err, ERR_DUP_SOURCE);  // R2
        } else {
          claim = true;
          deg = off[x + 1] - off[x];
          atomicAdd((unsigned long long*)&bstats[c * 4 + 1], 1ULL);
          atomicAdd((unsigned long long*)&bstats[c * 4 + 2], deg);
          atomicAdd((unsigned long long*)&bstats[c * 4 + 3], deg);
          atomicMax((unsigned long long*)&bstats[c * 4 + 0], 1ULL);
          if (rstats && R) {
            atomicAdd((unsigned long long*)&rstats[(uint64_t)c * R * 2], 1ULL);
            atomicAdd((unsigned long long*)&rstats[(uint64_t)c * R * 2 + 1], deg);
          }
        }
      }
    }
  }
  warp_append(claim, e, list, &ctr[0]);
  unsigned long long nu = warp_set_bit(claim, x, ubits0);
  deg = warp_sum(claim ? deg : 0);
  nu = warp_sum(nu);
  if (lane_id() == 0 && deg) atomicAdd(&ctr[1], deg);
  if (lane_id() == 0 && nu) atomicAdd(&ctr[3], nu);
}

template <int SL>
__global__ void k_seed(BState* __restrict__ S) {
  const BState& P = c_bs[SL];
  seed_body(P.sources, P.sizes, P.nb, P.n, P.inv, P.off, P.pend, P.list[0], P.ubits, P.bstats, S->cnt[0], &S->err,
            P.allow_empty, P.rstats, P.R);
}

// ---- kernel-level profile of the device-side loop: the first block of a
// launch to start takes the start time, the last to finish adds the launch's
// duration (globaltimer ns) and its work counts to the slot's BState
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void prof_begin(BState* S, bool on, int kind) {
  if (!on || threadIdx.x != 0) return;
  if (atomicAdd(&S->p_arrive[kind], 1u) == 0) S->p_t0[kind] = gtimer();
}
__device__ __forceinline__ void prof_end(BState* S, bool on, int kind, unsigned long long entries,
                                         unsigned long long arcs, unsigned long long uin, bool uout) {
  if (!on) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(&S->p_leave[kind], 1u) != gridDim.x - 1) return;
  __threadfence();
  volatile BState* V = S;
  V->p_ns[kind] += gtimer() - V->p_t0[kind];
  V->p_launch[kind] += 1;
  V->p_entries[kind] += entries;
  V->p_arcs[kind] += arcs;
  V->p_uin[kind] += uin;
  if (uout) V->p_uout[kind] += V->cnt[(V->i + 1) & 1][3];
  V->p_arrive[kind] = 0;
  V->p_leave[kind] = 0;
}

// ------------------------------------------------------------------ fold
// Vertex phase: S_new = S_next[u] \ S_seen[u] (= pend), set
// Delta_u on first visit, S_u[i - Delta_u] = S_new, S_seen[u] |= S_new; plus
// the output writes and the degrees for the push scan.  Independent per
// entry; FOLD_ILP entries per thread are loaded before any is used.
#ifndef CBFS_FOLD_ILP
#define CBFS_FOLD_ILP 4
#endif
constexpr int FOLD_ILP = CBFS_FOLD_ILP;
// "subset full" bit updates: 0 = aggregate every ILP step, 1 = one atomic per
// event, 2 (default) = aggregate only steps where some lane has an event
// (config 2: 69.9 / 72.4 / 68.9 ms)
#ifndef CBFS_FOLD_FULL
#define CBFS_FOLD_FULL 2
#endif
#ifndef CBFS_FOLD_PF  // prefetch the next iteration's frontier entries
#define CBFS_FOLD_PF 1
#endif
#ifndef CBFS_FOLD_MINB  // blocks per SM the register budget must allow (0: no bound)
#define CBFS_FOLD_MINB 4
#endif
#if CBFS_FOLD_MINB
#define CBFS_FOLD_BOUNDS __launch_bounds__(256, CBFS_FOLD_MINB)
#else
#define CBFS_FOLD_BOUNDS __launch_bounds__(256)
#endif

template <int DB, bool WIDE>
__device__ __forceinline__ void fold_body(const uint32_t* __restrict__ F, uint32_t nF, uint32_t i,
                                          uint64_t* __restrict__ seen, uint64_t* __restrict__ pend,
                                          uint16_t* __restrict__ dist, const uint64_t* __restrict__ off,
                                          const uint32_t* __restrict__ perm, uint32_t n, uint32_t C, uint32_t cbase,
                                          uint32_t planes, void* __restrict__ out_dist, void* __restrict__ out_masks,
                                          uint32_t mb, uint64_t* __restrict__ pre, int write_pre,
                                          const uint8_t* __restrict__ sizes, uint64_t* __restrict__ fullm,
                                          unsigned long long* __restrict__ err, uint32_t W) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t lane = lane_id();
  bool overflow = false;
#if CBFS_FOLD_PF
  // the next iteration's frontier entries are loaded before this one's
  // states, so an iteration waits on one dependent access instead of two
  uint32_t en[FOLD_ILP];
#pragma unroll
  for (int q = 0; q < FOLD_ILP; ++q) {
    const uint64_t t = tid + q * nth;
    en[q] = t < nF ? F[t] : 0xFFFFFFFFu;
  }
#endif
  for (uint64_t t0 = tid; t0 < nF; t0 += nth * FOLD_ILP) {
    uint32_t e[FOLD_ILP];
    uint64_t nw[FOLD_ILP], sv[FOLD_ILP];
    uint32_t dv[FOLD_ILP];
    uint32_t fvx[FOLD_ILP];  // vertex whose subset of cluster c just became full, else ~0
#if CBFS_FOLD_PF
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q) {
      e[q] = en[q];
      const uint64_t t = t0 + nth * FOLD_ILP + q * nth;
      en[q] = t < nF ? F[t] : 0xFFFFFFFFu;
    }
#else
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q) {
      const uint64_t t = t0 + q * nth;
      e[q] = t < nF ? F[t] : 0xFFFFFFFFu;
    }
#endif
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q) {
      if (e[q] != 0xFFFFFFFFu) {
        nw[q] = pend[e[q]];
        sv[q] = seen[e[q]];
        dv[q] = dist[e[q]];
      }
    }
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q) {
      fvx[q] = 0xFFFFFFFFu;
      if (e[q] == 0xFFFFFFFFu) continue;
      const uint32_t v = e[q] >> LSHIFT, c = e[q] & (LANES - 1);
      CBFS_DCHECK(v < n && (W > 1 || (sizes[c] >= 1 && sizes[c] <= 64)));
      pend[e[q]] = 0;
      seen[e[q]] = sv[q] | nw[q];
      if ((sv[q] | nw[q]) == full_mask(sizes[c])) fvx[q] = v;
      const bool first = dv[q] == INF16;
      if (first) { dv[q] = i; dist[e[q]] = (uint16_t)i; }
      if (write_pre) pre[t0 + q * nth] = off[v + 1] - off[v];
      const uint32_t orig = perm ? perm[v] : v;
      const uint64_t col = (uint64_t)orig * C + cbase + c;
      // wide clusters (k > 64, cbfs_run_wide): the W lanes of a cluster are
      // its 64-source words, each traversed as its own sub-cluster; the
      // cluster's Delta_v is the least over its lanes (all in lockstep
      // rounds, so a lane reaching v later has a larger Delta) and every
      // lane's subsets are placed relative to it
      uint32_t dc = dv[q];
      uint64_t dcol = col;
      if (WIDE) {
        const uint32_t b0 = e[q] & ~(W - 1);
        for (uint32_t x = 0; x < W; ++x) dc = min(dc, (uint32_t)dist[b0 + x]);
        dcol = (uint64_t)orig * (C / W) + (cbase + c) / W;
      }
      if (first && out_dist && (!WIDE || dc == i)) {
        if (DB == 1) {
          overflow |= i > 254;
          ((uint8_t*)out_dist)[dcol] = (uint8_t)(i > 254 ? 254 : i);
        } else {
          ((uint16_t*)out_dist)[dcol] = (uint16_t)i;
        }
      }
      const uint32_t oi = i - dc;
      CBFS_DCHECK(!out_masks || (orig < n && cbase + c < C));
      if (out_masks && oi < planes) {
        if (WIDE || mb != 8) store_mask(out_masks, (uint64_t)oi * n * C + col, nw[q], mb);
        else ((uint64_t*)out_masks)[(uint64_t)oi * n * C + col] = nw[q];
      }
    }
    // per-vertex "subset full" bits (read by the dense pull instead of the
    // whole S_seen row): one 64-bit atomic per distinct vertex in the warp
#if CBFS_FOLD_FULL == 1  // experiments: one atomic per event, no aggregation
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q)
      if (fvx[q] != 0xFFFFFFFFu) atomicOr((unsigned long long*)&fullm[fvx[q]], 1ULL << (e[q] & (LANES - 1)));
#elif CBFS_FOLD_FULL == 2  // experiments: aggregate only when some lane has an event
    const unsigned am = __activemask();
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q) {
      const bool f = fvx[q] != 0xFFFFFFFFu;
      if (!__any_sync(am, f)) continue;
      const uint64_t bit = f ? (1ULL << (e[q] & (LANES - 1))) : 0ULL;
      const unsigned grp = __match_any_sync(am, fvx[q]);
      const uint32_t lo = __reduce_or_sync(grp, (uint32_t)bit), hi = __reduce_or_sync(grp, (uint32_t)(bit >> 32));
      if (f && lane == (uint32_t)(__ffs(grp) - 1))
        atomicOr((unsigned long long*)&fullm[fvx[q]], ((unsigned long long)hi << 32) | lo);
    }
#else
    const unsigned am = __activemask();
#pragma unroll
    for (int q = 0; q < FOLD_ILP; ++q) {
      const bool f = fvx[q] != 0xFFFFFFFFu;
      const uint64_t bit = f ? (1ULL << (e[q] & (LANES - 1))) : 0ULL;
      const unsigned grp = __match_any_sync(am, fvx[q]);
      const uint32_t lo = __reduce_or_sync(grp, (uint32_t)bit), hi = __reduce_or_sync(grp, (uint32_t)(bit >> 32));
      if (f && lane == (uint32_t)(__ffs(grp) - 1))
        atomicOr((unsigned long long*)&fullm[fvx[q]], ((unsigned long long)hi << 32) | lo);
    }
#endif
  }
  if (overflow) atomicOr(err, ERR_OVERFLOW);
}

// the vertex phase of round S->i over F_i = list[i & 1]
template <int DB, bool WIDE, int SL>
__global__ void CBFS_FOLD_BOUNDS k_fold(BState* __restrict__ S) {
  const BState& P = c_bs[SL];
  prof_begin(S, P.prof_on, PK_FOLD);
  const uint32_t i = (uint32_t)S->i, cur = i & 1;
  const uint32_t nF = (uint32_t)S->cnt[cur][0];
  fold_body<DB, WIDE>(P.list[cur], nF, i, P.seen, P.pend, P.dist, P.off, P.perm, P.n, P.C, P.cbase, P.planes,
                      P.out_dist, P.out_masks, P.mb, P.pre, S->pull == 0, P.sizes, P.fullm, &S->err, P.W);
  prof_end(S, P.prof_on, PK_FOLD, nF, 0, 0, false);
}

// ------------------------------------------------------------------ push
// EdgeMap-Sparse with Edge_F = Fetch_And_Or: the
// frontier's (entry, arc) pairs form one virtual array of `total` arcs
// (exclusive prefix `pre`, pre[nF] = total); each warp takes PUSH_CHUNK
// consecutive arcs, so hubs and degree-4 grid vertices balance alike.
constexpr uint32_t PUSH_CHUNK = 256;

__device__ __forceinline__ void push_body(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols,
                                          const uint32_t* __restrict__ F, const uint64_t* __restrict__ pre,
                                          uint32_t nF, uint64_t total, const uint64_t* __restrict__ seen,
                                          const uint16_t* __restrict__ dist, uint64_t* __restrict__ pend,
                                          uint32_t* __restrict__ out_list, uint32_t* __restrict__ ubits_next,
                                          uint64_t* __restrict__ bstats, unsigned long long* __restrict__ ctr,
                                          uint32_t i, uint32_t d, uint64_t* __restrict__ rstats, uint32_t R) {
  __shared__ unsigned long long sF[LANES], sE[LANES], sM[LANES];
  __shared__ uint32_t s_out[8][PUSH_CHUNK];  // per-warp claims of the current chunk
  for (uint32_t c = threadIdx.x; c < LANES; c += blockDim.x) sF[c] = sE[c] = sM[c] = 0;
  __syncthreads();
  const uint32_t lane = lane_id();
  uint32_t* obuf = s_out[threadIdx.x >> 5];
  const unsigned lt = (1u << lane) - 1;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  unsigned long long degsum = 0, nu = 0;
  for (uint64_t w = warp; w * PUSH_CHUNK < total; w += nwarps) {
    const uint64_t start = w * PUSH_CHUNK;
    const uint64_t end = min(start + PUSH_CHUNK, total);
    // largest idx with pre[idx] <= start: 32-ary warp search (log32 steps)
    uint32_t lo = 0, hi = nF;  // answer in [lo, hi)
    while (hi - lo > 1) {
      const uint32_t step = (hi - lo + 31) / 32;
      const uint32_t pos = lo + lane * step;
      const bool le = pos < hi && pre[pos] <= start;
      const uint32_t cntle = __popc(__ballot_sync(FULLW, le));  // probes at or before the answer
      const uint32_t nlo = lo + (cntle - 1) * step;
      hi = min(nlo + step, hi);
      lo = nlo;
    }
    uint32_t idx = lo;
    uint32_t nout = 0;
    for (uint64_t p0 = start; p0 < end; p0 += 32) {
      const uint64_t p = p0 + lane;
      bool claim = false;
      uint32_t ev = 0, v = 0;
      if (p < end) {
        while (pre[idx + 1] <= p) ++idx;
        const uint32_t e = F[idx];
        const uint32_t u = e >> LSHIFT, c = e & (LANES - 1);
        v = cols[off[u] + (p - pre[idx])];
        ev = (v << LSHIFT) + c;
        const uint32_t dv = dist[ev];
        if (dv == INF16 || (int)i - (int)dv < (int)d) {  // P:722, R3
          const uint64_t x = seen[e] & ~seen[ev];
          if (x) {
            const unsigned long long old = atomicOr((unsigned long long*)&pend[ev], (unsigned long long)x);
            claim = old == 0;  // first setter wins (R4)
            if (claim) {
              const unsigned long long deg = off[v + 1] - off[v];
              degsum += deg;
              atomicAdd(&sF[c], 1ULL);
              atomicAdd(&sE[c], deg);
              if (dv == INF16) atomicAdd(&sM[c], deg);
            }
          }
        }
      }
      const unsigned cm = __ballot_sync(FULLW, claim);
      if (claim) obuf[nout + __popc(cm & lt)] = ev;
      nout += __popc(cm);
      nu += warp_set_bit(claim, v, ubits_next);
    }
    // one global reservation per chunk
    __syncwarp();
    if (nout) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(&ctr[0], (unsigned long long)nout);
      base = __shfl_sync(FULLW, base, 0);
      CBFS_DCHECK(nout <= PUSH_CHUNK);
      for (uint32_t t = lane; t < nout; t += 32) out_list[base + t] = obuf[t];
    }
    __syncwarp();
  }
  degsum = warp_sum(degsum);
  nu = warp_sum(nu);
  if (lane == 0 && degsum) atomicAdd(&ctr[1], degsum);
  if (lane == 0 && nu) atomicAdd(&ctr[3], nu);
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < LANES; c += blockDim.x)
    stats_flush(bstats, c, sF[c], sE[c], sM[c], i + 2, rstats, R);
}

// the sparse edge phase of round S->i (pre = the exclusive prefix of the
// frontier's degrees, pre[nF] = E_i)
template <int SL>
__global__ void __launch_bounds__(256) k_push(BState* __restrict__ S) {
  const BState& P = c_bs[SL];
  prof_begin(S, P.prof_on, PK_PUSH);
  const uint32_t i = (uint32_t)S->i, cur = i & 1;
  const uint32_t nF = (uint32_t)S->cnt[cur][0];
  const uint64_t E = S->cnt[cur][1];
  push_body(P.off, P.cols, P.list[cur], P.pre, nF, E, P.seen, P.dist, P.pend, P.list[cur ^ 1],
            P.ubits + (uint64_t)(cur ^ 1) * P.ub_words, P.bstats, S->cnt[cur ^ 1], i, P.d, P.rstats, P.R);
  prof_end(S, P.prof_on, PK_PUSH, nF, E, S->cnt[cur][3], true);
}

// ------------------------------------------------------------------ pull
// EdgeMap-Dense: every vertex v that can still receive (cap
// P:722 and S_seen[v] != S) ORs S_seen[u] over its neighbours u in the union
// frontier.  No first-hit break (R7): a vertex stops only when its
// accumulated subset is full.  Neighbours not in F_i^c contribute only bits v
// already holds (R7a), so one union-frontier test per arc
// serves all 64 clusters.  Lane l owns clusters 2l, 2l+1 (one 16-byte word
// pair per state row).
//
// A warp owns a PULL_CHUNK-arc slice of the CSR; its vertices are handled in
// groups of up to 32:
//   (1) one coalesced load gives the group's 32 offsets;
//   (2) the group's per-vertex state (Delta row, "subset full" word) is
//       loaded back to back; cap and first-visit bits are kept in registers;
//   (3) pass A streams the group's arcs 32 at a time (coalesced columns +
//       union-frontier bits), finds each arc's vertex by a shuffle binary
//       search and compacts the useful neighbours into a shared-memory list
//       that is sorted by vertex, with per-vertex counts;
//   (4) pass B walks each active vertex's segment of the list, gathering
//       PULL_MLP neighbour rows at a time into a register accumulator, with
//       the R7 full-subset exit checked after every batch;
//   (5) the group's claims are appended with one atomic.
#ifndef CBFS_PULL_MLP
#define CBFS_PULL_MLP 8
#endif
#ifndef CBFS_PULL_MINB
#define CBFS_PULL_MINB 8
#endif
constexpr int PULL_MLP = CBFS_PULL_MLP;  // neighbour rows in flight per warp
#ifndef CBFS_PULL_PA
#define CBFS_PULL_PA 2
#endif
constexpr int PULL_PA = CBFS_PULL_PA;  // pass-A 32-arc steps whose loads are in flight together
#ifndef CBFS_PULL_WARPS
#define CBFS_PULL_WARPS 4
#endif
constexpr int PULL_WARPS = CBFS_PULL_WARPS;  // warps per block
#ifndef CBFS_PULL_SKIP
#define CBFS_PULL_SKIP 0
#endif

#ifdef CBFS_PULL_STATS
__device__ unsigned long long g_dbg[32];
extern "C" int cbfs_debug_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_dbg, sizeof(g_dbg));
  unsigned long long z[32] = {0};
  cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
  return 0;
}
#endif

struct U2 {
  uint64_t a, b;
};

// L2 eviction-priority hints for the pull (CBFS_PULL_HINT, default on):
// the hub rows (lowest internal ids, gathered by most vertices) are loaded
// with an evict_last policy, the other gathered rows and the streamed CSR
// columns with evict_first, so the one-touch traffic does not push the hub
// rows out of L2.
#ifndef CBFS_PULL_HINT
#define CBFS_PULL_HINT 1
#endif
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ ulonglong2 ld_row_hint(const ulonglong2* p, uint64_t pol) {
  ulonglong2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ld_u32_hint(const uint32_t* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ U2 ld2(const uint64_t* p) {
  const ulonglong2 x = __ldg(reinterpret_cast<const ulonglong2*>(p));
  return {x.x, x.y};
}

__device__ __forceinline__ void pull_body(
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, const uint32_t* __restrict__ chunk_v,
    uint64_t n_chunks, uint64_t m, uint32_t n, const uint64_t* __restrict__ seen, const uint16_t* __restrict__ dist,
    uint64_t* __restrict__ pend, const uint32_t* __restrict__ ubits, uint32_t* __restrict__ ubits_next,
    const uint8_t* __restrict__ sizes, uint32_t nb, uint32_t* __restrict__ out_list, uint64_t* __restrict__ bstats,
    unsigned long long* __restrict__ ctr, const uint64_t* __restrict__ fullm, uint32_t i, uint32_t d,
    uint64_t* __restrict__ rstats, uint32_t R, uint32_t hub_rows) {
  __shared__ uint32_t s_list[PULL_WARPS][PULL_CHUNK + 32];
#if CBFS_PULL_HINT
  const uint64_t pol_last = l2_policy_last(), pol_first = l2_policy_first();
#endif
  __shared__ uint32_t s_cnt[PULL_WARPS][32];
  __shared__ unsigned long long s_stat[PULL_WARPS][3][LANES];  // per-warp F / E / M per cluster
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  uint32_t* list = s_list[wib];
  uint32_t* cnt = s_cnt[wib];
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint32_t c0 = 2 * lane, c1 = 2 * lane + 1;
  const uint64_t full0 = c0 < nb ? full_mask(sizes[c0]) : 0ULL;
  const uint64_t full1 = c1 < nb ? full_mask(sizes[c1]) : 0ULL;
  const unsigned lt = (1u << lane) - 1;
  unsigned long long degsum = 0, nu = 0;
  unsigned long long(*stat)[LANES] = s_stat[wib];
  stat[0][c0] = stat[0][c1] = stat[1][c0] = stat[1][c1] = stat[2][c0] = stat[2][c1] = 0;
  const uint64_t* seen2 = seen + 2 * lane;  // lane's word pair of row 0
  const ulonglong2* rows2 = reinterpret_cast<const ulonglong2*>(seen) + lane;
  const uint32_t* dist2 = reinterpret_cast<const uint32_t*>(dist) + lane;

  for (uint64_t w = warp; w < n_chunks; w += nwarps) {
    const uint64_t e0 = w * PULL_CHUNK;
    const uint64_t e1 = min(e0 + PULL_CHUNK, m);
    uint32_t v = chunk_v[w];
    uint64_t e = e0;
    while (e < e1) {
      // ---- (1) offsets of up to 32 vertices v .. v+31
      const uint32_t vj = v + lane;
      const uint64_t ob = vj < n ? off[vj] : m;
      const uint64_t oe = vj < n ? off[vj + 1] : m;
      const uint32_t nv = __popc(__ballot_sync(FULLW, vj < n && ob < e1));  // a prefix of lanes
      const uint64_t lo_j = max(ob, e0), hi_j = min(oe, e1);
      const unsigned hasarcs = __ballot_sync(FULLW, lane < nv && lo_j < hi_j);
      const uint64_t ge = __shfl_sync(FULLW, hi_j, nv - 1);  // group arc end
      // ---- (2) per-vertex state rows
      unsigned cap0 = 0, cap1 = 0, inf0 = 0, inf1 = 0, actv = 0;
      for (uint32_t j0 = 0; j0 < nv; j0 += 4) {
        uint32_t dq[4];
        uint64_t fq[4];  // "subset full" bits of the vertex (one broadcast load)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t j = j0 + q;
          dq[q] = 0xFFFFFFFFu;
          fq[q] = ~0ULL;
          if (j < nv && ((hasarcs >> j) & 1u)) {
            dq[q] = dist2[(uint64_t)(v + j) * (LANES / 2)];
            fq[q] = fullm[v + j];
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t j = j0 + q;
          if (j < nv && ((hasarcs >> j) & 1u)) {
            const uint32_t d0 = dq[q] & 0xFFFFu, d1 = dq[q] >> 16;
            const bool k0 = full0 != 0 && (d0 == INF16 || (int)i - (int)d0 < (int)d) && !((fq[q] >> c0) & 1ULL);
            const bool k1 = full1 != 0 && (d1 == INF16 || (int)i - (int)d1 < (int)d) && !((fq[q] >> c1) & 1ULL);
            cap0 |= (unsigned)k0 << j;
            cap1 |= (unsigned)k1 << j;
            inf0 |= (unsigned)(d0 == INF16) << j;
            inf1 |= (unsigned)(d1 == INF16) << j;
            if (__ballot_sync(FULLW, k0 || k1)) actv |= 1u << j;
          }
        }
      }
      if (actv) {
        // ---- (3) pass A: compact useful neighbours (ids u, grouped by vertex),
        // sorted by vertex, and count them per vertex
        cnt[lane] = 0;
        __syncwarp();
        uint32_t nl = 0;
#if CBFS_PULL_PA > 1
        // pass A in groups of PULL_PA 32-arc steps: the group's column loads,
        // then its union-frontier word loads, are issued before any is used
        // (two dependent round trips per group instead of two per step)
        for (uint64_t wg = e; wg < ge; wg += 32 * PULL_PA) {
          uint32_t uq[PULL_PA], bq[PULL_PA], jq[PULL_PA];
#pragma unroll
          for (int k = 0; k < PULL_PA; ++k) {
            const uint64_t a = wg + 32 * k + lane;
            const bool inr = a < ge;
#if CBFS_PULL_HINT
            uq[k] = inr ? ld_u32_hint(cols + a, pol_first) : 0u;
#else
            uq[k] = inr ? cols[a] : 0u;
#endif
            uint32_t jv = 0;  // largest j < nv with ob_j <= a
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
              const uint32_t cand = jv + step;
              const uint64_t oc = __shfl_sync(FULLW, ob, cand & 31);
              if (cand < nv && oc <= a) jv = cand;
            }
            jq[k] = inr && ((actv >> jv) & 1u) ? jv : 0xFFFFFFFFu;
          }
#pragma unroll
          for (int k = 0; k < PULL_PA; ++k) bq[k] = jq[k] != 0xFFFFFFFFu ? __ldg(&ubits[uq[k] >> 5]) : 0u;
#pragma unroll
          for (int k = 0; k < PULL_PA; ++k) {
            if (wg + 32 * k >= ge) break;  // warp-uniform
            const uint32_t u = uq[k], jv = jq[k];
            const bool want = jv != 0xFFFFFFFFu && ((bq[k] >> (u & 31)) & 1u);
            const unsigned fm = __ballot_sync(FULLW, want);
            CBFS_DCHECK(!want || (u < n && nl + __popc(fm & lt) < PULL_CHUNK + 32));
            if (want) list[nl + __popc(fm & lt)] = u;  // segments are contiguous per vertex (arc order)
            const unsigned grp = __match_any_sync(FULLW, want ? jv : 0xFFFFFFFFu);
            if (want && lane == (uint32_t)(__ffs(grp) - 1)) cnt[jv] += __popc(grp);
            nl += __popc(fm);
            __syncwarp();
          }
        }
#else
        for (uint64_t wb = e; wb < ge; wb += 32) {
          const uint64_t a = wb + lane;
          const bool inr = a < ge;
#if CBFS_PULL_HINT
          const uint32_t u = inr ? ld_u32_hint(cols + a, pol_first) : 0u;
#else
          const uint32_t u = inr ? cols[a] : 0u;
#endif
          uint32_t jv = 0;  // largest j < nv with ob_j <= a
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t cand = jv + step;
            const uint64_t oc = __shfl_sync(FULLW, ob, cand & 31);
            if (cand < nv && oc <= a) jv = cand;
          }
          const bool want = inr && ((actv >> jv) & 1u) && ((__ldg(&ubits[u >> 5]) >> (u & 31)) & 1u);
          const unsigned fm = __ballot_sync(FULLW, want);
          CBFS_DCHECK(!want || (u < n && nl + __popc(fm & lt) < PULL_CHUNK + 32));
          if (want) list[nl + __popc(fm & lt)] = u;  // segments are contiguous per vertex (arc order)
          const unsigned grp = __match_any_sync(FULLW, want ? jv : 0xFFFFFFFFu);
          if (want && lane == (uint32_t)(__ffs(grp) - 1)) cnt[jv] += __popc(grp);
          nl += __popc(fm);
          __syncwarp();
        }
#endif
        const uint32_t myc = cnt[lane];
        uint32_t incl = myc;  // per-vertex segment ends (inclusive scan, lane = vertex)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULLW, incl, o);
          if (lane >= (uint32_t)o) incl += y;
        }
        __syncwarp();
        // ---- (4) pass B: per active vertex, OR its neighbours' contributions
        // into a register accumulator, checking the R7 full-subset exit after
        // every batch, then decide the vertex's claims
        unsigned myb0 = 0, myb1 = 0;  // lane j: claim ballots of vertex j
        unsigned rem = actv;
        while (rem) {
          const uint32_t j = __ffs(rem) - 1;
          rem &= rem - 1;
          const uint32_t s1 = __shfl_sync(FULLW, incl, j);
          const uint32_t s0 = s1 - __shfl_sync(FULLW, myc, j);
          const uint64_t row = (uint64_t)(v + j) * LANES;
          const U2 sv = ld2(seen2 + row);
          const bool k0 = (cap0 >> j) & 1u, k1 = (cap1 >> j) & 1u;
          uint64_t acc0 = 0, acc1 = 0;
          {
            for (uint32_t q = s0; q < s1; q += PULL_MLP) {
              // CBFS_PULL_SKIP: a lane loads its 16 bytes of the rows only while
              // one of its clusters is capped and not yet full (config 3: 52% of
              // the sectors are needed in the first dense round, 1% in the
              // second; measured slower on configs 2 and 3, off by default)
              const bool need = CBFS_PULL_SKIP == 0 || (k0 && ((acc0 | sv.a) & full0) != full0) ||
                                (k1 && ((acc1 | sv.b) & full1) != full1);
              U2 g[PULL_MLP];
#pragma unroll
              for (int r = 0; r < PULL_MLP; ++r) {
                const uint32_t x = q + r < s1 ? list[q + r] : n;  // past the segment: the zero row
                ulonglong2 y = make_ulonglong2(0ULL, 0ULL);
#if CBFS_PULL_HINT
                if (need) y = ld_row_hint(rows2 + x * (LANES / 2), x < hub_rows ? pol_last : pol_first);
#else
                if (need) y = __ldg(rows2 + x * (LANES / 2));  // 32-bit index: x * 32 < 2^31
#endif
                g[r] = {y.x, y.y};
              }
#pragma unroll
              for (int r = 0; r < PULL_MLP; ++r) { acc0 |= g[r].a; acc1 |= g[r].b; }
#ifdef CBFS_PULL_STATS
              {  // per round: [hub, other] x {rows, non-zero words, set bits} of the gathered S_seen rows
                unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
                for (int r = 0; r < PULL_MLP; ++r) {
                  if (q + r >= s1) break;
                  const int o = list[q + r] < hub_rows ? 0 : 3;
                  const unsigned long long words = warp_sum((g[r].a != 0) + (g[r].b != 0));
                  const unsigned long long bits = warp_sum(__popcll(g[r].a) + __popcll(g[r].b));
                  cnt[o] += 1;
                  cnt[o + 1] += words;
                  cnt[o + 2] += bits;
                }
                if (lane == 0 && i < 4)
                  for (int k = 0; k < 6; ++k) atomicAdd(&g_dbg[i * 8 + k], cnt[k]);
              }
#endif
              // R7: stop once every capped lane holds its full subset
              if (q + PULL_MLP < s1 &&
                  !__ballot_sync(FULLW, (k0 && ((acc0 | sv.a) & full0) != full0) ||
                                            (k1 && ((acc1 | sv.b) & full1) != full1)))
                break;
            }
          }
          const uint64_t nw0 = k0 ? (acc0 & ~sv.a) : 0, nw1 = k1 ? (acc1 & ~sv.b) : 0;
          bool cl0 = false, cl1 = false;
          const uint64_t ob_j = __shfl_sync(FULLW, ob, j), oe_j = __shfl_sync(FULLW, oe, j);
          if (nw0 | nw1) {
            uint64_t* pp = pend + row + 2 * lane;
            if (ob_j >= e0 && oe_j <= e1) {  // this warp owns all of v's arcs
              *reinterpret_cast<ulonglong2*>(pp) = make_ulonglong2(nw0, nw1);
              cl0 = nw0 != 0;
              cl1 = nw1 != 0;
            } else {
              if (nw0) cl0 = atomicOr((unsigned long long*)pp, (unsigned long long)nw0) == 0;
              if (nw1) cl1 = atomicOr((unsigned long long*)(pp + 1), (unsigned long long)nw1) == 0;
            }
            const unsigned long long deg = oe_j - ob_j;
            if (cl0) { stat[0][c0] += 1; stat[1][c0] += deg; if ((inf0 >> j) & 1u) stat[2][c0] += deg; degsum += deg; }
            if (cl1) { stat[0][c1] += 1; stat[1][c1] += deg; if ((inf1 >> j) & 1u) stat[2][c1] += deg; degsum += deg; }
          }
          const unsigned b0 = __ballot_sync(FULLW, cl0), b1 = __ballot_sync(FULLW, cl1);
          if (lane == j) { myb0 = b0; myb1 = b1; }
        }
        // ---- (5) one append for the group; entries of a vertex in cluster order
        const uint32_t ccount = __popc(myb0) + __popc(myb1);
        uint32_t cinc = ccount;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULLW, cinc, o);
          if (lane >= (uint32_t)o) cinc += y;
        }
        const uint32_t total = __shfl_sync(FULLW, cinc, 31);
        if (total) {
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(&ctr[0], (unsigned long long)total);
          base = __shfl_sync(FULLW, base, 0);
          const uint32_t cexcl = cinc - ccount;
          unsigned rem2 = __ballot_sync(FULLW, ccount != 0);
          while (rem2) {
            const uint32_t j = __ffs(rem2) - 1;
            rem2 &= rem2 - 1;
            const unsigned b0 = __shfl_sync(FULLW, myb0, j), b1 = __shfl_sync(FULLW, myb1, j);
            const uint32_t oj = __shfl_sync(FULLW, cexcl, j);
            const bool h0 = (b0 >> lane) & 1u, h1 = (b1 >> lane) & 1u;
            const uint32_t r = oj + __popc(b0 & lt) + __popc(b1 & lt);
            const uint32_t ebase = ((v + j) << LSHIFT) + 2 * lane;
            CBFS_DCHECK(base + r + h0 + h1 <= (uint64_t)n * LANES);
            if (h0) out_list[base + r] = ebase;
            if (h1) out_list[base + r + h0] = ebase + 1;
          }
        }
        nu += warp_set_bit(ccount != 0, v + lane, ubits_next);
        __syncwarp();
      }
      e = ge;
      v += nv;
    }
  }
  degsum = warp_sum(degsum);
  nu = warp_sum(nu);
  if (lane == 0 && degsum) atomicAdd(&ctr[1], degsum);
  if (lane == 0 && nu) atomicAdd(&ctr[3], nu);
  stats_flush(bstats, c0, stat[0][c0], stat[1][c0], stat[2][c0], i + 2, rstats, R);
  stats_flush(bstats, c1, stat[0][c1], stat[1][c1], stat[2][c1], i + 2, rstats, R);
}

// the dense edge phase of round S->i
template <int SL>
__global__ void __launch_bounds__(PULL_WARPS * 32, CBFS_PULL_MINB) k_pull(BState* __restrict__ S) {
  const BState& P = c_bs[SL];
  prof_begin(S, P.prof_on, PK_PULL);
  const uint32_t i = (uint32_t)S->i, cur = i & 1;
  const uint32_t n = P.n;
  pull_body(P.off, P.cols, P.chunk_v, P.n_chunks, P.m, n, P.seen, P.dist, P.pend, P.ubits + (uint64_t)cur * P.ub_words,
            P.ubits + (uint64_t)(cur ^ 1) * P.ub_words, P.sizes, P.nb, P.list[cur ^ 1], P.bstats, S->cnt[cur ^ 1],
            P.fullm, i, P.d, P.rstats, P.R, min(n, P.hub_rows));
  prof_end(S, P.prof_on, PK_PULL, S->cnt[cur][0], S->cnt[cur][1], S->cnt[cur][3], true);
}

// ------------------------------------------------------------------ round loop
// The batch's round loop runs on the device as one CUDA graph per slot:
//   WHILE (go) { k_begin; k_fold; IF (pull) { k_pull } ELSE { k_scan_*; k_push }; k_end }
// k_begin decides the round's direction (R8: pull when the
// frontier's (cluster, arc) pairs exceed m * nb / alpha) and clears the next
// frontier's counters; k_end clears U_i and ends the round (Alg. 1's loop,
// continue while F_{i+1} is non-empty).
constexpr uint32_t SCAN_THREADS = 512;

template <int SL>
__global__ void k_begin(BState* __restrict__ S, cudaGraphConditionalHandle h_if) {
  const BState& P = c_bs[SL];
  const uint32_t cur = (uint32_t)(S->i & 1);
  const uint32_t t = threadIdx.x;
  if (t < 4) S->cnt[cur ^ 1][t] = 0;
  if (t == 0) {
    const unsigned long long E = S->cnt[cur][1];
    const bool pull = P.direction == CBFS_DIR_PULL ||
                      (P.direction == CBFS_DIR_AUTO && (double)E > P.pull_threshold);
    S->pull = pull;
    S->launches += pull ? 4 : 7;  // begin, fold, pull | 3 scan kernels + push, end
    if (h_if) cudaGraphSetConditional(h_if, pull ? 1u : 0u);
  }
}

// exclusive prefix of pre[0 .. nF) in place, pre[nF] = E_i: block sums,
// one block scans them, blocks rescan their tiles with the offsets
template <int SL>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_sums(BState* __restrict__ S) {
  typedef cub::BlockReduce<unsigned long long, SCAN_THREADS> BR;
  __shared__ typename BR::TempStorage tmp;
  const BState& P = c_bs[SL];
  const uint64_t nF = S->cnt[S->i & 1][0];
  const uint64_t tile = (nF + SCAN_BLOCKS - 1) / SCAN_BLOCKS;
  const uint64_t b0 = blockIdx.x * tile, b1 = min(b0 + tile, nF);
  unsigned long long x = 0;
  for (uint64_t k = b0 + threadIdx.x; k < b1; k += SCAN_THREADS) x += P.pre[k];
  x = BR(tmp).Sum(x);
  if (threadIdx.x == 0) P.scan_tmp[blockIdx.x] = x;
}

template <int SL>
__global__ void __launch_bounds__(1024) k_scan_top(BState* __restrict__ S) {
  typedef cub::BlockScan<unsigned long long, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  const BState& P = c_bs[SL];
  unsigned long long x = threadIdx.x < SCAN_BLOCKS ? P.scan_tmp[threadIdx.x] : 0ULL;
  BS(tmp).ExclusiveSum(x, x);
  if (threadIdx.x < SCAN_BLOCKS) P.scan_tmp[threadIdx.x] = x;
}

template <int SL>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(BState* __restrict__ S) {
  typedef cub::BlockScan<unsigned long long, SCAN_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned long long s_run;
  const BState& P = c_bs[SL];
  const uint32_t cur = (uint32_t)(S->i & 1);
  const uint64_t nF = S->cnt[cur][0];
  const uint64_t tile = (nF + SCAN_BLOCKS - 1) / SCAN_BLOCKS;
  const uint64_t b0 = blockIdx.x * tile, b1 = min(b0 + tile, nF);
  if (threadIdx.x == 0) s_run = P.scan_tmp[blockIdx.x];
  __syncthreads();
  for (uint64_t k0 = b0; k0 < b1; k0 += SCAN_THREADS) {
    const uint64_t k = k0 + threadIdx.x;
    unsigned long long x = k < b1 ? P.pre[k] : 0ULL, total;
    BS(tmp).ExclusiveSum(x, x, total);
    const unsigned long long run = s_run;
    if (k < b1) P.pre[k] = run + x;
    __syncthreads();
    if (threadIdx.x == 0) s_run = run + total;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.pre[nF] = S->cnt[cur][1];
}

template <int SL>
__global__ void k_end(BState* __restrict__ S, cudaGraphConditionalHandle h_while) {
  const BState& P = c_bs[SL];
  const uint32_t cur = (uint32_t)(S->i & 1);
  uint32_t* ub = P.ubits + (uint64_t)cur * P.ub_words;  // U_i consumed
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < P.ub_words;
       w += (uint64_t)gridDim.x * blockDim.x)
    ub[w] = 0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(&S->end_done, 1u) != gridDim.x - 1) return;
  __threadfence();
  volatile BState* V = S;
  V->end_done = 0;
  const unsigned long long i = V->i + 1;
  V->i = i;
  bool go = V->cnt[i & 1][0] > 0;
  if (go && i >= 0xFFFEull) {
    atomicOr(&S->err, (unsigned long long)ERR_ROUNDS);
    go = false;
  }
  if (V->err & (ERR_ROUNDS | ERR_BAD_SOURCE | ERR_DUP_SOURCE | ERR_BAD_SIZE)) go = false;
  V->go = go;
  if (h_while) cudaGraphSetConditional(h_while, go ? 1u : 0u);
}

// ------------------------------------------------------------------ driver
#ifndef CBFS_FOLD_GRID_PER_SM
#define CBFS_FOLD_GRID_PER_SM 32
#endif
constexpr unsigned FOLD_GRID = 148u * CBFS_FOLD_GRID_PER_SM;  // grid-stride kernels of the round loop (fixed grids:
constexpr unsigned PUSH_GRID = 148u * 8u * 4u;   // the loop's kernel nodes are launched with the same
constexpr unsigned END_GRID = 148u * 2u;         // configuration every round)

static int b_add(cudaGraph_t body, cudaGraphNode_t* node, const cudaGraphNode_t* dep, void* fn, unsigned grid,
                 unsigned block, void** args) {
  cudaKernelNodeParams kp = {};
  kp.func = fn;
  kp.gridDim = dim3(grid);
  kp.blockDim = dim3(block);
  kp.kernelParams = args;
  CBFS_CUDA(cudaGraphAddKernelNode(node, body, dep, dep ? 1 : 0, &kp));
  return CBFS_OK;
}

// the round-loop kernels of slot SL
struct BFns {
  void *seed, *fold[2][2], *push, *pull, *begin, *end, *scan_sums, *scan_top, *scan_apply;
};
template <int SL>
static BFns bfns() {
  BFns f;
  f.seed = (void*)k_seed<SL>;
  f.fold[0][0] = (void*)k_fold<1, false, SL>;
  f.fold[0][1] = (void*)k_fold<1, true, SL>;
  f.fold[1][0] = (void*)k_fold<2, false, SL>;
  f.fold[1][1] = (void*)k_fold<2, true, SL>;
  f.push = (void*)k_push<SL>;
  f.pull = (void*)k_pull<SL>;
  f.begin = (void*)k_begin<SL>;
  f.end = (void*)k_end<SL>;
  f.scan_sums = (void*)k_scan_sums<SL>;
  f.scan_top = (void*)k_scan_top<SL>;
  f.scan_apply = (void*)k_scan_apply<SL>;
  return f;
}
static const BFns& fns_of(int slot) {
  static const BFns t[BS_MAX] = {bfns<0>(), bfns<1>(), bfns<2>(), bfns<3>(),
                                 bfns<4>(), bfns<5>(), bfns<6>(), bfns<7>()};
  return t[slot];
}

// The slot's round-loop graph for (Delta width, wide):
//   WHILE (go) { k_begin -> k_fold -> IF (pull) { k_pull } ELSE { k_scan_sums -> k_scan_top -> k_scan_apply ->
//   k_push } -> k_end }
static int b_build(Slot* w, int db, bool wide) {
  cudaGraph_t g;
  CBFS_CUDA(cudaGraphCreate(&g, 0));
  w->b_graph[db - 1][wide] = g;
  cudaGraphConditionalHandle hw, hi;
  CBFS_CUDA(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  CBFS_CUDA(cudaGraphConditionalHandleCreate(&hi, g, 0, 0));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  CBFS_CUDA(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  BState* S = w->bs;
  const BFns& F = fns_of(w->idx);
  void* a_s[] = {&S};
  void* a_if[] = {&S, &hi};
  void* a_wh[] = {&S, &hw};
  cudaGraphNode_t nb, nf, nif, ne;
  int rc = b_add(body, &nb, nullptr, F.begin, 1, 32, a_if);
  if (!rc) rc = b_add(body, &nf, &nb, F.fold[db - 1][wide], FOLD_GRID, 256, a_s);
  if (rc) return rc;
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = hi;
  ip.conditional.type = cudaGraphCondTypeIf;
  ip.conditional.size = 2;  // [0] then (pull), [1] else (push)
  CBFS_CUDA(cudaGraphAddNode(&nif, body, &nf, 1, &ip));
  cudaGraph_t g_pull = ip.conditional.phGraph_out[0], g_push = ip.conditional.phGraph_out[1];
  cudaGraphNode_t np, s1, s2, s3, nq;
  rc = b_add(g_pull, &np, nullptr, F.pull, 148u * CBFS_PULL_MINB, PULL_WARPS * 32, a_s);
  if (!rc) rc = b_add(g_push, &s1, nullptr, F.scan_sums, SCAN_BLOCKS, SCAN_THREADS, a_s);
  if (!rc) rc = b_add(g_push, &s2, &s1, F.scan_top, 1, 1024, a_s);
  if (!rc) rc = b_add(g_push, &s3, &s2, F.scan_apply, SCAN_BLOCKS, SCAN_THREADS, a_s);
  if (!rc) rc = b_add(g_push, &nq, &s3, F.push, PUSH_GRID, 256, a_s);
  if (!rc) rc = b_add(body, &ne, &nif, F.end, END_GRID, 256, a_wh);
  if (rc) return rc;
  CBFS_CUDA(cudaGraphInstantiate(&w->b_exec[db - 1][wide], g, 0));
  return CBFS_OK;
}

// queue init + seeding of batch `a` on the slot's stream; the seeding's
// error bits come back to the host before the round loop is launched
static int slot_start(Graph* g, Slot* w, const RunArgs& a) {
  const uint32_t n = g->n;
  cudaStream_t st = w->s;
  w->a = a;
  w->busy = true;
  w->seeding = true;
  w->overflow = false;
  w->i = 0;
  w->engine = a.engine;
  if (a.engine == ENGINE_SPARSE) {
    w->pend_clean_cells = 0;  // the 32-byte cells overwrite the batched arrays
    return sparse_start(g, w, a);
  }
  const uint64_t cells = (uint64_t)n * LANES;
  if (w->pend_clean_cells < cells) {  // pend must be zero over this graph's cells
    CBFS_CUDA(cudaMemsetAsync(w->pend, 0, cells * sizeof(uint64_t), st));
    w->pend_clean_cells = cells;
  }
  BState* h = w->bs_h;  // the slot's previous batch (and its copy) finished before this one starts
  std::memset(h, 0, sizeof(BState));
  h->off = g->off;
  h->cols = g->cols;
  h->chunk_v = g->chunk_v;
  h->perm = a.out_internal ? nullptr : g->perm;
  h->inv = g->inv;
  h->n_chunks = g->n_chunks;
  h->m = g->m;
  h->sources = a.sources;
  h->sizes = a.sizes;
  h->out_dist = a.out_dist;
  h->out_masks = a.out_masks;
  h->rstats = a.out_rounds;
  h->R = a.out_rounds ? a.max_rounds : 0;
  h->n = n;
  h->nb = a.nb;
  h->d = a.d;
  h->planes = a.planes;
  h->C = a.C;
  h->cbase = a.cbase;
  h->mb = a.mask_bytes ? a.mask_bytes : 8;
  h->W = a.wide > 1 ? a.wide : 1;
  h->direction = a.direction;
  h->hub_rows = g_hub_rows;
  h->allow_empty = a.wide > 1;
  h->pull_threshold = (double)g->m * (double)a.nb / g_alpha;  // R8: E_i * alpha > m * nb
  h->seen = w->seen;
  h->pend = w->pend;
  h->pre = w->pre;
  h->fullm = w->fullm;
  h->bstats = w->bstats;
  h->scan_tmp = reinterpret_cast<uint64_t*>(w->scan_tmp);
  h->dist = w->dist;
  h->list[0] = w->listA;
  h->list[1] = w->listB;
  h->ubits = w->ubits;
  h->ub_words = (n >> 5) + 1;
  h->prof_on = g_prof.on;
  CBFS_CUDA(cudaMemcpyAsync(w->bs, h, sizeof(BState), cudaMemcpyHostToDevice, st));
  CBFS_CUDA(cudaMemcpyToSymbolAsync(c_bs, h, sizeof(BState), (size_t)w->idx * sizeof(BState), cudaMemcpyHostToDevice,
                                    st));
  CBFS_CUDA(cudaMemsetAsync(w->seen, 0, (uint64_t)(n + 1) * LANES * sizeof(uint64_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->dist, 0xFF, (uint64_t)n * LANES * sizeof(uint16_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->bstats, 0, LANES * 4 * sizeof(uint64_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->fullm, 0, (uint64_t)(n + 1) * sizeof(uint64_t), st));
  {
    BState* S = w->bs;
    void* args[] = {&S};
    CBFS_CUDA(cudaLaunchKernel(fns_of(w->idx).seed, dim3((a.nb * 64 + 255) / 256), dim3(256), args, 0, st));
  }
  CBFS_LAUNCHED();
  CBFS_CUDA(cudaMemcpyAsync(w->bs_h, w->bs, sizeof(BState), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaEventRecord(w->ready, st));
  return CBFS_OK;
}

// Profiling aid (env CBFS_BATCHED_HOSTLOOP=1): the loop's kernels launched
// from the host round by round (ncu cannot profile kernel nodes of graphs with
// conditional nodes).  Synchronous.
static int batched_hostloop(Slot* w) {
  cudaStream_t st = w->s;
  BState* S = w->bs;
  const BFns& F = fns_of(w->idx);
  const int db = w->a.dist_bytes;
  const bool wide = w->a.wide > 1;
  unsigned long long flag = 0;
  cudaGraphConditionalHandle none = 0;
  void* a_s[] = {&S};
  void* a_h[] = {&S, &none};
  for (;;) {
    CBFS_CUDA(cudaLaunchKernel(F.begin, dim3(1), dim3(32), a_h, 0, st));
    CBFS_CUDA(cudaLaunchKernel(F.fold[db - 1][wide], dim3(FOLD_GRID), dim3(256), a_s, 0, st));
    CBFS_CUDA(cudaMemcpyAsync(&flag, &S->pull, sizeof(flag), cudaMemcpyDeviceToHost, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    if (flag) {
      CBFS_CUDA(cudaLaunchKernel(F.pull, dim3(148u * CBFS_PULL_MINB), dim3(PULL_WARPS * 32), a_s, 0, st));
    } else {
      CBFS_CUDA(cudaLaunchKernel(F.scan_sums, dim3(SCAN_BLOCKS), dim3(SCAN_THREADS), a_s, 0, st));
      CBFS_CUDA(cudaLaunchKernel(F.scan_top, dim3(1), dim3(1024), a_s, 0, st));
      CBFS_CUDA(cudaLaunchKernel(F.scan_apply, dim3(SCAN_BLOCKS), dim3(SCAN_THREADS), a_s, 0, st));
      CBFS_CUDA(cudaLaunchKernel(F.push, dim3(PUSH_GRID), dim3(256), a_s, 0, st));
    }
    CBFS_CUDA(cudaLaunchKernel(F.end, dim3(END_GRID), dim3(256), a_h, 0, st));
    CBFS_CUDA(cudaGetLastError());
    CBFS_CUDA(cudaMemcpyAsync(&flag, &S->go, sizeof(flag), cudaMemcpyDeviceToHost, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    if (!flag) break;
  }
  return CBFS_OK;
}

// the batch's whole round loop (one graph launch) + the state readback
static int batched_launch(Slot* w) {
  static const bool hostloop = getenv("CBFS_BATCHED_HOSTLOOP") != nullptr;
  cudaStream_t st = w->s;
  const int db = w->a.dist_bytes == 1 ? 1 : 2;
  const bool wide = w->a.wide > 1;
  if (hostloop) {
    int rc = batched_hostloop(w);
    if (rc) return rc;
  } else {
    if (!w->b_exec[db - 1][wide]) {
      int rc = b_build(w, db, wide);
      if (rc) return rc;
    }
    CBFS_CUDA(cudaGraphLaunch(w->b_exec[db - 1][wide], st));
  }
  CBFS_CUDA(cudaMemcpyAsync(w->bs_h, w->bs, sizeof(BState), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaEventRecord(w->ready, st));
  return CBFS_OK;
}

// The slot's counters arrived: account the finished round, then queue the
// next one or finish the batch.  Returns 1 when the batch finished.
static int finish_batch(Slot* w, BatchSource& src, int slot, int* err) {
  if (w->a.out_stats)
    CBFS_CUDA(cudaMemcpyAsync(w->a.out_stats, w->bstats, (uint64_t)w->a.nb * 4 * sizeof(uint64_t),
                              cudaMemcpyDeviceToDevice, w->s));
  int rc = src.finished(w->a, slot, w->s);
  w->busy = false;
  if (rc) *err = rc;
  if (w->overflow && !*err) *err = fail(CBFS_EOVERFLOW, "a distance exceeds 254 with dist_bytes == 1");
  return 1;
}

static int seed_error(Slot* w, unsigned long long bits, int* err) {
  w->busy = false;
  if (bits & ERR_BAD_SIZE) *err = fail(CBFS_EINVAL, "cluster size must be 1..64");
  else if (bits & ERR_BAD_SOURCE) *err = fail(CBFS_EINVAL, "source id >= n");
  else *err = fail(CBFS_EINVAL, "duplicate source in a cluster");
  return 1;
}

// sparse engine: seeding checked -> the device-side round loop -> done
static int sparse_step(Graph* g, Slot* w, BatchSource& src, int slot, int* err) {
  const SpCtl& h = *w->sp_ctl_h;
  if (w->seeding) {
    w->seeding = false;
    if (h.err) return seed_error(w, h.err, err);  // bad sources (every batch re-initialises its cells)
    int rc = sparse_launch(w);
    if (rc) { *err = rc; w->busy = false; return 1; }
    return 0;
  }
  const uint64_t per_round = w->sp_fused ? 1 : 2;  // (fold +) push per round, launched by the graph
  count_launch(per_round * h.i);
  if (g_prof.on) {
    float ms = 0;
    CBFS_CUDA(cudaEventElapsedTime(&ms, w->sp_t0, w->sp_t1));
    g_prof.ms[PK_SPARSE] += ms; g_prof.launches[PK_SPARSE] += per_round * h.i;
    g_prof.entries[PK_SPARSE] += h.listed;
  }
  w->i = (uint32_t)h.i;
  if (h.err & ERR_ROUNDS) {
    w->busy = false;
    *err = fail(CBFS_EOVERFLOW, "more than 65534 rounds");
    return 1;
  }
  if (h.err & ERR_OVERFLOW) w->overflow = true;
  return finish_batch(w, src, slot, err);
}

static int slot_step(Graph* g, Slot* w, BatchSource& src, int slot, int* err) {
  if (w->engine == ENGINE_SPARSE) return sparse_step(g, w, src, slot, err);
  const uint32_t n = g->n;
  const BState& h = *w->bs_h;
  if (w->seeding) {
    w->seeding = false;
    if (h.err) {  // bad sources: restore the zero invariants, report
      CBFS_CUDA(cudaMemsetAsync(w->pend, 0, (uint64_t)n * LANES * sizeof(uint64_t), w->s));
      CBFS_CUDA(cudaMemsetAsync(w->ubits, 0, 2 * ((n >> 5) + 1) * sizeof(uint32_t), w->s));
      CBFS_CUDA(cudaStreamSynchronize(w->s));
      return seed_error(w, h.err, err);
    }
    int rc = batched_launch(w);
    if (rc) { *err = rc; w->busy = false; return 1; }
    return 0;
  }
  count_launch(h.launches);
  if (g_prof.on) {
    for (int k = PK_FOLD; k <= PK_PULL; ++k) {
      g_prof.ms[k] += h.p_ns[k] * 1e-6;
      g_prof.launches[k] += h.p_launch[k];
      g_prof.entries[k] += h.p_entries[k];
      g_prof.arcs[k] += h.p_arcs[k];
      g_prof.u_in[k] += h.p_uin[k];
      g_prof.u_out[k] += h.p_uout[k];
    }
  }
  w->i = (uint32_t)h.i;
  if (h.err & ERR_ROUNDS) {
    w->busy = false;
    *err = fail(CBFS_EOVERFLOW, "more than 65534 rounds");
    return 1;  // pend is left non-zero only for this slot's pending entries; cleared by run_batches
  }
  if (h.err & ERR_OVERFLOW) w->overflow = true;
  return finish_batch(w, src, slot, err);
}

// Drive all batches of `src` through the device's slots; every slot stream
// first waits for the caller's prior work on `st`, and `st` waits for all of
// them at the end.
int run_batches(Graph* g, BatchSource& src, cudaStream_t st, int max_slots) {
  DevSlots& D = *reinterpret_cast<DevSlots*>(g->work);
  const int P = max_slots > 0 ? std::min<int>(max_slots, (int)D.slots.size()) : (int)D.slots.size();
  cudaEvent_t start;
  CBFS_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CBFS_CUDA(cudaEventRecord(start, st));
  for (int k = 0; k < P; ++k) CBFS_CUDA(cudaStreamWaitEvent(D.slots[k]->s, start, 0));
  CBFS_CUDA(cudaEventDestroy(start));
  int err = CBFS_OK;
  bool exhausted = false;
  for (;;) {
    bool progressed = false, any_busy = false;
    for (int k = 0; k < P; ++k) {
      Slot* w = D.slots[k];
      if (w->busy) {
        const cudaError_t q = cudaEventQuery(w->ready);
        if (q == cudaSuccess) {
          slot_step(g, w, src, k, &err);
          progressed = true;
        } else if (q != cudaErrorNotReady) {
          err = cuda_fail(q, "batch round");
          w->busy = false;
        }
      }
      if (!w->busy && !exhausted && err == CBFS_OK) {
        RunArgs a{};
        const int got = src.next(a);
        if (got < 0) exhausted = true;
        if (got > 0) {
          int rc = src.bind(a, k, w->s);
          if (rc == CBFS_OK) rc = slot_start(g, w, a);
          if (rc) err = rc;
          progressed = true;
        }
      }
      any_busy |= w->busy;
    }
    if (!any_busy && (exhausted || err != CBFS_OK)) break;
    if (!progressed) std::this_thread::yield();
  }
  cudaEvent_t done;
  CBFS_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  for (int k = 0; k < P; ++k) {
    CBFS_CUDA(cudaEventRecord(done, D.slots[k]->s));
    CBFS_CUDA(cudaStreamWaitEvent(st, done, 0));
  }
  CBFS_CUDA(cudaEventDestroy(done));
  if (err != CBFS_OK) {
    // restore the zero invariants of every slot for the next call
    CBFS_CUDA(cudaDeviceSynchronize());
    for (Slot* w : D.slots) {
      CBFS_CUDA(cudaMemset(w->pend, 0, D.cap * sizeof(uint64_t)));
      CBFS_CUDA(cudaMemset(w->ubits, 0, 2 * ((D.cap / LANES >> 5) + 1) * sizeof(uint32_t)));
      w->busy = false;
      }
  }
  return err;
}

int ArraySource::next(RunArgs& a) {
  if (next_c >= n_clusters) return -1;
  a = proto;
  a.sources = sources + (uint64_t)next_c * 64;
  a.sizes = sizes + next_c;
  a.nb = std::min<uint32_t>(LANES, n_clusters - next_c);
  a.cbase = proto.cbase + next_c;
  a.out_stats = out_stats ? out_stats + (uint64_t)next_c * 4 : nullptr;
  a.out_rounds = out_rounds ? out_rounds + (uint64_t)next_c * max_rounds * 2 : nullptr;
  a.max_rounds = max_rounds;
  next_c += a.nb;
  return 1;
}

int num_slots(const Graph* g) { return (int)reinterpret_cast<const DevSlots*>(g->work)->slots.size(); }

int check_run_args(const Graph* g, const void* sources, const void* sizes, uint32_t n_clusters, uint32_t d,
                   uint32_t dist_bytes, uint32_t planes, uint32_t direction) {
  if (!g) return fail(CBFS_EINVAL, "null graph");
  if (n_clusters && (!sources || !sizes)) return fail(CBFS_EINVAL, "null sources/sizes");
  if (d > CBFS_MAX_D) return fail(CBFS_EUNSUPPORTED, "d > CBFS_MAX_D");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (planes != d + 1 && !(planes == d && d > 0)) return fail(CBFS_EINVAL, "planes must be d+1 or d");
  if (direction > CBFS_DIR_PULL) return fail(CBFS_EINVAL, "bad direction");
  return CBFS_OK;
}

// cbfs_run_wide: split each cluster of k <= 64 W sources into W lane sizes
// (lane w holds sources 64w .. 64w+63) and check the cluster (R2: no
// duplicate across its words; 1 <= k <= 64 W; ids < n).  One block per
// cluster, one thread per source slot.
__global__ void k_wide_prep(const uint32_t* __restrict__ sources, const uint16_t* __restrict__ sizes, uint32_t C,
                            uint32_t W, uint32_t n, uint8_t* __restrict__ lane_sizes, int* __restrict__ bad) {
  __shared__ uint32_t s_src[64 * CBFS_WIDE_MAX_W];
  const uint32_t c = blockIdx.x, j = threadIdx.x, K = 64 * W;
  const uint32_t k = sizes[c];
  const uint32_t s = sources[(uint64_t)c * K + j];
  s_src[j] = s;
  __syncthreads();
  if (k == 0 || k > K) {
    if (j == 0) atomicOr(bad, 1);
    return;
  }
  if (j < W) lane_sizes[(uint64_t)c * W + j] = (uint8_t)(k > 64 * j ? min(64u, k - 64 * j) : 0u);
  if (j >= k) return;
  if (s >= n) atomicOr(bad, 2);
  for (uint32_t x = 0; x < j; ++x)
    if (s_src[x] == s) atomicOr(bad, 4);
}

int run_arrays(Graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
               uint32_t dist_bytes, void* out_dist, void* out_masks, uint32_t mask_bytes, uint32_t planes,
               uint64_t* out_stats, uint32_t direction, cudaStream_t st) {
  int rc = check_run_args(g, sources, sizes, n_clusters, d, dist_bytes, planes, direction);
  if (rc) return rc;
  if (mask_bytes != 1 && mask_bytes != 2 && mask_bytes != 4 && mask_bytes != 8)
    return fail(CBFS_EINVAL, "mask word must be 1, 2, 4 or 8 bytes");
  CBFS_CUDA(cudaSetDevice(g->device));
  const int engine = choose_engine(g, direction);
  if (engine < 0) return CBFS_ECUDA;
  WorkLease lease(g, engine);
  if (lease.rc) return lease.rc;
  const uint64_t C = n_clusters;
  if (out_dist) CBFS_CUDA(cudaMemsetAsync(out_dist, 0xFF, (uint64_t)g->n * C * dist_bytes, st));
  if (out_masks) CBFS_CUDA(cudaMemsetAsync(out_masks, 0, (uint64_t)planes * g->n * C * mask_bytes, st));
  ArraySource src;
  src.proto = RunArgs{};
  src.proto.d = d;
  src.proto.planes = planes;
  src.proto.dist_bytes = dist_bytes;
  src.proto.C = n_clusters;
  src.proto.direction = direction;
  src.proto.engine = engine;
  src.proto.out_dist = out_dist;
  src.proto.out_masks = out_masks;
  src.proto.mask_bytes = mask_bytes;
  src.sources = sources;
  src.sizes = sizes;
  src.n_clusters = n_clusters;
  src.out_stats = out_stats;
  rc = run_batches(g, src, st);
  if (rc) return rc;
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}
}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_run(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
             uint32_t dist_bytes, void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
             uint32_t direction, cbfs_stream stream) {
  return run_arrays(reinterpret_cast<Graph*>(gh), sources, sizes, n_clusters, d, dist_bytes, out_dist, out_masks, 8,
                    planes, out_stats, direction, (cudaStream_t)stream);
}

// A1 overlapped with A2-A8: the selection CTA runs on a side stream and
// publishes each finished cluster through mapped host memory; a batch of
// LANES clusters is started as soon as its clusters exist.  With world > 1
// the caller's rank owns the clusters c = rank, rank + world, ... (SURVEY
// §8(e)); a batch's rows are gathered into slot-local contiguous buffers.
struct SelectSource : ArraySource {
  volatile uint32_t* prog;
  cudaStream_t side;
  uint32_t r;
  uint32_t world = 1, rank = 0;
  std::vector<uint32_t*> slot_src;
  std::vector<uint8_t*> slot_sz;
  uint32_t local_of(uint32_t global_count) const {  // this rank's clusters among the first global_count
    return global_count > rank ? (global_count - rank + world - 1) / world : 0;
  }
  int next(RunArgs& a) override {
    const uint32_t total = local_of(r);
    if (next_c >= total) return -1;
    const uint32_t want_end = std::min<uint32_t>(total, next_c + LANES);
    const uint32_t need = rank + world * (want_end - 1) + 1;  // global clusters that must exist
    const uint32_t p = prog[0];
    const bool done = prog[1] != 0;
    if (p < need && !done) {
      if (cudaStreamQuery(side) != cudaErrorNotReady && prog[0] < need && !prog[1]) return -1;  // selection died
      return 0;
    }
    const uint32_t avail = local_of(std::min<uint32_t>((uint32_t)prog[0], r));
    if (next_c >= avail) return -1;  // the selection ran out of vertices
    a = proto;
    a.nb = std::min<uint32_t>(LANES, avail - next_c);
    const uint64_t g0 = rank + (uint64_t)world * next_c;  // global index of the batch's first cluster
    a.sources = sources + g0 * 64;
    a.sizes = sizes + g0;
    a.cbase = proto.cbase + next_c;
    a.out_stats = out_stats ? out_stats + (uint64_t)next_c * 4 : nullptr;
    a.out_rounds = out_rounds ? out_rounds + (uint64_t)next_c * max_rounds * 2 : nullptr;
    a.max_rounds = max_rounds;
    next_c += a.nb;
    return 1;
  }
  int bind(RunArgs& a, int slot, cudaStream_t st) override {
    if (world == 1) return CBFS_OK;
    CBFS_CUDA(cudaMemcpy2DAsync(slot_src[slot], 64 * sizeof(uint32_t), a.sources, (uint64_t)world * 64 * sizeof(uint32_t),
                                64 * sizeof(uint32_t), a.nb, cudaMemcpyDeviceToDevice, st));
    CBFS_CUDA(cudaMemcpy2DAsync(slot_sz[slot], 1, a.sizes, world, 1, a.nb, cudaMemcpyDeviceToDevice, st));
    a.sources = slot_src[slot];
    a.sizes = slot_sz[slot];
    return CBFS_OK;
  }
};

int cbfs_select_and_run_shard(cbfs_graph* gh, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                              uint64_t seed, uint32_t world, uint32_t rank, uint32_t* out_sources,
                              uint8_t* out_sizes, uint32_t* out_r, uint32_t dist_bytes, void* out_dist,
                              uint64_t* out_masks, uint32_t planes, uint64_t* out_stats, uint32_t direction,
                              cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (world == 0 || rank >= world) return fail(CBFS_EINVAL, "rank must be < world");
  int rc = check_select_args(g, r, k, d, root_policy, out_sources, out_sizes);
  if (rc) return rc;
  rc = check_run_args(g, out_sources, out_sizes, r, d, dist_bytes, planes, direction);
  if (rc) return rc;
  if (!out_r) return fail(CBFS_EINVAL, "null out_r");
  *out_r = 0;
  if (r == 0 || g->n == 0) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int engine = choose_engine(g, direction);
  if (engine < 0) return CBFS_ECUDA;
  WorkLease lease(g, engine);
  if (lease.rc) return lease.rc;
  static cudaStream_t side[MAX_DEV];
  static volatile uint32_t* prog_h[MAX_DEV];
  static uint32_t* prog_d[MAX_DEV];
  static uint32_t* count_d[MAX_DEV];
  const int dv = g->device;
  if (!side[dv]) {  // guarded by the device lease
    CBFS_CUDA(cudaStreamCreateWithFlags(&side[dv], cudaStreamNonBlocking));
    void* hp = nullptr;
    CBFS_CUDA(cudaHostAlloc(&hp, 2 * sizeof(uint32_t), cudaHostAllocMapped));
    prog_h[dv] = (volatile uint32_t*)hp;
    CBFS_CUDA(cudaHostGetDevicePointer((void**)&prog_d[dv], hp, 0));
    CBFS_CUDA(cudaMalloc(&count_d[dv], sizeof(uint32_t)));
  }
  volatile uint32_t* prog = prog_h[dv];
  prog[0] = 0;
  prog[1] = 0;
  cudaEvent_t ready;
  CBFS_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  CBFS_CUDA(cudaEventRecord(ready, st));  // selection after the caller's prior work (graph build)
  CBFS_CUDA(cudaStreamWaitEvent(side[dv], ready, 0));
  CBFS_CUDA(cudaEventDestroy(ready));
  rc = select_launch(g, r, k, d, root_policy, seed, out_sources, out_sizes, count_d[dv], prog_d[dv], side[dv]);
  if (rc) return rc;
  SelectSource src;
  src.world = world;
  src.rank = rank;
  const uint64_t C = src.local_of(r);  // this rank's output columns
  if (out_dist) CBFS_CUDA(cudaMemsetAsync(out_dist, 0xFF, (uint64_t)g->n * C * dist_bytes, st));
  if (out_masks) CBFS_CUDA(cudaMemsetAsync(out_masks, 0, (uint64_t)planes * g->n * C * sizeof(uint64_t), st));
  src.proto = RunArgs{};
  src.proto.d = d;
  src.proto.planes = planes;
  src.proto.dist_bytes = dist_bytes;
  src.proto.C = (uint32_t)C;
  src.proto.direction = direction;
  src.proto.engine = engine;
  src.proto.out_dist = out_dist;
  src.proto.out_masks = out_masks;
  src.sources = out_sources;
  src.sizes = out_sizes;
  src.n_clusters = 0;
  src.out_stats = out_stats;
  src.prog = prog;
  src.side = side[dv];
  src.r = r;
  const int P = num_slots(g);
  if (world > 1) {
    src.slot_src.assign(P, nullptr);
    src.slot_sz.assign(P, nullptr);
    for (int q = 0; q < P; ++q) {
      CBFS_CUDA(cudaMallocAsync(&src.slot_src[q], LANES * 64 * sizeof(uint32_t), st));
      CBFS_CUDA(cudaMallocAsync(&src.slot_sz[q], LANES, st));
    }
  }
  rc = run_batches(g, src, st);
  cudaError_t e2 = cudaStreamSynchronize(side[dv]);
  for (int q = 0; q < (int)src.slot_src.size(); ++q) {
    cudaFreeAsync(src.slot_src[q], st);
    cudaFreeAsync(src.slot_sz[q], st);
  }
  if (rc) return rc;
  if (e2 != cudaSuccess) return cuda_fail(e2, "cluster selection");
  if (!prog[1]) return fail(CBFS_ECUDA, "cluster selection ended without publishing");
  CBFS_CUDA(cudaStreamSynchronize(st));
  *out_r = prog[0];
  return CBFS_OK;
}

int cbfs_run_wide(cbfs_graph* gh, const uint32_t* sources, const uint16_t* sizes, uint32_t n_clusters,
                  uint32_t words, uint32_t d, uint32_t dist_bytes, void* out_dist, uint64_t* out_masks,
                  uint32_t planes, uint64_t* out_stats, uint32_t direction, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (words != 1 && words != 2 && words != 4 && words != 8) return fail(CBFS_EUNSUPPORTED, "words must be 1, 2, 4 or 8");
  int rc = check_run_args(g, sources, sizes, n_clusters, d, dist_bytes, planes, direction);
  if (rc) return rc;
  if ((uint64_t)n_clusters * words > 0xFFFFFFFFull) return fail(CBFS_EINVAL, "too many clusters");
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  WorkLease lease(g);
  if (lease.rc) return lease.rc;
  const uint64_t C = n_clusters, L = C * words;
  if (out_dist) CBFS_CUDA(cudaMemsetAsync(out_dist, 0xFF, (uint64_t)g->n * C * dist_bytes, st));
  if (out_masks) CBFS_CUDA(cudaMemsetAsync(out_masks, 0, (uint64_t)planes * g->n * L * sizeof(uint64_t), st));
  if (C == 0) {
    CBFS_CUDA(cudaStreamSynchronize(st));
    return CBFS_OK;
  }
  uint8_t* lane_sizes = nullptr;
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&lane_sizes, L, st));
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  k_wide_prep<<<(unsigned)C, 64 * words, 0, st>>>(sources, sizes, n_clusters, words, g->n, lane_sizes, bad);
  CBFS_LAUNCHED();
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (hbad) {
    cudaFreeAsync(lane_sizes, st);
    cudaFreeAsync(bad, st);
    cudaStreamSynchronize(st);
    return fail(CBFS_EINVAL, (hbad & 1) ? "cluster size must be 1..64*words"
                             : (hbad & 2) ? "source id >= n" : "duplicate source in a cluster");
  }
  ArraySource src;
  src.proto = RunArgs{};
  src.proto.d = d;
  src.proto.planes = planes;
  src.proto.dist_bytes = dist_bytes;
  src.proto.C = (uint32_t)L;
  src.proto.direction = direction;
  src.proto.engine = choose_engine(g, direction);  // both engines advance a batch's lanes in lockstep rounds
  if (src.proto.engine < 0) return CBFS_ECUDA;
  src.proto.out_dist = out_dist;
  src.proto.out_masks = out_masks;
  src.proto.mask_bytes = 8;
  src.proto.wide = words;
  src.sources = sources;  // [C][64 W] is [C W][64]: lane c W + w = word w of cluster c
  src.sizes = lane_sizes;
  src.n_clusters = (uint32_t)L;
  src.out_stats = out_stats;
  rc = run_batches(g, src, st);
  cudaFreeAsync(lane_sizes, st);
  cudaFreeAsync(bad, st);
  if (rc) return rc;
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

int cbfs_select_and_run(cbfs_graph* gh, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy, uint64_t seed,
                        uint32_t* out_sources, uint8_t* out_sizes, uint32_t* out_r, uint32_t dist_bytes,
                        void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
                        uint32_t direction, cbfs_stream stream) {
  return cbfs_select_and_run_shard(gh, r, k, d, root_policy, seed, 1, 0, out_sources, out_sizes, out_r, dist_bytes,
                                   out_dist, out_masks, planes, out_stats, direction, stream);
}

int cbfs_profile_enable(int on) {
  g_prof.on = on != 0;
  return CBFS_OK;
}

int cbfs_release_workspace(int device) {
  if (device < 0 || device >= MAX_DEV) return fail(CBFS_EINVAL, "bad device");
  std::lock_guard<std::mutex> lk(g_work_mu[device]);
  if (g_dev[device].slots.empty()) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(device));
  CBFS_CUDA(cudaDeviceSynchronize());
  work_release(g_dev[device]);
  return CBFS_OK;
}

int cbfs_set_concurrency(int batches) {
  if (batches < 1 || batches > BS_MAX) return fail(CBFS_EINVAL, "concurrency must be 1..8");
  for (int dv = 0; dv < MAX_DEV; ++dv) {  // re-size the slot sets lazily
    std::lock_guard<std::mutex> lk(g_work_mu[dv]);
    if ((int)g_dev[dv].slots.size() != batches && !g_dev[dv].slots.empty()) {
      cudaSetDevice(dv);
      work_release(g_dev[dv]);
    }
  }
  g_max_slots = batches;
  return CBFS_OK;
}

int cbfs_profile_read(double* ms, uint64_t* launches, uint64_t* arcs, uint64_t* entries, uint64_t* u_in,
                      uint64_t* u_out, int reset) {
  for (int k = 0; k < PK_N; ++k) {
    if (ms) ms[k] = g_prof.ms[k];
    if (launches) launches[k] = g_prof.launches[k];
    if (arcs) arcs[k] = g_prof.arcs[k];
    if (entries) entries[k] = g_prof.entries[k];
    if (u_in) u_in[k] = g_prof.u_in[k];
    if (u_out) u_out[k] = g_prof.u_out[k];
  }
  if (reset)
    for (int k = 0; k < PK_N; ++k)
      g_prof.ms[k] = 0, g_prof.launches[k] = g_prof.arcs[k] = g_prof.entries[k] = g_prof.u_in[k] = g_prof.u_out[k] = 0;
  return CBFS_OK;
}

int cbfs_set_pull_hub_rows(uint32_t rows) {
  g_hub_rows = rows;
  return CBFS_OK;
}

int cbfs_set_direction_alpha(double alpha) {
  if (!(alpha > 0)) return fail(CBFS_EINVAL, "alpha must be > 0");
  g_alpha = alpha;
  return CBFS_OK;
}

}  // extern "C"
