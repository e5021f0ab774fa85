// sparse.cu — the SPARSE C-BFS engine: Alg. 1 for a batch of
// LANES = 64 clusters on graphs whose clusters' wavefronts do not overlap
// (high diameter: the road-like grid and the k-NN graph of BASELINE.json
// configs 4 and 5).
//
// Why a second engine: in the BATCHED engine (cbfs.cu) the 64 clusters of a
// batch share one 512-byte state row per vertex, which pays off when their
// frontiers cover the same vertices in the same round (social/web graphs).
// On a 4096^2 grid the 64 clusters' frontiers are 64 disjoint rings, so each
// 32-byte sector of a row carries one useful 8-byte word, and the ~7,400
// rounds each cost a host round trip.  Here:
//  * state is CLUSTER-major: cell[c][v] = {S_seen, Delta, P_0, P_1} in one
//    32-byte sector (P = S_next \ S_seen, double-buffered by round parity);
//    a cluster's frontier band is contiguous along rows of the grid;
//  * rounds are push-only (EdgeMap-Sparse): per frontier entry
//    (c, v) the bits S_new[v] are pushed to the neighbours (R7a: older bits of
//    S_seen[v] reached them in earlier rounds), 64-bit atomicOr into the NEXT
//    pending buffer; the first setter claims the entry (R4);
//  * the round loop runs on the device: one CUDA graph per slot whose
//    conditional WHILE node repeats {fold, push, tail} until the next
//    frontier is empty — no host synchronisation per round.
// Phase order (H9): the fold of round i completes (kernel boundary) before
// the push of round i reads S_seen / Delta of its neighbours, and the push
// writes only the other pending buffer, so the cap (R3) and the
// claim see exactly Alg. 1's post-fold state.
#include <cstdlib>

#include "engine.cuh"

namespace cbfs {

int g_engine_policy = CBFS_ENGINE_AUTO;
// ordered-frontier threshold (cbfs_set_sparse_order): -1 = default, else the
// |F_i| from which claims go to the bitmap (0 = never); env CBFS_SP_BM_MIN
long long g_sp_order_min = getenv("CBFS_SP_BM_MIN") ? atoll(getenv("CBFS_SP_BM_MIN")) : -1;

constexpr uint32_t VBITS = 26;  // list entry = c << 26 | v  (n <= CBFS_MAX_N = 2^26 - 1: never all-ones)
constexpr uint32_t VMASK = (1u << VBITS) - 1;
constexpr int SP_THREADS = 256;
constexpr int SP_WARPS = SP_THREADS / 32;
constexpr uint32_t SP_OUTBUF = 256;  // per-warp claim buffer (entries)
#ifndef CBFS_SP_ILP
#define CBFS_SP_ILP 4
#endif
#ifndef CBFS_SP_GRID_PER_SM
#define CBFS_SP_GRID_PER_SM 8
#endif
constexpr int SP_ILP = CBFS_SP_ILP;  // neighbours per lane in flight (push)
constexpr int SP_FOLD_ILP = 4;       // frontier entries per lane in flight (fold)
// CBFS_SP_DYN (default on): the warps of a round kernel take their chunks of
// the frontier list from a per-round counter (one atomic per chunk) instead of
// a fixed grid stride, and the grid is one wave of resident blocks — degree
// skew (k-NN) and uneven chunk costs no longer leave SMs idle at the tail.
#ifndef CBFS_SP_DYN
#define CBFS_SP_DYN 1
#endif
// Two shapes of the push (measured, configs 4 and 5, 256 clusters): 2
// frontier entries per lane per warp step at 3 blocks / SM for sparse graphs
// (average degree < SP_DEG_SPLIT: the grid, 3.8 — a step then still holds ~240
// arcs), 1 entry per lane at 4 blocks / SM for denser ones (the k-NN graph,
// 11.5: more resident warps, 13% faster there, 13% slower on the grid).
constexpr double SP_DEG_SPLIT = 8.0;
#ifndef CBFS_SP_MINB
#define CBFS_SP_MINB 3
#endif
#ifndef CBFS_SP_EPL
#define CBFS_SP_EPL 2
#endif
template <int V>
struct SpShape;
template <>
struct SpShape<0> {  // low degree
  static constexpr int EPL = CBFS_SP_EPL, MINB = CBFS_SP_MINB;
};
template <>
struct SpShape<1> {  // average degree >= SP_DEG_SPLIT
  static constexpr int EPL = 1, MINB = 4;
};
static unsigned sp_grid(int minb) { return CBFS_SP_DYN ? 148u * minb : 148u * CBFS_SP_GRID_PER_SM; }

// The warp's next chunk [b, b + step) of the round's list: from the shared
// counter (dynamic) or by grid stride.
__device__ __forceinline__ uint64_t sp_next_chunk(unsigned long long* take, uint64_t b, uint64_t step,
                                                  uint64_t stride) {
#if CBFS_SP_DYN
  unsigned long long x = 0;
  if (lane_id() == 0) x = atomicAdd(take, (unsigned long long)step);
  return __shfl_sync(FULLW, x, 0);
#else
  return b + stride;
#endif
}
__device__ __forceinline__ uint64_t sp_first_chunk(unsigned long long* take, uint64_t warp, uint64_t step) {
#if CBFS_SP_DYN
  return sp_next_chunk(take, 0, step, 0);
#else
  return warp * step;
#endif
}

// ------------------------------------------------------------------ init
// Per batch: every cell = {S_seen = 0, Delta = inf, P_0 = P_1 = 0} (A2).
__global__ void k_sp_init(SpCell* __restrict__ cells, uint64_t count) {
  const ulonglong2 a = make_ulonglong2(0ULL, (unsigned long long)INF16), z = make_ulonglong2(0ULL, 0ULL);
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < count;
       t += (uint64_t)gridDim.x * blockDim.x) {
    ulonglong2* p = reinterpret_cast<ulonglong2*>(cells + t);
    p[0] = a;
    p[1] = z;
  }
}

// ------------------------------------------------------------------ seeding
// R1 (S_next[s_j] = {j}, F_0 = S): P_0 of cell (c, s_j) = bit j.
__global__ void k_sp_seed(const uint32_t* __restrict__ sources, const uint8_t* __restrict__ sizes, uint32_t nb,
                          uint32_t n, const uint32_t* __restrict__ inv, SpCell* __restrict__ cells,
                          uint32_t* __restrict__ list0, SpCtl* __restrict__ ctl, int allow_empty) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // 64 threads per cluster
  const uint32_t c = t >> 6, j = t & 63;
  bool claim = false;
  uint32_t e = 0;
  if (c < nb) {
    const uint32_t k = sizes[c];
    if ((k == 0 && !allow_empty) || k > 64) {
      if (j == 0) atomicOr(&ctl->err, ERR_BAD_SIZE);
    } else if (j < k) {
      const uint32_t s = sources[(uint64_t)c * 64 + j];
      if (s >= n) {
        atomicOr(&ctl->err, ERR_BAD_SOURCE);
      } else {
        const uint32_t x = inv ? inv[s] : s;
        const unsigned long long old =
            atomicOr((unsigned long long*)&cells[(uint64_t)c * n + x].p[0], 1ULL << j);
        if (old != 0) atomicOr(&ctl->err, ERR_DUP_SOURCE);  // R2
        else { claim = true; e = (c << VBITS) | x; }
      }
    }
  }
  const unsigned m = __ballot_sync(FULLW, claim);
  if (!m) return;
  unsigned long long base = 0;
  const int leader = __ffs(m) - 1;
  if ((int)lane_id() == leader) base = atomicAdd(&ctl->nF[0], (unsigned long long)__popc(m));
  base = __shfl_sync(FULLW, base, leader);
  if (claim) list0[base + __popc(m & ((1u << lane_id()) - 1))] = e;
}

// ------------------------------------------------------------------ fold
// Vertex phase of round i for every entry of F_i: S_new =
// P_i \ S_seen; Delta on first visit; S_v[i - Delta] = S_new; S_seen |=
// S_new; the output writes; per-cluster statistics.  P_i keeps S_new for the
// push of the same round.

// Output of one folded entry (cluster lane c, vertex v, first visit in round
// dv): Delta on the first visit, S_new into plane i - Delta.  With wide
// clusters (W > 1, cbfs_run_wide, R28) the cluster's Delta is the least first
// visit over its W lanes (their cells at the same vertex; lanes advance in
// lockstep rounds) and out_dist has one column per cluster.
template <int DB>
__device__ __forceinline__ void sp_output(const SpDesc* __restrict__ D, const SpCell* __restrict__ cells, uint32_t n,
                                          uint32_t c, uint32_t v, uint32_t i, uint32_t dv, bool first, uint64_t nw,
                                          bool& overflow) {
  const uint32_t orig = D->perm ? D->perm[v] : v;
  const uint64_t col = (uint64_t)orig * D->C + D->cbase + c;
  uint32_t dc = dv;
  uint64_t dcol = col;
  const uint32_t W = D->wide;
  if (W > 1) {
    const uint32_t c0 = c & ~(W - 1);
    for (uint32_t x = 0; x < W; ++x) dc = min(dc, (uint32_t)cells[(uint64_t)(c0 + x) * n + v].dist);
    dcol = (uint64_t)orig * (D->C / W) + (D->cbase + c) / W;
  }
  if (D->out_cmajor) {  // library staging: Delta at c * n + row, subset i at (i * C + c) * n + row
    dcol = (D->cbase + c) * (uint64_t)n + orig;
    if (DB == 1) overflow |= first && dc == i && i > 254;  // the caller asked for u8 Delta (staging keeps u16)
    if (first && D->out_dist && dc == i) ((uint16_t*)D->out_dist)[dcol] = (uint16_t)i;
    const uint32_t oi = i - dc;
    if (D->out_masks && oi < D->planes)
      store_mask(D->out_masks, ((uint64_t)oi * D->C + D->cbase + c) * n + orig, nw, D->mask_bytes);
    return;
  }
  if (first && D->out_dist && dc == i) {
    if (DB == 1) {
      overflow |= i > 254;
      ((uint8_t*)D->out_dist)[dcol] = (uint8_t)(i > 254 ? 254 : i);
    } else {
      ((uint16_t*)D->out_dist)[dcol] = (uint16_t)i;
    }
  }
  const uint32_t oi = i - dc;
  if (D->out_masks && oi < D->planes) store_mask(D->out_masks, (uint64_t)oi * n * D->C + col, nw, D->mask_bytes);
}

// {S_seen, Delta} of a neighbour's cell in the push.  In the FUSED kernel the
// cell may be folded by another thread of the same launch, so the read is a
// relaxed (coherent, non-.nc) load: each 64-bit half is the value before or
// after that fold, and either is harmless (see the FUSED note at k_sp_push).
// Without fusion no cell is written during the push: read-only path.
__device__ __forceinline__ ulonglong2 ld_cell(const SpCell* p, bool fused) {
  if (!fused) return __ldg(reinterpret_cast<const ulonglong2*>(p));
  ulonglong2 r;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
  return r;
}

// per-round record {|F_i|, E_i} of cluster lane c (cbfs_run_rounds)
__device__ __forceinline__ void sp_round_record(const SpDesc* __restrict__ D, uint32_t c, uint32_t i,
                                                unsigned long long f, unsigned long long e) {
  if (!D->rounds || i >= D->max_rounds) return;
  uint64_t* r = D->rounds + ((uint64_t)c * D->max_rounds + i) * 2;
  atomicAdd((unsigned long long*)&r[0], f);
  atomicAdd((unsigned long long*)&r[1], e);
}

template <int DB>
__global__ void __launch_bounds__(SP_THREADS) k_sp_fold(const SpDesc* __restrict__ D, SpCtl* __restrict__ ctl,
                                                        SpCell* __restrict__ cells,
                                                        const uint32_t* __restrict__ list0,
                                                        const uint32_t* __restrict__ list1,
                                                        uint64_t* __restrict__ bstats) {
  __shared__ unsigned long long sF[LANES], sE[LANES], sM[LANES];
  for (uint32_t c = threadIdx.x; c < LANES; c += blockDim.x) sF[c] = sE[c] = sM[c] = 0;
  __syncthreads();
  const uint32_t i = (uint32_t)ctl->i;
  const uint32_t cur = i & 1;
  const uint32_t* __restrict__ L = cur ? list1 : list0;
  const uint64_t nF = ctl->nF[cur];
  const uint32_t n = D->n;
  const uint64_t* __restrict__ off = D->off;
  void* __restrict__ out_dist = D->out_dist;
  void* __restrict__ out_masks = D->out_masks;
  const uint32_t lane = lane_id();
  bool overflow = false;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b = sp_first_chunk(&ctl->take[0], warp, 32 * SP_FOLD_ILP); b < nF;
       b = sp_next_chunk(&ctl->take[0], b, 32 * SP_FOLD_ILP, nwarps * 32 * SP_FOLD_ILP)) {
    // SP_FOLD_ILP entries per lane: all their loads are issued before any is used
    uint32_t e[SP_FOLD_ILP];
    ulonglong2 sd[SP_FOLD_ILP];
    uint64_t p[SP_FOLD_ILP], o0[SP_FOLD_ILP], o1[SP_FOLD_ILP];
#pragma unroll
    for (int q = 0; q < SP_FOLD_ILP; ++q) {
      const uint64_t t = b + q * 32 + lane;
      e[q] = t < nF ? L[t] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int q = 0; q < SP_FOLD_ILP; ++q) {
      if (e[q] == 0xFFFFFFFFu) continue;
      const uint32_t v = e[q] & VMASK;
      const SpCell* cell = cells + (uint64_t)(e[q] >> VBITS) * n + v;
      sd[q] = *reinterpret_cast<const ulonglong2*>(cell);  // {S_seen, Delta}
      p[q] = cell->p[cur];
      o0[q] = off[v];
      o1[q] = off[v + 1];
    }
#pragma unroll
    for (int q = 0; q < SP_FOLD_ILP; ++q) {
      uint32_t c = LANES, deg = 0;
      bool act = false, first = false;
      if (e[q] != 0xFFFFFFFFu) {
        c = e[q] >> VBITS;
        const uint32_t v = e[q] & VMASK;
        SpCell* cell = cells + (uint64_t)c * n + v;
        const uint64_t nw = p[q] & ~sd[q].x;
        if (nw != p[q]) cell->p[cur] = nw;
        if (nw) {
          act = true;
          uint32_t dv = (uint32_t)sd[q].y;
          first = dv == INF16;
          if (first) dv = i;
          *reinterpret_cast<ulonglong2*>(cell) = make_ulonglong2(sd[q].x | nw, (unsigned long long)dv);
          deg = (uint32_t)(o1[q] - o0[q]);
          if (out_dist || out_masks) sp_output<DB>(D, cells, n, c, v, i, dv, first, nw, overflow);
        }
      }
      // per-cluster statistics, one shared atomic per distinct cluster in the warp
      const unsigned grp = __match_any_sync(FULLW, act ? c : 0xFFFFFFFFu);
      const uint32_t fsum = __reduce_add_sync(grp, act ? 1u : 0u);
      const uint32_t esum = __reduce_add_sync(grp, act ? deg : 0u);
      const uint32_t msum = __reduce_add_sync(grp, act && first ? deg : 0u);
      if (act && lane == (uint32_t)(__ffs(grp) - 1)) {
        atomicAdd(&sF[c], (unsigned long long)fsum);
        atomicAdd(&sE[c], (unsigned long long)esum);
        if (msum) atomicAdd(&sM[c], (unsigned long long)msum);
      }
    }
  }
  if (overflow) atomicOr(&ctl->err, ERR_OVERFLOW);
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < LANES; c += blockDim.x) {
    if (!sF[c]) continue;
    atomicAdd((unsigned long long*)&bstats[c * 4 + 1], sF[c]);
    atomicAdd((unsigned long long*)&bstats[c * 4 + 2], sE[c]);
    if (sM[c]) atomicAdd((unsigned long long*)&bstats[c * 4 + 3], sM[c]);
    atomicMax((unsigned long long*)&bstats[c * 4 + 0], (unsigned long long)(i + 1));
    sp_round_record(D, c, i, sF[c], sE[c]);
  }
}

// ------------------------------------------------------------------ round end
// End of round i, run by the last block of the push to finish (no separate
// tail kernel): F_i is consumed, i advances, and the graph's WHILE node
// repeats while F_{i+1} is non-empty (Alg. 1's loop).
// Ordered frontiers (CBFS_SP_ORDER, default on): when F_i is large (>=
// SpDesc::bm_min entries) the push of round i records its claims as bits of a
// cluster-major bitmap instead of appending them to the list in claim order,
// and a compaction kernel turns the bitmap into F_{i+1} sorted by (cluster,
// vertex) runs — the next round's pushes then walk each cluster's band in id
// order, so the neighbour cells they read and OR share L2 lines instead of
// arriving in scattered order.  Which entries F_{i+1} holds is unchanged
// (each claim is the unique 0 -> non-zero transition of P_{i+1}), only their
// order, and every consumer of a frontier is order-independent.
#ifndef CBFS_SP_ORDER
#define CBFS_SP_ORDER 1
#endif

__device__ __forceinline__ void sp_round_end(SpCtl* __restrict__ ctl, cudaGraphConditionalHandle h,
                                             cudaGraphConditionalHandle h_bm, uint64_t bm_min) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  __threadfence();
  const unsigned prev = atomicAdd(&ctl->done, 1u);
  if (prev != gridDim.x - 1) return;
  __threadfence();
  volatile SpCtl* v = ctl;
  const unsigned long long i = v->i;
  const uint32_t cur = i & 1;
  v->listed = v->listed + v->nF[cur];
  v->nF[cur] = 0;
  const unsigned long long nn = v->nF[cur ^ 1];
  v->i = i + 1;
  v->done = 0;
  v->take[0] = 0;  // every block of this round's kernels has left its chunk loop
  v->take[1] = 0;
  bool go = nn > 0;
  if (go && i + 1 >= 0xFFFEull) {
    atomicOr(&ctl->err, ERR_ROUNDS);
    go = false;
  }
  v->go = go;
  v->bm_fill = 0;
  const bool bm = bm_min && nn >= bm_min;  // the claim target of round i + 1
  v->bm = bm ? 1 : 0;
  if (h) cudaGraphSetConditional(h, go ? 1u : 0u);  // h == 0: host-driven loop (profiling mode)
  if (h_bm) cudaGraphSetConditional(h_bm, bm ? 1u : 0u);
}

// Bitmap -> list F_{i+1} (after round i's push, which advanced ctl->i): warp
// per 32 consecutive bitmap words, entries appended as one run per warp in
// (cluster, vertex) order; the words are cleared (the bitmap is zero between
// rounds).
__global__ void __launch_bounds__(256) k_sp_compact(const SpDesc* __restrict__ D, SpCtl* __restrict__ ctl,
                                                    uint32_t* __restrict__ list0, uint32_t* __restrict__ list1) {
  const uint32_t nw32 = D->nw32;
  const uint64_t words = (uint64_t)D->nb * nw32;
  uint32_t* __restrict__ bits = D->bits;
  uint32_t* __restrict__ Ln = (ctl->i & 1) ? list1 : list0;  // ctl->i is already i + 1
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w0 = warp * 32; w0 < words; w0 += nwarps * 32) {
    const uint64_t wi = w0 + lane;
    uint32_t x = 0;
    if (wi < words) {
      x = bits[wi];
      if (x) bits[wi] = 0;
    }
    const uint32_t k = __popc(x);
    uint32_t inc = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULLW, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    const uint32_t tot = __shfl_sync(FULLW, inc, 31);
    if (!tot) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&ctl->bm_fill, (unsigned long long)tot);
    base = __shfl_sync(FULLW, base, 0) + (inc - k);
    if (x) {
      const uint32_t c = (uint32_t)(wi / nw32), v0 = (uint32_t)(wi - (uint64_t)c * nw32) * 32;
      while (x) {
        const uint32_t b = __ffs(x) - 1;
        x &= x - 1;
        CBFS_DCHECK(v0 + b < D->n && c < LANES);
        Ln[base++] = (c << VBITS) | (v0 + b);
      }
    }
  }
}

// ------------------------------------------------------------------ push
// Edge phase of round i: for every entry (c, v) of F_i and u in
// N(v) with cap(u) (Delta_u = inf or i - Delta_u < d, R3): x =
// S_new[v] \ S_seen[u]; if x != 0, atomicOr(P_{i+1}[c][u], x); the op that
// turns P_{i+1}[c][u] non-zero appends (c, u) to F_{i+1} (R4).  P_i[c][v] is
// cleared once read, so both pending buffers are zero when the batch ends.
// S_seen and Delta are not written during the push: read-only loads.
// The warp takes SP_EPL * 32 frontier entries at a time, loads their S_new
// and degree ranges together, and then walks the concatenation of their
// neighbour lists SP_ILP * 32 arcs at a time (each lane finds its arcs'
// entries by a binary search over the warp's degree prefix in shared memory),
// so every lane keeps several independent memory operations in flight and
// hubs and degree-4 grid vertices are balanced alike.

//
// FUSED (d >= 1): the fold of each entry runs in the same thread right before
// its push, so a round is one kernel.  A pusher may then read a neighbour's
// {S_seen, Delta} before that neighbour's own fold of this round: a stale
// Delta = inf passes the cap exactly like the post-fold Delta = i does when d
// >= 1 (H9), and bits the neighbour is folding this round may be pushed into
// its P_{i+1} again — they are masked by the next fold (S_new = P \ S_seen),
// and an entry whose S_new comes out empty is skipped (no output, statistic
// or push), so outputs and round statistics are exactly Alg. 1's.  d = 0 uses
// the separate fold kernel (there the post-fold cap differs).
template <int DB, bool FUSED, int V, bool BM>
__global__ void __launch_bounds__(SP_THREADS, SpShape<V>::MINB) k_sp_push(const SpDesc* __restrict__ D, SpCtl* __restrict__ ctl,
                                                        SpCell* __restrict__ cells, uint32_t* __restrict__ list0,
                                                        uint32_t* __restrict__ list1, uint64_t* __restrict__ bstats,
                                                        cudaGraphConditionalHandle hcond,
                                                        cudaGraphConditionalHandle hbm) {
  constexpr int SP_EPL = SpShape<V>::EPL;  // frontier entries per lane per warp step
  constexpr int W = 32 * SP_EPL;           // entries per warp step
  __shared__ unsigned long long sF[FUSED ? LANES : 1], sE[FUSED ? LANES : 1], sM[FUSED ? LANES : 1];
  if (FUSED) {
    for (uint32_t c = threadIdx.x; c < LANES; c += blockDim.x) sF[c] = sE[c] = sM[c] = 0;
    __syncthreads();
  }
  bool overflow = false;
  __shared__ uint32_t s_out[SP_WARPS][SP_OUTBUF];
  __shared__ uint32_t s_pre[SP_WARPS][W + 1];
  __shared__ uint32_t s_c[SP_WARPS][W];
  __shared__ uint64_t s_beg[SP_WARPS][W];
  __shared__ uint64_t s_nw[SP_WARPS][W];
  const uint32_t wib = threadIdx.x >> 5;
  uint32_t* pre = s_pre[wib];
  uint32_t* sc = s_c[wib];
  uint64_t* sbeg = s_beg[wib];
  uint64_t* snw = s_nw[wib];
  const uint32_t i = (uint32_t)ctl->i;
  const uint32_t cur = i & 1, nxt = cur ^ 1;
  const uint32_t* __restrict__ L = cur ? list1 : list0;
  uint32_t* __restrict__ Ln = cur ? list0 : list1;
  unsigned long long* cnt = &ctl->nF[nxt];
  const uint64_t nF = ctl->nF[cur];
  const uint32_t n = D->n, d = D->d;
  const uint64_t* __restrict__ off = D->off;
  const uint32_t* __restrict__ cols = D->cols;
  const uint32_t lane = lane_id();
  const unsigned lt = (1u << lane) - 1;
  uint32_t* obuf = s_out[wib];
  uint32_t nout = 0;
  constexpr bool bm = BM;  // this round's claims go to the ordered bitmap
  auto emit = [&](bool claim, uint32_t val) {
    const unsigned m = __ballot_sync(FULLW, claim);
    if (bm) {  // nout counts the warp's bitmap claims (added to F_{i+1}'s size at the end)
      if (claim) {
        const uint32_t c = val >> VBITS, u = val & VMASK;
        atomicOr(&D->bits[(uint64_t)c * D->nw32 + (u >> 5)], 1u << (u & 31));
      }
      nout += __popc(m);
      return;
    }
    if (claim) obuf[nout + __popc(m & lt)] = val;
    nout += __popc(m);
    if (nout > SP_OUTBUF - 32) {
      __syncwarp();
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(cnt, (unsigned long long)nout);
      base = __shfl_sync(FULLW, base, 0);
      CBFS_DCHECK(base + nout <= (uint64_t)n * LANES);
      for (uint32_t q = lane; q < nout; q += 32) Ln[base + q] = obuf[q];
      __syncwarp();
      nout = 0;
    }
  };
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b = sp_first_chunk(&ctl->take[1], warp, W); b < nF; b = sp_next_chunk(&ctl->take[1], b, W, nwarps * W)) {
    // ---- the step's entries: S_new (cleared once read) and neighbour ranges
    uint32_t e[SP_EPL];
    uint64_t nw[SP_EPL], o0[SP_EPL], o1[SP_EPL];
#pragma unroll
    for (int q = 0; q < SP_EPL; ++q) {
      const uint64_t t = b + q * 32 + lane;
      e[q] = t < nF ? L[t] : 0xFFFFFFFFu;
    }
    ulonglong2 sd0[SP_EPL];
#pragma unroll
    for (int q = 0; q < SP_EPL; ++q) {
      nw[q] = 0;
      o0[q] = o1[q] = 0;
      if (e[q] != 0xFFFFFFFFu) {
        const uint32_t v = e[q] & VMASK;
        const SpCell* cell = cells + (uint64_t)(e[q] >> VBITS) * n + v;
        nw[q] = cell->p[cur];
        if (FUSED) sd0[q] = *reinterpret_cast<const ulonglong2*>(cell);  // {S_seen, Delta}
        o0[q] = off[v];
        o1[q] = off[v + 1];
      }
    }
    if (FUSED) {  // the fold of the step's entries
#pragma unroll
      for (int q = 0; q < SP_EPL; ++q) {
        uint32_t c = LANES, deg = 0;
        bool act = false, first = false;
        if (e[q] != 0xFFFFFFFFu) {
          c = e[q] >> VBITS;
          const uint32_t v = e[q] & VMASK;
          SpCell* cell = cells + (uint64_t)c * n + v;
          const uint64_t p = nw[q];
          nw[q] = p & ~sd0[q].x;
          if (nw[q]) {
            act = true;
            uint32_t dv = (uint32_t)sd0[q].y;
            first = dv == INF16;
            if (first) dv = i;
            *reinterpret_cast<ulonglong2*>(cell) = make_ulonglong2(sd0[q].x | nw[q], (unsigned long long)dv);
            deg = (uint32_t)(o1[q] - o0[q]);
            if (D->out_dist || D->out_masks) sp_output<DB>(D, cells, n, c, v, i, dv, first, nw[q], overflow);
          }
          if (p) cell->p[cur] = 0;
        }
        const unsigned grp = __match_any_sync(FULLW, act ? c : 0xFFFFFFFFu);
        const uint32_t fsum = __reduce_add_sync(grp, act ? 1u : 0u);
        const uint32_t esum = __reduce_add_sync(grp, act ? deg : 0u);
        const uint32_t msum = __reduce_add_sync(grp, act && first ? deg : 0u);
        if (act && lane == (uint32_t)(__ffs(grp) - 1)) {
          atomicAdd(&sF[c], (unsigned long long)fsum);
          atomicAdd(&sE[c], (unsigned long long)esum);
          if (msum) atomicAdd(&sM[c], (unsigned long long)msum);
        }
      }
    }
    uint32_t base = 0;
#pragma unroll
    for (int q = 0; q < SP_EPL; ++q) {
      if (!FUSED && nw[q]) cells[(uint64_t)(e[q] >> VBITS) * n + (e[q] & VMASK)].p[cur] = 0;
      const uint32_t deg = nw[q] ? (uint32_t)(o1[q] - o0[q]) : 0u;
      uint32_t inc = deg;  // inclusive warp scan of the degrees
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULLW, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      const int idx = q * 32 + lane;
      pre[idx] = base + inc - deg;
      sc[idx] = e[q] >> VBITS;
      sbeg[idx] = o0[q];
      snw[idx] = nw[q];
      base += __shfl_sync(FULLW, inc, 31);
    }
    if (lane == 0) pre[W] = base;
    __syncwarp();
    // ---- the step's arcs, SP_ILP * 32 at a time
    for (uint32_t a0 = 0; a0 < base; a0 += 32 * SP_ILP) {
      uint32_t u[SP_ILP], cq[SP_ILP];
      uint64_t nq[SP_ILP];
      ulonglong2 sd[SP_ILP];
      bool claim[SP_ILP];
#pragma unroll
      for (int r = 0; r < SP_ILP; ++r) {
        const uint32_t a = a0 + r * 32 + lane;
        u[r] = 0xFFFFFFFFu;
        if (a < base) {
          int lo = 0, hi = W;  // largest idx with pre[idx] <= a
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pre[mid] <= a) lo = mid; else hi = mid;
          }
          cq[r] = sc[lo];
          nq[r] = snw[lo];
          u[r] = cols[sbeg[lo] + (a - pre[lo])];
          CBFS_DCHECK(u[r] < n && cq[r] < LANES);
        }
      }
#pragma unroll
      for (int r = 0; r < SP_ILP; ++r)
        if (u[r] != 0xFFFFFFFFu) sd[r] = ld_cell(cells + (uint64_t)cq[r] * n + u[r], FUSED);
#pragma unroll
      for (int r = 0; r < SP_ILP; ++r) {
        claim[r] = false;
        if (u[r] == 0xFFFFFFFFu) continue;
        const uint32_t du = (uint32_t)sd[r].y;
        if (du != INF16 && (int)i - (int)du >= (int)d) continue;  // cap, R3
        const uint64_t x = nq[r] & ~sd[r].x;
        if (x)
          claim[r] = atomicOr((unsigned long long*)&cells[(uint64_t)cq[r] * n + u[r]].p[nxt],
                              (unsigned long long)x) == 0ULL;
      }
#pragma unroll
      for (int r = 0; r < SP_ILP; ++r) emit(claim[r], claim[r] ? ((cq[r] << VBITS) | u[r]) : 0u);
    }
    __syncwarp();
  }
  __syncwarp();
  if (bm) {
    if (lane == 0 && nout) atomicAdd(cnt, (unsigned long long)nout);
    nout = 0;
  }
  if (nout) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cnt, (unsigned long long)nout);
    base = __shfl_sync(FULLW, base, 0);
    for (uint32_t q = lane; q < nout; q += 32) Ln[base + q] = obuf[q];
  }
  if (FUSED) {
    if (overflow) atomicOr(&ctl->err, ERR_OVERFLOW);
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < LANES; c += blockDim.x) {
      if (!sF[c]) continue;
      atomicAdd((unsigned long long*)&bstats[c * 4 + 1], sF[c]);
      atomicAdd((unsigned long long*)&bstats[c * 4 + 2], sE[c]);
      if (sM[c]) atomicAdd((unsigned long long*)&bstats[c * 4 + 3], sM[c]);
      atomicMax((unsigned long long*)&bstats[c * 4 + 0], (unsigned long long)(i + 1));
      sp_round_record(D, c, i, sF[c], sE[c]);
    }
  }
  sp_round_end(ctl, hcond, hbm, D->bm_min);
}

// ------------------------------------------------------------------ host
static int sp_add_kernel(cudaGraph_t body, cudaGraphNode_t* node, const cudaGraphNode_t* dep, void* fn, unsigned grid,
                         unsigned block, void** args) {
  cudaKernelNodeParams kp = {};
  kp.func = fn;
  kp.gridDim = dim3(grid);
  kp.blockDim = dim3(block);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  CBFS_CUDA(cudaGraphAddKernelNode(node, body, dep, dep ? 1 : 0, &kp));
  return CBFS_OK;
}

// The per-slot round-loop graph: WHILE (F_i non-empty) { [fold;] push } (the
// push's last block ends the round).
// Two graphs per slot would be needed for the two Delta output widths; the
// fold instance is chosen by dist_bytes when the graph is (re)built.
// The push instance of (Delta width, fusion, shape, ordered claims).
template <bool BM>
static void* sp_push_fn_bm(uint32_t dist_bytes, bool fused, int shape) {
  if (!fused) return shape ? (void*)k_sp_push<2, false, 1, BM> : (void*)k_sp_push<2, false, 0, BM>;
  if (dist_bytes == 1) return shape ? (void*)k_sp_push<1, true, 1, BM> : (void*)k_sp_push<1, true, 0, BM>;
  return shape ? (void*)k_sp_push<2, true, 1, BM> : (void*)k_sp_push<2, true, 0, BM>;
}
static void* sp_push_fn(uint32_t dist_bytes, bool fused, int shape, bool bm) {
  return bm ? sp_push_fn_bm<true>(dist_bytes, fused, shape) : sp_push_fn_bm<false>(dist_bytes, fused, shape);
}
static int sp_minb(int shape) { return shape ? SpShape<1>::MINB : SpShape<0>::MINB; }

constexpr unsigned SP_COMPACT_GRID = 148u * 8u;

static int sp_build(Slot* w, uint32_t dist_bytes, bool fused, int shape, bool ordered) {
  if (w->sp_exec) {
    CBFS_CUDA(cudaGraphExecDestroy(w->sp_exec));
    w->sp_exec = nullptr;
  }
  if (w->sp_graph) {
    CBFS_CUDA(cudaGraphDestroy(w->sp_graph));
    w->sp_graph = nullptr;
  }
  cudaGraph_t g;
  CBFS_CUDA(cudaGraphCreate(&g, 0));
  w->sp_graph = g;
  cudaGraphConditionalHandle h, hc = 0;  // hc == 0: no ordered-frontier branch (the push sets no IF handle)
  CBFS_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  if (ordered)  // round 0 claims into the list
    CBFS_CUDA(cudaGraphConditionalHandleCreate(&hc, g, 0, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond;
  CBFS_CUDA(cudaGraphAddNode(&cond, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  SpDesc* D = w->sp_desc;
  SpCtl* ctl = w->sp_ctl;
  SpCell* cells = reinterpret_cast<SpCell*>(w->blk);
  uint32_t* l0 = w->listA;
  uint32_t* l1 = w->listB;
  void* fa[] = {&D, &ctl, &cells, &l0, &l1, &w->bstats};
  void* pa[] = {&D, &ctl, &cells, &l0, &l1, &w->bstats, &h, &hc};
  void* ca[] = {&D, &ctl, &l0, &l1};
  cudaGraphNode_t nf, ni, np1, nc, np0;
  int rc;
  if (!fused) {  // d = 0: the fold is its own kernel
    rc = sp_add_kernel(body, &nf, nullptr, dist_bytes == 1 ? (void*)k_sp_fold<1> : (void*)k_sp_fold<2>,
                       sp_grid(CBFS_SP_MINB), SP_THREADS, fa);
    if (rc) return rc;
  }
  const uint32_t pdb = fused ? dist_bytes : 2;
  if (!ordered) {  // list frontiers only: the push alone
    rc = sp_add_kernel(body, &np0, fused ? nullptr : &nf, sp_push_fn(pdb, fused, shape, false),
                       sp_grid(sp_minb(shape)), SP_THREADS, pa);
    if (rc) return rc;
  } else {  // IF (round i's claims go to the ordered bitmap) { push; compact into F_{i+1} } ELSE { push }
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hc;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 2;
    CBFS_CUDA(cudaGraphAddNode(&ni, body, fused ? nullptr : &nf, fused ? 0 : 1, &ip));
    cudaGraph_t g_bm = ip.conditional.phGraph_out[0], g_list = ip.conditional.phGraph_out[1];
    rc = sp_add_kernel(g_bm, &np1, nullptr, sp_push_fn(pdb, fused, shape, true), sp_grid(sp_minb(shape)),
                       SP_THREADS, pa);
    if (!rc) rc = sp_add_kernel(g_bm, &nc, &np1, (void*)k_sp_compact, SP_COMPACT_GRID, 256, ca);
    if (!rc)
      rc = sp_add_kernel(g_list, &np0, nullptr, sp_push_fn(pdb, fused, shape, false), sp_grid(sp_minb(shape)),
                         SP_THREADS, pa);
    if (rc) return rc;
  }
  CBFS_CUDA(cudaGraphInstantiate(&w->sp_exec, g, 0));
  w->sp_db = dist_bytes;
  w->sp_fused = fused;
  w->sp_shape = shape;
  w->sp_ordered = ordered;
  return CBFS_OK;
}

int sparse_alloc(Slot* w) {
  CBFS_CUDA(cudaMalloc(&w->sp_desc, sizeof(SpDesc)));
  CBFS_CUDA(cudaMallocHost(&w->sp_desc_h, sizeof(SpDesc)));
  CBFS_CUDA(cudaMalloc(&w->sp_ctl, sizeof(SpCtl)));
  CBFS_CUDA(cudaMallocHost(&w->sp_ctl_h, sizeof(SpCtl)));
  CBFS_CUDA(cudaEventCreate(&w->sp_t0));
  CBFS_CUDA(cudaEventCreate(&w->sp_t1));
  return CBFS_OK;
}

void sparse_free(Slot* w) {
  if (w->sp_exec) cudaGraphExecDestroy(w->sp_exec);
  if (w->sp_graph) cudaGraphDestroy(w->sp_graph);
  cudaFree(w->sp_desc);
  cudaFreeHost(w->sp_desc_h);
  cudaFree(w->sp_ctl);
  cudaFreeHost(w->sp_ctl_h);
  if (w->sp_t0) cudaEventDestroy(w->sp_t0);
  if (w->sp_t1) cudaEventDestroy(w->sp_t1);
  if (w->sp_bits) cudaFree(w->sp_bits);
}

int sparse_start(const Graph* g, Slot* w, const RunArgs& a) {
  const uint32_t n = g->n;
  cudaStream_t st = w->s;
  const bool fused = a.d >= 1;
  const int shape = g->m >= SP_DEG_SPLIT * (double)n ? 1 : 0;
  // ordered frontiers for the denser shape only: on low-degree graphs (the
  // grid: thousands of small rounds) the compaction never pays (measured at
  // every threshold) and the IF node alone costs ~1%
  const long long bm_set = g_sp_order_min;
  const uint64_t bm_min = bm_set >= 0 ? (uint64_t)bm_set
                                      : (CBFS_SP_ORDER && shape == 1 ? std::max<uint64_t>(n / 4, 1u << 16) : 0);
  const bool ordered = bm_min != 0;
  if (!w->sp_exec || w->sp_db != a.dist_bytes || w->sp_fused != fused || w->sp_shape != shape ||
      w->sp_ordered != ordered) {
    int rc = sp_build(w, a.dist_bytes, fused, shape, ordered);
    if (rc) return rc;
  }
  SpDesc* h = w->sp_desc_h;  // the slot's previous batch (and its copy) finished before this one starts
  h->off = g->off;
  h->cols = g->cols;
  h->perm = a.out_internal ? nullptr : g->perm;  // output rows: original ids unless library staging
  h->inv = g->inv;
  h->sources = a.sources;
  h->sizes = a.sizes;
  h->out_dist = a.out_dist;
  h->out_masks = a.out_masks;
  h->C = a.C;
  h->cbase = a.cbase;
  h->n = n;
  h->nb = a.nb;
  h->d = a.d;
  h->planes = a.planes;
  h->dist_bytes = a.dist_bytes;
  h->mask_bytes = a.mask_bytes ? a.mask_bytes : 8;
  h->wide = a.wide > 1 ? a.wide : 1;
  h->out_cmajor = a.out_cmajor;
  h->rounds = a.out_rounds;
  h->max_rounds = a.out_rounds ? a.max_rounds : 0;
  // the ordered-frontier bitmap (zero between rounds; sized for this graph)
  h->nw32 = (n + 31) / 32;
  const uint64_t words = (uint64_t)LANES * h->nw32;
  if (bm_min && w->sp_bits_words < words) {
    if (w->sp_bits) CBFS_CUDA(cudaFree(w->sp_bits));
    w->sp_bits = nullptr;
    w->sp_bits_words = 0;
    CBFS_CUDA(cudaMalloc(&w->sp_bits, words * sizeof(uint32_t)));
    CBFS_CUDA(cudaMemsetAsync(w->sp_bits, 0, words * sizeof(uint32_t), st));
    w->sp_bits_words = words;
  }
  h->bits = bm_min ? w->sp_bits : nullptr;
  h->bm_min = bm_min;
  CBFS_CUDA(cudaMemcpyAsync(w->sp_desc, h, sizeof(SpDesc), cudaMemcpyHostToDevice, st));
  const uint64_t ncell = (uint64_t)n * LANES;
  k_sp_init<<<grid_for(ncell, 256, 148u * 16u), 256, 0, st>>>(reinterpret_cast<SpCell*>(w->blk), ncell);
  CBFS_LAUNCHED();
  CBFS_CUDA(cudaMemsetAsync(w->bstats, 0, LANES * 4 * sizeof(uint64_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->sp_ctl, 0, sizeof(SpCtl), st));
  k_sp_seed<<<(a.nb * 64 + 255) / 256, 256, 0, st>>>(a.sources, a.sizes, a.nb, n, g->inv,
                                                     reinterpret_cast<SpCell*>(w->blk), w->listA, w->sp_ctl,
                                                     a.wide > 1);
  CBFS_LAUNCHED();
  CBFS_CUDA(cudaMemcpyAsync(w->sp_ctl_h, w->sp_ctl, sizeof(SpCtl), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaEventRecord(w->ready, st));
  return CBFS_OK;
}

// Profiling aid (env CBFS_SPARSE_HOSTLOOP=1): the same kernels launched one
// by one with a host round trip per round, so that ncu (which cannot profile
// kernel nodes of graphs with conditional nodes) sees them.  Synchronous.
static int sparse_hostloop(Slot* w) {
  cudaStream_t st = w->s;
  SpDesc* D = w->sp_desc;
  SpCtl* ctl = w->sp_ctl;
  CBFS_CUDA(cudaEventRecord(w->sp_t0, st));
  bool bm_next = false;  // round 0 claims into the list (as the graph's IF handle default)
  for (;;) {
    SpCell* cells = reinterpret_cast<SpCell*>(w->blk);
    cudaGraphConditionalHandle h0 = 0;
    void* pa[] = {&D, &ctl, &cells, &w->listA, &w->listB, &w->bstats, &h0, &h0};
    void* ca[] = {&D, &ctl, &w->listA, &w->listB};
    void* fa[] = {&D, &ctl, &cells, &w->listA, &w->listB, &w->bstats};
    if (!w->sp_fused)
      CBFS_CUDA(cudaLaunchKernel(w->sp_db == 1 ? (void*)k_sp_fold<1> : (void*)k_sp_fold<2>, sp_grid(CBFS_SP_MINB),
                                 SP_THREADS, fa, 0, st));
    const bool bm = bm_next;
    CBFS_CUDA(cudaLaunchKernel(sp_push_fn(w->sp_fused ? w->sp_db : 2, w->sp_fused, w->sp_shape, bm),
                               sp_grid(sp_minb(w->sp_shape)), SP_THREADS, pa, 0, st));
    if (bm) CBFS_CUDA(cudaLaunchKernel((void*)k_sp_compact, SP_COMPACT_GRID, 256, ca, 0, st));
    CBFS_CUDA(cudaMemcpyAsync(w->sp_ctl_h, ctl, sizeof(SpCtl), cudaMemcpyDeviceToHost, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    bm_next = w->sp_ctl_h->bm != 0;
    if (!w->sp_ctl_h->go) break;
  }
  CBFS_CUDA(cudaEventRecord(w->sp_t1, st));
  CBFS_CUDA(cudaMemcpyAsync(w->sp_ctl_h, ctl, sizeof(SpCtl), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaEventRecord(w->ready, st));
  return CBFS_OK;
}

int sparse_launch(Slot* w) {
  static const bool hostloop = getenv("CBFS_SPARSE_HOSTLOOP") != nullptr;
  if (hostloop) return sparse_hostloop(w);
  cudaStream_t st = w->s;
  CBFS_CUDA(cudaEventRecord(w->sp_t0, st));
  CBFS_CUDA(cudaGraphLaunch(w->sp_exec, st));
  CBFS_CUDA(cudaEventRecord(w->sp_t1, st));
  CBFS_CUDA(cudaMemcpyAsync(w->sp_ctl_h, w->sp_ctl, sizeof(SpCtl), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaEventRecord(w->ready, st));
  return CBFS_OK;
}

// ------------------------------------------------------------------ engine choice
// AUTO: a graph with a vertex of degree > PROBE_MAX_DEGREE is taken as low
// diameter (BATCHED); otherwise a plain BFS from the highest-degree vertex
// decides: if it is still running after PROBE_ROUNDS levels the graph is
// "high diameter" and the clusters' wavefronts will not share state rows ->
// SPARSE, else BATCHED.  Cached per graph handle.  Parity-neutral: both
// engines compute Alg. 1 exactly.
constexpr uint32_t PROBE_ROUNDS = 48;
constexpr uint32_t PROBE_MAX_DEGREE = 256;

// One bottom-up BFS level (P:1769-1782 for a single source): every
// unvisited vertex looks for a neighbour on level `lvl` (first hit wins), so
// no thread walks a hub's whole neighbour list.
__global__ void k_probe_level(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, uint32_t n,
                              uint8_t* __restrict__ level, uint32_t lvl, unsigned long long* __restrict__ cnt) {
  uint32_t found = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    if (level[v] != 0xFF) continue;
    for (uint64_t a = off[v]; a < off[v + 1]; ++a)
      if (level[cols[a]] == lvl) {
        level[v] = (uint8_t)(lvl + 1);  // read only as "== lvl" in this launch: no race
        ++found;
        break;
      }
  }
  const unsigned long long s = warp_sum(found);
  if (lane_id() == 0 && s) atomicAdd(cnt, s);
}

static int probe_high_diameter(Graph* g, int* out) {
  const uint32_t n = g->n;
  *out = 0;
  if (n == 0 || g->m == 0) return CBFS_OK;
  cudaStream_t st;
  CBFS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  uint8_t* level = nullptr;
  unsigned long long* cnt = nullptr;
  unsigned long long* h = nullptr;
  CBFS_CUDA(cudaMallocAsync(&level, n, st));
  CBFS_CUDA(cudaMallocAsync(&cnt, sizeof(unsigned long long), st));
  CBFS_CUDA(cudaMallocHost(&h, sizeof(unsigned long long)));
  CBFS_CUDA(cudaMemsetAsync(level, 0xFF, n, st));
  // root: the highest-degree vertex (position 0 of the degree order), level 0
  CBFS_CUDA(cudaMemcpyAsync(h, g->order, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  const uint32_t root = (uint32_t)(*h & 0xFFFFFFFFu);
  CBFS_CUDA(cudaMemsetAsync(level + root, 0, 1, st));
  unsigned long long found = 1;
  uint32_t lvl = 0;
  for (; found && lvl < PROBE_ROUNDS; ++lvl) {
    CBFS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    k_probe_level<<<grid_for(n, 256), 256, 0, st>>>(g->off, g->cols, n, level, lvl, cnt);
    CBFS_LAUNCHED();
    CBFS_CUDA(cudaMemcpyAsync(h, cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    found = *h;
  }
  *out = found > 0 ? 1 : 0;  // still growing after PROBE_ROUNDS levels
  CBFS_CUDA(cudaFreeAsync(level, st));
  CBFS_CUDA(cudaFreeAsync(cnt, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  CBFS_CUDA(cudaFreeHost(h));
  CBFS_CUDA(cudaStreamDestroy(st));
  return CBFS_OK;
}

int choose_engine(Graph* g, uint32_t direction) {
  if (direction == CBFS_DIR_PULL) return ENGINE_BATCHED;  // pull exists in the batched engine only
  if (g_engine_policy == CBFS_ENGINE_BATCHED) return ENGINE_BATCHED;
  if (g_engine_policy == CBFS_ENGINE_SPARSE) return ENGINE_SPARSE;
  if (g->high_diameter < 0) {
    int hd = 0;
    // graphs with hubs (power-law degree tails: social / web) have low
    // diameter; only hub-free graphs (meshes, roads, k-NN) pay for the probe
    if (g->max_degree <= PROBE_MAX_DEGREE && probe_high_diameter(g, &hd) != CBFS_OK) return -1;
    g->high_diameter = hd;
  }
  return g->high_diameter ? ENGINE_SPARSE : ENGINE_BATCHED;
}

}  // namespace cbfs

extern "C" int cbfs_set_sparse_order(int64_t min_entries) {
  if (min_entries < -1) return cbfs::fail(CBFS_EINVAL, "min_entries must be >= -1");
  cbfs::g_sp_order_min = min_entries;
  return CBFS_OK;
}

extern "C" int cbfs_set_engine(int engine) {
  if (engine < CBFS_ENGINE_AUTO || engine > CBFS_ENGINE_SPARSE) return cbfs::fail(CBFS_EINVAL, "bad engine");
  cbfs::g_engine_policy = engine;
  return CBFS_OK;
}
