// cbfs.cu — the C-BFS engine (§8(a) rows A2-A8): Alg. 1 of PAPER.md
// with the direction-optimised EdgeMap, run for a
// batch of 32 clusters at once in lock-step rounds.
//
// B200 design:
//  * vertex-major state: for vertex v the 32 clusters of a batch own the 32
//    consecutive words seen[v*32 + c] / pend[v*32 + c] (u64 bit-subsets,
//    P:641-645) and dist[v*32 + c] (u16 Delta).  A warp with lane c =
//    cluster c reads one neighbour's state for all clusters as one coalesced
//    256-byte access, so random neighbour gathers use whole sectors.
//  * S_next of Alg. 1 is kept as `pend` = S_next \ S_seen (the bits that
//    arrived this round and are not yet folded).  pend is zero outside the
//    pending entries; the first writer that turns a pend word non-zero owns
//    the claim (R4), so no separate r[] array is needed.
//  * a frontier is a list of packed (v*32 + c) entries; the pending list of
//    round i IS F_i.
//  * round i = fold kernel (vertex phase P:714-720) -> push kernel (sparse,
//    P:1758-1768, edge-balanced over the frontier's arcs, 64-bit atomicOr)
//    or pull kernel (dense, warp per 256-arc CSR chunk, lane per
//    cluster, no atomics except on chunk-boundary vertices).  Kernel
//    boundaries are the barriers that H9 requires between the two phases.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace cbfs {

struct Work {
  uint64_t cap = 0;       // n * LANES
  uint64_t* seen = nullptr;
  uint64_t* pend = nullptr;
  uint16_t* dist = nullptr;
  uint32_t* listA = nullptr;
  uint32_t* listB = nullptr;
  uint64_t* pre = nullptr;   // [cap + 1]
  uint32_t* ubits = nullptr; // [n/32 + 1]
  unsigned long long* ctr = nullptr;  // [0] next count, [1] next E, [2] error bits
  unsigned long long* h_ctr = nullptr; // pinned mirror
  uint64_t* bstats = nullptr; // [LANES][4]
  void* scan_tmp = nullptr;
  size_t scan_bytes = 0;
};

static double g_alpha = 20.0;

void work_free(Graph* g) {
  Work* w = g->work;
  if (!w) return;
  cudaFree(w->seen); cudaFree(w->pend); cudaFree(w->dist); cudaFree(w->listA); cudaFree(w->listB);
  cudaFree(w->pre); cudaFree(w->ubits); cudaFree(w->ctr); cudaFreeHost(w->h_ctr); cudaFree(w->bstats);
  cudaFree(w->scan_tmp);
  delete w;
  g->work = nullptr;
}

int ensure_work(Graph* g) {
  if (g->work) return CBFS_OK;
  Work* w = new Work();
  g->work = w;
  const uint64_t cap = (uint64_t)(g->n ? g->n : 1) * LANES;
  w->cap = cap;
  CBFS_CUDA(cudaMalloc(&w->seen, cap * sizeof(uint64_t)));
  CBFS_CUDA(cudaMalloc(&w->pend, cap * sizeof(uint64_t)));
  CBFS_CUDA(cudaMalloc(&w->dist, cap * sizeof(uint16_t)));
  CBFS_CUDA(cudaMalloc(&w->listA, cap * sizeof(uint32_t)));
  CBFS_CUDA(cudaMalloc(&w->listB, cap * sizeof(uint32_t)));
  CBFS_CUDA(cudaMalloc(&w->pre, (cap + 1) * sizeof(uint64_t)));
  CBFS_CUDA(cudaMalloc(&w->ubits, ((g->n >> 5) + 1) * sizeof(uint32_t)));
  CBFS_CUDA(cudaMalloc(&w->ctr, 4 * sizeof(unsigned long long)));
  CBFS_CUDA(cudaMallocHost(&w->h_ctr, 4 * sizeof(unsigned long long)));
  CBFS_CUDA(cudaMalloc(&w->bstats, LANES * 4 * sizeof(uint64_t)));
  CBFS_CUDA(cudaMemset(w->pend, 0, cap * sizeof(uint64_t)));  // zero-invariant from here on
  CBFS_CUDA(cudaMemset(w->ubits, 0, ((g->n >> 5) + 1) * sizeof(uint32_t)));
  CBFS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, w->scan_bytes, w->pre, w->pre, cap));
  CBFS_CUDA(cudaMalloc(&w->scan_tmp, w->scan_bytes ? w->scan_bytes : 1));
  return CBFS_OK;
}

enum : unsigned long long { ERR_BAD_SOURCE = 1, ERR_DUP_SOURCE = 2, ERR_BAD_SIZE = 4, ERR_OVERFLOW = 8 };

// warp-aggregated append of `e` for lanes with `flag`
__device__ __forceinline__ void warp_append(bool flag, uint32_t e, uint32_t* __restrict__ list,
                                            unsigned long long* __restrict__ count) {
  const unsigned FULL = 0xFFFFFFFFu;
  unsigned mask = __ballot_sync(FULL, flag);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(mask));
  base = __shfl_sync(FULL, base, leader);
  if (flag) list[base + __popc(mask & ((1u << lane) - 1))] = e;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
  return x;
}

// ------------------------------------------------------------------ init
// R1 seeding (S_next[s_j] = {s_j}; F_0 = S): pend[s_j, c] = bit j.
__global__ void k_seed(const uint32_t* __restrict__ sources, const uint8_t* __restrict__ sizes, uint32_t nb,
                       uint32_t n, const uint32_t* __restrict__ inv, const uint64_t* __restrict__ off,
                       uint64_t* __restrict__ pend, uint32_t* __restrict__ list, unsigned long long* __restrict__ ctr) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // one warp per (cluster, 32 sources)
  const uint32_t c = t >> 6, j = t & 63;
  bool claim = false;
  uint32_t e = 0;
  unsigned long long degsum = 0;
  if (c < nb) {
    const uint32_t k = sizes[c];
    if (k == 0 || k > 64) {
      if (j == 0) atomicOr(&ctr[2], ERR_BAD_SIZE);
    } else if (j < k) {
      const uint32_t s = sources[(uint64_t)c * 64 + j];
      if (s >= n) {
        atomicOr(&ctr[2], ERR_BAD_SOURCE);
      } else {
        const uint32_t x = inv ? inv[s] : s;
        e = x * LANES + c;
        unsigned long long old = atomicOr((unsigned long long*)&pend[e], 1ULL << j);
        if (old != 0) atomicOr(&ctr[2], ERR_DUP_SOURCE);  // R2
        else { claim = true; degsum = off[x + 1] - off[x]; }
      }
    }
  }
  warp_append(claim, e, list, &ctr[0]);
  degsum = warp_sum(degsum);
  if ((threadIdx.x & 31) == 0 && degsum) atomicAdd(&ctr[1], degsum);
}

// ------------------------------------------------------------------ fold
// Vertex phase: S_new = S_next[u] \ S_seen[u] (= pend), set
// Delta_u on first visit, S_u[i - Delta_u] = S_new, S_seen[u] |= S_new.
// Also: outputs, union-frontier bitmap, per-cluster stats, degrees for the
// push scan.
template <int DB>
__global__ void __launch_bounds__(256) k_fold(const uint32_t* __restrict__ F, uint32_t nF, uint32_t i,
                                              uint64_t* __restrict__ seen, uint64_t* __restrict__ pend,
                                              uint16_t* __restrict__ dist, const uint64_t* __restrict__ off,
                                              const uint32_t* __restrict__ perm, uint32_t n, uint32_t C,
                                              uint32_t cbase, uint32_t planes, void* __restrict__ out_dist,
                                              uint64_t* __restrict__ out_masks, uint32_t* __restrict__ ubits,
                                              uint64_t* __restrict__ pre, uint64_t* __restrict__ bstats,
                                              unsigned long long* __restrict__ ctr) {
  __shared__ unsigned long long sF[LANES], sE[LANES], sM[LANES];
  __shared__ unsigned sR[LANES];
  if (threadIdx.x < LANES) { sF[threadIdx.x] = sE[threadIdx.x] = sM[threadIdx.x] = 0; sR[threadIdx.x] = 0; }
  __syncthreads();
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nF; t += gridDim.x * blockDim.x) {
    const uint32_t e = F[t];
    const uint32_t v = e >> 5, c = e & 31;
    const uint64_t nw = pend[e];
    pend[e] = 0;
    uint32_t dv = dist[e];
    const bool first = dv == INF16;
    if (first) { dv = i; dist[e] = (uint16_t)i; }
    seen[e] |= nw;
    const uint64_t deg = off[v + 1] - off[v];
    pre[t] = deg;
    atomicOr(&ubits[v >> 5], 1u << (v & 31));
    const uint32_t orig = perm ? perm[v] : v;
    const uint64_t col = (uint64_t)orig * C + cbase + c;
    if (first && out_dist) {
      if (DB == 1) {
        if (i > 254) atomicOr(&ctr[2], ERR_OVERFLOW);
        ((uint8_t*)out_dist)[col] = (uint8_t)(i > 254 ? 254 : i);
      } else {
        ((uint16_t*)out_dist)[col] = (uint16_t)i;
      }
    }
    const uint32_t oi = i - dv;
    if (out_masks && oi < planes) out_masks[(uint64_t)oi * n * C + col] = nw;
    atomicAdd(&sF[c], 1ULL);
    atomicAdd(&sE[c], (unsigned long long)deg);
    if (first) atomicAdd(&sM[c], (unsigned long long)deg);
    atomicMax(&sR[c], i + 1);
  }
  __syncthreads();
  if (threadIdx.x < LANES) {
    const uint32_t c = threadIdx.x;
    if (sF[c]) {
      atomicAdd((unsigned long long*)&bstats[c * 4 + 1], sF[c]);
      atomicAdd((unsigned long long*)&bstats[c * 4 + 2], sE[c]);
      if (sM[c]) atomicAdd((unsigned long long*)&bstats[c * 4 + 3], sM[c]);
      atomicMax((unsigned long long*)&bstats[c * 4 + 0], (unsigned long long)sR[c]);
    }
  }
}

// ------------------------------------------------------------------ push
// EdgeMap-Sparse with Edge_F = Fetch_And_Or: the
// frontier's (entry, arc) pairs form one virtual array of `total` arcs
// (exclusive prefix `pre`, pre[nF] = total); each warp takes PUSH_CHUNK
// consecutive arcs, so hubs and degree-4 grid vertices balance alike.
constexpr uint32_t PUSH_CHUNK = 256;

__global__ void __launch_bounds__(256) k_push(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols,
                                              const uint32_t* __restrict__ F, const uint64_t* __restrict__ pre,
                                              uint32_t nF, uint64_t total, const uint64_t* __restrict__ seen,
                                              const uint16_t* __restrict__ dist, uint64_t* __restrict__ pend,
                                              uint32_t* __restrict__ out_list, unsigned long long* __restrict__ ctr,
                                              uint32_t i, uint32_t d) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  unsigned long long degsum = 0;
  for (uint64_t w = warp; w * PUSH_CHUNK < total; w += nwarps) {
    const uint64_t start = w * PUSH_CHUNK;
    const uint64_t end = min(start + PUSH_CHUNK, total);
    uint32_t idx = 0;
    if (lane == 0) {  // largest idx with pre[idx] <= start
      uint32_t lo = 0, hi = nF - 1;
      while (lo < hi) {
        uint32_t mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= start) lo = mid; else hi = mid - 1;
      }
      idx = lo;
    }
    idx = __shfl_sync(0xFFFFFFFFu, idx, 0);
    for (uint64_t p0 = start; p0 < end; p0 += 32) {
      const uint64_t p = p0 + lane;
      bool claim = false;
      uint32_t ev = 0;
      if (p < end) {
        while (pre[idx + 1] <= p) ++idx;
        const uint32_t e = F[idx];
        const uint32_t u = e >> 5, c = e & 31;
        const uint32_t v = cols[off[u] + (p - pre[idx])];
        ev = v * LANES + c;
        const uint32_t dv = dist[ev];
        if (dv == INF16 || (int)i - (int)dv < (int)d) {  // P:722, R3
          const uint64_t x = seen[e] & ~seen[ev];
          if (x) {
            const unsigned long long old = atomicOr((unsigned long long*)&pend[ev], (unsigned long long)x);
            claim = old == 0;  // first setter wins (R4)
            if (claim) degsum += off[v + 1] - off[v];
          }
        }
      }
      warp_append(claim, ev, out_list, &ctr[0]);
    }
  }
  degsum = warp_sum(degsum);
  if (lane == 0 && degsum) atomicAdd(&ctr[1], degsum);
}

// ------------------------------------------------------------------ pull
// EdgeMap-Dense: every vertex v that can still receive (cap
// P:722 and S_seen[v] != S) ORs S_seen[u] over its neighbours u in the union
// frontier; lane c = cluster c.  No first-hit break (R7): stop only when the
// accumulated subset is full.  Neighbours not in F_i^c contribute only bits v
// already holds (reading R7a), so one union-frontier test per
// arc serves all 32 clusters.
constexpr int PULL_MLP = 8;

__global__ void __launch_bounds__(256) k_pull(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols,
                                              const uint32_t* __restrict__ chunk_v, uint64_t n_chunks, uint64_t m,
                                              const uint64_t* __restrict__ seen, const uint16_t* __restrict__ dist,
                                              uint64_t* __restrict__ pend, const uint32_t* __restrict__ ubits,
                                              const uint8_t* __restrict__ sizes, uint32_t nb,
                                              uint32_t* __restrict__ out_list, unsigned long long* __restrict__ ctr,
                                              uint32_t i, uint32_t d) {
  const unsigned FULLW = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint64_t full = (uint32_t)lane < nb ? full_mask(sizes[lane]) : 0ULL;
  unsigned long long degsum = 0;
  for (uint64_t w = warp; w < n_chunks; w += nwarps) {
    uint64_t e0 = w * PULL_CHUNK;
    const uint64_t e1 = min(e0 + PULL_CHUNK, m);
    uint32_t v = chunk_v[w];
    while (e0 < e1) {
      const uint64_t vb = off[v], ve = off[v + 1];
      const uint64_t lo = max(vb, e0), hi = min(ve, e1);
      if (lo >= hi) { ++v; continue; }
      const uint64_t x = (uint64_t)v * LANES + lane;
      const uint32_t dv = dist[x];
      const uint64_t sv = seen[x];
      const bool cap = full != 0 && (dv == INF16 || (int)i - (int)dv < (int)d) && sv != full;
      if (__ballot_sync(FULLW, cap)) {
        uint64_t acc = 0;
        for (uint64_t e = lo; e < hi; e += 32) {
          const uint32_t myu = (e + lane < hi) ? cols[e + lane] : 0xFFFFFFFFu;
          const bool inF = myu != 0xFFFFFFFFu && ((__ldg(&ubits[myu >> 5]) >> (myu & 31)) & 1u);
          unsigned fm = __ballot_sync(FULLW, inF);
          while (fm) {
            uint64_t g[PULL_MLP];
#pragma unroll
            for (int q = 0; q < PULL_MLP; ++q) {
              g[q] = 0;
              if (fm) {
                const int j = __ffs(fm) - 1;
                fm &= fm - 1;
                const uint32_t u = __shfl_sync(FULLW, myu, j);
                g[q] = seen[(uint64_t)u * LANES + lane];
              }
            }
#pragma unroll
            for (int q = 0; q < PULL_MLP; ++q) acc |= g[q];
          }
          if (!__ballot_sync(FULLW, cap && ((acc | sv) != full))) break;
        }
        const uint64_t nw = acc & ~sv;
        bool claim = false;
        if (cap && nw) {
          if (vb >= e0 && ve <= e1) {  // this warp owns all of v's arcs
            pend[x] = nw;
            claim = true;
          } else {
            claim = atomicOr((unsigned long long*)&pend[x], (unsigned long long)nw) == 0;
          }
          if (claim) degsum += ve - vb;
        }
        warp_append(claim, (uint32_t)x, out_list, &ctr[0]);
      }
      e0 = hi;
      ++v;
    }
  }
  degsum = warp_sum(degsum);
  if (lane == 0 && degsum) atomicAdd(&ctr[1], degsum);
}

__global__ void k_set_u64(uint64_t* p, uint64_t v) { *p = v; }

// ------------------------------------------------------------------ driver

static int sync_ctr(Work* w, cudaStream_t st) {
  CBFS_CUDA(cudaMemcpyAsync(w->h_ctr, w->ctr, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

int run_batch(Graph* g, const RunArgs& a, cudaStream_t st) {
  Work* w = g->work;
  const uint32_t n = g->n;
  CBFS_CUDA(cudaMemsetAsync(w->seen, 0, (uint64_t)n * LANES * sizeof(uint64_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->dist, 0xFF, (uint64_t)n * LANES * sizeof(uint16_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->bstats, 0, LANES * 4 * sizeof(uint64_t), st));
  CBFS_CUDA(cudaMemsetAsync(w->ctr, 0, 3 * sizeof(unsigned long long), st));
  k_seed<<<(a.nb * 64 + 255) / 256, 256, 0, st>>>(a.sources, a.sizes, a.nb, n, g->inv, g->off, w->pend, w->listA,
                                                   w->ctr);
  CBFS_LAUNCHED();
  int rc = sync_ctr(w, st);
  if (rc) return rc;
  if (w->h_ctr[2]) {
    // leave pend zero-invariant for the next call
    CBFS_CUDA(cudaMemsetAsync(w->pend, 0, (uint64_t)n * LANES * sizeof(uint64_t), st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    if (w->h_ctr[2] & ERR_BAD_SIZE) return fail(CBFS_EINVAL, "cluster size must be 1..64");
    if (w->h_ctr[2] & ERR_BAD_SOURCE) return fail(CBFS_EINVAL, "source id >= n");
    return fail(CBFS_EINVAL, "duplicate source in a cluster");
  }
  uint64_t nF = w->h_ctr[0], E = w->h_ctr[1];
  uint32_t* cur = w->listA;
  uint32_t* nxt = w->listB;
  bool overflow = false;
  for (uint32_t i = 0; nF > 0; ++i) {
    if (i >= 0xFFFEu) return fail(CBFS_EOVERFLOW, "more than 65534 rounds");
    const unsigned fb = grid_for(nF, 256);
    if (a.dist_bytes == 1)
      k_fold<1><<<fb, 256, 0, st>>>(cur, (uint32_t)nF, i, w->seen, w->pend, w->dist, g->off, g->perm, n, a.C, a.cbase,
                                    a.planes, a.out_dist, a.out_masks, w->ubits, w->pre, w->bstats, w->ctr);
    else
      k_fold<2><<<fb, 256, 0, st>>>(cur, (uint32_t)nF, i, w->seen, w->pend, w->dist, g->off, g->perm, n, a.C, a.cbase,
                                    a.planes, a.out_dist, a.out_masks, w->ubits, w->pre, w->bstats, w->ctr);
    CBFS_LAUNCHED();
    CBFS_CUDA(cudaMemsetAsync(w->ctr, 0, 2 * sizeof(unsigned long long), st));
    bool pull = a.direction == CBFS_DIR_PULL ||
                (a.direction == CBFS_DIR_AUTO && (double)E * g_alpha > (double)g->m * (double)a.nb);
    if (pull) {
      const unsigned pb = grid_for(g->n_chunks * 32, 256, 148u * 8u * 4u);
      k_pull<<<pb, 256, 0, st>>>(g->off, g->cols, g->chunk_v, g->n_chunks, g->m, w->seen, w->dist, w->pend, w->ubits,
                                 a.sizes, a.nb, nxt, w->ctr, i, a.d);
      CBFS_LAUNCHED();
    } else if (E > 0) {
      CBFS_CUDA(cub::DeviceScan::ExclusiveSum(w->scan_tmp, w->scan_bytes, w->pre, w->pre, nF, st));
      count_launch(2);
      k_set_u64<<<1, 1, 0, st>>>(w->pre + nF, E);
      CBFS_LAUNCHED();
      const uint64_t warps = (E + PUSH_CHUNK - 1) / PUSH_CHUNK;
      const unsigned pb = grid_for(warps * 32, 256, 148u * 8u * 4u);
      k_push<<<pb, 256, 0, st>>>(g->off, g->cols, cur, w->pre, (uint32_t)nF, E, w->seen, w->dist, w->pend, nxt,
                                 w->ctr, i, a.d);
      CBFS_LAUNCHED();
    }
    CBFS_CUDA(cudaMemsetAsync(w->ubits, 0, ((n >> 5) + 1) * sizeof(uint32_t), st));
    rc = sync_ctr(w, st);
    if (rc) return rc;
    if (w->h_ctr[2] & ERR_OVERFLOW) overflow = true;
    nF = w->h_ctr[0];
    E = w->h_ctr[1];
    std::swap(cur, nxt);
  }
  if (a.out_stats)
    CBFS_CUDA(cudaMemcpyAsync(a.out_stats, w->bstats, (uint64_t)a.nb * 4 * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                              st));
  if (overflow) return fail(CBFS_EOVERFLOW, "a distance exceeds 254 with dist_bytes == 1");
  return CBFS_OK;
}

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

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_run(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
             uint32_t dist_bytes, void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
             uint32_t direction, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  int rc = check_run_args(g, sources, sizes, n_clusters, d, dist_bytes, planes, direction);
  if (rc) return rc;
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  rc = ensure_work(g);
  if (rc) return rc;
  const uint64_t C = n_clusters;
  if (out_dist) CBFS_CUDA(cudaMemsetAsync(out_dist, 0xFF, (uint64_t)g->n * C * dist_bytes, st));
  if (out_masks) CBFS_CUDA(cudaMemsetAsync(out_masks, 0, (uint64_t)planes * g->n * C * sizeof(uint64_t), st));
  for (uint32_t cb = 0; cb < n_clusters; cb += LANES) {
    RunArgs a;
    a.sources = sources + (uint64_t)cb * 64;
    a.sizes = sizes + cb;
    a.nb = std::min<uint32_t>(LANES, n_clusters - cb);
    a.d = d;
    a.planes = planes;
    a.dist_bytes = dist_bytes;
    a.C = n_clusters;
    a.cbase = cb;
    a.direction = direction;
    a.out_dist = out_dist;
    a.out_masks = out_masks;
    a.out_stats = out_stats ? out_stats + (uint64_t)cb * 4 : nullptr;
    rc = run_batch(g, a, st);
    if (rc) return rc;
  }
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

int cbfs_set_direction_alpha(double alpha) {
  if (!(alpha > 0)) return fail(CBFS_EINVAL, "alpha must be > 0");
  g_alpha = alpha;
  return CBFS_OK;
}

}  // extern "C"
