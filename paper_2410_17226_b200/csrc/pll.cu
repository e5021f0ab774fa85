// pll.cu — exact 2-hop distance oracle: Pruned
// Landmark Labeling with a C-BFS first phase, reading R29
// (DESIGN.md §2).
//
//   phase 1  the caller's r clusters (diameter <= d) run as C-BFS batches
//            (cbfs_run's engines): their labels are every vertex's cluster
//            distance vector, kept with rows by internal id;
//   phase 2  the uncovered vertices in (degree desc, id asc) order, in
//            batches b_0 = first, b_{i+1} = min(bmax, floor(3 b_i / 2))
//            (200 x 1.5^i up to 1000).  Every root of a batch
//            runs a BFS pruned against the index as it was when the batch
//            started (R29), so a batch's BFSs are independent and run in
//            parallel: one CTA per root (persistent CTAs pull roots from a
//            counter), one warp per frontier vertex for the pruning query,
//            then the warp expands the vertex if it was not pruned.
//
// Pruning query(r, u) <= delta: the root's snapshot label is
// scattered into a per-CTA dense map hub -> distance, so the explicit part is
// one map probe per label entry of u; the cluster part skips every cluster
// with Delta_r + Delta_u > delta before touching a subset word.
//
// A root appends (pos << 8 | dist) to L(u) beyond u's batch-start length
// (invisible to the batch's own queries); batches follow each other on the
// stream with no host round trip, and one bitonic sort per list at the end
// makes every list ascending by hub position (a deterministic layout; the
// query binary-searches one list for the hubs of the other).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.cuh"

namespace cbfs {

#ifndef CBFS_PLL_THREADS
#define CBFS_PLL_THREADS 1024
#endif
constexpr int PLL_THREADS = CBFS_PLL_THREADS;
constexpr int PLL_WARPS = PLL_THREADS / 32;
constexpr uint32_t PLL_SMEM_MAX = 200u << 10;  // the root's cluster labels staged in shared memory
enum : unsigned { PLL_ERR_CAP = 1, PLL_ERR_DIST = 4 };
constexpr uint32_t PLL_MAX_CAP = 8192;  // a list is sorted in shared memory at the end

struct Pll {
  int device = 0;
  Graph* g = nullptr;
  uint32_t n = 0, C = 0, d = 0, planes = 0, cap = 0, first = 0, bmax = 0;
  uint32_t roots = 0, batches = 0, max_count = 0;
  uint64_t total = 0;
  float ms_cbfs = 0.f, ms_pbfs = 0.f;
  uint16_t* cdist = nullptr;  // [n][C] Delta, internal rows
  uint64_t* cmask = nullptr;  // [planes][n][C]
  uint32_t* counts = nullptr; // [n] internal rows
  uint32_t* entries = nullptr;  // [n][cap] pos << 8 | dist, ascending
};

// R15 scan of cluster c restricted to values <= bound: true iff some
// t* <= bound - Delta_a - Delta_b exists (subsets of a from shared memory)
__device__ __forceinline__ bool cluster_within(const uint64_t* __restrict__ sa, uint32_t C, const uint64_t* __restrict__ cmask,
                                               uint64_t n, uint32_t b, uint32_t c, uint32_t d, int slack) {
  const int tmax = min(slack, (int)(2 * d));
  for (int tt = 0; tt <= tmax; ++tt) {
    const int i0 = tt > (int)d ? tt - (int)d : 0, i1 = tt < (int)d ? tt : (int)d;
    for (int i = i0; i <= i1; ++i)
      if (sa[i * C + c] & cmask[((uint64_t)(tt - i) * n + b) * C + c]) return true;
  }
  return false;
}

__global__ void __launch_bounds__(PLL_THREADS) k_pll_bfs(
    const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, const uint32_t* __restrict__ rank,
    uint32_t n, const uint32_t* __restrict__ roots, uint32_t nb, uint32_t tag_base, uint32_t C, uint32_t d,
    const uint16_t* __restrict__ cdist, const uint64_t* __restrict__ cmask, uint32_t* __restrict__ counts,
    const uint32_t* __restrict__ snap, const uint32_t* entries, uint32_t cap,
    uint32_t* entries_w /* == entries: appends land beyond the batch-start lengths this batch reads */,
    unsigned long long* __restrict__ ctl,
    uint32_t* __restrict__ visited_all, uint8_t* __restrict__ tmp_all, uint32_t* __restrict__ q_all) {
  extern __shared__ uint64_t s_dyn[];  // the root's cluster labels: subsets [d+1][C], then Delta [C]
  uint64_t* s_mask = s_dyn;
  uint32_t* s_da = reinterpret_cast<uint32_t*>(s_dyn + (uint64_t)(d + 1) * C);
  __shared__ uint32_t s_ri, s_nf;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  uint32_t* visited = visited_all + (uint64_t)blockIdx.x * n;
  uint8_t* tmp = tmp_all + (uint64_t)blockIdx.x * n;
  uint32_t* qa = q_all + (uint64_t)blockIdx.x * 2 * n;
  uint32_t* qb = qa + n;
  for (;;) {
    if (tid == 0) s_ri = (uint32_t)atomicAdd(&ctl[0], 1ULL);
    __syncthreads();
    const uint32_t ri = s_ri;
    if (ri >= nb) break;
    const uint32_t r = roots[ri];
    const uint32_t tag = tag_base + ri + 1;
    const uint32_t pos_r = rank[r];
    for (uint32_t c = tid; c < C; c += PLL_THREADS) {
      s_da[c] = cdist[(uint64_t)r * C + c];
      for (uint32_t i = 0; i <= d; ++i) s_mask[i * C + c] = cmask[((uint64_t)i * n + r) * C + c];
    }
    const uint32_t sr = min(snap[r], cap);  // a list that overflowed cap (reported as EOVERFLOW) holds cap entries
    for (uint32_t a = tid; a < sr; a += PLL_THREADS) {
      const uint32_t e = entries[(uint64_t)r * cap + a];
      tmp[e >> 8] = (uint8_t)(e & 255u);
    }
    if (tid == 0) {
      qa[0] = r;
      visited[r] = tag;
      s_nf = 1;
    }
    __syncthreads();
    uint32_t nfr = s_nf;
    for (uint32_t delta = 0; nfr > 0; ++delta) {
      __syncthreads();
      if (tid == 0) s_nf = 0;
      __syncthreads();
      for (uint32_t fi = wib; fi < nfr; fi += PLL_WARPS) {
        const uint32_t u = qa[fi];
        // ---- pruning query against the batch-start index
        bool hit = false;
        const uint32_t su = min(snap[u], cap);
        for (uint32_t a0 = 0; a0 < su && !hit; a0 += 32) {
          bool h = false;
          if (a0 + lane < su) {
            const uint32_t e = entries[(uint64_t)u * cap + a0 + lane];
            const uint32_t x = tmp[e >> 8];
            h = x != 0xFFu && x + (e & 255u) <= delta;
          }
          hit = __any_sync(FULLW, h);
        }
        for (uint32_t c0 = 0; c0 < C && !hit; c0 += 32) {
          bool h = false;
          const uint32_t c = c0 + lane;
          if (c < C) {
            const uint32_t da = s_da[c], db = cdist[(uint64_t)u * C + c];
            if (da != INF16 && db != INF16 && da + db <= delta)
              h = cluster_within(s_mask, C, cmask, n, u, c, d, (int)(delta - da - db));
          }
          hit = __any_sync(FULLW, h);
        }
        if (hit) continue;  // pruned: no label, not expanded
        if (lane == 0) {
          const uint32_t slot = atomicAdd(&counts[u], 1u);
          if (slot >= cap) {
            atomicOr(&ctl[2], (unsigned long long)PLL_ERR_CAP);
          } else if (delta > 254) {
            atomicOr(&ctl[2], (unsigned long long)PLL_ERR_DIST);
          } else {  // beyond u's batch-start length: invisible to this batch's queries
            entries_w[(uint64_t)u * cap + slot] = (pos_r << 8) | delta;
          }
        }
        const uint64_t e0 = off[u], e1 = off[u + 1];
        for (uint64_t a0 = e0; a0 < e1; a0 += 32) {
          const uint64_t a = a0 + lane;
          bool fresh = false;
          uint32_t x = 0;
          if (a < e1) {
            x = cols[a];
            fresh = visited[x] != tag && atomicExch(&visited[x], tag) != tag;
          }
          const unsigned m = __ballot_sync(FULLW, fresh);
          uint32_t base = 0;
          if (lane == 0 && m) base = atomicAdd(&s_nf, (uint32_t)__popc(m));
          base = __shfl_sync(FULLW, base, 0);
          if (fresh) qb[base + __popc(m & ((1u << lane) - 1))] = x;
        }
      }
      __syncthreads();
      nfr = s_nf;
      uint32_t* t = qa; qa = qb; qb = t;
    }
    for (uint32_t a = tid; a < sr; a += PLL_THREADS) tmp[entries[(uint64_t)r * cap + a] >> 8] = 0xFFu;
    __syncthreads();
  }
}

// Each list holds its batches' segments in batch order, each segment in
// arrival order; one bitonic sort per list (block per vertex, shared memory
// of the next power of two >= the list) makes it ascending by hub position.
__global__ void __launch_bounds__(256) k_pll_sort(uint32_t* __restrict__ entries, const uint32_t* __restrict__ counts,
                                                  uint32_t n, uint32_t cap) {
  extern __shared__ uint32_t s_key[];
  for (uint32_t v = blockIdx.x; v < n; v += gridDim.x) {
    const uint32_t L = min(counts[v], cap);
    if (L < 2) continue;
    uint32_t P = 1;
    while (P < L) P <<= 1;
    uint32_t* row = entries + (uint64_t)v * cap;
    for (uint32_t x = threadIdx.x; x < P; x += blockDim.x) s_key[x] = x < L ? row[x] : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1)
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t x = threadIdx.x; x < P; x += blockDim.x) {
          const uint32_t y = x ^ j;
          if (y > x) {
            const uint32_t a = s_key[x], b = s_key[y];
            if (((x & k) == 0) == (a > b)) { s_key[x] = b; s_key[y] = a; }
          }
        }
        __syncthreads();
      }
    for (uint32_t x = threadIdx.x; x < L; x += blockDim.x) row[x] = s_key[x];
    __syncthreads();
  }
}

__global__ void k_pll_flags(const uint32_t* __restrict__ sources, const uint8_t* __restrict__ sizes, uint32_t C,
                            const uint32_t* __restrict__ inv, uint32_t n, uint8_t* __restrict__ covered,
                            int* __restrict__ bad) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t c = t >> 6, j = t & 63;
  if (c >= C) return;
  const uint32_t k = sizes[c];
  if (k == 0 || k > 64) { if (j == 0) atomicOr(bad, 1); return; }
  if (j >= k) return;
  const uint32_t s = sources[(uint64_t)c * 64 + j];
  if (s >= n) { atomicOr(bad, 2); return; }
  covered[inv ? inv[s] : s] = 1;
}

__global__ void k_pll_root_flags(const uint32_t* __restrict__ order, const uint8_t* __restrict__ covered, uint32_t n,
                                 uint8_t* __restrict__ flag) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    flag[p] = !covered[order[p]];
}

__global__ void k_pll_stats(const uint32_t* __restrict__ counts, uint32_t n, unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  uint32_t mx = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    s += counts[v];
    mx = max(mx, counts[v]);
  }
  s = warp_sum(s);
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULLW, mx, o));
  if (lane_id() == 0) {
    atomicAdd(&out[0], s);
    atomicMax(&out[1], (unsigned long long)mx);
  }
}

// one warp per query: cluster part (lanes over clusters, R15 scan) and the
// common hubs of two ascending lists (lanes over L(a), binary search in L(b))
__global__ void __launch_bounds__(256) k_pll_query(const uint32_t* __restrict__ inv, uint32_t n, uint32_t C,
                                                   uint32_t d, const uint16_t* __restrict__ cdist,
                                                   const uint64_t* __restrict__ cmask,
                                                   const uint32_t* __restrict__ counts,
                                                   const uint32_t* __restrict__ entries, uint32_t cap,
                                                   const uint32_t* __restrict__ s, const uint32_t* __restrict__ t,
                                                   uint64_t q, int32_t* __restrict__ out, int* __restrict__ bad) {
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t qi = warp; qi < q; qi += nwarps) {
    uint32_t a = s[qi], b = t[qi];
    if (a >= n || b >= n) {
      if (lane == 0) *bad = 1;
      continue;
    }
    if (inv) { a = inv[a]; b = inv[b]; }
    int32_t best = INT32_MAX;
    const uint32_t ca = min(counts[a], cap), cbn = min(counts[b], cap);
    const uint32_t* A = entries + (uint64_t)a * cap;
    const uint32_t* B = entries + (uint64_t)b * cap;
    for (uint32_t x = lane; x < ca; x += 32) {
      const uint32_t e = A[x], key = e & ~255u;
      uint32_t lo = 0, hi = cbn;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (B[mid] < key) lo = mid + 1; else hi = mid;
      }
      if (lo < cbn && (B[lo] & ~255u) == key) best = min(best, (int32_t)((e & 255u) + (B[lo] & 255u)));
    }
    for (uint32_t c = lane; c < C; c += 32) {
      const uint32_t da = cdist[(uint64_t)a * C + c], db = cdist[(uint64_t)b * C + c];
      if (da == INF16 || db == INF16 || (int32_t)(da + db) >= best) continue;
      for (uint32_t tt = 0; tt <= 2 * d; ++tt) {
        bool h = false;
        const uint32_t i0 = tt > d ? tt - d : 0, i1 = tt < d ? tt : d;
        for (uint32_t i = i0; i <= i1 && !h; ++i)
          h = (cmask[((uint64_t)i * n + a) * C + c] & cmask[((uint64_t)(tt - i) * n + b) * C + c]) != 0;
        if (h) {
          best = min(best, (int32_t)(da + db + tt));
          break;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(FULLW, best, o));
    if (lane == 0) out[qi] = best;
  }
}

__global__ void k_pll_export(const uint32_t* __restrict__ perm, uint32_t n, uint32_t cap,
                             const uint32_t* __restrict__ counts, const uint32_t* __restrict__ entries,
                             uint32_t* __restrict__ out_counts, uint32_t* __restrict__ out_entries) {
  const uint32_t lane = lane_id();
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = warp; v < n; v += nwarps) {
    const uint32_t o = perm ? perm[v] : (uint32_t)v;
    const uint32_t cv = counts[v];
    if (lane == 0 && out_counts) out_counts[o] = cv;
    if (out_entries)
      for (uint32_t a = lane; a < cap; a += 32)
        out_entries[(uint64_t)o * cap + a] = a < cv ? entries[(uint64_t)v * cap + a] : 0u;
  }
}

struct PllScratch {
  std::vector<void*> ptrs;
  cudaStream_t st;
  ~PllScratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <class T>
  int alloc(T** p, uint64_t count) {
    void* x = nullptr;
    if (cudaMallocAsync(&x, sizeof(T) * (count ? count : 1), st) != cudaSuccess) {
      cudaGetLastError();
      return fail(CBFS_ENOMEM, "PLL scratch allocation");
    }
    ptrs.push_back(x);
    *p = reinterpret_cast<T*>(x);
    return CBFS_OK;
  }
};

static void pll_free(Pll* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  cudaFree(P->cdist);
  cudaFree(P->cmask);
  cudaFree(P->counts);
  cudaFree(P->entries);
  delete P;
}

static int pll_build(Graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t C, Pll* P, cudaStream_t st) {
  const uint32_t n = g->n;
  const uint64_t N = n ? n : 1;
  struct Events {  // destroyed on every return path
    cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    ~Events() {
      for (cudaEvent_t x : e)
        if (x) cudaEventDestroy(x);
    }
  } E;
  cudaEvent_t* ev = E.e;
  for (int k = 0; k < 3; ++k) CBFS_CUDA(cudaEventCreate(&ev[k]));
  CBFS_CUDA(cudaEventRecord(ev[0], st));
  if (cudaMalloc(&P->cdist, sizeof(uint16_t) * N * (C ? C : 1)) != cudaSuccess ||
      cudaMalloc(&P->cmask, sizeof(uint64_t) * P->planes * N * (C ? C : 1)) != cudaSuccess ||
      cudaMalloc(&P->counts, sizeof(uint32_t) * N) != cudaSuccess ||
      cudaMalloc(&P->entries, sizeof(uint32_t) * N * P->cap) != cudaSuccess) {
    cudaGetLastError();
    return fail(CBFS_ENOMEM, "PLL index allocation");
  }
  CBFS_CUDA(cudaMemsetAsync(P->counts, 0, sizeof(uint32_t) * N, st));
  PllScratch S;
  S.st = st;
  int* bad = nullptr;
  uint8_t *covered = nullptr, *rflag = nullptr;
  int rc;
  if ((rc = S.alloc(&bad, 1)) || (rc = S.alloc(&covered, N)) || (rc = S.alloc(&rflag, N))) return rc;
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(covered, 0, N, st));
  // ---- phase 1: the clusters' C-BFS (one batch of <= 64 lanes), rows by internal id
  if (C) {
    k_pll_flags<<<(unsigned)(((uint64_t)C * 64 + 255) / 256), 256, 0, st>>>(sources, sizes, C, g->inv, n, covered, bad);
    CBFS_LAUNCHED();
    int hbad = 0;
    CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    if (hbad) return fail(CBFS_EINVAL, (hbad & 1) ? "cluster size must be 1..64" : "source id >= n");
    CBFS_CUDA(cudaMemsetAsync(P->cdist, 0xFF, sizeof(uint16_t) * N * C, st));
    CBFS_CUDA(cudaMemsetAsync(P->cmask, 0, sizeof(uint64_t) * P->planes * N * C, st));
    WorkLease lease(g);
    if (lease.rc) return lease.rc;
    ArraySource src;
    src.proto = RunArgs{};
    src.proto.d = P->d;
    src.proto.planes = P->planes;
    src.proto.dist_bytes = 2;
    src.proto.C = C;
    src.proto.direction = CBFS_DIR_AUTO;
    src.proto.engine = choose_engine(g, CBFS_DIR_AUTO);
    if (src.proto.engine < 0) return CBFS_ECUDA;
    src.proto.out_internal = 1;
    src.proto.out_dist = P->cdist;
    src.proto.out_masks = P->cmask;
    src.sources = sources;
    src.sizes = sizes;
    src.n_clusters = C;
    rc = run_batches(g, src, st);
    if (rc) return rc;
    CBFS_CUDA(cudaStreamSynchronize(st));  // the workspace lease ends here
  }
  CBFS_CUDA(cudaEventRecord(ev[1], st));
  // ---- phase 2 roots: uncovered vertices in position order
  uint32_t* roots = nullptr;
  uint32_t* nroots_d = nullptr;
  if ((rc = S.alloc(&roots, N)) || (rc = S.alloc(&nroots_d, 1))) return rc;
  k_pll_root_flags<<<grid_for(n, 256), 256, 0, st>>>(g->order, covered, n, rflag);
  CBFS_LAUNCHED();
  size_t tb = 0;
  CBFS_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, g->order, rflag, roots, nroots_d, (int64_t)n, st));
  void* tsel = nullptr;
  if ((rc = S.alloc(reinterpret_cast<uint8_t**>(&tsel), tb))) return rc;
  CBFS_CUDA(cub::DeviceSelect::Flagged(tsel, tb, g->order, rflag, roots, nroots_d, (int64_t)n, st));
  uint32_t nroots = 0;
  CBFS_CUDA(cudaMemcpyAsync(&nroots, nroots_d, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  P->roots = nroots;
  // ---- per-CTA scratch: visited stamps, hub map, two frontier queues (13 n bytes)
  size_t fr = 0, tot = 0;
  CBFS_CUDA(cudaMemGetInfo(&fr, &tot));
  const uint64_t per_cta = 13ull * N;
  uint64_t want_ctas = 148ull * (2048 / PLL_THREADS);  // persistent CTAs: one resident set
  if (const char* e = getenv("CBFS_PLL_CTAS")) want_ctas = std::max(1, atoi(e));  // experiments
  uint32_t ctas = std::min<uint64_t>(want_ctas, std::max<uint64_t>(1, (fr / 4) / per_cta));
  ctas = std::min<uint32_t>(ctas, std::max<uint32_t>(1, std::min(P->bmax, nroots)));
  uint32_t *visited = nullptr, *queues = nullptr, *snap = nullptr;
  uint8_t* tmpmap = nullptr;
  unsigned long long *ctl = nullptr, *stats = nullptr;
  if ((rc = S.alloc(&visited, (uint64_t)ctas * N)) || (rc = S.alloc(&tmpmap, (uint64_t)ctas * N)) ||
      (rc = S.alloc(&queues, 2ull * ctas * N)) || (rc = S.alloc(&snap, N)) || (rc = S.alloc(&ctl, 4)) ||
      (rc = S.alloc(&stats, 2)))
    return rc;
  CBFS_CUDA(cudaMemsetAsync(visited, 0, sizeof(uint32_t) * ctas * N, st));
  CBFS_CUDA(cudaMemsetAsync(tmpmap, 0xFF, (uint64_t)ctas * N, st));
  CBFS_CUDA(cudaMemsetAsync(ctl, 0, 4 * sizeof(unsigned long long), st));
  const size_t smem = (size_t)C * (8 * (P->d + 1) + 4);
  CBFS_CUDA(cudaFuncSetAttribute(k_pll_bfs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLL_SMEM_MAX));
  // batches run back to back on the stream (no host round trip): each takes
  // a snapshot of the list lengths, then its roots' pruned BFSs; errors
  // accumulate in ctl[2] and are checked once at the end
  uint32_t b = std::min(P->first, P->bmax);
  uint32_t batches = 0;
  for (uint32_t r0 = 0; r0 < nroots; r0 += b, b = std::min<uint32_t>(P->bmax, b * 3 / 2)) {
    const uint32_t nb = std::min(b, nroots - r0);
    ++batches;
    CBFS_CUDA(cudaMemcpyAsync(snap, P->counts, sizeof(uint32_t) * N, cudaMemcpyDeviceToDevice, st));
    CBFS_CUDA(cudaMemsetAsync(ctl, 0, sizeof(unsigned long long), st));  // the batch's root counter
    k_pll_bfs<<<std::min(ctas, nb), PLL_THREADS, smem, st>>>(g->off, g->cols, g->rank, n, roots + r0, nb, r0, C, P->d,
                                                             P->cdist, P->cmask, P->counts, snap, P->entries, P->cap,
                                                             P->entries, ctl, visited, tmpmap, queues);
    CBFS_LAUNCHED();
  }
  unsigned long long hctl[4];
  CBFS_CUDA(cudaMemcpyAsync(hctl, ctl, sizeof(hctl), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (hctl[2] & PLL_ERR_CAP) return fail(CBFS_EOVERFLOW, "a PLL label list exceeds cap");
  if (hctl[2] & PLL_ERR_DIST) return fail(CBFS_EOVERFLOW, "a PLL label distance exceeds 254");
  uint32_t P2 = 1;
  while (P2 < P->cap) P2 <<= 1;
  CBFS_CUDA(cudaFuncSetAttribute(k_pll_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(P2 * 4)));
  k_pll_sort<<<148 * 8, 256, P2 * 4, st>>>(P->entries, P->counts, n, P->cap);
  CBFS_LAUNCHED();
  P->batches = batches;
  CBFS_CUDA(cudaEventRecord(ev[2], st));
  CBFS_CUDA(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), st));
  k_pll_stats<<<grid_for(n, 256), 256, 0, st>>>(P->counts, n, stats);
  CBFS_LAUNCHED();
  unsigned long long hs[2] = {0, 0};
  CBFS_CUDA(cudaMemcpyAsync(hs, stats, sizeof(hs), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  P->total = hs[0];
  P->max_count = (uint32_t)hs[1];
  CBFS_CUDA(cudaEventElapsedTime(&P->ms_cbfs, ev[0], ev[1]));
  CBFS_CUDA(cudaEventElapsedTime(&P->ms_pbfs, ev[1], ev[2]));
  return CBFS_OK;
}

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_pll_build(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                   uint32_t first, uint32_t bmax, uint32_t cap, cbfs_pll** out, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (!out) return fail(CBFS_EINVAL, "null out");
  *out = nullptr;
  if (!g) return fail(CBFS_EINVAL, "null graph");
  if (d > CBFS_MAX_D) return fail(CBFS_EUNSUPPORTED, "d > CBFS_MAX_D");
  if ((uint64_t)n_clusters * (8ull * (d + 1) + 4) > PLL_SMEM_MAX)
    return fail(CBFS_EUNSUPPORTED, "too many first-phase clusters for d (n_clusters * (8 (d+1) + 4) > 200 KB)");
  if (n_clusters && (!sources || !sizes)) return fail(CBFS_EINVAL, "null sources/sizes");
  if (first == 0 || bmax == 0 || cap == 0) return fail(CBFS_EINVAL, "first, bmax and cap must be >= 1");
  if (cap > PLL_MAX_CAP) return fail(CBFS_EUNSUPPORTED, "cap > 8192 label entries per vertex");
  if (g->n >= (1u << 24)) return fail(CBFS_EUNSUPPORTED, "PLL hub positions are 24-bit (n < 2^24)");
  CBFS_CUDA(cudaSetDevice(g->device));
  Pll* P = new Pll();
  P->device = g->device;
  P->g = g;
  P->n = g->n;
  P->C = n_clusters;
  P->d = d;
  P->planes = d + 1;
  P->cap = cap;
  P->first = first;
  P->bmax = bmax;
  int rc = pll_build(g, sources, sizes, n_clusters, P, (cudaStream_t)stream);
  if (rc != CBFS_OK) {
    cudaStreamSynchronize((cudaStream_t)stream);
    pll_free(P);
    return rc;
  }
  *out = reinterpret_cast<cbfs_pll*>(P);
  return CBFS_OK;
}

int cbfs_pll_info(const cbfs_pll* ph, uint64_t* total_labels, uint32_t* max_labels, uint32_t* roots,
                  uint32_t* batches, float* ms_cbfs, float* ms_pbfs) {
  const Pll* P = reinterpret_cast<const Pll*>(ph);
  if (!P) return fail(CBFS_EINVAL, "null PLL index");
  if (total_labels) *total_labels = P->total;
  if (max_labels) *max_labels = P->max_count;
  if (roots) *roots = P->roots;
  if (batches) *batches = P->batches;
  if (ms_cbfs) *ms_cbfs = P->ms_cbfs;
  if (ms_pbfs) *ms_pbfs = P->ms_pbfs;
  return CBFS_OK;
}

int cbfs_pll_export(const cbfs_pll* ph, uint32_t* counts, uint32_t* entries, cbfs_stream stream) {
  const Pll* P = reinterpret_cast<const Pll*>(ph);
  if (!P) return fail(CBFS_EINVAL, "null PLL index");
  if (!counts && !entries) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  k_pll_export<<<grid_for((uint64_t)P->n * 32, 256), 256, 0, st>>>(P->g->perm, P->n, P->cap, P->counts, P->entries,
                                                                  counts, entries);
  CBFS_LAUNCHED();
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

int cbfs_pll_query(const cbfs_pll* ph, const uint32_t* s, const uint32_t* t, uint64_t q, int32_t* out,
                   cbfs_stream stream) {
  const Pll* P = reinterpret_cast<const Pll*>(ph);
  if (!P) return fail(CBFS_EINVAL, "null PLL index");
  if (q == 0) return CBFS_OK;
  if (!s || !t || !out) return fail(CBFS_EINVAL, "null query arrays");
  CBFS_CUDA(cudaSetDevice(P->device));
  cudaStream_t st = (cudaStream_t)stream;
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  k_pll_query<<<grid_for(q * 32, 256, 148u * 64u), 256, 0, st>>>(P->g->inv, P->n, P->C, P->d, P->cdist, P->cmask,
                                                                  P->counts, P->entries, P->cap, s, t, q, out, bad);
  CBFS_LAUNCHED();
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaFreeAsync(bad, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (hbad) return fail(CBFS_EINVAL, "query vertex id >= n");
  return CBFS_OK;
}

int cbfs_pll_destroy(cbfs_pll* ph) {
  pll_free(reinterpret_cast<Pll*>(ph));
  return CBFS_OK;
}

}  // extern "C"
