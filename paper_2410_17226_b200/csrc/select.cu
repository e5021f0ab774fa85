// select.cu — cluster selection (§8(a) row A1): "Selecting Landmarks in
// Clusters", with reading R12.
//
// The greedy rule is inherently sequential (each cluster's marks constrain
// the next), so one 1024-thread CTA runs the cluster loop and parallelises
// inside a cluster: the root scan over the (degree desc, id asc) order (warp
// 0, 32 positions per step), the floor(d/2)-hop ball expansion, and the k-1
// best candidates (rank = position in that order; ranks are unique): up to
// 1024 candidates each thread counts the candidates ranked before its own,
// which is its position; beyond that a block radix select of the (k-1)-th
// smallest rank gives an exact threshold.  About three block barriers per
// cluster: the loop is barrier-latency bound.
#include <algorithm>

#include "common.cuh"

namespace cbfs {

constexpr int SEL_THREADS = 1024;
constexpr uint32_t SEL_PUBLISH = 8;

struct SelScratch {
  uint8_t* marked;
  uint32_t* stamp;
  uint32_t* fa;    // BFS level lists
  uint32_t* fb;
  uint32_t* cand;  // candidate ranks
};

__global__ void __launch_bounds__(SEL_THREADS, 1)
k_select(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, const uint32_t* __restrict__ rank,
         const uint32_t* __restrict__ order, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ inv,
         uint32_t n, uint32_t r, uint32_t k, uint32_t d, uint32_t policy, uint64_t seed, SelScratch S,
         uint32_t* __restrict__ out_sources, uint8_t* __restrict__ out_sizes, uint32_t* __restrict__ out_count,
         volatile uint32_t* progress, uint32_t stride, uint16_t* __restrict__ out_sizes16) {
  __shared__ unsigned s_na, s_nb, s_nc, s_nsel, s_root;
  __shared__ unsigned long long s_avail;
  __shared__ unsigned hist[256];
  __shared__ unsigned s_need, s_prefix, s_pmask;
  __shared__ unsigned sel[64 * CBFS_WIDE_MAX_W];
  __shared__ unsigned s_cand[SEL_THREADS];  // the first SEL_THREADS candidate ranks (the common case)
  const unsigned tid = threadIdx.x, lane = tid & 31;
  const uint32_t h = d / 2;
  const unsigned want = k - 1;
  const int rank_bits = max(1, 32 - __clz((int)max(n, 2u) - 1));  // ranks < n
  // available = unmarked non-isolated vertices
  if (tid == 0) s_avail = 0;
  __syncthreads();
  unsigned long long loc = 0;
  for (uint32_t v = tid; v < n; v += SEL_THREADS) loc += off[v + 1] > off[v];
  atomicAdd(&s_avail, loc);
  __syncthreads();
  uint32_t produced = 0;
  unsigned long long cursor = 0, tdraw = 0;  // warp 0's root-scan state
  uint32_t* fa = S.fa;
  uint32_t* fb = S.fb;
  for (uint32_t c = 0; c < r; ++c) {
    const uint32_t tag = c + 1;
    // ---- root (R12), by warp 0; the ball's first level is set up with it
    if (tid < 32) {
      uint32_t root = 0xFFFFFFFFu;
      if (s_avail != 0) {
        if (policy == CBFS_ROOT_DEGREE) {
          while (cursor < n) {  // next unmarked non-isolated vertex in (degree desc, id asc) order
            const unsigned long long p = cursor + lane;
            bool ok = false;
            if (p < n) {
              const uint32_t x = order[p];
              ok = !S.marked[x] && off[x + 1] > off[x];
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
            if (m) {
              cursor += __ffs(m) - 1;
              root = order[cursor];
              break;
            }
            cursor += 32;
          }
        } else if (lane == 0) {
          for (;;) {
            const uint32_t v = (uint32_t)bounded(crand(seed, 1, tdraw++), n);
            const uint32_t x = inv ? inv[v] : v;
            if (!S.marked[x] && off[x + 1] > off[x]) { root = x; break; }
          }
        }
      }
      if (lane == 0) {
        s_root = root;
        s_na = 1;
        s_nb = 0;
        s_nc = 0;
        s_nsel = 0;
        if (root != 0xFFFFFFFFu) {
          fa[0] = root;
          S.stamp[root] = tag;
        }
      }
    }
    __syncthreads();
    const uint32_t root = s_root;
    if (root == 0xFFFFFFFFu) break;
    // ---- floor(d/2)-hop ball through all vertices; unmarked ones are candidates
    for (uint32_t lev = 1; lev <= h; ++lev) {
      const unsigned na = s_na;
      for (unsigned q = 0; q < na; ++q) {
        const uint32_t u = fa[q];
        const uint64_t b = off[u], e = off[u + 1];
        for (uint64_t t = b + tid; t < e; t += SEL_THREADS) {
          const uint32_t v = cols[t];
          if (atomicExch(&S.stamp[v], tag) != tag) {
            if (lev < h) fb[atomicAdd(&s_nb, 1u)] = v;
            if (!S.marked[v]) {
              const unsigned ci = atomicAdd(&s_nc, 1u);
              const unsigned rk = rank[v];
              S.cand[ci] = rk;
              if (ci < SEL_THREADS) s_cand[ci] = rk;
            }
          }
        }
      }
      uint32_t* tmp = fa; fa = fb; fb = tmp;
      __syncthreads();
      if (lev < h) {
        if (tid == 0) { s_na = s_nb; s_nb = 0; }
        __syncthreads();
      }
    }
    // ---- the best k-1 candidates by rank (degree desc, id asc), in rank order
    const unsigned nc = s_nc;
    const unsigned ns = min(nc, want);
    uint32_t* outS = out_sources + (uint64_t)c * stride;
    unsigned long long dec = 0;
    if (nc <= SEL_THREADS) {
      // rank by counting (ranks are unique): candidate t is selected iff fewer
      // than `want` candidates precede it, and that count is its position
      if (tid < nc) {
        const unsigned rk = s_cand[tid];
        unsigned pos = 0;
        for (unsigned j = 0; j < nc && pos < want; ++j) pos += s_cand[j] < rk;
        if (pos < want) {
          const uint32_t x = order[rk];
          outS[1 + pos] = perm ? perm[x] : x;
          S.marked[x] = 1;
          dec += off[x + 1] > off[x];
        }
      }
    } else {
      // radix select of the want-th smallest rank (8-bit digits over the rank bits)
      if (tid == 0) { s_need = want; s_prefix = 0; s_pmask = 0; }
      __syncthreads();
      const int passes = (rank_bits + 7) / 8;
      for (int pass = 0; pass < passes; ++pass) {
        const int shift = 8 * (passes - 1 - pass);
        for (unsigned b = tid; b < 256; b += SEL_THREADS) hist[b] = 0;
        __syncthreads();
        const unsigned pre = s_prefix, pm = s_pmask;
        for (unsigned t = tid; t < nc; t += SEL_THREADS) {
          const unsigned rk = S.cand[t];
          if ((rk & pm) == pre) atomicAdd(&hist[(rk >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {  // the bucket holding the need-th smallest: warp prefix over 8 buckets per lane
          unsigned lc[8], sum = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) { lc[q] = hist[tid * 8 + q]; sum += lc[q]; }
          unsigned incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (tid >= (unsigned)o) incl += y;
          }
          const unsigned need = s_need;
          unsigned cum = incl - sum;
          if (cum < need && incl >= need) {
            unsigned b = tid * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (cum + lc[q] >= need) { b = tid * 8 + q; break; }
              cum += lc[q];
            }
            s_need = need - cum;
            s_prefix = pre | (b << shift);
            s_pmask = pm | (255u << shift);
          }
        }
        __syncthreads();
      }
      const unsigned thr = s_prefix;  // the want-th smallest rank
      for (unsigned t = tid; t < nc; t += SEL_THREADS) {
        const unsigned rk = S.cand[t];
        if (rk <= thr) sel[atomicAdd(&s_nsel, 1u)] = rk;
      }
      __syncthreads();
      if (tid < ns) {
        const unsigned rk = sel[tid];
        unsigned pos = 0;
        for (unsigned j = 0; j < ns; ++j) pos += sel[j] < rk;
        const uint32_t x = order[rk];
        outS[1 + pos] = perm ? perm[x] : x;
        S.marked[x] = 1;
        dec += off[x + 1] > off[x];
      }
    }
    if (tid == 0) {
      outS[0] = perm ? perm[root] : root;
      S.marked[root] = 1;
      dec += 1;  // root is non-isolated
      if (out_sizes16) out_sizes16[c] = (uint16_t)(1 + ns);
      else out_sizes[c] = (uint8_t)(1 + ns);
    }
    if (dec) atomicAdd(&s_avail, (unsigned long long)0 - dec);  // subtract
    ++produced;
    // publish to a concurrent traversal (cbfs_select_and_run*) every
    // SEL_PUBLISH clusters (a system-scope fence per cluster costs more than
    // the batches, which need 64 clusters at a time, can use)
    const bool publish = progress && (produced % SEL_PUBLISH) == 0;
    if (publish) __threadfence();
    __syncthreads();
    if (publish && tid == 0) {
      __threadfence_system();
      progress[0] = produced;
    }
  }
  if (tid == 0) {
    *out_count = produced;
    if (progress) {
      __threadfence_system();
      progress[0] = produced;
      progress[1] = 1;
    }
  }
}

}  // namespace cbfs

using namespace cbfs;

namespace cbfs {
// Queue the selection on `st`; the count lands in device memory *d_count and,
// if `progress` (mapped pinned host memory) is given, is published after
// every cluster.
int select_launch(const Graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy, uint64_t seed,
                  uint32_t* out_sources, uint8_t* out_sizes, uint32_t* d_count, volatile uint32_t* progress,
                  cudaStream_t st, uint32_t words, uint16_t* out_sizes16) {
  const uint32_t n = g->n;
  SelScratch S;
  CBFS_CUDA(cudaMallocAsync(&S.marked, n, st));
  CBFS_CUDA(cudaMallocAsync(&S.stamp, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMallocAsync(&S.fa, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMallocAsync(&S.fb, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMallocAsync(&S.cand, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMemsetAsync(S.marked, 0, n, st));
  CBFS_CUDA(cudaMemsetAsync(S.stamp, 0, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMemsetAsync(out_sources, 0xFF, sizeof(uint32_t) * 64ULL * words * r, st));
  if (out_sizes16) CBFS_CUDA(cudaMemsetAsync(out_sizes16, 0, sizeof(uint16_t) * (uint64_t)r, st));
  else CBFS_CUDA(cudaMemsetAsync(out_sizes, 0, r, st));
  k_select<<<1, SEL_THREADS, 0, st>>>(g->off, g->cols, g->rank, g->order, g->perm, g->inv, n, r, k, d, root_policy,
                                      seed, S, out_sources, out_sizes, d_count, progress, 64 * words, out_sizes16);
  CBFS_LAUNCHED();
  CBFS_CUDA(cudaFreeAsync(S.marked, st));
  CBFS_CUDA(cudaFreeAsync(S.stamp, st));
  CBFS_CUDA(cudaFreeAsync(S.fa, st));
  CBFS_CUDA(cudaFreeAsync(S.fb, st));
  CBFS_CUDA(cudaFreeAsync(S.cand, st));
  return CBFS_OK;
}

int check_select_args(const Graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                      const void* out_sources, const void* out_sizes) {
  if (!g || (r && (!out_sources || !out_sizes))) return fail(CBFS_EINVAL, "null argument");
  if (k == 0) return fail(CBFS_EINVAL, "k must be >= 1");
  if (k > CBFS_MAX_K) return fail(CBFS_EUNSUPPORTED, "k > 64");
  if (d > CBFS_MAX_D) return fail(CBFS_EUNSUPPORTED, "d > CBFS_MAX_D");
  if (root_policy > CBFS_ROOT_RANDOM) return fail(CBFS_EINVAL, "bad root policy");
  return CBFS_OK;
}
}  // namespace cbfs

extern "C" int cbfs_select_clusters_wide(const cbfs_graph* gh, uint32_t r, uint32_t k, uint32_t d,
                                         uint32_t root_policy, uint64_t seed, uint32_t words, uint32_t* out_sources,
                                         uint16_t* out_sizes, uint32_t* out_r, cbfs_stream stream) {
  const Graph* g = reinterpret_cast<const Graph*>(gh);
  if (words != 1 && words != 2 && words != 4 && words != 8) return fail(CBFS_EUNSUPPORTED, "words must be 1, 2, 4 or 8");
  if (k > 64 * words) return fail(CBFS_EINVAL, "k > 64 * words");
  int rc = check_select_args(g, r, k <= CBFS_MAX_K ? k : 1, d, root_policy, out_sources, out_sizes);
  if (rc) return rc;
  if (k == 0) return fail(CBFS_EINVAL, "k must be >= 1");
  if (!out_r) return fail(CBFS_EINVAL, "null out_r");
  *out_r = 0;
  if (r == 0 || g->n == 0) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* d_count = nullptr;
  CBFS_CUDA(cudaMallocAsync(&d_count, sizeof(uint32_t), st));
  rc = select_launch(g, r, k, d, root_policy, seed, out_sources, nullptr, d_count, nullptr, st, words, out_sizes);
  if (rc) return rc;
  CBFS_CUDA(cudaMemcpyAsync(out_r, d_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaFreeAsync(d_count, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

extern "C" int cbfs_select_clusters(const cbfs_graph* gh, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                                    uint64_t seed, uint32_t* out_sources, uint8_t* out_sizes, uint32_t* out_r,
                                    cbfs_stream stream) {
  const Graph* g = reinterpret_cast<const Graph*>(gh);
  int rc = check_select_args(g, r, k, d, root_policy, out_sources, out_sizes);
  if (rc) return rc;
  if (!out_r) return fail(CBFS_EINVAL, "null out_r");
  *out_r = 0;
  if (r == 0 || g->n == 0) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* d_count = nullptr;
  CBFS_CUDA(cudaMallocAsync(&d_count, sizeof(uint32_t), st));
  rc = select_launch(g, r, k, d, root_policy, seed, out_sources, out_sizes, d_count, nullptr, st, 1, nullptr);
  if (rc) return rc;
  CBFS_CUDA(cudaMemcpyAsync(out_r, d_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaFreeAsync(d_count, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}
