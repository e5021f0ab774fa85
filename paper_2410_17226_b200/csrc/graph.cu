// graph.cu — device CSR builder (§8(a) row A0, R17, R18).
//
// Undirected pairs -> 64-bit arc keys (u<<32|v and v<<32|u; self loops map to
// a sentinel row n) -> CUB radix sort over the low 32+ceil(log2(n+1)) bits ->
// unique -> CSR (u64 offsets, u32 cols).  Optional degree relabelling: order
// vertices by (degree desc, original id asc), rebuild the CSR in that order
// (hubs get small ids, so their vertex-major rows share cache lines and L2
// sets).  The rank array used by cluster selection is the same order.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace cbfs {

// ------------------------------------------------------------- errors
static thread_local std::string g_err;
static thread_local uint64_t g_launches = 0;
void set_error(const std::string& m) { g_err = m; }
int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? CBFS_ENOMEM : CBFS_ECUDA;
}
void count_launch(uint64_t k) { g_launches += k; }
uint64_t launches(int reset) {
  uint64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

// Keep freed memory in the device's stream-ordered pool: with the default
// release threshold (0) every synchronisation hands the pool back to the
// driver and the next allocation pays for page mapping again.
void keep_pool(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

// ------------------------------------------------------------- kernels
__global__ void k_make_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t P,
                            uint32_t n, uint64_t* __restrict__ keys, int* __restrict__ bad) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < P; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u = src[e], v = dst[e];
    uint64_t a, b;
    if (u >= n || v >= n) {
      *bad = 1;
      a = b = (uint64_t)n << 32;
    } else if (u == v) {
      a = b = (uint64_t)n << 32;  // self loop -> sentinel row n, dropped after unique
    } else {
      a = ((uint64_t)u << 32) | v;
      b = ((uint64_t)v << 32) | u;
    }
    keys[2 * e] = a;
    keys[2 * e + 1] = b;
  }
}

// CSR arcs -> pair keys (each arc u->v contributes u<<32|v and v<<32|u)
__global__ void k_csr_keys(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, uint32_t n,
                           uint64_t* __restrict__ keys, int* __restrict__ bad) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
    for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t v = cols[e];
      uint64_t a, b;
      if (v >= n) { *bad = 1; a = b = (uint64_t)n << 32; }
      else if (v == u) { a = b = (uint64_t)n << 32; }
      else { a = ((uint64_t)u << 32) | v; b = ((uint64_t)v << 32) | u; }
      keys[2 * e] = a;
      keys[2 * e + 1] = b;
    }
  }
}

// sorted (row << 32 | col) keys -> cols; the row offsets come from
// k_row_offsets (a binary search per row: runs of empty rows — the isolated
// vertices, all at the end after the degree relabel — cost nothing extra)
__global__ void k_split_keys(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ cols) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
    cols[e] = (uint32_t)keys[e];
}
// off[x] = first e with row(keys[e]) >= x, x = 0..n
__global__ void k_row_offsets(const uint64_t* __restrict__ keys, uint64_t m, uint32_t n, uint64_t* __restrict__ off) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x <= n; x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if ((keys[mid] >> 32) < x) lo = mid + 1; else hi = mid;
    }
    off[x] = lo;
  }
}

__global__ void k_degree_keys(const uint64_t* __restrict__ off, uint32_t n, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ maxdeg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t deg = (uint32_t)(off[v + 1] - off[v]);
    keys[v] = ((uint64_t)(0xFFFFFFFFu - deg) << 32) | v;  // ascending = degree desc, id asc
    atomicMax(maxdeg, deg);
    if (deg) atomicAdd(maxdeg + 1, 1u);  // non-isolated count
  }
}

__global__ void k_order_from_keys(const uint64_t* __restrict__ keys, uint32_t n, uint32_t* __restrict__ order,
                                  uint32_t* __restrict__ rank) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = (uint32_t)keys[p];
    order[p] = v;
    rank[v] = (uint32_t)p;
  }
}

// arc-parallel: (u<<32|v) -> (inv[u]<<32 | inv[v])
__global__ void k_relabel_keys(const uint64_t* __restrict__ arcs, uint64_t m, const uint32_t* __restrict__ inv,
                               uint64_t* __restrict__ keys) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = arcs[e];
    keys[e] = ((uint64_t)inv[a >> 32] << 32) | inv[(uint32_t)a];
  }
}

// ---- locality order (CBFS_RELABEL_LOCALITY): a deterministic
// Cuthill-McKee-like BFS order.  Level L+1 is sorted by (smallest position of
// a parent in level L, original id), so vertices near each other in the graph
// get nearby ids and a cluster's wavefront touches contiguous state.
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Every BFS level runs inside one cooperative kernel (no host round trip
// and no sort per level; config 4's 4096^2 grid has ~6,000 BFS levels):
// (1) every unplaced neighbour v of the level's parents (positions p in
// [lo, hi)) gets key[v] = min p; (2) each warp owns a contiguous run of
// parents and counts, 32 parents at a time, the neighbours whose key is that
// parent — a parent's children are its own adjacency (sorted by id) filtered
// by key, so the level's (key, id) order needs no sort — and warp / block /
// grid prefix sums give each warp its first position; (3) the warp places its
// parents' children in (parent, id) order.  Three grid barriers per level.
constexpr int BO_THREADS = 256, BO_WARPS = BO_THREADS / 32;

__device__ __forceinline__ uint32_t bo_children(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols,
                                                const uint32_t* __restrict__ perm, const uint32_t* __restrict__ pos,
                                                const uint32_t* __restrict__ key, uint64_t p) {
  const uint32_t u = __ldcg(&perm[p]);
  uint32_t c = 0;
  for (uint64_t a = __ldg(&off[u]), e = __ldg(&off[u + 1]); a < e; ++a) {
    const uint32_t v = __ldg(&cols[a]);
    c += (__ldcg(&pos[v]) == 0xFFFFFFFFu && __ldcg(&key[v]) == (uint32_t)p) ? 1u : 0u;
  }
  return c;
}

__global__ void __launch_bounds__(BO_THREADS) k_bfsord_coop(const uint64_t* __restrict__ off,
                                                            const uint32_t* __restrict__ cols, uint32_t* __restrict__ perm,
                                                            uint32_t* __restrict__ pos, uint32_t* __restrict__ key,
                                                            unsigned long long* __restrict__ blk,
                                                            uint32_t* __restrict__ out_hi) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long s_w[BO_WARPS];
  __shared__ unsigned long long s_red[BO_THREADS];
  __shared__ unsigned long long s_base, s_total;
  const uint32_t nb = gridDim.x, b = blockIdx.x, t = threadIdx.x, lane = t & 31, wib = t >> 5;
  const uint64_t nw = (uint64_t)nb * BO_WARPS, w = (uint64_t)b * BO_WARPS + wib;
  const uint64_t nth = (uint64_t)nb * BO_THREADS, tid = (uint64_t)b * BO_THREADS + t;
  uint32_t lo = 0, hi = 1;
  while (lo < hi) {
    const uint64_t np = hi - lo;
    // (1) keys, thread per parent
    for (uint64_t p = lo + tid; p < hi; p += nth) {
      const uint32_t u = __ldcg(&perm[p]);
      for (uint64_t a = __ldg(&off[u]), e = __ldg(&off[u + 1]); a < e; ++a) {
        const uint32_t v = __ldg(&cols[a]);
        if (__ldcg(&pos[v]) == 0xFFFFFFFFu) atomicMin(&key[v], (uint32_t)p);
      }
    }
    grid.sync();
    // (2) the warp's run of parents [wp0, wp1), children counted 32 parents at a time
    const uint64_t per_w = (np + nw - 1) / nw;
    const uint64_t wp0 = lo + umin64(np, w * per_w), wp1 = lo + umin64(np, (w + 1) * per_w);
    unsigned long long wsum = 0;
    for (uint64_t c0 = wp0; c0 < wp1; c0 += 32) {
      const uint64_t p = c0 + lane;
      const uint32_t c = p < wp1 ? bo_children(off, cols, perm, pos, key, p) : 0u;
      uint32_t cs = c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xFFFFFFFFu, cs, o);
      wsum += cs;
    }
    if (lane == 0) s_w[wib] = wsum;
    __syncthreads();
    if (t == 0) {
      unsigned long long x = 0;
      for (int k = 0; k < BO_WARPS; ++k) {
        const unsigned long long y = s_w[k];
        s_w[k] = x;  // exclusive prefix of the block's warps
        x += y;
      }
      blk[b] = x;
    }
    grid.sync();
    {  // this block's base and the level's total (block-parallel sums of the block totals)
      unsigned long long base = 0, tot = 0;
      for (uint32_t k = t; k < nb; k += BO_THREADS) {
        const unsigned long long x = __ldcg(&blk[k]);
        if (k < b) base += x;
        tot += x;
      }
      s_red[t] = base;
      __syncthreads();
      for (uint32_t o = BO_THREADS / 2; o > 0; o >>= 1) {
        if (t < o) s_red[t] += s_red[t + o];
        __syncthreads();
      }
      if (t == 0) s_base = s_red[0];
      __syncthreads();
      s_red[t] = tot;
      __syncthreads();
      for (uint32_t o = BO_THREADS / 2; o > 0; o >>= 1) {
        if (t < o) s_red[t] += s_red[t + o];
        __syncthreads();
      }
      if (t == 0) s_total = s_red[0];
      __syncthreads();
    }
    // (3) place, 32 parents at a time: lane offsets by a warp scan of the counts
    unsigned long long q = hi + s_base + s_w[wib];
    for (uint64_t c0 = wp0; c0 < wp1; c0 += 32) {
      const uint64_t p = c0 + lane;
      const uint32_t c = p < wp1 ? bo_children(off, cols, perm, pos, key, p) : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      if (c) {
        uint64_t r = q + inc - c;
        const uint32_t u = __ldcg(&perm[p]);
        for (uint64_t a = __ldg(&off[u]), e = __ldg(&off[u + 1]); a < e; ++a) {
          const uint32_t v = __ldg(&cols[a]);
          if (__ldcg(&pos[v]) == 0xFFFFFFFFu && __ldcg(&key[v]) == (uint32_t)p) {
            perm[r] = v;
            pos[v] = (uint32_t)r;
            ++r;
          }
        }
      }
      q += __shfl_sync(0xFFFFFFFFu, inc, 31);
    }
    const uint32_t total = (uint32_t)s_total;
    grid.sync();
    lo = hi;
    hi += total;
  }
  if (b == 0 && t == 0) *out_hi = hi;
}

// vertices the BFS did not reach (other components), appended in id order
__global__ void k_bfsord_flags(const uint32_t* __restrict__ pos, uint32_t n, uint32_t* __restrict__ f) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    f[v] = pos[v] == 0xFFFFFFFFu ? 1u : 0u;
}
__global__ void k_bfsord_rest(const uint32_t* __restrict__ f, const uint32_t* __restrict__ x, uint32_t n,
                              uint32_t base, uint32_t* __restrict__ order, uint32_t* __restrict__ pos) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    if (f[v]) {
      order[base + x[v]] = (uint32_t)v;
      pos[v] = base + x[v];
    }
}
// degree order (sorted keys of original ids) expressed in internal ids
__global__ void k_order_map(const uint64_t* __restrict__ keys, uint32_t n, const uint32_t* __restrict__ inv,
                            uint32_t* __restrict__ order, uint32_t* __restrict__ rank) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = inv[(uint32_t)keys[p]];
    order[p] = x;
    rank[x] = (uint32_t)p;
  }
}

__global__ void k_identity(uint32_t* a, uint32_t n) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    a[v] = (uint32_t)v;
}

__global__ void k_chunk_table(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ chunk_v) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = (off[v] + PULL_CHUNK - 1) / PULL_CHUNK, hi = (off[v + 1] + PULL_CHUNK - 1) / PULL_CHUNK;
    for (uint64_t w = lo; w < hi; ++w) chunk_v[w] = (uint32_t)v;
  }
}

// ------------------------------------------------------------- helpers
static int bits_for(uint64_t x) {
  int b = 0;
  while ((1ULL << b) <= x && b < 63) ++b;
  return b;
}

// sort + unique the 2P keys in `keys` (device, length L); returns arcs in
// `*out_keys` (device, freshly allocated, caller frees) and m.
static int sort_unique(uint64_t* keys, uint64_t L, uint32_t n, cudaStream_t st, uint64_t** out_keys, uint64_t* m) {
  uint64_t* alt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int64_t* d_num = nullptr;
  int end_bit = 32 + bits_for(n);
  if (end_bit > 64) end_bit = 64;
  CBFS_CUDA(cudaMallocAsync(&alt, sizeof(uint64_t) * (L ? L : 1), st));
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  CBFS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, L, 0, end_bit, st));
  CBFS_CUDA(cudaMallocAsync(&tmp, tb, st));
  CBFS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, db, L, 0, end_bit, st));
  count_launch(end_bit / 7);
  CBFS_CUDA(cudaFreeAsync(tmp, st));
  uint64_t* sorted = db.Current();
  uint64_t* other = db.Alternate();
  size_t tb2 = 0;
  CBFS_CUDA(cudaMallocAsync(&d_num, sizeof(int64_t), st));
  CBFS_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, sorted, other, d_num, (int64_t)L, st));
  CBFS_CUDA(cudaMallocAsync(&tmp, tb2, st));
  CBFS_CUDA(cub::DeviceSelect::Unique(tmp, tb2, sorted, other, d_num, (int64_t)L, st));
  count_launch(2);
  CBFS_CUDA(cudaFreeAsync(tmp, st));
  int64_t num = 0;
  CBFS_CUDA(cudaMemcpyAsync(&num, d_num, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  uint64_t last = 0;
  if (num > 0) {
    CBFS_CUDA(cudaMemcpyAsync(&last, other + num - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    if ((last >> 32) == n) --num;  // sentinel row of self loops
  }
  CBFS_CUDA(cudaFreeAsync(d_num, st));
  // `keys` and `alt` are both ours now: keep the unique keys, free the other
  CBFS_CUDA(cudaFreeAsync(sorted, st));
  *out_keys = other;
  *m = (uint64_t)num;
  return CBFS_OK;
}

static int keys_to_csr(const uint64_t* keys, uint64_t m, uint32_t n, cudaStream_t st, uint64_t** off, uint32_t** cols) {
  CBFS_CUDA(cudaMallocAsync(off, sizeof(uint64_t) * (n + 1ULL), st));
  CBFS_CUDA(cudaMallocAsync(cols, sizeof(uint32_t) * (m ? m : 1), st));
  if (m == 0) {
    CBFS_CUDA(cudaMemsetAsync(*off, 0, sizeof(uint64_t) * (n + 1ULL), st));
    return CBFS_OK;
  }
  k_split_keys<<<grid_for(m, 256), 256, 0, st>>>(keys, m, *cols);
  CBFS_LAUNCHED();
  k_row_offsets<<<grid_for(n + 1ull, 256), 256, 0, st>>>(keys, m, n, *off);
  CBFS_LAUNCHED();
  return CBFS_OK;
}

int graph_free(Graph* g) {
  if (!g) return CBFS_OK;
  cudaSetDevice(g->device);
  // all graph arrays come from the stream-ordered pool; free them in order
  // on the legacy stream (after any work that used them)
  cudaStream_t s0 = 0;
  if (g->off_orig && g->off_orig != g->off) cudaFreeAsync(g->off_orig, s0);
  if (g->cols_orig && g->cols_orig != g->cols) cudaFreeAsync(g->cols_orig, s0);
  void* ps[] = {g->off, g->cols, g->perm, g->inv, g->rank, g->order, g->chunk_v};
  for (void* p : ps)
    if (p) cudaFreeAsync(p, s0);
  extern void work_free(Graph*);
  work_free(g);
  delete g;
  return CBFS_OK;
}

// perm (internal -> original) = the locality order from `root`, inv = its inverse
static int locality_order(const uint64_t* off, const uint32_t* cols, uint32_t n, uint32_t root, cudaStream_t st,
                          uint32_t* perm, uint32_t* inv) {
  uint32_t *key = nullptr, *flag = nullptr, *d_hi = nullptr, *h_hi = nullptr;
  unsigned long long* blk = nullptr;
  int dev = 0, nsm = 0, per_sm = 0;
  CBFS_CUDA(cudaGetDevice(&dev));
  CBFS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CBFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfsord_coop, BO_THREADS, 0));
  // four blocks per SM (4,736 warps): enough for the large levels (k-NN),
  // few enough that the three grid barriers per level stay cheap (the grid's
  // ~6,000 levels)
  const unsigned grid = (unsigned)std::max(1, nsm * std::min(4, std::max(1, per_sm)));
  CBFS_CUDA(cudaMallocAsync(&key, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMallocAsync(&flag, sizeof(uint32_t) * n, st));
  CBFS_CUDA(cudaMallocAsync(&blk, sizeof(unsigned long long) * grid, st));
  CBFS_CUDA(cudaMallocAsync(&d_hi, sizeof(uint32_t), st));
  CBFS_CUDA(cudaMallocHost(&h_hi, sizeof(uint32_t)));
  CBFS_CUDA(cudaMemsetAsync(inv, 0xFF, sizeof(uint32_t) * n, st));  // pos = inv
  CBFS_CUDA(cudaMemsetAsync(key, 0xFF, sizeof(uint32_t) * n, st));
  const uint32_t zero = 0;
  CBFS_CUDA(cudaMemcpyAsync(perm, &root, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  CBFS_CUDA(cudaMemcpyAsync(inv + root, &zero, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  uint32_t* pos = inv;
  void* args[] = {(void*)&off, (void*)&cols, (void*)&perm, (void*)&pos, (void*)&key, (void*)&blk, (void*)&d_hi};
  CBFS_CUDA(cudaLaunchCooperativeKernel((void*)k_bfsord_coop, grid, BO_THREADS, args, 0, st));
  CBFS_LAUNCHED();
  CBFS_CUDA(cudaMemcpyAsync(h_hi, d_hi, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  const uint32_t hi = *h_hi;
  if (hi < n) {  // unreached vertices (other components, isolated) in id order
    uint32_t *f = key, *x = flag;  // reuse as scratch
    k_bfsord_flags<<<grid_for(n, 256), 256, 0, st>>>(inv, n, f);
    CBFS_LAUNCHED();
    size_t sb = 0;
    CBFS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, f, x, n, st));
    void* stmp = nullptr;
    CBFS_CUDA(cudaMallocAsync(&stmp, sb ? sb : 1, st));
    CBFS_CUDA(cub::DeviceScan::ExclusiveSum(stmp, sb, f, x, n, st));
    count_launch(2);
    k_bfsord_rest<<<grid_for(n, 256), 256, 0, st>>>(f, x, n, hi, perm, inv);
    CBFS_LAUNCHED();
    CBFS_CUDA(cudaFreeAsync(stmp, st));
  }
  CBFS_CUDA(cudaFreeAsync(key, st));
  CBFS_CUDA(cudaFreeAsync(flag, st));
  CBFS_CUDA(cudaFreeAsync(blk, st));
  CBFS_CUDA(cudaFreeAsync(d_hi, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  CBFS_CUDA(cudaFreeHost(h_hi));
  return CBFS_OK;
}

// build from device keys buffer (length L = 2 * pairs), consumes `keys`
static int build_from_keys(uint64_t* keys, uint64_t L, uint32_t n, uint32_t flags, int device, cudaStream_t st,
                           cbfs_graph** out) {
  Graph* g = new Graph();
  g->device = device;
  g->n = n;
  uint64_t* uk = nullptr;
  int rc = sort_unique(keys, L, n, st, &uk, &g->m);
  if (rc) { delete g; return rc; }
  // Let the stream-ordered frees of each phase complete before the next
  // phase allocates: measured on the 16.7M-vertex graphs, a build issued
  // right after a traversal otherwise spent 0.3-0.6 s in allocation instead
  // of ~8 ms (the pool could not reuse blocks whose frees were still queued).
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (g->m > 0xFFFFFFFFull) { cudaFreeAsync(uk, st); delete g; return fail(CBFS_EUNSUPPORTED, "more than 2^32-1 arcs"); }
  rc = keys_to_csr(uk, g->m, n, st, &g->off, &g->cols);
  if (rc) { delete g; return rc; }
  CBFS_CUDA(cudaStreamSynchronize(st));
  // degree order (deg desc, original id asc)
  uint64_t* dk = nullptr;
  uint32_t* d_max = nullptr;
  CBFS_CUDA(cudaMallocAsync(&dk, sizeof(uint64_t) * (n ? n : 1), st));
  CBFS_CUDA(cudaMallocAsync(&d_max, 2 * sizeof(uint32_t), st));
  CBFS_CUDA(cudaMemsetAsync(d_max, 0, 2 * sizeof(uint32_t), st));
  CBFS_CUDA(cudaMallocAsync(&g->rank, sizeof(uint32_t) * (n ? n : 1), st));
  CBFS_CUDA(cudaMallocAsync(&g->order, sizeof(uint32_t) * (n ? n : 1), st));
  if (n) {
    k_degree_keys<<<grid_for(n, 256), 256, 0, st>>>(g->off, n, dk, d_max);
    CBFS_LAUNCHED();
    uint64_t* alt = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CBFS_CUDA(cudaMallocAsync(&alt, sizeof(uint64_t) * n, st));
    cub::DoubleBuffer<uint64_t> db(dk, alt);
    CBFS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (uint64_t)n, 0, 64, st));
    CBFS_CUDA(cudaMallocAsync(&tmp, tb, st));
    CBFS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, db, (uint64_t)n, 0, 64, st));
    count_launch(8);
    CBFS_CUDA(cudaFreeAsync(tmp, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    const bool by_degree = (flags & CBFS_RELABEL_DEGREE) != 0;
    const bool by_locality = !by_degree && (flags & CBFS_RELABEL_LOCALITY) != 0 && g->m > 0;
    if (by_degree || by_locality) {
      CBFS_CUDA(cudaMallocAsync(&g->perm, sizeof(uint32_t) * n, st));
      CBFS_CUDA(cudaMallocAsync(&g->inv, sizeof(uint32_t) * n, st));
      if (by_degree) {  // perm = degree order (internal x -> original), inv = rank
        k_order_from_keys<<<grid_for(n, 256), 256, 0, st>>>(db.Current(), n, g->perm, g->inv);
        CBFS_LAUNCHED();
      } else {  // perm = BFS order from the highest-degree vertex
        uint64_t k0 = 0;
        CBFS_CUDA(cudaMemcpyAsync(&k0, db.Current(), sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CBFS_CUDA(cudaStreamSynchronize(st));
        int rcl = locality_order(g->off, g->cols, n, (uint32_t)k0, st, g->perm, g->inv);
        if (rcl) return rcl;
      }
      // internal CSR: keys (inv[u] << 32 | inv[v]) sorted; the original
      // arc keys' buffer is reused as the sort's alternate buffer
      uint64_t* rk = nullptr;
      CBFS_CUDA(cudaMallocAsync(&rk, sizeof(uint64_t) * (g->m ? g->m : 1), st));
      if (g->m) {
        k_relabel_keys<<<grid_for(g->m, 256), 256, 0, st>>>(uk, g->m, g->inv, rk);
        CBFS_LAUNCHED();
      }
      uint64_t* ralt = uk;
      uk = nullptr;
      cub::DoubleBuffer<uint64_t> rdb(rk, ralt);
      int end_bit = 32 + bits_for(n);
      size_t tb3 = 0;
      CBFS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb3, rdb, g->m, 0, end_bit, st));
      CBFS_CUDA(cudaMallocAsync(&tmp, tb3, st));
      CBFS_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb3, rdb, g->m, 0, end_bit, st));
      count_launch(end_bit / 7);
      CBFS_CUDA(cudaFreeAsync(tmp, st));
      g->off_orig = g->off;
      g->cols_orig = g->cols;
      g->off = nullptr;
      g->cols = nullptr;
      int rc2 = keys_to_csr(rdb.Current(), g->m, n, st, &g->off, &g->cols);
      if (rc2) return rc2;
      CBFS_CUDA(cudaFreeAsync(rk, st));
      CBFS_CUDA(cudaFreeAsync(ralt, st));
      if (by_degree) {  // in internal ids the degree order is the identity
        k_identity<<<grid_for(n, 256), 256, 0, st>>>(g->rank, n);
        CBFS_LAUNCHED();
        k_identity<<<grid_for(n, 256), 256, 0, st>>>(g->order, n);
        CBFS_LAUNCHED();
      } else {  // the degree order (ties by original id, R12/R18) mapped to internal ids
        k_order_map<<<grid_for(n, 256), 256, 0, st>>>(db.Current(), n, g->inv, g->order, g->rank);
        CBFS_LAUNCHED();
      }
      g->relabeled = true;
    } else {
      k_order_from_keys<<<grid_for(n, 256), 256, 0, st>>>(db.Current(), n, g->order, g->rank);
      CBFS_LAUNCHED();
      g->off_orig = g->off;
      g->cols_orig = g->cols;
    }
    CBFS_CUDA(cudaFreeAsync(alt, st));
  } else {
    g->off_orig = g->off;
    g->cols_orig = g->cols;
  }
  CBFS_CUDA(cudaFreeAsync(dk, st));
  if (uk) CBFS_CUDA(cudaFreeAsync(uk, st));
  uint32_t hm[2] = {0, 0};
  CBFS_CUDA(cudaMemcpyAsync(hm, d_max, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  g->max_degree = hm[0];
  g->n_nonisolated = hm[1];
  CBFS_CUDA(cudaFreeAsync(d_max, st));
  // pull chunk table
  g->n_chunks = (g->m + PULL_CHUNK - 1) / PULL_CHUNK;
  CBFS_CUDA(cudaMallocAsync(&g->chunk_v, sizeof(uint32_t) * (g->n_chunks ? g->n_chunks : 1), st));
  if (g->n_chunks) {
    k_chunk_table<<<grid_for(n, 256), 256, 0, st>>>(g->off, n, g->chunk_v);
    CBFS_LAUNCHED();
  }
  CBFS_CUDA(cudaStreamSynchronize(st));
  *out = reinterpret_cast<cbfs_graph*>(g);
  return CBFS_OK;
}

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_graph_create(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t n_pairs, uint32_t flags,
                      int device, cbfs_stream stream, cbfs_graph** out) {
  if (!out) return fail(CBFS_EINVAL, "out is null");
  *out = nullptr;
  if (n_pairs && (!src || !dst)) return fail(CBFS_EINVAL, "null edge arrays");
  if (n > CBFS_MAX_N) return fail(CBFS_EUNSUPPORTED, "n exceeds CBFS_MAX_N");
  CBFS_CUDA(cudaSetDevice(device));
  keep_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t *ds = src, *dd = dst;
  uint32_t *tmp_s = nullptr, *tmp_d = nullptr;
  if (!(flags & CBFS_INPUT_DEVICE) && n_pairs) {
    CBFS_CUDA(cudaMallocAsync(&tmp_s, sizeof(uint32_t) * n_pairs, st));
    CBFS_CUDA(cudaMallocAsync(&tmp_d, sizeof(uint32_t) * n_pairs, st));
    CBFS_CUDA(cudaMemcpyAsync(tmp_s, src, sizeof(uint32_t) * n_pairs, cudaMemcpyHostToDevice, st));
    CBFS_CUDA(cudaMemcpyAsync(tmp_d, dst, sizeof(uint32_t) * n_pairs, cudaMemcpyHostToDevice, st));
    ds = tmp_s;
    dd = tmp_d;
  }
  uint64_t L = 2 * n_pairs;
  uint64_t* keys = nullptr;
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * (L ? L : 1), st));
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  if (n_pairs) {
    k_make_keys<<<grid_for(n_pairs, 256), 256, 0, st>>>(ds, dd, n_pairs, n, keys, bad);
    CBFS_LAUNCHED();
  }
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  CBFS_CUDA(cudaFreeAsync(bad, st));
  if (tmp_s) CBFS_CUDA(cudaFreeAsync(tmp_s, st));
  if (tmp_d) CBFS_CUDA(cudaFreeAsync(tmp_d, st));
  if (hbad) {
    cudaFreeAsync(keys, st);
    return fail(CBFS_EINVAL, "edge endpoint >= n");
  }
  return build_from_keys(keys, L, n, flags, device, st, out);
}

int cbfs_graph_create_csr(uint32_t n, const uint64_t* offsets, const uint32_t* cols, uint64_t m, uint32_t flags,
                          int device, cbfs_stream stream, cbfs_graph** out) {
  if (!out || !offsets || (m && !cols)) return fail(CBFS_EINVAL, "null argument");
  *out = nullptr;
  if (n > CBFS_MAX_N) return fail(CBFS_EUNSUPPORTED, "n exceeds CBFS_MAX_N");
  CBFS_CUDA(cudaSetDevice(device));
  keep_pool(device);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t* doff = offsets;
  const uint32_t* dcols = cols;
  uint64_t* to = nullptr;
  uint32_t* tc = nullptr;
  if (!(flags & CBFS_INPUT_DEVICE)) {
    if (offsets[n] != m) return fail(CBFS_EINVAL, "offsets[n] != m");
    CBFS_CUDA(cudaMallocAsync(&to, sizeof(uint64_t) * (n + 1ULL), st));
    CBFS_CUDA(cudaMallocAsync(&tc, sizeof(uint32_t) * (m ? m : 1), st));
    CBFS_CUDA(cudaMemcpyAsync(to, offsets, sizeof(uint64_t) * (n + 1ULL), cudaMemcpyHostToDevice, st));
    if (m) CBFS_CUDA(cudaMemcpyAsync(tc, cols, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
    doff = to;
    dcols = tc;
  }
  uint64_t L = 2 * m;
  uint64_t* keys = nullptr;
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&keys, sizeof(uint64_t) * (L ? L : 1), st));
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  if (n) {
    k_csr_keys<<<grid_for(n, 256), 256, 0, st>>>(doff, dcols, n, keys, bad);
    CBFS_LAUNCHED();
  }
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  CBFS_CUDA(cudaFreeAsync(bad, st));
  if (to) CBFS_CUDA(cudaFreeAsync(to, st));
  if (tc) CBFS_CUDA(cudaFreeAsync(tc, st));
  if (hbad) {
    cudaFreeAsync(keys, st);
    return fail(CBFS_EINVAL, "column id >= n");
  }
  return build_from_keys(keys, L, n, flags, device, st, out);
}

int cbfs_graph_info(const cbfs_graph* gh, uint32_t* n, uint64_t* m, uint32_t* max_degree) {
  const Graph* g = reinterpret_cast<const Graph*>(gh);
  if (!g) return fail(CBFS_EINVAL, "null graph");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (max_degree) *max_degree = g->max_degree;
  return CBFS_OK;
}

int cbfs_graph_nonisolated(const cbfs_graph* gh, uint32_t* count) {
  const Graph* g = reinterpret_cast<const Graph*>(gh);
  if (!g || !count) return fail(CBFS_EINVAL, "null argument");
  *count = g->n_nonisolated;
  return CBFS_OK;
}

int cbfs_graph_export_csr(const cbfs_graph* gh, uint64_t* offsets, uint32_t* cols) {
  const Graph* g = reinterpret_cast<const Graph*>(gh);
  if (!g || !offsets || (g->m && !cols)) return fail(CBFS_EINVAL, "null argument");
  CBFS_CUDA(cudaSetDevice(g->device));
  CBFS_CUDA(cudaMemcpy(offsets, g->off_orig, sizeof(uint64_t) * (g->n + 1ULL), cudaMemcpyDeviceToHost));
  if (g->m) CBFS_CUDA(cudaMemcpy(cols, g->cols_orig, sizeof(uint32_t) * g->m, cudaMemcpyDeviceToHost));
  return CBFS_OK;
}

int cbfs_graph_internal_order(const cbfs_graph* gh, uint32_t* out_perm) {
  const Graph* g = reinterpret_cast<const Graph*>(gh);
  if (!g || (g->n && !out_perm)) return fail(CBFS_EINVAL, "null argument");
  if (g->n == 0) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(g->device));
  if (!g->perm) {
    for (uint32_t x = 0; x < g->n; ++x) out_perm[x] = x;
    return CBFS_OK;
  }
  CBFS_CUDA(cudaMemcpy(out_perm, g->perm, sizeof(uint32_t) * g->n, cudaMemcpyDeviceToHost));
  return CBFS_OK;
}

int cbfs_graph_destroy(cbfs_graph* gh) { return graph_free(reinterpret_cast<Graph*>(gh)); }

const char* cbfs_last_error(void) { return g_err.c_str(); }
const char* cbfs_version(void) { return "cbfs-b200 0.1 (sm_100a)"; }
uint64_t cbfs_launch_count(int reset) { return launches(reset); }

}  // extern "C"
