// query.cu — distance decode (§8(a) A9), landmark query (A11,
// P:1013-1021 and P:1074-1086, R14-R16), the fused streaming build+query
// used when the label store cannot be resident (H3), and the host-buffer
// variant of cbfs_run used for end-to-end timing.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "engine.cuh"

namespace cbfs {

constexpr unsigned FULLW_Q = 0xFFFFFFFFu;


template <int DB>
__device__ __forceinline__ uint32_t load_dist(const void* p, uint64_t idx) {
  if (DB == 1) {
    const uint8_t x = ((const uint8_t*)p)[idx];
    return x == 0xFFu ? 0xFFFFFFFFu : x;
  } else {
    const uint16_t x = ((const uint16_t*)p)[idx];
    return x == 0xFFFFu ? 0xFFFFFFFFu : x;
  }
}

// one bit-subset word of a store with MB-byte words (w = 8 * MB)
template <int MB>
__device__ __forceinline__ uint64_t load_mask(const void* p, uint64_t idx) {
  if (MB == 1) return ((const uint8_t*)p)[idx];
  if (MB == 2) return ((const uint16_t*)p)[idx];
  if (MB == 4) return ((const uint32_t*)p)[idx];
  return ((const uint64_t*)p)[idx];
}

// ------------------------------------------------------------------ decode
template <int DB>
__global__ void k_decode(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* __restrict__ dist,
                         const uint64_t* __restrict__ masks, uint32_t c, uint32_t k, uint16_t* __restrict__ out) {
  const uint64_t full = full_mask(k);
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t dv = load_dist<DB>(dist, v * C + c);
    uint64_t S[CBFS_MAX_D + 1];
    uint64_t uni = 0;
    for (uint32_t i = 0; i < planes; ++i) { S[i] = masks[((uint64_t)i * n + v) * C + c]; uni |= S[i]; }
    if (planes == d) S[d] = dv == 0xFFFFFFFFu ? 0 : (full & ~uni);  // R14
    for (uint32_t j = 0; j < k; ++j) {
      uint32_t r = 0xFFFFu;
      if (dv != 0xFFFFFFFFu)
        for (uint32_t i = 0; i <= d; ++i)
          if ((S[i] >> j) & 1ULL) { r = dv + i; break; }
      out[(uint64_t)j * n + v] = (uint16_t)(r > 0xFFFFu ? 0xFFFFu : r);
    }
  }
}

// ------------------------------------------------------------------ query
// One warp per query pair, lane over clusters.  Per cluster: skip when
// either Delta is unreachable (R16); else the smallest i+j with
// S_s[i] & S_t[j] != 0, scanning i+j = 0..2d; S_x[d] is
// rebuilt from the other subsets when the store keeps only d (R14).  MB is
// the store's word: 8 bytes, or 1/2/4 for the packed w = 8/16/32 stores.
// CM: the subsets are cluster-major (subset i of cluster c at (i * C + c) *
// n + v) — the streaming query's staging when the sparse engine (cluster-
// major frontier) writes them; Delta is vertex-major (transposed after the
// batch, k_transpose_dist), so the per-query Delta rows stay coalesced.
template <int DB, int MB, bool CM = false>
__global__ void __launch_bounds__(256) k_query(uint32_t n, uint32_t C, uint32_t d, uint32_t planes,
                                               const void* __restrict__ dist, const void* __restrict__ masks,
                                               const uint8_t* __restrict__ sizes, const uint32_t* __restrict__ s,
                                               const uint32_t* __restrict__ t, uint64_t q,
                                               int32_t* __restrict__ best, int* __restrict__ bad,
                                               const uint32_t* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  for (uint64_t qi = warp; qi < q; qi += nwarps) {
    uint32_t a = s[qi], b = t[qi];
    if (a >= n || b >= n) {
      if (lane == 0) *bad = 1;
      continue;
    }
    if (inv) {  // label rows in internal ids (the streaming store)
      a = inv[a];
      b = inv[b];
    }
    // start from the answer so far (earlier batches / label shards): a
    // cluster whose Delta sum cannot beat it is skipped before its subsets
    // are read
    const int32_t prev = best[qi];
    int32_t mine = prev;
    for (uint32_t c = lane; c < C; c += 32) {
      const uint32_t da = load_dist<DB>(dist, (uint64_t)a * C + c);
      const uint32_t db = load_dist<DB>(dist, (uint64_t)b * C + c);
      if (da == 0xFFFFFFFFu || db == 0xFFFFFFFFu) continue;
      if ((int32_t)(da + db) >= mine) continue;  // cannot improve (value >= da + db)
      uint64_t Sa[CBFS_MAX_D + 1], Sb[CBFS_MAX_D + 1];
      uint64_t ua = 0, ub = 0;
      for (uint32_t i = 0; i < planes; ++i) {
        Sa[i] = load_mask<MB>(masks, CM ? ((uint64_t)i * C + c) * n + a : ((uint64_t)i * n + a) * C + c);
        Sb[i] = load_mask<MB>(masks, CM ? ((uint64_t)i * C + c) * n + b : ((uint64_t)i * n + b) * C + c);
        ua |= Sa[i];
        ub |= Sb[i];
      }
      if (planes == d) {
        const uint64_t full = full_mask(sizes[c]);
        Sa[d] = full & ~ua;
        Sb[d] = full & ~ub;
      }
      for (uint32_t tt = 0; tt <= 2 * d; ++tt) {
        bool hit = false;
        const uint32_t i0 = tt > d ? tt - d : 0, i1 = tt < d ? tt : d;
        for (uint32_t i = i0; i <= i1; ++i)
          if (Sa[i] & Sb[tt - i]) { hit = true; break; }
        if (hit) {
          const int32_t val = (int32_t)(da + db + tt);
          if (val < mine) mine = val;
          break;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, o));
    if (lane == 0 && mine < prev) atomicMin(&best[qi], mine);  // concurrent batches min-merge
  }
}

template <int DB>
static void launch_query_db(unsigned blocks, uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist,
                            const void* masks, uint32_t mask_bytes, const uint8_t* sizes, const uint32_t* s,
                            const uint32_t* t, uint64_t q, int32_t* best, int* bad, cudaStream_t st,
                            const uint32_t* inv) {
  switch (mask_bytes) {
    case 1: k_query<DB, 1><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad, inv); break;
    case 2: k_query<DB, 2><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad, inv); break;
    case 4: k_query<DB, 4><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad, inv); break;
    default: k_query<DB, 8><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad, inv);
  }
}

// ------------------------------------------------------------------ wide clusters (k > 64)
// The cbfs_run_wide layout: dist [n][C], masks [planes][n][C W] (word w of
// cluster c in column c W + w), sizes [C] uint16.  Bit j of the cluster is
// bit j % 64 of word j / 64 (R11).
__device__ __forceinline__ uint64_t wide_full(uint32_t k, uint32_t w) {
  return k > 64 * w ? full_mask(k - 64 * w) : 0ULL;
}

template <int DB>
__global__ void k_decode_wide(uint32_t n, uint32_t C, uint32_t W, uint32_t d, uint32_t planes,
                              const void* __restrict__ dist, const uint64_t* __restrict__ masks, uint32_t c,
                              uint32_t k, uint16_t* __restrict__ out) {
  const uint64_t CW = (uint64_t)C * W;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t dv = load_dist<DB>(dist, v * C + c);
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t w = j >> 6;
      const uint64_t* col = masks + v * CW + (uint64_t)c * W + w;  // plane i at col[i * n * CW]
      uint32_t r = 0xFFFFu;
      if (dv != 0xFFFFFFFFu) {
        uint64_t uni = 0;
        for (uint32_t i = 0; i <= d; ++i) {
          const uint64_t S = i < planes ? col[(uint64_t)i * n * CW] : (wide_full(k, w) & ~uni);  // R14
          uni |= S;
          if ((S >> (j & 63)) & 1ULL) { r = dv + i; break; }
        }
      }
      out[(uint64_t)j * n + v] = (uint16_t)(r > 0xFFFFu ? 0xFFFFu : r);
    }
  }
}

// One warp per query pair, lane over clusters, as k_query; the subsets are
// W words, S_x[d] rebuilt word by word when the store keeps d planes.
template <int DB, int W>
__global__ void __launch_bounds__(256) k_query_wide(uint32_t n, uint32_t C, uint32_t d, uint32_t planes,
                                                    const void* __restrict__ dist,
                                                    const uint64_t* __restrict__ masks,
                                                    const uint16_t* __restrict__ sizes,
                                                    const uint32_t* __restrict__ s, const uint32_t* __restrict__ t,
                                                    uint64_t q, int32_t* __restrict__ best, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const uint64_t CW = (uint64_t)C * W, plane = (uint64_t)n * CW;
  for (uint64_t qi = warp; qi < q; qi += nwarps) {
    const uint32_t a = s[qi], b = t[qi];
    if (a >= n || b >= n) {
      if (lane == 0) *bad = 1;
      continue;
    }
    const int32_t prev = best[qi];
    int32_t mine = prev;
    for (uint32_t c = lane; c < C; c += 32) {
      const uint32_t da = load_dist<DB>(dist, (uint64_t)a * C + c);
      const uint32_t db = load_dist<DB>(dist, (uint64_t)b * C + c);
      if (da == 0xFFFFFFFFu || db == 0xFFFFFFFFu) continue;
      if ((int32_t)(da + db) >= mine) continue;
      const uint64_t* ca = masks + (uint64_t)a * CW + (uint64_t)c * W;
      const uint64_t* cb = masks + (uint64_t)b * CW + (uint64_t)c * W;
      uint64_t ra[W], rb[W];  // S_x[d] per word (only read when planes == d)
      if (planes == d) {
        const uint32_t k = sizes[c];
#pragma unroll
        for (int w = 0; w < W; ++w) {
          uint64_t ua = 0, ub = 0;
          for (uint32_t i = 0; i < planes; ++i) { ua |= ca[i * plane + w]; ub |= cb[i * plane + w]; }
          ra[w] = wide_full(k, w) & ~ua;
          rb[w] = wide_full(k, w) & ~ub;
        }
      }
      for (uint32_t tt = 0; tt <= 2 * d; ++tt) {
        bool hit = false;
        const uint32_t i0 = tt > d ? tt - d : 0, i1 = tt < d ? tt : d;
        for (uint32_t i = i0; i <= i1 && !hit; ++i) {
          const uint32_t j = tt - i;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const uint64_t x = i < planes ? ca[i * plane + w] : ra[w];
            const uint64_t y = j < planes ? cb[j * plane + w] : rb[w];
            hit |= (x & y) != 0;
          }
        }
        if (hit) {
          const int32_t val = (int32_t)(da + db + tt);
          if (val < mine) mine = val;
          break;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(0xFFFFFFFFu, mine, o));
    if (lane == 0 && mine < prev) atomicMin(&best[qi], mine);
  }
}

template <int DB>
static void launch_query_wide_db(unsigned blocks, uint32_t n, uint32_t C, uint32_t W, uint32_t d, uint32_t planes,
                                 const void* dist, const uint64_t* masks, const uint16_t* sizes, const uint32_t* s,
                                 const uint32_t* t, uint64_t q, int32_t* best, int* bad, cudaStream_t st) {
  switch (W) {
    case 1: k_query_wide<DB, 1><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad); break;
    case 2: k_query_wide<DB, 2><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad); break;
    case 4: k_query_wide<DB, 4><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad); break;
    default: k_query_wide<DB, 8><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad);
  }
}

// [LANES][n] u16 -> [n][LANES]: 32 vertices x 64 clusters per block through
// shared memory, both sides coalesced
__global__ void __launch_bounds__(256) k_transpose_dist(const uint16_t* __restrict__ in, uint32_t n,
                                                        uint16_t* __restrict__ out) {
  __shared__ uint16_t tile[LANES][33];
  for (uint64_t v0 = (uint64_t)blockIdx.x * 32; v0 < n; v0 += (uint64_t)gridDim.x * 32) {
    for (uint32_t x = threadIdx.x; x < LANES * 32; x += blockDim.x) {
      const uint32_t c = x >> 5, j = x & 31;
      tile[c][j] = v0 + j < n ? in[(uint64_t)c * n + v0 + j] : 0xFFFFu;
    }
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < LANES * 32; x += blockDim.x) {
      const uint32_t j = x >> 6, c = x & 63;
      if (v0 + j < n) out[(v0 + j) * LANES + c] = tile[c][j];
    }
    __syncthreads();
  }
}

static int launch_query(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                        const void* masks, const uint8_t* sizes, const uint32_t* s, const uint32_t* t, uint64_t q,
                        int32_t* best, int* bad, cudaStream_t st, const uint32_t* inv = nullptr,
                        uint32_t mask_bytes = 8, bool cmajor = false) {
  if (q == 0 || C == 0) return CBFS_OK;
  const unsigned blocks = grid_for(q * 32, 256, 148u * 8u * 8u);
  if (cmajor) {  // the streaming query's cluster-major staging (u16 Delta, u64 subsets)
    k_query<2, 8, true><<<blocks, 256, 0, st>>>(n, C, d, planes, dist, masks, sizes, s, t, q, best, bad, inv);
    CBFS_LAUNCHED();
    return CBFS_OK;
  }
  if (dist_bytes == 1)
    launch_query_db<1>(blocks, n, C, d, planes, dist, masks, mask_bytes, sizes, s, t, q, best, bad, st, inv);
  else
    launch_query_db<2>(blocks, n, C, d, planes, dist, masks, mask_bytes, sizes, s, t, q, best, bad, st, inv);
  CBFS_LAUNCHED();
  return CBFS_OK;
}

// ------------------------------------------------------------------ bidirectional refinement
// Appendix B, reading R27: from each endpoint a BFS in the
// order of the sorted ORIGINAL-id CSR visits vertices in discovery order (the
// endpoint first) until tau are visited; the answer is min over vertices
// visited by both sides of dist_s + dist_t, min-merged into best.  One warp
// per query pair; each side keeps its visited list (id, hop) and an
// open-addressing hash of the visited ids in shared memory.  A neighbour
// chunk of 32 arcs is tested by 32 lanes at once and the new vertices are
// appended in arc order (ballot prefix), so the visited sets are exactly the
// sequential BFS's.
constexpr uint32_t BIDIR_EMPTY = 0xFFFFFFFFu;

struct BidirSide {
  uint32_t* ids;   // [tau] visited, discovery order
  uint32_t* hop;   // [tau]
  uint32_t* keys;  // [H] hash keys
  uint32_t* pos;   // [H] position in ids
};

__device__ __forceinline__ uint32_t bidir_hash(uint32_t x, uint32_t mask) { return (x * 0x9E3779B1u) & mask; }

__device__ __forceinline__ int bidir_find(const BidirSide& S, uint32_t x, uint32_t mask) {
  for (uint32_t h = bidir_hash(x, mask);; h = (h + 1) & mask) {
    const uint32_t k = S.keys[h];
    if (k == x) return (int)S.pos[h];
    if (k == BIDIR_EMPTY) return -1;
  }
}

__device__ __forceinline__ void bidir_insert(const BidirSide& S, uint32_t x, uint32_t p, uint32_t mask) {
  for (uint32_t h = bidir_hash(x, mask);; h = (h + 1) & mask) {
    if (atomicCAS(&S.keys[h], BIDIR_EMPTY, x) == BIDIR_EMPTY) {
      S.pos[h] = p;
      return;
    }
  }
}

// visits up to tau vertices from src; returns how many
__device__ uint32_t bidir_bfs(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, uint32_t src,
                              uint32_t tau, const BidirSide& S, uint32_t H) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t mask = H - 1;
  for (uint32_t h = lane; h < H; h += 32) S.keys[h] = BIDIR_EMPTY;
  __syncwarp();
  if (tau == 0) return 0;
  if (lane == 0) {
    S.ids[0] = src;
    S.hop[0] = 0;
    bidir_insert(S, src, 0, mask);
  }
  __syncwarp();
  uint32_t cnt = 1, head = 0;
  while (head < cnt && cnt < tau) {
    const uint32_t x = S.ids[head], hx = S.hop[head];
    ++head;
    const uint64_t e1 = off[x + 1];
    for (uint64_t a0 = off[x]; a0 < e1 && cnt < tau; a0 += 32) {
      const uint64_t a = a0 + lane;
      const uint32_t u = a < e1 ? cols[a] : 0u;
      const bool isnew = a < e1 && bidir_find(S, u, mask) < 0;
      const unsigned m = __ballot_sync(FULLW_Q, isnew);
      const uint32_t rank = __popc(m & ((1u << lane) - 1));
      if (isnew && cnt + rank < tau) {
        S.ids[cnt + rank] = u;
        S.hop[cnt + rank] = hx + 1;
        bidir_insert(S, u, cnt + rank, mask);
      }
      cnt = min(cnt + (uint32_t)__popc(m), tau);
      __syncwarp();
    }
  }
  return cnt;
}

__global__ void k_bidir(const uint64_t* __restrict__ off, const uint32_t* __restrict__ cols, uint32_t n,
                        const uint32_t* __restrict__ s, const uint32_t* __restrict__ t, uint64_t q, uint32_t tau,
                        uint32_t H, int32_t* __restrict__ best, int* __restrict__ bad) {
  extern __shared__ uint32_t smem[];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t per_side = 2 * tau + 2 * H;
  uint32_t* base = smem + (uint64_t)wib * 2 * per_side;
  BidirSide A{base, base + tau, base + 2 * tau, base + 2 * tau + H};
  uint32_t* b2 = base + per_side;
  BidirSide B{b2, b2 + tau, b2 + 2 * tau, b2 + 2 * tau + H};
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t qi = warp; qi < q; qi += nwarps) {
    const uint32_t a = s[qi], b = t[qi];
    if (a >= n || b >= n) {
      if (lane == 0) *bad = 1;
      continue;
    }
    const uint32_t ca = bidir_bfs(off, cols, a, tau, A, H);
    bidir_bfs(off, cols, b, tau, B, H);
    int32_t mine = 0x7FFFFFFF;
    for (uint32_t p = lane; p < ca; p += 32) {
      const int k = bidir_find(B, A.ids[p], H - 1);
      if (k >= 0) mine = min(mine, (int32_t)(A.hop[p] + B.hop[k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(FULLW_Q, mine, o));
    if (lane == 0 && mine < best[qi]) atomicMin(&best[qi], mine);
    __syncwarp();
  }
}

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_decode(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                const uint64_t* masks, uint32_t c, uint32_t k, uint16_t* out, cbfs_stream stream) {
  if (!dist || !masks || !out) return fail(CBFS_EINVAL, "null argument");
  if (c >= C || k == 0 || k > CBFS_MAX_K) return fail(CBFS_EINVAL, "bad cluster index or k");
  if (d > CBFS_MAX_D || (planes != d + 1 && !(planes == d && d > 0))) return fail(CBFS_EINVAL, "bad d/planes");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (n == 0) return CBFS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dist_bytes == 1)
    k_decode<1><<<grid_for(n, 256), 256, 0, st>>>(n, C, d, planes, dist, masks, c, k, out);
  else
    k_decode<2><<<grid_for(n, 256), 256, 0, st>>>(n, C, d, planes, dist, masks, c, k, out);
  CBFS_LAUNCHED();
  return CBFS_OK;
}

int cbfs_decode_wide(uint32_t n, uint32_t C, uint32_t words, uint32_t d, uint32_t planes, const void* dist,
                     uint32_t dist_bytes, const uint64_t* masks, uint32_t c, uint32_t k, uint16_t* out,
                     cbfs_stream stream) {
  if (!dist || !masks || !out) return fail(CBFS_EINVAL, "null argument");
  if (words != 1 && words != 2 && words != 4 && words != 8) return fail(CBFS_EUNSUPPORTED, "words must be 1, 2, 4 or 8");
  if (c >= C || k == 0 || k > 64 * words) return fail(CBFS_EINVAL, "bad cluster index or k");
  if (d > CBFS_MAX_D || (planes != d + 1 && !(planes == d && d > 0))) return fail(CBFS_EINVAL, "bad d/planes");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (n == 0) return CBFS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dist_bytes == 1)
    k_decode_wide<1><<<grid_for(n, 256), 256, 0, st>>>(n, C, words, d, planes, dist, masks, c, k, out);
  else
    k_decode_wide<2><<<grid_for(n, 256), 256, 0, st>>>(n, C, words, d, planes, dist, masks, c, k, out);
  CBFS_LAUNCHED();
  return CBFS_OK;
}

int cbfs_query_distance_wide(uint32_t n, uint32_t C, uint32_t words, uint32_t d, uint32_t planes, const void* dist,
                             uint32_t dist_bytes, const uint64_t* masks, const uint16_t* sizes, const uint32_t* s,
                             const uint32_t* t, uint64_t q, int32_t* inout_best, cbfs_stream stream) {
  if (q && (!s || !t || !inout_best)) return fail(CBFS_EINVAL, "null query arrays");
  if (C && (!dist || !masks || !sizes)) return fail(CBFS_EINVAL, "null label arrays");
  if (words != 1 && words != 2 && words != 4 && words != 8) return fail(CBFS_EUNSUPPORTED, "words must be 1, 2, 4 or 8");
  if (d > CBFS_MAX_D || (planes != d + 1 && !(planes == d && d > 0))) return fail(CBFS_EINVAL, "bad d/planes");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (q == 0 || C == 0) return CBFS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const unsigned blocks = grid_for(q * 32, 256, 148u * 8u * 8u);
  if (dist_bytes == 1)
    launch_query_wide_db<1>(blocks, n, C, words, d, planes, dist, masks, sizes, s, t, q, inout_best, bad, st);
  else
    launch_query_wide_db<2>(blocks, n, C, words, d, planes, dist, masks, sizes, s, t, q, inout_best, bad, st);
  CBFS_LAUNCHED();
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaFreeAsync(bad, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (hbad) return fail(CBFS_EINVAL, "query vertex id >= n");
  return CBFS_OK;
}

int cbfs_query_bidir(cbfs_graph* gh, const uint32_t* s, const uint32_t* t, uint64_t q, uint32_t tau,
                     int32_t* inout_best, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (!g) return fail(CBFS_EINVAL, "null graph");
  if (q && (!s || !t || !inout_best)) return fail(CBFS_EINVAL, "null query arrays");
  if (tau > CBFS_BIDIR_MAX_TAU) return fail(CBFS_EUNSUPPORTED, "tau > CBFS_BIDIR_MAX_TAU");
  if (q == 0 || tau == 0) return CBFS_OK;
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t H = 1;
  while (H < 2 * tau) H <<= 1;
  const uint32_t warps = 4;
  const size_t smem = (size_t)warps * 2 * (2 * tau + 2 * H) * sizeof(uint32_t);
  CBFS_CUDA(cudaFuncSetAttribute(k_bidir, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const unsigned blocks = grid_for(q * 32, warps * 32, 148u * 16u);
  k_bidir<<<blocks, warps * 32, smem, st>>>(g->off_orig, g->cols_orig, g->n, s, t, q, tau, H, inout_best, bad);
  CBFS_LAUNCHED();
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaFreeAsync(bad, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (hbad) return fail(CBFS_EINVAL, "query vertex id >= n");
  return CBFS_OK;
}

}  // extern "C"

namespace cbfs {
// cbfs_query_distance over a store whose bit-subset words are mask_bytes wide
int query_store(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                const void* masks, uint32_t mask_bytes, const uint8_t* sizes, const uint32_t* s, const uint32_t* t,
                uint64_t q, int32_t* inout_best, cudaStream_t st) {
  if (q && (!s || !t || !inout_best)) return fail(CBFS_EINVAL, "null query arrays");
  // planes = d = 0: plain landmarks (single-source clusters, Delta only; S_v[0]
  // = FULL is rebuilt like any S_v[d], R14)
  if (C && (!dist || (!masks && planes) || !sizes)) return fail(CBFS_EINVAL, "null label arrays");
  if (d > CBFS_MAX_D || (planes != d + 1 && planes != d)) return fail(CBFS_EINVAL, "bad d/planes");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (mask_bytes != 1 && mask_bytes != 2 && mask_bytes != 4 && mask_bytes != 8)
    return fail(CBFS_EINVAL, "mask word must be 1, 2, 4 or 8 bytes");
  int* bad = nullptr;
  CBFS_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  int rc = launch_query(n, C, d, planes, dist, dist_bytes, masks, sizes, s, t, q, inout_best, bad, st, nullptr,
                        mask_bytes);
  if (rc) return rc;
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CBFS_CUDA(cudaFreeAsync(bad, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (hbad) return fail(CBFS_EINVAL, "query vertex id >= n");
  return CBFS_OK;
}
}  // namespace cbfs

extern "C" {

int cbfs_query_distance(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                        const uint64_t* masks, const uint8_t* sizes, const uint32_t* s, const uint32_t* t, uint64_t q,
                        int32_t* inout_best, cbfs_stream stream) {
  return query_store(n, C, d, planes, dist, dist_bytes, masks, 8, sizes, s, t, q, inout_best, (cudaStream_t)stream);
}

// per-slot label staging; the query runs on the slot's stream when its batch ends
struct QuerySource : ArraySource {
  uint32_t n = 0, d = 0, planes = 0;
  std::vector<uint16_t*> sd, sdt;  // Delta staging (cluster-major when the sparse engine writes it) + transposed
  std::vector<uint64_t*> sm;
  const uint32_t *s = nullptr, *t = nullptr;
  uint64_t q = 0;
  int32_t* best = nullptr;
  int* bad = nullptr;
  const uint32_t* inv = nullptr;  // the graph's original -> internal map (label rows are internal ids)
  int bind(RunArgs& a, int slot, cudaStream_t st) override {
    a.out_dist = sd[slot];
    a.out_masks = sm[slot];
    a.C = LANES;
    a.cbase = 0;
    a.out_internal = 1;  // rows by internal id: the fold's writes follow the traversal's locality
    // the sparse engine's frontier is cluster-major: its label writes coalesce
    // in a cluster-major staging (the batched engine's are vertex-grouped)
    a.out_cmajor = a.engine == ENGINE_SPARSE && !getenv("CBFS_QUERY_VMAJOR");
    CBFS_CUDA(cudaMemsetAsync(sd[slot], 0xFF, sizeof(uint16_t) * (uint64_t)n * LANES, st));
    CBFS_CUDA(cudaMemsetAsync(sm[slot], 0, sizeof(uint64_t) * (uint64_t)planes * n * LANES, st));
    return CBFS_OK;
  }
  int finished(const RunArgs& a, int slot, cudaStream_t st) override {
    // lanes >= nb stay unreachable (dist 0xFFFF), so the query skips them
    const uint16_t* dq = sd[slot];
    if (a.out_cmajor && q) {
      k_transpose_dist<<<grid_for((n + 31ull) / 32, 1, 148u * 16u), 256, 0, st>>>(sd[slot], n, sdt[slot]);
      CBFS_LAUNCHED();
      dq = sdt[slot];
    }
    return launch_query(n, LANES, d, planes, dq, 2, sm[slot], a.sizes, s, t, q, best, bad, st, inv, 8,
                        a.out_cmajor != 0);
  }
};

int cbfs_query_stream(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                      const uint32_t* s, const uint32_t* t, uint64_t q, int32_t* inout_best, uint64_t* out_stats,
                      cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  int rc = check_run_args(g, sources, sizes, n_clusters, d, 2, d + 1, CBFS_DIR_AUTO);
  if (rc) return rc;
  if (q && (!s || !t || !inout_best)) return fail(CBFS_EINVAL, "null query arrays");
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int engine = choose_engine(g, CBFS_DIR_AUTO);
  if (engine < 0) return CBFS_ECUDA;
  const uint64_t stage = (uint64_t)g->n * LANES * (2 * sizeof(uint16_t) + sizeof(uint64_t) * (d > 0 ? d : 1)) + 64;
  WorkLease lease(g, engine, stage);
  if (lease.rc) return lease.rc;
  const uint32_t n = g->n;
  // label records keep S_v[0..d-1] only (R14): S_v[d] is rebuilt
  // by the query from the cluster size; d = 0 keeps its single subset
  const uint32_t planes = d > 0 ? d : 1;
  const int P = num_slots(g);
  QuerySource src;
  src.proto.d = d;
  src.proto.planes = planes;
  src.proto.dist_bytes = 2;
  src.proto.direction = CBFS_DIR_AUTO;
  src.proto.engine = engine;
  src.sources = sources;
  src.sizes = sizes;
  src.n_clusters = n_clusters;
  src.out_stats = out_stats;
  src.n = n; src.d = d; src.planes = planes; src.s = s; src.t = t; src.q = q; src.best = inout_best;
  src.inv = g->inv;
  src.sd.assign(P, nullptr);
  src.sdt.assign(P, nullptr);
  src.sm.assign(P, nullptr);
  for (int k = 0; k < P; ++k) {
    CBFS_CUDA(cudaMallocAsync(&src.sd[k], sizeof(uint16_t) * (uint64_t)n * LANES + 16, st));
    CBFS_CUDA(cudaMallocAsync(&src.sdt[k], sizeof(uint16_t) * (uint64_t)n * LANES + 16, st));
    CBFS_CUDA(cudaMallocAsync(&src.sm[k], sizeof(uint64_t) * (uint64_t)planes * n * LANES + 16, st));
  }
  CBFS_CUDA(cudaMallocAsync(&src.bad, sizeof(int), st));
  CBFS_CUDA(cudaMemsetAsync(src.bad, 0, sizeof(int), st));
  rc = run_batches(g, src, st);
  int hbad = 0;
  CBFS_CUDA(cudaMemcpyAsync(&hbad, src.bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  for (int k = 0; k < P; ++k) {
    CBFS_CUDA(cudaFreeAsync(src.sd[k], st));
    CBFS_CUDA(cudaFreeAsync(src.sdt[k], st));
    CBFS_CUDA(cudaFreeAsync(src.sm[k], st));
  }
  CBFS_CUDA(cudaFreeAsync(src.bad, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  if (rc) return rc;
  if (hbad) return fail(CBFS_EINVAL, "query vertex id >= n");
  return CBFS_OK;
}

// per-slot output staging copied to the caller's host arrays when a batch ends
struct HostSource : ArraySource {
  uint32_t n = 0, planes = 0, dist_bytes = 0;
  uint64_t C = 0;
  void* h_dist = nullptr;
  uint64_t* h_masks = nullptr;
  std::vector<void*> sd;
  std::vector<uint64_t*> sm;
  int bind(RunArgs& a, int slot, cudaStream_t st) override {
    a.out_dist = sd[slot];
    a.out_masks = sm[slot];
    a.C = LANES;
    a.cbase = 0;
    if (sd[slot]) CBFS_CUDA(cudaMemsetAsync(sd[slot], 0xFF, (uint64_t)n * LANES * dist_bytes, st));
    if (sm[slot]) CBFS_CUDA(cudaMemsetAsync(sm[slot], 0, sizeof(uint64_t) * (uint64_t)planes * n * LANES, st));
    return CBFS_OK;
  }
  int finished(const RunArgs& a, int slot, cudaStream_t st) override {
    const uint64_t cb = (uint64_t)(a.sizes - sizes);  // first cluster of the batch
    if (h_dist)
      CBFS_CUDA(cudaMemcpy2DAsync((uint8_t*)h_dist + cb * dist_bytes, C * dist_bytes, sd[slot],
                                  (uint64_t)LANES * dist_bytes, (uint64_t)a.nb * dist_bytes, n,
                                  cudaMemcpyDeviceToHost, st));
    if (h_masks)
      CBFS_CUDA(cudaMemcpy2DAsync(h_masks + cb, C * sizeof(uint64_t), sm[slot], LANES * sizeof(uint64_t),
                                  (uint64_t)a.nb * sizeof(uint64_t), (uint64_t)planes * n, cudaMemcpyDeviceToHost,
                                  st));
    return CBFS_OK;
  }
};

int cbfs_run_host(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                  uint32_t dist_bytes, void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
                  uint32_t direction, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  int rc = check_run_args(g, sources, sizes, n_clusters, d, dist_bytes, planes, direction);
  if (rc) return rc;
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int engine = choose_engine(g, direction);
  if (engine < 0) return CBFS_ECUDA;
  WorkLease lease(g, engine);
  if (lease.rc) return lease.rc;
  const uint32_t n = g->n;
  const uint64_t C = n_clusters;
  const int P = num_slots(g);
  uint32_t* dsrc = nullptr;
  uint8_t* dsz = nullptr;
  uint64_t* dstats = nullptr;
  CBFS_CUDA(cudaMallocAsync(&dsrc, sizeof(uint32_t) * 64 * (C ? C : 1), st));
  CBFS_CUDA(cudaMallocAsync(&dsz, C ? C : 1, st));
  CBFS_CUDA(cudaMallocAsync(&dstats, sizeof(uint64_t) * 4 * (C ? C : 1), st));
  if (C) {
    CBFS_CUDA(cudaMemcpyAsync(dsrc, sources, sizeof(uint32_t) * 64 * C, cudaMemcpyHostToDevice, st));
    CBFS_CUDA(cudaMemcpyAsync(dsz, sizes, C, cudaMemcpyHostToDevice, st));
  }
  // When the whole output fits next to the workspace, traverse into a
  // device-resident [n][C] store and copy it out with one contiguous DMA per
  // array (the per-batch path below copies 64-column strips: 64..512-byte
  // rows, far below PCIe efficiency).
  const uint64_t dbytes = out_dist ? (uint64_t)n * C * dist_bytes : 0;
  const uint64_t mbytes = out_masks ? (uint64_t)planes * n * C * sizeof(uint64_t) : 0;
  size_t fr = 0, tot = 0;
  CBFS_CUDA(cudaMemGetInfo(&fr, &tot));
  const bool force_staging = getenv("CBFS_HOST_STAGING") != nullptr;  // tests: exercise the per-batch path
  if (!force_staging && C && (dbytes + mbytes) > 0 && dbytes + mbytes + (2ull << 30) < fr) {
    void* dd = nullptr;
    uint64_t* dm = nullptr;
    if (dbytes) CBFS_CUDA(cudaMallocAsync(&dd, dbytes, st));
    if (mbytes) CBFS_CUDA(cudaMallocAsync(&dm, mbytes, st));
    if (dd) CBFS_CUDA(cudaMemsetAsync(dd, 0xFF, dbytes, st));
    if (dm) CBFS_CUDA(cudaMemsetAsync(dm, 0, mbytes, st));
    ArraySource as;
    as.proto = RunArgs{};
    as.proto.d = d;
    as.proto.planes = planes;
    as.proto.dist_bytes = dist_bytes;
    as.proto.C = n_clusters;
    as.proto.direction = direction;
    as.proto.engine = engine;
    as.proto.out_dist = dd;
    as.proto.out_masks = dm;
    as.sources = dsrc;
    as.sizes = dsz;
    as.n_clusters = n_clusters;
    as.out_stats = dstats;
    rc = run_batches(g, as, st);
    if (rc == CBFS_OK) {
      if (dd) CBFS_CUDA(cudaMemcpyAsync(out_dist, dd, dbytes, cudaMemcpyDeviceToHost, st));
      if (dm) CBFS_CUDA(cudaMemcpyAsync(out_masks, dm, mbytes, cudaMemcpyDeviceToHost, st));
      if (out_stats) CBFS_CUDA(cudaMemcpyAsync(out_stats, dstats, sizeof(uint64_t) * 4 * C, cudaMemcpyDeviceToHost, st));
    }
    if (dd) CBFS_CUDA(cudaFreeAsync(dd, st));
    if (dm) CBFS_CUDA(cudaFreeAsync(dm, st));
    CBFS_CUDA(cudaFreeAsync(dsrc, st));
    CBFS_CUDA(cudaFreeAsync(dsz, st));
    CBFS_CUDA(cudaFreeAsync(dstats, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    return rc;
  }
  HostSource src;
  src.proto.d = d;
  src.proto.planes = planes;
  src.proto.dist_bytes = dist_bytes;
  src.proto.direction = direction;
  src.proto.engine = engine;
  src.sources = dsrc;
  src.sizes = dsz;
  src.n_clusters = n_clusters;
  src.out_stats = dstats;
  src.n = n; src.planes = planes; src.dist_bytes = dist_bytes; src.C = C;
  src.h_dist = out_dist;
  src.h_masks = out_masks;
  src.sd.assign(P, nullptr);
  src.sm.assign(P, nullptr);
  for (int k = 0; k < P; ++k) {
    if (out_dist) CBFS_CUDA(cudaMallocAsync(&src.sd[k], (uint64_t)n * LANES * dist_bytes + 16, st));
    if (out_masks) CBFS_CUDA(cudaMallocAsync(&src.sm[k], sizeof(uint64_t) * (uint64_t)planes * n * LANES + 16, st));
  }
  rc = run_batches(g, src, st);
  if (rc == CBFS_OK && out_stats && C)
    CBFS_CUDA(cudaMemcpyAsync(out_stats, dstats, sizeof(uint64_t) * 4 * C, cudaMemcpyDeviceToHost, st));
  for (int k = 0; k < P; ++k) {
    if (src.sd[k]) CBFS_CUDA(cudaFreeAsync(src.sd[k], st));
    if (src.sm[k]) CBFS_CUDA(cudaFreeAsync(src.sm[k], st));
  }
  CBFS_CUDA(cudaFreeAsync(dsrc, st));
  CBFS_CUDA(cudaFreeAsync(dsz, st));
  CBFS_CUDA(cudaFreeAsync(dstats, st));
  CBFS_CUDA(cudaStreamSynchronize(st));
  return rc;
}

}  // extern "C"
