// digest.cu — full-size output consumers of the C-BFS engines:
//  * cbfs_run_digest: every batch of 64 clusters writes its full output
//    vectors <Delta_v, S_v[0..planes-1]> into a per-slot staging
//    store in HBM (the fold's ordinary output path); when the batch's last
//    round is queued, k_digest reads the store back on the slot's stream,
//    reduces every cluster to its 64-bit digest and resets the store for the
//    slot's next batch.  This is how configurations whose whole output does
//    not fit HBM (config 3: 1.7 TB) are run with every output written and
//    consumed inside the call, and compared with the oracle at full size;
//  * cbfs_digest_store: the same digest over a caller's [n][C] store;
//  * cbfs_run_rounds: per-round frontier statistics {|F_i|, E_i}.
// The digest definition is in include/cbfs.h (cbfs_digest_store); the oracle
// computes it independently (oracle.c or_digest_cluster).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.cuh"

namespace cbfs {

__device__ __forceinline__ uint64_t dg_fin(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// One 64-column strip [c0, c0 + 64) of a vertex-major store (row stride L
// columns): a warp per row, lane l owns columns c0 + 2l and c0 + 2l + 1, so
// every Delta / subset load of the warp is one contiguous row segment.  Each
// lane accumulates its two clusters' sums over its rows in registers and adds
// them to out[] once.  With `clear`, the strip is reset to the unreached state
// (Delta = sentinel, subsets 0) after it is read (staging reuse).
// Staging rows by internal id (the fold's writes follow the traversal's
// vertex order; the digest keys perm[v]): 0 never, 1 always, 2 (default) for
// the sparse engine only — measured: batched engine on config 3 slower
// (fold +45 ms, consume +57 ms per step), see profiles/r02_*.
#ifndef CBFS_DIGEST_INTERNAL
#define CBFS_DIGEST_INTERNAL 2
#endif
constexpr uint32_t DG_MAXP = 4;  // planes held in registers per row (more are streamed)
#ifndef CBFS_DG_ROWS
#define CBFS_DG_ROWS 2
#endif
#ifndef CBFS_DG_MINB
#define CBFS_DG_MINB 3
#endif
constexpr int DG_ROWS = CBFS_DG_ROWS;  // rows in flight per warp

template <int DB>
__global__ void __launch_bounds__(256, CBFS_DG_MINB) k_digest(void* __restrict__ dist, uint64_t* __restrict__ masks, uint32_t n,
                                                uint64_t L, uint32_t c0, uint32_t nc, uint32_t planes,
                                                uint64_t* __restrict__ out, int clear,
                                                const uint32_t* __restrict__ perm) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cb = c0 + 64 * blockIdx.y;  // this block's strip
  const uint32_t ca = cb + 2 * lane, cc = ca + 1;
  const bool ha = ca < nc, hb = cc < nc;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t plane_stride = (uint64_t)n * L;
  uint64_t sa = 0, sb = 0;
  if (ha || hb) {
    // DG_ROWS rows per warp step: all their loads are issued before any hash
    for (uint64_t v0 = warp; v0 < n; v0 += nwarps * DG_ROWS) {
      uint64_t da[DG_ROWS], db[DG_ROWS], ma[DG_ROWS][DG_MAXP], mb[DG_ROWS][DG_MAXP];
#pragma unroll
      for (int r = 0; r < DG_ROWS; ++r) {
        const uint64_t v = v0 + r * nwarps;
        da[r] = db[r] = 0xFFFF;
        if (v >= n) continue;
        const uint64_t row = v * L;
        CBFS_DCHECK(!hb || cc < L);
        if (DB == 1) {
          const uint8_t* p = (const uint8_t*)dist + row;
          if (ha) { const uint8_t x = p[ca]; da[r] = x == 0xFF ? 0xFFFFu : x; }
          if (hb) { const uint8_t x = p[cc]; db[r] = x == 0xFF ? 0xFFFFu : x; }
        } else {
          const uint16_t* p = (const uint16_t*)dist + row;
          if (ha) da[r] = p[ca];
          if (hb) db[r] = p[cc];
        }
#pragma unroll
        for (uint32_t i = 0; i < DG_MAXP; ++i) {
          ma[r][i] = mb[r][i] = 0;
          if (i < planes) {
            const uint64_t* mp = masks + i * plane_stride + row;
            if (ha) ma[r][i] = mp[ca];
            if (hb) mb[r][i] = mp[cc];
          }
        }
      }
#pragma unroll
      for (int r = 0; r < DG_ROWS; ++r) {
        const uint64_t v = v0 + r * nwarps;
        if (v >= n) continue;
        const uint64_t row = v * L;
        const uint64_t vo = perm ? perm[v] : v;  // internal-id rows: the digest keys original ids
        const uint64_t key = vo * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL;
        uint64_t xa = dg_fin(key ^ (da[r] << 48)), xb = dg_fin(key ^ (db[r] << 48));
#pragma unroll
        for (uint32_t i = 0; i < DG_MAXP; ++i) {
          if (i >= planes) break;
          uint64_t* mp = masks + i * plane_stride + row;
          xa = dg_fin(xa ^ ma[r][i]);
          xb = dg_fin(xb ^ mb[r][i]);
          if (clear) {
            if (ha && ma[r][i]) mp[ca] = 0;
            if (hb && mb[r][i]) mp[cc] = 0;
          }
        }
        for (uint32_t i = DG_MAXP; i < planes; ++i) {  // d > 3: streamed
          uint64_t* mp = masks + i * plane_stride + row;
          const uint64_t wa = ha ? mp[ca] : 0, wb = hb ? mp[cc] : 0;
          xa = dg_fin(xa ^ wa);
          xb = dg_fin(xb ^ wb);
          if (clear) {
            if (ha && wa) mp[ca] = 0;
            if (hb && wb) mp[cc] = 0;
          }
        }
        if (clear) {
          if (DB == 1) {
            uint8_t* p = (uint8_t*)dist + row;
            if (ha && da[r] != 0xFFFF) p[ca] = 0xFF;
            if (hb && db[r] != 0xFFFF) p[cc] = 0xFF;
          } else {
            uint16_t* p = (uint16_t*)dist + row;
            if (ha && da[r] != 0xFFFF) p[ca] = 0xFFFF;
            if (hb && db[r] != 0xFFFF) p[cc] = 0xFFFF;
          }
        }
        sa += xa;
        sb += xb;
      }
    }
  }
  if (ha) atomicAdd((unsigned long long*)&out[ca], (unsigned long long)sa);
  if (hb) atomicAdd((unsigned long long*)&out[cc], (unsigned long long)sb);
}

// The same digest over a CLUSTER-major staging store (the sparse engine's
// outputs: its frontier is cluster-major, so its writes coalesce there):
// Delta (u16) at [c][v], subset i at [i][64][v].  Block row y = cluster c,
// thread per vertex, block-reduced sum added once per block.
__global__ void __launch_bounds__(256) k_digest_cm(uint16_t* __restrict__ dist, uint64_t* __restrict__ masks,
                                                   uint32_t n, uint32_t planes, uint64_t* __restrict__ out,
                                                   const uint32_t* __restrict__ perm) {
  __shared__ unsigned long long s_sum[8];
  const uint32_t c = blockIdx.y;
  uint16_t* dc = dist + (uint64_t)c * n;
  uint64_t sum = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t dv = dc[v];
    const uint64_t vo = perm ? perm[v] : v;
    uint64_t x = dg_fin((vo * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL) ^ (dv << 48));
    for (uint32_t i = 0; i < planes; ++i) {
      uint64_t* mp = masks + ((uint64_t)i * LANES + c) * n + v;
      const uint64_t m = *mp;
      x = dg_fin(x ^ m);
      if (m) *mp = 0;
    }
    if (dv != 0xFFFF) dc[v] = 0xFFFF;
    sum += x;
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_sum[k];
    atomicAdd((unsigned long long*)&out[c], t);
  }
}

static int launch_digest(const void* dist, uint32_t dist_bytes, const uint64_t* masks, uint32_t n, uint64_t L,
                         uint32_t nc, uint32_t planes, uint64_t* out, int clear, const uint32_t* perm,
                         cudaStream_t st) {
  if (nc == 0 || n == 0) return CBFS_OK;
  const uint32_t strips = (nc + 63) / 64;
  const unsigned bx = std::max(1u, grid_for((uint64_t)n * 32, 256, 148u * CBFS_DG_MINB) / std::max(1u, std::min(strips, 8u)));
  const dim3 grid(bx, strips);
  if (dist_bytes == 1)
    k_digest<1><<<grid, 256, 0, st>>>(const_cast<void*>(dist), const_cast<uint64_t*>(masks), n, L, 0, nc, planes, out,
                                      clear, perm);
  else
    k_digest<2><<<grid, 256, 0, st>>>(const_cast<void*>(dist), const_cast<uint64_t*>(masks), n, L, 0, nc, planes, out,
                                      clear, perm);
  CBFS_LAUNCHED();
  return CBFS_OK;
}

// per-slot staging store: the batch writes its outputs there; the digest
// reads (and resets) it on the slot's stream when the batch ends
struct DigestSource : ArraySource {
  uint32_t n = 0, planes = 0, dist_bytes = 0;
  uint64_t* digest = nullptr;  // [n_clusters]
  std::vector<void*> sd;
  std::vector<uint64_t*> sm;
  bool cmajor = false;  // sparse engine: cluster-major staging, u16 Delta (sd sized for u16)
  const uint32_t* perm = nullptr;  // staging rows are internal ids; the digest keys perm[v]
  int bind(RunArgs& a, int slot, cudaStream_t) override {
    if (sd.empty()) return CBFS_OK;  // statistics only (cbfs_run_rounds)
    a.out_dist = sd[slot];
    a.out_masks = sm[slot];
    a.C = LANES;
    a.cbase = 0;
    a.out_cmajor = cmajor;
    return CBFS_OK;
  }
  int launch(const RunArgs& a, int slot, uint64_t* out, cudaStream_t st) {
    if (!cmajor) return launch_digest(sd[slot], dist_bytes, sm[slot], n, LANES, a.nb, planes, out, 1, perm, st);
    if (n == 0 || a.nb == 0) return CBFS_OK;
    const dim3 grid(std::max(1u, grid_for(n, 256, 148u * 8u) / std::max(1u, a.nb / 8u)), a.nb);
    k_digest_cm<<<grid, 256, 0, st>>>(reinterpret_cast<uint16_t*>(sd[slot]), sm[slot], n, planes, out, perm);
    CBFS_LAUNCHED();
    return CBFS_OK;
  }
  int finished(const RunArgs& a, int slot, cudaStream_t st) override {
    if (sd.empty()) return CBFS_OK;
    const uint64_t c0 = (uint64_t)(a.sizes - sizes);  // first cluster of the batch
    if (!prof_on()) return launch(a, slot, digest + c0, st);
    if (!ev[0]) {
      CBFS_CUDA(cudaEventCreate(&ev[0]));
      CBFS_CUDA(cudaEventCreate(&ev[1]));
    }
    CBFS_CUDA(cudaEventRecord(ev[0], st));
    int rc = launch(a, slot, digest + c0, st);
    if (rc) return rc;
    CBFS_CUDA(cudaEventRecord(ev[1], st));
    CBFS_CUDA(cudaEventSynchronize(ev[1]));
    float ms = 0;
    CBFS_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    prof_add(PK_CONSUME, ms, 1, (uint64_t)n * a.nb);
    return CBFS_OK;
  }
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~DigestSource() override {
    if (ev[0]) cudaEventDestroy(ev[0]);
    if (ev[1]) cudaEventDestroy(ev[1]);
  }
};

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_digest_store(uint32_t n, uint32_t C, uint32_t planes, const void* dist, uint32_t dist_bytes,
                      const uint64_t* masks, uint64_t* out_digest, cbfs_stream stream) {
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (planes > CBFS_MAX_D + 1) return fail(CBFS_EINVAL, "planes must be <= CBFS_MAX_D + 1");
  if (C && (!out_digest || (n && (!dist || (planes && !masks))))) return fail(CBFS_EINVAL, "null store / digest");
  cudaStream_t st = (cudaStream_t)stream;
  if (C == 0) return CBFS_OK;
  CBFS_CUDA(cudaMemsetAsync(out_digest, 0, sizeof(uint64_t) * C, st));
  int rc = launch_digest(dist, dist_bytes, masks, n, C, C, planes, out_digest, 0, nullptr, st);
  if (rc) return rc;
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

// one staging store per slot used: as many slots as fit next to the stores
static int run_consumed(Graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                        uint32_t dist_bytes, uint32_t planes, uint64_t* out_digest, uint64_t* out_stats,
                        uint64_t* out_rounds, uint32_t max_rounds, uint32_t direction, cudaStream_t st) {
  const int engine = choose_engine(g, direction);
  if (engine < 0) return CBFS_ECUDA;
  const bool cmajor = engine == ENGINE_SPARSE;
  const uint32_t sdb = cmajor ? 2 : dist_bytes;  // cluster-major staging keeps u16 Delta
  const uint64_t stage = out_digest ? (uint64_t)g->n * LANES * (sdb + 8ull * planes) + 64 : 0;
  WorkLease lease(g, engine, stage);
  if (lease.rc) return lease.rc;
  const uint32_t n = g->n;
  const uint64_t C = n_clusters;
  if (out_digest && C) CBFS_CUDA(cudaMemsetAsync(out_digest, 0, sizeof(uint64_t) * C, st));
  if (out_rounds && C) CBFS_CUDA(cudaMemsetAsync(out_rounds, 0, sizeof(uint64_t) * 2 * max_rounds * C, st));
  DigestSource src;
  src.proto = RunArgs{};
  src.proto.d = d;
  src.proto.planes = planes;
  src.proto.dist_bytes = dist_bytes;
  src.proto.C = n_clusters;
  src.proto.direction = direction;
  src.proto.engine = engine;
  // outputs staged by internal id: the fold's writes follow the traversal
  // (no dependent perm[v] load per entry); the digest maps rows back
  const bool internal = CBFS_DIGEST_INTERNAL == 1 || (CBFS_DIGEST_INTERNAL == 2 && cmajor);
  src.proto.out_internal = internal;
  src.perm = internal ? g->perm : nullptr;
  src.sources = sources;
  src.sizes = sizes;
  src.n_clusters = n_clusters;
  src.out_stats = out_stats;
  src.out_rounds = out_rounds;
  src.max_rounds = max_rounds;
  src.n = n;
  src.planes = planes;
  src.dist_bytes = dist_bytes;
  src.digest = out_digest;
  src.cmajor = cmajor;
  int P = num_slots(g);
  const double ta = getenv("CBFS_TRACE") ? std::chrono::duration<double, std::milli>(
                                              std::chrono::steady_clock::now().time_since_epoch()).count() : 0;
  if (out_digest) {
    const uint64_t per = stage;
    size_t fr = 0, tot = 0;
    CBFS_CUDA(cudaMemGetInfo(&fr, &tot));
    const uint64_t margin = 1ull << 30;
    const uint64_t fit = fr > margin ? (fr - margin) / per : 0;
    if (fit == 0) return fail(CBFS_ENOMEM, "no room for one output staging store");
    P = (int)std::min<uint64_t>((uint64_t)P, fit);
    src.sd.assign(P, nullptr);
    src.sm.assign(P, nullptr);
    for (int k = 0; k < P; ++k) {
      CBFS_CUDA(cudaMallocAsync(&src.sd[k], (uint64_t)n * LANES * sdb + 16, st));
      CBFS_CUDA(cudaMemsetAsync(src.sd[k], 0xFF, (uint64_t)n * LANES * sdb, st));
      if (planes) {
        CBFS_CUDA(cudaMallocAsync(&src.sm[k], sizeof(uint64_t) * planes * (uint64_t)n * LANES + 16, st));
        CBFS_CUDA(cudaMemsetAsync(src.sm[k], 0, sizeof(uint64_t) * planes * (uint64_t)n * LANES, st));
      }
    }
  }
  static const bool trace = getenv("CBFS_TRACE") != nullptr;  // measurements: phase times with syncs
  if (trace) {
    cudaStreamSynchronize(st);
    fprintf(stderr, "[cbfs trace] run_consumed: staging allocated + cleared in %.1f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count() - ta);
  }
  auto now_ms = [&]() {
    cudaStreamSynchronize(st);
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = trace ? now_ms() : 0;
  int rc = run_batches(g, src, st, P);
  if (trace) fprintf(stderr, "[cbfs trace] run_consumed: %d slots, staging %.1f GB each, batches %.1f ms\n", P,
                     stage / 1e9, now_ms() - t0);
  for (int k = 0; k < (int)src.sd.size(); ++k) {
    cudaFreeAsync(src.sd[k], st);
    if (src.sm[k]) cudaFreeAsync(src.sm[k], st);
  }
  if (rc) return rc;
  CBFS_CUDA(cudaStreamSynchronize(st));
  return CBFS_OK;
}

int cbfs_run_digest(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                    uint32_t dist_bytes, uint32_t planes, uint64_t* out_digest, uint64_t* out_stats,
                    uint32_t direction, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  int rc = check_run_args(g, sources, sizes, n_clusters, d, dist_bytes, planes, direction);
  if (rc) return rc;
  if (n_clusters && !out_digest) return fail(CBFS_EINVAL, "null out_digest");
  CBFS_CUDA(cudaSetDevice(g->device));
  return run_consumed(g, sources, sizes, n_clusters, d, dist_bytes, planes, out_digest, out_stats, nullptr, 0,
                      direction, (cudaStream_t)stream);
}

int cbfs_run_rounds(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                    uint64_t* out_rounds, uint32_t max_rounds, uint64_t* out_stats, uint32_t direction,
                    cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  int rc = check_run_args(g, sources, sizes, n_clusters, d, 2, d + 1, direction);
  if (rc) return rc;
  if (n_clusters && (!out_rounds || max_rounds == 0)) return fail(CBFS_EINVAL, "null out_rounds / max_rounds == 0");
  CBFS_CUDA(cudaSetDevice(g->device));
  return run_consumed(g, sources, sizes, n_clusters, d, 2, d + 1, nullptr, out_stats, out_rounds, max_rounds,
                      direction, (cudaStream_t)stream);
}

}  // extern "C"
