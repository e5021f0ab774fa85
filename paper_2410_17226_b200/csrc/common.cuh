// common.cuh — shared internals of libcbfs.so (product side only; the oracle
// under oracle/ shares nothing with this file).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include <atomic>
#include <string>

#include "../../include/cbfs.h"

namespace cbfs {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(uint64_t k = 1);

#define CBFS_CUDA(call)                                  \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::cbfs::cuda_fail(_e, #call); \
  } while (0)

#define CBFS_LAUNCHED()                                           \
  do {                                                            \
    ::cbfs::count_launch();                                       \
    cudaError_t _e = cudaGetLastError();                          \
    if (_e != cudaSuccess) return ::cbfs::cuda_fail(_e, "kernel launch"); \
  } while (0)

// Device-side bounds checks of the hot kernels (build with
// -DCBFS_DEBUG_CHECKS: tools/build_variant.sh checks -DCBFS_DEBUG_CHECKS);
// a failed check prints the condition and traps.  Compiled out by default.
#ifdef CBFS_DEBUG_CHECKS
#define CBFS_DCHECK(cond)                                                                                   \
  do {                                                                                                      \
    if (!(cond)) {                                                                                          \
      printf("CBFS_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,          \
             (int)blockIdx.x, (int)threadIdx.x);                                                            \
      __trap();                                                                                             \
    }                                                                                                       \
  } while (0)
#else
#define CBFS_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

constexpr uint16_t INF16 = 0xFFFFu;
constexpr uint32_t LANES = 64;  // clusters per batch (vertex-major state rows of 64 words)

// ---------------------------------------------------------------- graph
struct Graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t m = 0;            // arcs
  uint32_t max_degree = 0;
  uint32_t n_nonisolated = 0;
  bool relabeled = false;
  // internal CSR (internal ids; == original ids unless relabeled)
  uint64_t* off = nullptr;   // [n+1]
  uint32_t* cols = nullptr;  // [m]
  // original-id CSR (only when relabeled; else aliases off/cols)
  uint64_t* off_orig = nullptr;
  uint32_t* cols_orig = nullptr;
  uint32_t* perm = nullptr;  // internal -> original (null if identity)
  uint32_t* inv = nullptr;   // original -> internal (null if identity)
  uint32_t* rank = nullptr;  // internal id -> position in (deg desc, orig id asc) order
  uint32_t* order = nullptr; // position -> internal id
  // pull-kernel chunk table: first vertex of every PULL_CHUNK arcs
  uint32_t* chunk_v = nullptr;
  uint64_t n_chunks = 0;
  // diameter class for the engine choice (-1 unknown, 0 low, 1 high; sparse.cu)
  int high_diameter = -1;
  // traversal workspace (lazily allocated, sized n*LANES)
  struct Work* work = nullptr;
};

#ifndef CBFS_PULL_CHUNK
#define CBFS_PULL_CHUNK 1024
#endif
constexpr uint32_t PULL_CHUNK = CBFS_PULL_CHUNK;  // arcs per warp task in the dense pull kernel

int graph_free(Graph* g);

// RAII lease of the device's cached traversal workspace (sets g->work)
struct WorkLease {
  // engine: ENGINE_* the call runs (-1: either; sizes the state block);
  // extra_per_slot: bytes the caller will allocate per slot (staging)
  explicit WorkLease(Graph* g, int engine = -1, uint64_t extra_per_slot = 0);
  ~WorkLease();
  int rc = CBFS_OK;
 private:
  Graph* g_;
  bool locked_ = false;
};

// one batch (<= LANES clusters) of cbfs_run; outputs use row stride C and
// start at column cbase
struct RunArgs {
  const uint32_t* sources;  // device, batch base ([nb][64])
  const uint8_t* sizes;     // device, batch base ([nb])
  uint32_t nb, d, planes, dist_bytes, C, cbase, direction;
  int engine;               // ENGINE_BATCHED / ENGINE_SPARSE (engine.cuh)
  int out_internal;         // output rows are internal ids (library-internal staging), not original ids
  void* out_dist;           // device [n][C] or null
  void* out_masks;          // device [planes][n][C] words of mask_bytes, or null
  uint64_t* out_stats;      // device [nb][4] or null
  uint32_t mask_bytes;      // 8 (cbfs_run) or 1/2/4 (packed label stores, w = 8 * mask_bytes; 0 reads as 8)
  uint32_t out_cmajor;      // outputs cluster-major (Delta at col * n + row; library-internal staging, sparse engine)
  uint32_t wide;            // W > 1: lanes are the 64-source words of clusters of W lanes (cbfs_run_wide); out_dist
                            // has C / W columns
  uint64_t* out_rounds;     // device [nb][max_rounds][2] {|F_i|, E_i} per round, or null (added to: zeroed by the caller)
  uint32_t max_rounds;      // rounds recorded per cluster in out_rounds
};
// A producer of batches for run_batches (several batches run concurrently,
// one per workspace slot, each on its own stream).
struct BatchSource {
  virtual ~BatchSource() = default;
  // fill `a` with the next batch: 1 = got one, 0 = none available yet, -1 = exhausted
  virtual int next(RunArgs& a) = 0;
  // before the batch starts on slot `slot` (may redirect outputs to slot-local buffers on stream s)
  virtual int bind(RunArgs& a, int slot, cudaStream_t s) { (void)a; (void)slot; (void)s; return CBFS_OK; }
  // after the batch's last kernel has been queued on stream s
  virtual int finished(const RunArgs& a, int slot, cudaStream_t s) { (void)a; (void)slot; (void)s; return CBFS_OK; }
};
// batches of an array of clusters in device memory
struct ArraySource : BatchSource {
  RunArgs proto{};
  const uint32_t* sources = nullptr;
  const uint8_t* sizes = nullptr;
  uint32_t n_clusters = 0, next_c = 0;
  uint64_t* out_stats = nullptr;
  uint64_t* out_rounds = nullptr;  // [n_clusters][max_rounds][2] or null
  uint32_t max_rounds = 0;
  int next(RunArgs& a) override;
};
// Drive all batches of `src` through the device's slots (at most max_slots of
// them when > 0: callers that stage outputs per slot bound their memory).
int run_batches(Graph* g, BatchSource& src, cudaStream_t st, int max_slots = 0);
int num_slots(const Graph* g);  // concurrent batches of the leased workspace
int select_launch(const Graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy, uint64_t seed,
                  uint32_t* out_sources, uint8_t* out_sizes, uint32_t* d_count, volatile uint32_t* progress,
                  cudaStream_t st, uint32_t words = 1, uint16_t* out_sizes16 = nullptr);
int check_select_args(const Graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                      const void* out_sources, const void* out_sizes);
// cbfs_run with the output bit-subset words mask_bytes wide (1/2/4/8)
int run_arrays(Graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
               uint32_t dist_bytes, void* out_dist, void* out_masks, uint32_t mask_bytes, uint32_t planes,
               uint64_t* out_stats, uint32_t direction, cudaStream_t st);
// cbfs_query_distance over a store whose bit-subset words are mask_bytes wide
int query_store(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                const void* masks, uint32_t mask_bytes, const uint8_t* sizes, const uint32_t* s, const uint32_t* t,
                uint64_t q, int32_t* inout_best, cudaStream_t st);
int check_run_args(const Graph* g, const void* sources, const void* sizes, uint32_t n_clusters, uint32_t d,
                   uint32_t dist_bytes, uint32_t planes, uint32_t direction);

// ---------------------------------------------------------------- RNG
// Counter-based SplitMix64 with the same definition as the input generator
// (implemented here independently of the generator library).
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t crand(uint64_t seed, uint64_t stream, uint64_t index) {
  uint64_t key = mix64(seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL);
  return mix64(key + (index + 1) * 0x9E3779B97F4A7C15ULL);
}
__host__ __device__ inline uint64_t bounded(uint64_t x, uint64_t n) {
#ifdef __CUDA_ARCH__
  return __umul64hi(x, n);
#else
  return (uint64_t)(((unsigned __int128)x * n) >> 64);
#endif
}

// one output bit-subset word: a full u64, or the low 8/16/32 bits of a packed
// w-bit label store (the cluster has <= w sources, so nothing is dropped)
__device__ __forceinline__ void store_mask(void* p, uint64_t idx, uint64_t v, uint32_t mb) {
  switch (mb) {
    case 1: ((uint8_t*)p)[idx] = (uint8_t)v; break;
    case 2: ((uint16_t*)p)[idx] = (uint16_t)v; break;
    case 4: ((uint32_t*)p)[idx] = (uint32_t)v; break;
    default: ((uint64_t*)p)[idx] = v; break;
  }
}

__host__ __device__ inline uint64_t full_mask(uint32_t k) { return k >= 64 ? ~0ULL : ((1ULL << k) - 1); }

inline unsigned grid_for(uint64_t items, unsigned block, unsigned cap = 148u * 64u) {
  uint64_t g = (items + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace cbfs
