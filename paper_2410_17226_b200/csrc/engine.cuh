// engine.cuh — internals shared by the two C-BFS engines of libcbfs.so:
//  * the BATCHED engine (cbfs.cu): vertex-major state rows of 64 clusters,
//    host-driven rounds with a push/pull switch — for low-diameter graphs,
//    where the 64 clusters' frontiers overlap round by round;
//  * the SPARSE engine (sparse.cu): cluster-major state, push-only rounds,
//    the whole round loop on the device (CUDA-graph while-node) — for
//    high-diameter graphs, where the clusters' wavefronts are disjoint.
// Both run Alg. 1 and produce identical outputs (R8, R25).
#pragma once
#include <vector>

#include "common.cuh"

namespace cbfs {

enum : unsigned long long { ERR_BAD_SOURCE = 1, ERR_DUP_SOURCE = 2, ERR_BAD_SIZE = 4, ERR_OVERFLOW = 8,
                            ERR_ROUNDS = 16 };
enum { ENGINE_BATCHED = 0, ENGINE_SPARSE = 1 };
// kernel-level profiling (cbfs_profile_*): kinds of cbfs_profile_read
enum { PK_FOLD = 0, PK_PUSH = 1, PK_PULL = 2, PK_SPARSE = 3, PK_CONSUME = 4, PK_N = 5 };
bool prof_on();
void prof_add(int kind, double ms, uint64_t launches, uint64_t entries);

constexpr unsigned FULLW = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULLW, x, o);
  return x;
}

// Sparse-engine state of one (cluster, vertex) cell: S_seen, Delta and the
// two pending buffers P_i / P_{i+1} (S_next \ S_seen) in one 32-byte sector,
// so the push touches one sector per arc (the cap test and the atomicOr hit
// the same sector).
struct __align__(32) SpCell {
  uint64_t seen;
  uint32_t dist;  // Delta, INF16 = unreached
  uint32_t pad;
  uint64_t p[2];
};
constexpr uint64_t SPARSE_CELL_BYTES = sizeof(SpCell);
static_assert(sizeof(SpCell) == 32, "one sector per cell");

// Device-resident description of the batch a sparse-engine slot runs: the
// instantiated CUDA graph reads everything that changes per batch from here,
// so one graph per slot serves every batch and every graph handle.
struct SpDesc {
  const uint64_t* off;
  const uint32_t* cols;
  const uint32_t* perm;      // internal -> original id (null: identity)
  const uint32_t* inv;       // original -> internal id (null: identity)
  const uint32_t* sources;   // [nb][64]
  const uint8_t* sizes;      // [nb]
  void* out_dist;            // [n][C] or null
  void* out_masks;           // [planes][n][C] words of mask_bytes, or null
  uint64_t C, cbase;
  uint32_t n, nb, d, planes, dist_bytes, mask_bytes;
  uint32_t wide;             // W > 1: lanes are the 64-source words of clusters of W lanes (cbfs_run_wide)
  uint32_t out_cmajor;       // outputs cluster-major (RunArgs::out_cmajor)
  uint64_t* rounds;          // [nb][max_rounds][2] per-round {|F_i|, E_i}, or null
  uint32_t max_rounds;
  uint32_t nw32;             // words per cluster of the ordered frontier bitmap (ceil(n / 32))
  uint32_t* bits;            // ordered frontier bitmap [nb][nw32] (null: list frontiers only)
  uint64_t bm_min;           // |F_{i+1}| from which round i+1's claims go to the bitmap
};
// Round state of a sparse-engine batch (device-resident).
struct SpCtl {
  unsigned long long nF[2];  // frontier list sizes: list (i & 1) holds F_i
  unsigned long long err;    // ERR_* bits
  unsigned long long i;      // current round
  unsigned long long listed; // frontier list entries processed (incl. entries whose S_new came out empty)
  unsigned long long go;     // the round loop continues (set at the end of each round)
  unsigned done;             // blocks of the round's push that finished
  unsigned pad;
  unsigned long long take[2];  // next unclaimed frontier entry of the round's fold / push (dynamic chunks)
  unsigned long long bm;       // the next round's push records its claims in the ordered bitmap (sparse.cu)
  unsigned long long bm_fill;  // append cursor of the bitmap -> list compaction
};

// Device-resident state of a BATCHED-engine slot: the graph and batch
// arguments (written by the host when a batch starts), the slot's arrays, and
// the round state the device-side round loop advances (cbfs.cu).  Kernels of
// the loop take only this pointer, so one instantiated CUDA graph per slot
// (and Delta width / wide flag) serves every batch and every graph handle.
struct BState {
  // graph
  const uint64_t* off;
  const uint32_t* cols;
  const uint32_t* chunk_v;
  const uint32_t* perm;  // output rows: internal -> original (null: identity or library-internal rows)
  const uint32_t* inv;   // original -> internal (sources)
  uint64_t n_chunks, m;
  // batch
  const uint32_t* sources;  // [nb][64]
  const uint8_t* sizes;     // [nb]
  void* out_dist;
  void* out_masks;
  uint64_t* rstats;         // [nb][R][2] or null
  uint32_t n, nb, d, planes, C, cbase, mb, W, R, direction, hub_rows, allow_empty;
  double pull_threshold;    // the edge phase pulls when the frontier's (cluster, arc) pairs exceed this
  // slot arrays
  uint64_t *seen, *pend, *pre, *fullm, *bstats, *scan_tmp;
  uint16_t* dist;
  uint32_t* list[2];
  uint32_t* ubits;          // [2][ub_words]: U_i of parity i & 1
  uint64_t ub_words;
  // round state: cnt[p] = {entries, E (degree sum), -, |U|} of the list of parity p
  unsigned long long cnt[2][4];
  unsigned long long err, i, pull, go, launches;
  unsigned end_done;
  unsigned prof_on;
  // per-kernel profile of the batch (PK_* kinds, globaltimer ns)
  unsigned long long p_t0[8], p_ns[8], p_launch[8], p_entries[8], p_arcs[8], p_uin[8], p_uout[8];
  unsigned p_arrive[8], p_leave[8];
};

// One in-flight batch of LANES clusters: its workspace, its stream, and the
// state of its round loop.  Several slots run concurrently (run_batches), so
// the small rounds and the latency-bound dense rounds of different batches
// overlap on the GPU.  The sparse engine reuses the same arrays with a
// cluster-major layout (see sparse.cu).
struct Slot {
  uint64_t cap = 0;                     // n * LANES entries
  void* blk = nullptr;                  // per-cell state of either engine (seen/pend/pre/dist or sparse cells)
  uint64_t* seen = nullptr;             // [n+1][64] S_seen (row n stays zero)
  uint64_t* pend = nullptr;             // [n][64] S_next \ S_seen (pending)
  uint16_t* dist = nullptr;             // [n][64] Delta
  uint32_t* listA = nullptr;            // frontier lists (packed v*64+c)
  uint32_t* listB = nullptr;
  uint64_t* pre = nullptr;              // [cap + 1] degrees -> exclusive prefix (push)
  uint32_t* ubits = nullptr;            // 2 x [n/32 + 1]: union frontier U_i, U_{i+1}
  uint64_t* bstats = nullptr;           // [LANES][4]
  uint64_t* fullm = nullptr;            // [n] bit c: S_seen[v][c] == S_c (maintained by the fold)
  void* scan_tmp = nullptr;             // [SCAN_BLOCKS] tile sums of the push's degree scan
  cudaStream_t s = nullptr;
  cudaEvent_t ready = nullptr;  // counters of the last queued round are on the host
  // round-loop state
  bool busy = false;
  bool seeding = false;
  RunArgs a{};
  uint32_t i = 0;
  bool overflow = false;
  // sparse engine
  int engine = ENGINE_BATCHED;  // engine of the batch in flight
  uint64_t pend_clean_cells = 0;  // the batched `pend` is zero over [0, pend_clean_cells)
  SpDesc* sp_desc = nullptr;    // device
  SpDesc* sp_desc_h = nullptr;  // pinned staging
  SpCtl* sp_ctl = nullptr;      // device
  SpCtl* sp_ctl_h = nullptr;    // pinned mirror
  cudaGraph_t sp_graph = nullptr;
  cudaGraphExec_t sp_exec = nullptr;
  cudaEvent_t sp_t0 = nullptr, sp_t1 = nullptr;  // profiling
  uint32_t sp_db = 0;                             // dist_bytes the graph was built for
  bool sp_fused = false;                          // fold fused into the push (d >= 1)
  int sp_shape = 0;                               // push shape (SpShape: by the graph's average degree)
  bool sp_ordered = false;                        // graph built with the ordered-frontier branch
  uint32_t* sp_bits = nullptr;                    // ordered frontier bitmap [LANES][nw32 * 32 bits]
  uint64_t sp_bits_words = 0;
  // batched engine (device-side round loop)
  int idx = 0;             // slot index on its device (constant-memory BState mirror c_bs[idx])
  BState* bs = nullptr;    // device
  BState* bs_h = nullptr;  // pinned mirror
  cudaGraph_t b_graph[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [dist_bytes == 2][wide]
  cudaGraphExec_t b_exec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
};

struct DevSlots {
  std::vector<Slot*> slots;
  uint64_t cap = 0;  // cells per slot (n * LANES)
  uint64_t blk = 0;  // bytes of each slot's state block (engine-dependent)
};

// sparse.cu
int sparse_alloc(Slot* w);
void sparse_free(Slot* w);
int sparse_start(const Graph* g, Slot* w, const RunArgs& a);  // queue init + seeding + counters readback
int sparse_launch(Slot* w);                                    // queue the whole round loop + readback
int choose_engine(Graph* g, uint32_t direction);               // ENGINE_* for this graph and direction
extern int g_engine_policy;                                    // CBFS_ENGINE_*

}  // namespace cbfs
