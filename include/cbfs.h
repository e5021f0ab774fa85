/*
 * cbfs.h — C-ABI of libcbfs.so, the B200 (sm_100a) Cluster-BFS library.
 *
 * Implements the data-parallel hot path of "Parallel Cluster-BFS and
 * Applications to Shortest Paths" (arXiv 2410.17226; citations P:n are lines
 * of its PAPER.md, R1..R26 the readings listed in DESIGN.md §2):
 *   graph build      -> cbfs_graph_create / cbfs_graph_create_csr
 *   cluster selection -> cbfs_select_clusters
 *   C-BFS, Alg. 1, direction-optimised EdgeMap,
 *     batched over clusters      -> cbfs_run
 *   distance decode  -> cbfs_decode
 *   landmark labels -> cbfs_run with planes = d,
 *                                  or the cbfs_labels_* handle (build, export
 *                                  / import for the multi-GPU gather, query)
 *   landmark query  -> cbfs_query_distance
 *   fused build + query (streaming index)      -> cbfs_query_stream
 *
 * Conventions (all functions):
 *  - Return CBFS_OK (0) or a negative cbfs_status; cbfs_last_error() gives a
 *    thread-local message.  Argument errors are detected on the host before
 *    any work is queued.  Device-side argument errors (duplicate / out of
 *    range sources held in device memory) and CUDA faults are reported by the
 *    call that detects them; the call then leaves outputs unspecified.
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream).  Calls
 *    are stream-ordered; every function that returns a host-visible value
 *    synchronises the stream before returning.  The traversals (cbfs_run and
 *    the calls built on it) run each batch's whole round loop on the device
 *    (one CUDA graph launch per batch of 64 clusters: a conditional WHILE
 *    over the rounds, an IF/ELSE for the push / pull direction); the host
 *    waits once per batch for the seeding's argument check and returns when
 *    the last batch is done.
 *  - Pointers documented "device" must be device memory of the graph's
 *    device; "host" pointers are ordinary host memory.  All caller buffers
 *    are caller-owned; the library never frees them.  Handles are
 *    library-owned and released with cbfs_graph_destroy.
 *  - Vertex ids at the API are ORIGINAL ids (R18); an internal degree
 *    relabelling (CBFS_RELABEL_DEGREE) is invisible to callers.
 *  - Bit j of a bit-subset is the j-th source of the cluster's source list,
 *    LSB first (R11); k <= 64 so a bit-subset is one uint64_t.
 *  - Traversals use a per-device cached workspace (several batch slots, each
 *    with its own CUDA stream); calls that traverse on the same device are
 *    serialised by a lock.  The calls order their work after the caller's
 *    prior work on `stream` and make `stream` wait for all of it.
 */
#ifndef CBFS_H
#define CBFS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct cbfs_graph cbfs_graph;
typedef struct cbfs_labels cbfs_labels; /* opaque, device-resident landmark label store */
typedef void* cbfs_stream; /* cudaStream_t */

enum cbfs_status {
  CBFS_OK = 0,
  CBFS_EINVAL = -1,        /* bad argument                                  */
  CBFS_ENOMEM = -2,        /* device allocation failed                      */
  CBFS_ECUDA = -3,         /* CUDA error (message in cbfs_last_error)       */
  CBFS_EOVERFLOW = -4,     /* a finite distance does not fit dist_bytes     */
  CBFS_EUNSUPPORTED = -5   /* k > 64, d > CBFS_MAX_D, n > CBFS_MAX_N ...    */
};

#define CBFS_MAX_K 64u
#define CBFS_WIDE_MAX_W 8u  /* cbfs_run_wide: up to 8 words = 512 sources per cluster */
#define CBFS_MAX_D 31u
#define CBFS_MAX_N ((1u << 26) - 1)    /* (vertex, cluster-in-batch) pairs pack into 32 bits below the
                                          all-ones empty-slot sentinel */
#define CBFS_PAD 0xFFFFFFFFu           /* source-list padding                */
#define CBFS_UNREACHED_U16 0xFFFFu     /* Delta sentinel, dist_bytes == 2    */
#define CBFS_UNREACHED_U8 0xFFu        /* Delta sentinel, dist_bytes == 1    */
#define CBFS_QUERY_UNREACHED 0x7FFFFFFF /* query answer when no cluster reaches both ends */
#define CBFS_BIDIR_MAX_TAU 1024u        /* vertices visited per side by cbfs_query_bidir */

/* graph flags */
enum { CBFS_RELABEL_DEGREE = 2, CBFS_INPUT_DEVICE = 4, CBFS_RELABEL_LOCALITY = 8 };
/* cluster root policies (R12) */
enum { CBFS_ROOT_DEGREE = 0, CBFS_ROOT_RANDOM = 1 };
/* EdgeMap direction policy (R8: parity-neutral) */
enum { CBFS_DIR_AUTO = 0, CBFS_DIR_PUSH = 1, CBFS_DIR_PULL = 2 };
/* traversal engines (cbfs_set_engine; identical outputs, R8/R25) */
enum { CBFS_ENGINE_AUTO = 0, CBFS_ENGINE_BATCHED = 1, CBFS_ENGINE_SPARSE = 2 };

/* --------------------------------------------------------------- graph
 * cbfs_graph_create — build the device CSR of an UNDIRECTED graph from an
 * edge list (R17): every pair {src[e], dst[e]} with src != dst
 * becomes arcs in both directions, self loops are dropped, duplicates
 * removed, neighbour lists sorted.  n vertices, ids in [0, n).
 *   src, dst : [n_pairs] uint32 — host, or device if flags & CBFS_INPUT_DEVICE
 *   flags    : CBFS_RELABEL_DEGREE (internal degree-descending order,
 *              ties by id: hubs packed, for power-law graphs) or
 *              CBFS_RELABEL_LOCALITY (internal BFS order from the highest-
 *              degree vertex, each level sorted by its first parent's
 *              position then id, other components appended by id: graph
 *              neighbours get nearby ids, for meshes / k-NN graphs; DEGREE
 *              wins if both are set) | CBFS_INPUT_DEVICE
 *   device   : CUDA ordinal; the handle lives there.
 * Errors: EINVAL (null out, id >= n), EUNSUPPORTED (n > CBFS_MAX_N or more
 * than 2^32-1 arcs), ENOMEM, ECUDA.  Synchronises. */
int cbfs_graph_create(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t n_pairs, uint32_t flags,
                      int device, cbfs_stream stream, cbfs_graph** out);

/* Same, from a CSR whose arcs are read as undirected pairs (offsets [n+1]
 * uint64, cols [m] uint32); the result is the normalised symmetric CSR. */
int cbfs_graph_create_csr(uint32_t n, const uint64_t* offsets, const uint32_t* cols, uint64_t m, uint32_t flags,
                          int device, cbfs_stream stream, cbfs_graph** out);

/* n, number of arcs m (directed CSR entries, R17), max degree (host outs, any may be NULL). */
int cbfs_graph_info(const cbfs_graph* g, uint32_t* n, uint64_t* m, uint32_t* max_degree);

/* Copy the normalised CSR in ORIGINAL-id order to host buffers
 * offsets [n+1] uint64, cols [m] uint32. Synchronises. */
int cbfs_graph_export_csr(const cbfs_graph* g, uint64_t* offsets, uint32_t* cols);

/* Copy the internal vertex order to a host buffer: out_perm[x] = the original
 * id of internal vertex x ([n] uint32; the identity without relabelling).
 * Inspection only — every output of the library is in original ids.
 * Synchronises.  Errors: EINVAL (null argument). */
int cbfs_graph_internal_order(const cbfs_graph* g, uint32_t* out_perm);

int cbfs_graph_destroy(cbfs_graph* g);

/* --------------------------------------------------------------- selection
 * cbfs_select_clusters — "Selecting Landmarks in Clusters" (R12):
 * repeat r times: root = best unmarked non-isolated vertex (policy DEGREE:
 * highest degree, ties by smaller id; policy RANDOM: draw
 * v_t = floor(rand(seed,1,t) * n / 2^64), t = 0,1,..., until unmarked and
 * non-isolated), members = up to k-1 unmarked vertices within floor(d/2) hops
 * (marked vertices may be passed through), best (degree desc, id asc) first;
 * mark them all.  Stops early when nothing unmarked and non-isolated is left.
 *   out_sources : device [r][64] uint32, row = [root, members...], padded
 *                 with CBFS_PAD
 *   out_sizes   : device [r] uint8 (cluster size k_c)
 *   out_r       : host, number of clusters produced (<= r)
 * Errors: EINVAL (k == 0, null outputs), EUNSUPPORTED (k > 64, d > MAX_D).
 * rand() is the counter-based SplitMix64 of include/cbfs_gen.h, implemented
 * independently in this library.  Synchronises. */
int cbfs_select_clusters(const cbfs_graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                         uint64_t seed, uint32_t* out_sources, uint8_t* out_sizes, uint32_t* out_r,
                         cbfs_stream stream);

/* cbfs_select_clusters_wide — the same rule for clusters of up to
 * k <= 64 * words sources (general k; input of cbfs_run_wide):
 *   out_sources : device [r][64 * words] uint32 (padding 0xFFFFFFFF)
 *   out_sizes   : device [r] uint16
 *   words       : 1, 2, 4 or 8
 * Errors: EINVAL (k == 0 or k > 64 * words, null outputs), EUNSUPPORTED
 * (words, d > MAX_D).  Synchronises. */
int cbfs_select_clusters_wide(const cbfs_graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                              uint64_t seed, uint32_t words, uint32_t* out_sources, uint16_t* out_sizes,
                              uint32_t* out_r, cbfs_stream stream);

/* --------------------------------------------------------------- C-BFS
 * cbfs_run — Cluster-BFS (Alg. 1, with R1 seeding, R3 cap, R4
 * claim, R5 output) from each of `n_clusters` clusters, d = the cluster
 * diameter bound.  For every cluster c and vertex v it produces the cluster
 * distance vector <S_v[0..d], Delta_v>.  A cluster whose true
 * diameter exceeds d is not an error (R9): the output is Alg. 1's, exactly.
 *   sources   : device [n_clusters][64] uint32 original ids, row c holds
 *               sizes[c] distinct ids then padding (ignored)
 *   sizes     : device [n_clusters] uint8, 1..64
 *   d         : 0..CBFS_MAX_D
 *   dist_bytes: 1 or 2 — width of out_dist entries (sentinel 0xFF / 0xFFFF)
 *   out_dist  : device [n][n_clusters] (row = original vertex id), Delta_v,
 *               or NULL
 *   out_masks : device [planes][n][n_clusters] uint64, S_v[i] for
 *               i < planes, or NULL
 *   planes    : d+1 (full vectors) or d (landmark-label records, R14: the
 *               last subset is implied, S_v[d] = S \ U_{i<d} S_v[i])
 *   out_stats : device [n_clusters][4] uint64 {rounds, sum_i |F_i|,
 *               sum_i E_i (E_i = sum of frontier degrees), sum of degrees of
 *               reached vertices}, or NULL
 *   direction : CBFS_DIR_AUTO / PUSH / PULL (identical outputs, R8)
 * Errors: EINVAL (k == 0, duplicate or out-of-range source, bad dist_bytes /
 * planes), EUNSUPPORTED (k > 64, d > MAX_D), EOVERFLOW (dist_bytes == 1 and a
 * Delta > 254), ENOMEM, ECUDA.  Synchronises at the end (and once per batch,
 * after its seeding, for the argument check). */
int cbfs_run(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
             uint32_t dist_bytes, void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
             uint32_t direction, cbfs_stream stream);

/* cbfs_run_digest — cbfs_run whose full outputs are consumed inside the
 * call: every batch of 64 clusters writes its cluster distance vectors
 * <Delta_v, S_v[0..planes-1]> (the same fold and the same layout
 * as cbfs_run's out_dist / out_masks, 64 columns) into a library-owned
 * staging store in HBM, and when the batch's last round has been queued a
 * kernel on the batch's stream reads the store back, reduces each cluster
 * to cbfs_digest_store's digest and resets the store for the next batch.
 * For configurations whose whole output does not fit HBM (n * C * (dist_bytes
 * + 8 planes) bytes) this is the full-output run; the digests are compared
 * with the oracle's (tests/golden).  As many batches run concurrently as
 * there are workspace slots with room for a staging store next to them
 * (n * 64 * (dist_bytes + 8 planes) bytes each).
 *   out_digest: device [n_clusters] uint64 (overwritten)
 *   out_stats : as cbfs_run, or NULL
 *   other arguments as cbfs_run.
 * Errors: as cbfs_run; ENOMEM when not even one staging store fits. */
int cbfs_run_digest(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                    uint32_t dist_bytes, uint32_t planes, uint64_t* out_digest, uint64_t* out_stats,
                    uint32_t direction, cbfs_stream stream);

/* cbfs_digest_store — 64-bit digest of every column c of a vertex-major
 * store (cbfs_run's output layout) dist [n][C] (dist_bytes 1 or 2, 0xFF /
 * 0xFFFF = unreached), masks [planes][n][C] uint64 (NULL if planes == 0),
 * all device:
 *   fin(z)  = SplitMix64 finaliser: z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
 *             z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31
 *   x_v     = fin((v * 0x9E3779B97F4A7C15 + 0xD1B54A32D192ED03) ^ (D_v << 48)),
 *             D_v = Delta_v as a 16-bit value (0xFFFF unreached, also for
 *             dist_bytes == 1); then x_v = fin(x_v ^ S_v[i]) for i = 0 ..
 *             planes-1
 *   digest  = sum over v = 0 .. n-1 of x_v, mod 2^64
 * (an order-independent sum, so it is formed in parallel).  Used to compare
 * whole outputs with the oracle (which implements the same definition
 * independently, oracle.c or_digest_cluster); not part of the method.
 *   out_digest: device [C] uint64 (overwritten).  Synchronises.
 * Errors: EINVAL (dist_bytes, planes > CBFS_MAX_D + 1, null pointers). */
int cbfs_digest_store(uint32_t n, uint32_t C, uint32_t planes, const void* dist, uint32_t dist_bytes,
                      const uint64_t* masks, uint64_t* out_digest, cbfs_stream stream);

/* cbfs_run_rounds — cbfs_run recording the frontier of every round: for
 * cluster c and round i < max_rounds, out_rounds[c][i] = {|F_i|, E_i} (the
 * frontier size and its degree sum; the per-round invariants of
 * a vertex appears in at most d+1 frontiers, and
 * the rounds executed are 1 + the largest source distance).  Rounds
 * past the cluster's last are 0.  No distance outputs.
 *   out_rounds: device [n_clusters][max_rounds][2] uint64 (overwritten)
 *   max_rounds: >= 1; rounds beyond it are counted in out_stats only
 *   out_stats, direction, stream: as cbfs_run.
 * Errors: as cbfs_run; EINVAL for a null out_rounds or max_rounds == 0. */
int cbfs_run_rounds(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                    uint64_t* out_rounds, uint32_t max_rounds, uint64_t* out_stats, uint32_t direction,
                    cbfs_stream stream);

/* cbfs_run_wide — C-BFS from clusters of more than 64 sources (k > w, the
 * paper's general k: P:448): each
 * bit-subset is `words` 64-bit words (bit j of the cluster = bit j % 64 of
 * word j / 64, R11).  Reading R28: the cluster's 64-source words are
 * traversed as sub-clusters in lanes of one batch, in lockstep rounds, and
 * the fold places each word's subsets relative to the cluster's Delta_v
 * (the least first-visit round over its words).  For a cluster of diameter
 * <= d this is the cluster distance vector, exactly; for d <
 * diameter the output is not specified (unlike cbfs_run's R9).
 *   sources   : device [n_clusters][64 * words] uint32 original ids, row c
 *               holds sizes[c] distinct ids then padding
 *   sizes     : device [n_clusters] uint16, 1..64 * words
 *   words     : 1, 2, 4 or 8 (CBFS_WIDE_MAX_W)
 *   out_dist  : device [n][n_clusters], Delta_v, or NULL
 *   out_masks : device [planes][n][n_clusters * words] uint64; word w of
 *               cluster c in column c * words + w; or NULL
 *   out_stats : device [n_clusters * words][4], the statistics of each
 *               64-source word (as cbfs_run's per cluster), or NULL
 *   other arguments as cbfs_run (either engine: both advance the lanes of a
 *   batch in lockstep rounds, which the Delta merge relies on).
 * Errors: EINVAL (size 0 or > 64 * words, duplicate or out-of-range source),
 * EUNSUPPORTED (words not 1/2/4/8, d > MAX_D), EOVERFLOW, ENOMEM, ECUDA. */
int cbfs_run_wide(cbfs_graph* g, const uint32_t* sources, const uint16_t* sizes, uint32_t n_clusters, uint32_t words,
                  uint32_t d, uint32_t dist_bytes, void* out_dist, uint64_t* out_masks, uint32_t planes,
                  uint64_t* out_stats, uint32_t direction, cbfs_stream stream);

/* cbfs_select_and_run — cbfs_select_clusters followed by cbfs_run over the
 * selected clusters, overlapped: the (sequential) selection runs on a side
 * stream and publishes each cluster as it is fixed, and each batch of 64
 * clusters is traversed as soon as its clusters exist.  Same arguments and
 * outputs as the two calls (out_sources / out_sizes device [r][64] / [r];
 * outputs use row stride C = r; columns >= *out_r stay unreached).
 * Synchronises. */
int cbfs_select_and_run(cbfs_graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy, uint64_t seed,
                        uint32_t* out_sources, uint8_t* out_sizes, uint32_t* out_r, uint32_t dist_bytes,
                        void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
                        uint32_t direction, cbfs_stream stream);

/* cbfs_select_and_run_shard — the same for rank `rank` of `world` ranks
 * (cluster c belongs to rank c mod world): every rank runs the
 * whole (deterministic, sequential) selection of r clusters on a side stream
 * into out_sources / out_sizes ([r][64] / [r], device) and traverses its own
 * clusters c = rank, rank + world, ... as soon as each batch of 64 of them
 * exists.  Outputs use this rank's columns: C_rank = ceil((r - rank) /
 * world), out_dist [n][C_rank], out_masks [planes][n][C_rank], out_stats
 * [C_rank][4], column j = global cluster rank + j * world.  world = 1 is
 * cbfs_select_and_run.  Errors: EINVAL (rank >= world) and as above. */
int cbfs_select_and_run_shard(cbfs_graph* g, uint32_t r, uint32_t k, uint32_t d, uint32_t root_policy,
                              uint64_t seed, uint32_t world, uint32_t rank, uint32_t* out_sources,
                              uint8_t* out_sizes, uint32_t* out_r, uint32_t dist_bytes, void* out_dist,
                              uint64_t* out_masks, uint32_t planes, uint64_t* out_stats, uint32_t direction,
                              cbfs_stream stream);

/* Same computation with HOST buffers (sources, sizes, out_dist, out_masks,
 * out_stats all host memory, pinned recommended): inputs are copied in; when
 * the whole output fits in free device memory it is built there and copied
 * out with one DMA per array, otherwise each batch of 64 clusters is
 * traversed into device staging and copied out while the next batch runs.
 * Used for the end-to-end measurement. */
int cbfs_run_host(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                  uint32_t dist_bytes, void* out_dist, uint64_t* out_masks, uint32_t planes, uint64_t* out_stats,
                  uint32_t direction, cbfs_stream stream);

/* cbfs_decode — distances of every source of ONE cluster:
 * delta(s_j, v) = Delta_v + i for the unique i with bit j in S_v[i]
 * (S_v[d] reconstructed when planes == d), CBFS_UNREACHED_U16 otherwise.
 *   dist, masks : device, the cbfs_run output layout ([n][C], [planes][n][C])
 *   c           : cluster column, k = sizes_host value for that cluster
 *   out         : device [k][n] uint16
 * Errors: EINVAL. */
int cbfs_decode(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                const uint64_t* masks, uint32_t c, uint32_t k, uint16_t* out, cbfs_stream stream);

/* cbfs_decode_wide / cbfs_query_distance_wide — cbfs_decode and
 * cbfs_query_distance over the cbfs_run_wide layout (dist [n][C], masks
 * [planes][n][C * words], sizes device [C] uint16; k <= 64 * words).
 * Same semantics, arguments and errors otherwise. */
int cbfs_decode_wide(uint32_t n, uint32_t C, uint32_t words, uint32_t d, uint32_t planes, const void* dist,
                     uint32_t dist_bytes, const uint64_t* masks, uint32_t c, uint32_t k, uint16_t* out,
                     cbfs_stream stream);
int cbfs_query_distance_wide(uint32_t n, uint32_t C, uint32_t words, uint32_t d, uint32_t planes, const void* dist,
                             uint32_t dist_bytes, const uint64_t* masks, const uint16_t* sizes, const uint32_t* s,
                             const uint32_t* t, uint64_t q, int32_t* inout_best, cbfs_stream stream);

/* --------------------------------------------------------------- queries
 * cbfs_query_distance — landmark query with clustered landmarks
 * (R15, R16): for each pair (s[q], t[q]),
 *   best = min over clusters c with both Delta finite of
 *          Delta_s + Delta_t + min{ i+j : S_s[i] & S_t[j] != 0 },
 * min-merged into inout_best[q] (initialise to CBFS_QUERY_UNREACHED).
 *   n, C, d, planes, dist, dist_bytes, masks : a label store in the
 *         cbfs_run layout (planes = d or d+1; planes = d = 0 with a null
 *         masks is a plain landmark store of single-source clusters)
 *   sizes : device [C] uint8 (needed for S_v[d] = FULL & ~U when planes == d)
 *   s, t  : device [q] uint32 original ids;  inout_best : device [q] int32
 * Errors: EINVAL (null pointers, planes not d or d+1).  Ids >= n: the
 * answer for that pair is left unchanged and the call returns EINVAL. */
int cbfs_query_distance(uint32_t n, uint32_t C, uint32_t d, uint32_t planes, const void* dist, uint32_t dist_bytes,
                        const uint64_t* masks, const uint8_t* sizes, const uint32_t* s, const uint32_t* t,
                        uint64_t q, int32_t* inout_best, cbfs_stream stream);

/* cbfs_query_stream — build the landmark labels of `n_clusters` clusters
 * batch by batch and answer the q queries against each batch as soon as it
 * is built, min-merging into inout_best; the full label store is never
 * resident (config 5).  Same semantics as cbfs_run (planes = d+1 internally)
 * followed by cbfs_query_distance over all clusters. */
int cbfs_query_stream(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                      const uint32_t* s, const uint32_t* t, uint64_t q, int32_t* inout_best, uint64_t* out_stats,
                      cbfs_stream stream);

/* --------------------------------------------------------------- label store handles
 * cbfs_labels_build — the landmark labels of n_clusters clusters (A10,
 * P:1001-1012 and P:1438-1447): one cbfs_run with planes = d (records Delta +
 * S_v[0..d-1], R14; d = 0 keeps S_v[0]) into a library-owned device image.
 *   sources, sizes : as cbfs_run (device);  dist_bytes : 1 or 2
 * Errors: as cbfs_run, ENOMEM.  Synchronises.
 * cbfs_labels_build_w — the same with the store's word size w = word_bits
 *   (8, 16, 32 or 64; the paper's w, P:1447 and Tables 4/8 at P:1379-1414 and
 *   P:1821-1848): each bit-subset is stored in w bits, so a record is
 *   dist_bytes + d * w / 8 bytes (3 B at w = 8, d = 2, u8 Delta; 17 B at
 *   w = 64).  Every cluster must have <= w sources (EINVAL otherwise; sizes
 *   are read back to the host for that check).  word_bits = 0 is the
 *   paper's plain landmark labeling: d = 0 and single-source
 *   clusters (EINVAL otherwise), records are Delta alone.  cbfs_labels_build
 *   is w = 64.
 * cbfs_labels_word_bits — the store's w.
 * cbfs_labels_info — n, clusters, d, dist_bytes and the image size in bytes.
 * cbfs_labels_export — copy the flat image (64-byte header, sizes, Delta
 *   rows, subset planes) to buf (device or host, >= image bytes): the unit
 *   an NCCL all-gather moves between ranks (A12).  EINVAL if buf is small.
 * cbfs_labels_import — a new handle on g's device from an exported image
 *   (device or host); EINVAL if the header is not a label image of a graph
 *   with g's n.
 * cbfs_labels_query — cbfs_query_distance over the store (min-merged into
 *   inout_best, device [q] int32; s, t device [q] uint32 original ids).
 * cbfs_labels_destroy — free the handle. */
int cbfs_labels_build(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                      uint32_t dist_bytes, cbfs_labels** out, cbfs_stream stream);
int cbfs_labels_build_w(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters,
                        uint32_t d, uint32_t dist_bytes, uint32_t word_bits, cbfs_labels** out, cbfs_stream stream);
int cbfs_labels_word_bits(const cbfs_labels* l, uint32_t* word_bits);
int cbfs_labels_info(const cbfs_labels* l, uint32_t* n, uint32_t* n_clusters, uint32_t* d, uint32_t* dist_bytes,
                     uint64_t* image_bytes);
int cbfs_labels_export(const cbfs_labels* l, void* buf, uint64_t bytes);
int cbfs_labels_import(cbfs_graph* g, const void* buf, uint64_t bytes, cbfs_labels** out);
int cbfs_labels_query(const cbfs_labels* l, const uint32_t* s, const uint32_t* t, uint64_t q, int32_t* inout_best,
                      cbfs_stream stream);
int cbfs_labels_destroy(cbfs_labels* l);

/* --------------------------------------------------------------- exact 2-hop oracle (PLL)
 * cbfs_pll_build — Pruned Landmark Labeling with a C-BFS first phase
 * (SURVEY §8(f) NEXT-4), reading R29:
 *   phase 1: the n_clusters given clusters (diameter <= d, as
 *     cbfs_run) are traversed by C-BFS; every vertex keeps its cluster
 *     distance vector (all d+1 subsets) as its cluster label;
 *   phase 2: every vertex not in a cluster, in (degree desc, original id
 *     asc) order, runs a BFS pruned by the index: at a vertex u at distance
 *     delta, if query(root, u) <= delta then u gets no label and is not
 *     expanded, else (root, delta) joins L(u).  Roots run in batches of
 *     first, floor(3/2 first), ... up to bmax (200 x 1.5^i up to
 *     1000); the roots of a batch run in parallel, each pruned against the
 *     index as it was when its batch started.
 *   sources, sizes : device [n_clusters][64] / [n_clusters] (cbfs_run layout)
 *   cap            : label entries per vertex (EOVERFLOW beyond; distances
 *                    above 254 are EOVERFLOW too)
 * The graph must outlive the index.  Errors: EINVAL, EUNSUPPORTED
 * (n_clusters * (8 (d+1) + 4) > 200 KB: a root's cluster labels live in
 * shared memory; n >= 2^24), EOVERFLOW, ENOMEM, ECUDA.  Synchronises.
 * cbfs_pll_info — phase-2 label count, largest list, roots, batches, and
 *   the device time of phase 1 (C-BFS) and phase 2 (pruned BFSs) in ms.
 * cbfs_pll_export — the phase-2 labels by original vertex id: counts
 *   device [n] uint32, entries device [n][cap] uint32 = hub position << 8 |
 *   distance (hub position in the degree order above), ascending, zero
 *   padded.  Either pointer may be NULL.
 * cbfs_pll_query — exact distances: out[i] = delta(s[i],
 *   t[i]) (int32 device [q], INT32_MAX = unreachable); s, t device [q]
 *   uint32 original ids; EINVAL on an id >= n.
 * cbfs_pll_destroy — free the index. */
typedef struct cbfs_pll cbfs_pll;
int cbfs_pll_build(cbfs_graph* g, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                   uint32_t first, uint32_t bmax, uint32_t cap, cbfs_pll** out, cbfs_stream stream);
int cbfs_pll_info(const cbfs_pll* p, uint64_t* total_labels, uint32_t* max_labels, uint32_t* roots,
                  uint32_t* batches, float* ms_cbfs, float* ms_pbfs);
int cbfs_pll_export(const cbfs_pll* p, uint32_t* counts, uint32_t* entries, cbfs_stream stream);
int cbfs_pll_query(const cbfs_pll* p, const uint32_t* s, const uint32_t* t, uint64_t q, int32_t* out,
                   cbfs_stream stream);
int cbfs_pll_destroy(cbfs_pll* p);

/* cbfs_query_bidir — the fixed-size bi-directional search of Appendix B
 * (P:1790-1800), reading R27: from each endpoint a BFS over the sorted
 * original-id CSR visits vertices in discovery order (the endpoint first)
 * until tau are visited; the answer is min over vertices visited by both
 * sides of dist_s + dist_t, min-merged into inout_best (so calling it after
 * cbfs_query_distance gives the combined query, "the minimum distance
 * obtained by the index and bi-directional search").  Disjoint visited sets
 * (or tau = 0) leave the answer unchanged.
 *   s, t : device [q] uint32 original ids; inout_best : device [q] int32
 *   tau  : 0..CBFS_BIDIR_MAX_TAU
 * Errors: EINVAL (null pointers, ids >= n: the call returns after the
 * kernel), EUNSUPPORTED (tau too large).  Synchronises. */
int cbfs_query_bidir(cbfs_graph* g, const uint32_t* s, const uint32_t* t, uint64_t q, uint32_t tau,
                     int32_t* inout_best, cbfs_stream stream);

/* --------------------------------------------------------------- misc */
/* Direction switch: pull when the frontier's (cluster, arc) pair count
 * exceeds batch_clusters * m / alpha (default 100; S:186 suggests 20 for a
 * single source; tunable, parity-neutral R8). */
int cbfs_set_direction_alpha(double alpha);
/* Traversal engine for later cbfs_run / cbfs_select_and_run / cbfs_run_host /
 * cbfs_query_stream calls (process-wide):
 *   CBFS_ENGINE_BATCHED — vertex-major state rows shared by the 64 clusters
 *     of a batch, host-driven rounds, push/pull switch (low-diameter graphs);
 *   CBFS_ENGINE_SPARSE  — cluster-major state, push-only rounds, the round
 *     loop on the device (CUDA-graph while node) (high-diameter graphs);
 *   CBFS_ENGINE_AUTO (default) — BATCHED when some vertex has degree > 256
 *     (hubs: low diameter); otherwise SPARSE when a BFS from the
 *     highest-degree vertex is still running after 48 levels, else BATCHED
 *     (cached per graph).
 * direction == CBFS_DIR_PULL always uses BATCHED.  Outputs are identical.
 * Errors: EINVAL (unknown engine). */
int cbfs_set_engine(int engine);
/* Dense-pull tuning (batched engine; outputs never change): the S_seen rows
 * of the `rows` lowest internal ids (the hubs under CBFS_RELABEL_DEGREE) are
 * gathered with an L2 evict_last hint, every other row and the CSR columns
 * with evict_first.  Default 131,072 rows (64 MiB of 512-byte rows). */
int cbfs_set_pull_hub_rows(uint32_t rows);
/* Sparse-engine frontier order (outputs never change): a round whose
 * frontier F_i holds >= min_entries entries records its claims in a
 * cluster-major bitmap that is compacted into F_{i+1} in (cluster, vertex)
 * order, so the next round's pushes read neighbour cells in id order; smaller
 * rounds append claims to the list in claim order.  min_entries = -1
 * (default): max(n / 4, 65,536) on graphs of average degree >= 8, never on
 * sparser ones (the grid's thousands of small rounds do not repay the
 * compaction); 0: never; k > 0: from k entries on, every graph.  Takes effect
 * at the next batch.  Errors: EINVAL (min_entries < -1). */
int cbfs_set_sparse_order(int64_t min_entries);

/* Free the device's cached traversal workspace (the batch slots; the next
 * traversal re-allocates them).  Errors: EINVAL (device out of range). */
int cbfs_release_workspace(int device);

/* Index budget arithmetic: bytes of one (cluster,
 * vertex) label record — Delta (dist_bytes: 1 as the paper counts, or 2) plus
 * d bit-subsets of word_bits bits (S_v[0..d-1], R14; d = 0 keeps S_v[0];
 * word_bits = 0: a plain landmark, Delta alone) — and the number
 * of clusters whose records fit t_bytes per vertex (t = 1,024, w = 64,
 * d = 2 -> 17 B, 60 clusters).  Host outputs.
 * Errors: EINVAL (word_bits not 0/8/16/32/64, dist_bytes, null out),
 * EUNSUPPORTED (d > CBFS_MAX_D). */
int cbfs_record_bytes(uint32_t word_bits, uint32_t d, uint32_t dist_bytes, uint64_t* out_bytes);
int cbfs_budget_clusters(uint64_t t_bytes, uint32_t word_bits, uint32_t d, uint32_t dist_bytes, uint64_t* out_r);

/* Kernel-level timing of the C-BFS engine (process-wide, not thread-safe):
 * when enabled, the batched engine's fold / push / pull kernels time every
 * launch on the device (%globaltimer from the first block to start to the
 * last to finish, inside the round-loop graph), the sparse engine's round
 * loop and the digest consumer are timed with CUDA events on their streams.
 * cbfs_profile_read fills arrays of 5 entries indexed {0 fold, 1 push,
 * 2 pull, 3 sparse-engine round loop (one graph launch per batch; its
 * "launches" count the kernels the loop ran), 4 output consumer of
 * cbfs_run_digest (per batch; the call synchronises the batch's stream
 * after it while profiling)}: total device ms, launches, frontier (cluster, arc) pairs,
 * frontier (vertex, cluster) entries, distinct frontier vertices |U_i| and
 * distinct vertices claimed for the next frontier |U_{i+1}| summed over the
 * launches (host pointers, any may be NULL). */
int cbfs_profile_enable(int on);
int cbfs_profile_read(double* ms, uint64_t* launches, uint64_t* arcs, uint64_t* entries, uint64_t* u_in,
                      uint64_t* u_out, int reset);
/* Number of vertices with at least one arc. */
int cbfs_graph_nonisolated(const cbfs_graph* g, uint32_t* count);
/* Maximum number of 64-cluster batches traversed concurrently (each with its
 * own workspace and stream; fewer if device memory is short).  1..8, default
 * 4.  Errors: EINVAL. */
int cbfs_set_concurrency(int batches);
/* Number of kernels this library launched on this thread since the last reset. */
uint64_t cbfs_launch_count(int reset);
const char* cbfs_last_error(void);
const char* cbfs_version(void);

#ifdef __cplusplus
}
#endif
#endif
