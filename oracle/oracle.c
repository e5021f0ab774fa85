/*
 * oracle.c — plain, slow, sequential CPU oracle for the C-BFS hot path.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke()
 *   and bench.py's cpu_baseline / --impl reference leg may load this file's
 *   library.  It shares no code, header, table or constant with the CUDA
 *   product (paper_2410_17226_b200/); the only common module is the input
 *   generator library cbfs_inputs/ (random numbers, no method arithmetic).
 *
 * Every function cites the PAPER.md passage (P:line) it follows; readings of
 * ambiguous passages are SURVEY.md §8(c) R1..R26, restated in DESIGN.md §2.
 * Graphs are CSR with 64-bit offsets, symmetric, sorted, deduplicated, no
 * self loops (built by oracle/__init__.py: csr_from_edges).
 *
 * Pins (tests/test_oracle_*.py, `-m "not gpu"`): scipy BFS distances encoded
 * by the definition, closed forms (path, cycle, star, complete,
 * intact grid), paper-printed budget numbers, the
 * Fig. 2 values, invariants.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_INF16 0xFFFFu
#define OR_INF32 0xFFFFFFFFu

/* ---------------------------------------------------------------------
 * plain_bfs — textbook queue BFS from one source (Alg. simpleBFS P:1708-1732,
 * run sequentially).  dist[v] = hop distance, OR_INF32 if unreachable.
 * ------------------------------------------------------------------- */
int or_plain_bfs(uint32_t n, const uint64_t* off, const uint32_t* cols, uint32_t s, uint32_t* dist) {
  if (s >= n) return -1;
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) dist[v] = OR_INF32;
  uint64_t head = 0, tail = 0;
  dist[s] = 0; q[tail++] = s;
  while (head < tail) {
    uint32_t u = q[head++];
    for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
      uint32_t v = cols[e];
      if (dist[v] == OR_INF32) { dist[v] = dist[u] + 1; q[tail++] = v; }
    }
  }
  free(q);
  return 0;
}

static int check_sources(uint32_t n, const uint32_t* S, uint32_t k) {
  if (k == 0 || k > 64) return -1;
  for (uint32_t j = 0; j < k; ++j) {
    if (S[j] >= n) return -1;
    for (uint32_t t = 0; t < j; ++t) if (S[t] == S[j]) return -1; /* R2: duplicates rejected */
  }
  return 0;
}

/* ---------------------------------------------------------------------
 * brute_cluster — the DEFINITION of the cluster distance vector
 * (P:630-639): k independent BFS runs, then
 *   Delta_v = min_j delta(s_j, v),  S_v[i] = { j : delta(s_j,v) = Delta_v + i }.
 * Sources whose offset exceeds d are not representable (cluster diameter > d,
 * Corollary 1 P:620-624 violated); the function then returns 1.
 * ------------------------------------------------------------------- */
int or_brute_cluster(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* S, uint32_t k,
                     uint32_t d, uint16_t* out_dist, uint64_t* out_sub) {
  if (check_sources(n, S, k)) return -1;
  uint32_t* dist = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n * k);
  for (uint32_t j = 0; j < k; ++j) or_plain_bfs(n, off, cols, S[j], dist + (size_t)j * n);
  int over = 0;
  memset(out_sub, 0, sizeof(uint64_t) * (size_t)(d + 1) * n);
  for (uint32_t v = 0; v < n; ++v) {
    uint32_t mn = OR_INF32;
    for (uint32_t j = 0; j < k; ++j) if (dist[(size_t)j * n + v] < mn) mn = dist[(size_t)j * n + v];
    out_dist[v] = (mn == OR_INF32) ? (uint16_t)OR_INF16 : (uint16_t)mn;
    if (mn == OR_INF32) continue;
    for (uint32_t j = 0; j < k; ++j) {
      uint32_t dj = dist[(size_t)j * n + v];
      if (dj == OR_INF32) continue;
      uint32_t i = dj - mn;
      if (i > d) { over = 1; continue; }
      out_sub[(size_t)i * n + v] |= 1ULL << j;
    }
  }
  free(dist);
  return over;
}

/* ---------------------------------------------------------------------
 * cluster_bfs — Alg. 1 "Cluster-BFS search from S", sequential,
 * step by step in the paper's order and notation:
 *   init with R1: S_next[s_j] = {s_j} (bit j), S_seen = {}, so the
 *        round-0 fold yields Delta_s = 0 and S_s[0] = {s};
 *   while F_i != {}:
 *     vertex phase: S_new = S_next[u] \ S_seen[u];
 *        if Delta_u = inf: Delta_u = i;  S_u[i - Delta_u] = S_new;
 *        S_seen[u] = S_seen[u] u S_new;
 *     edge phase: for v in N(u) with i - Delta_v < d (R3: an
 *        infinite Delta_v passes): Fetch_And_Or(S_next[v], S_seen[u]); if it
 *        set a bit, the first claim of r[v] for round i (R4) puts v in F_{i+1};
 *     i = i + 1
 *   return <S_v[0..d], Delta_v> (R5).
 * Outputs: out_dist[n] (OR_INF16 = unreachable), out_sub[(d+1)][n].
 * stats (optional) = {rounds, sum_i |F_i|, sum_i E_i, sum_{reached v} deg(v)}
 * where E_i = sum_{u in F_i} deg(u).  round_F/round_E (optional, length
 * max_rounds) receive |F_i| and E_i.
 * ------------------------------------------------------------------- */
int or_cluster_bfs(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* S, uint32_t k,
                   uint32_t d, uint16_t* out_dist, uint64_t* out_sub, uint64_t* stats, uint32_t* round_F,
                   uint64_t* round_E, uint32_t max_rounds) {
  if (check_sources(n, S, k)) return -1;
  uint64_t* seen = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  uint64_t* next = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  uint32_t* r = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* F = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* Fn = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  /* Initialization */
  for (uint32_t v = 0; v < n; ++v) { out_dist[v] = (uint16_t)OR_INF16; r[v] = OR_INF32; }
  memset(out_sub, 0, sizeof(uint64_t) * (size_t)(d + 1) * n);
  uint64_t nF = 0;
  for (uint32_t j = 0; j < k; ++j) { next[S[j]] = 1ULL << j; F[nF++] = S[j]; } /* R1, F_0 = S */
  uint64_t rounds = 0, sumF = 0, sumE = 0, mreach = 0;
  uint32_t i = 0;
  while (nF > 0) {
    /* vertex phase */
    uint64_t Ei = 0;
    for (uint64_t t = 0; t < nF; ++t) {
      uint32_t u = F[t];
      uint64_t Snew = next[u] & ~seen[u];
      if (out_dist[u] == OR_INF16) { out_dist[u] = (uint16_t)i; mreach += off[u + 1] - off[u]; }
      out_sub[(size_t)(i - out_dist[u]) * n + u] = Snew;
      seen[u] = seen[u] | Snew;
      Ei += off[u + 1] - off[u];
    }
    if (round_F && rounds < max_rounds) { round_F[rounds] = (uint32_t)nF; round_E[rounds] = Ei; }
    rounds++; sumF += nF; sumE += Ei;
    /* edge phase */
    uint64_t nFn = 0;
    for (uint64_t t = 0; t < nF; ++t) {
      uint32_t u = F[t];
      for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
        uint32_t v = cols[e];
        if (!(out_dist[v] == OR_INF16 || (int64_t)i - (int64_t)out_dist[v] < (int64_t)d)) continue; /* P:722, R3 */
        uint64_t old = next[v];
        next[v] = old | seen[u];                  /* Fetch_And_Or */
        if (next[v] != old) {
          if (r[v] != i) { r[v] = i; Fn[nFn++] = v; } /* claim r[v] (R4) */
        }
      }
    }
    uint32_t* tmp = F; F = Fn; Fn = tmp; nF = nFn;
    i = i + 1;
    if (i >= OR_INF16 - 1) break; /* Delta must stay below the sentinel */
  }
  if (stats) { stats[0] = rounds; stats[1] = sumF; stats[2] = sumE; stats[3] = mreach; }
  free(seen); free(next); free(r); free(F); free(Fn);
  return 0;
}

/* ---------------------------------------------------------------------
 * Many clusters, one sequential Alg. 1 per cluster, clusters spread over
 * host threads (each cluster is still the sequential function above).
 * sources [C][64] (pad ignored), sizes [C].  Outputs cluster-major:
 * out_dist [C][n], out_sub [C][d+1][n] (either may be NULL to skip),
 * stats [C][4].  out_hash [C] (may be NULL) = or_hash_cluster of each output.
 * ------------------------------------------------------------------- */
uint64_t or_hash_cluster(uint32_t n, uint32_t d, const uint16_t* dist, const uint64_t* sub);
uint64_t or_digest_cluster(uint32_t n, uint32_t planes, const uint16_t* dist, const uint64_t* sub);

typedef struct {
  uint32_t n; const uint64_t* off; const uint32_t* cols; const uint32_t* sources; const uint8_t* sizes;
  uint32_t C, d; uint16_t* out_dist; uint64_t* out_sub; uint64_t* stats; uint64_t* hash;
  int* status; uint32_t next_c; pthread_mutex_t* mu;
  uint64_t* digest; uint32_t* round_F; uint64_t* round_E; uint32_t max_rounds;
} many_job;

static void* many_worker(void* p) {
  many_job* J = (many_job*)p;
  uint16_t* dist = (uint16_t*)malloc(sizeof(uint16_t) * (J->n ? J->n : 1));
  uint64_t* sub = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(J->d + 1) * (J->n ? J->n : 1));
  for (;;) {
    pthread_mutex_lock(J->mu);
    uint32_t c = J->next_c++;
    pthread_mutex_unlock(J->mu);
    if (c >= J->C) break;
    uint64_t st[4];
    int rc = or_cluster_bfs(J->n, J->off, J->cols, J->sources + (size_t)c * 64, J->sizes[c], J->d, dist, sub, st,
                            J->round_F ? J->round_F + (size_t)c * J->max_rounds : NULL,
                            J->round_E ? J->round_E + (size_t)c * J->max_rounds : NULL,
                            J->round_F ? J->max_rounds : 0);
    J->status[c] = rc;
    if (rc) continue;
    if (J->stats) memcpy(J->stats + 4 * (size_t)c, st, sizeof st);
    if (J->out_dist) memcpy(J->out_dist + (size_t)c * J->n, dist, sizeof(uint16_t) * J->n);
    if (J->out_sub) memcpy(J->out_sub + (size_t)c * (J->d + 1) * J->n, sub, sizeof(uint64_t) * (size_t)(J->d + 1) * J->n);
    if (J->hash) J->hash[c] = or_hash_cluster(J->n, J->d, dist, sub);
    if (J->digest) J->digest[c] = or_digest_cluster(J->n, J->d + 1, dist, sub);
  }
  free(dist); free(sub);
  return NULL;
}

int or_cluster_bfs_many_ex(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* sources,
                           const uint8_t* sizes, uint32_t C, uint32_t d, int threads, uint16_t* out_dist,
                           uint64_t* out_sub, uint64_t* stats, uint64_t* hash, uint64_t* digest, uint32_t* round_F,
                           uint64_t* round_E, uint32_t max_rounds) {
  if (threads < 1) threads = 1;
  int* status = (int*)calloc(C ? C : 1, sizeof(int));
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  many_job J = {n, off, cols, sources, sizes, C, d, out_dist, out_sub, stats, hash, status, 0, &mu,
                digest, round_F, round_E, max_rounds};
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, many_worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  int rc = 0;
  for (uint32_t c = 0; c < C; ++c) if (status[c]) rc = -1;
  free(th); free(status);
  return rc;
}

int or_cluster_bfs_many(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* sources,
                        const uint8_t* sizes, uint32_t C, uint32_t d, int threads, uint16_t* out_dist,
                        uint64_t* out_sub, uint64_t* stats, uint64_t* hash) {
  return or_cluster_bfs_many_ex(n, off, cols, sources, sizes, C, d, threads, out_dist, out_sub, stats, hash, NULL,
                                NULL, NULL, 0);
}

/* Order-independent 64-bit digest of one cluster's output vector, used to
 * compare whole outputs at full size (not part of the method).  Written out:
 *   fin(z)  = the SplitMix64 finaliser (z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
 *             z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31);
 *   x       = fin((v * 0x9E3779B97F4A7C15 + 0xD1B54A32D192ED03) ^ (Delta_v << 48))
 *             (Delta_v as u16, 0xFFFF unreached; arithmetic mod 2^64);
 *   x       = fin(x ^ S_v[i]) for i = 0 .. planes-1 in order;
 *   digest  = sum over v = 0 .. n-1 of x, mod 2^64.
 * The product computes the same definition independently (include/cbfs.h,
 * cbfs_digest_store); a sum is used so that it can be formed in any order. */
static uint64_t dg_fin(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t or_digest_cluster(uint32_t n, uint32_t planes, const uint16_t* dist, const uint64_t* sub) {
  uint64_t sum = 0;
  for (uint32_t v = 0; v < n; ++v) {
    uint64_t x = dg_fin(((uint64_t)v * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL) ^ ((uint64_t)dist[v] << 48));
    for (uint32_t i = 0; i < planes; ++i) x = dg_fin(x ^ sub[(size_t)i * n + v]);
    sum += x;
  }
  return sum;
}

/* Order-dependent 64-bit digest of one cluster's output (dist[v], then the
 * d+1 subsets of v, v ascending); FNV-1a over the little-endian bytes.  Used
 * only to compare whole outputs compactly; not part of the method. */
uint64_t or_hash_cluster(uint32_t n, uint32_t d, const uint16_t* dist, const uint64_t* sub) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint32_t v = 0; v < n; ++v) {
    uint64_t w = dist[v];
    for (int b = 0; b < 2; ++b) { h ^= (w >> (8 * b)) & 0xFF; h *= 0x100000001b3ULL; }
    for (uint32_t i = 0; i <= d; ++i) {
      uint64_t x = sub[(size_t)i * n + v];
      for (int b = 0; b < 8; ++b) { h ^= (x >> (8 * b)) & 0xFF; h *= 0x100000001b3ULL; }
    }
  }
  return h;
}

/* ---------------------------------------------------------------------
 * select_clusters — "Selecting Landmarks in Clusters" with
 * reading R12: repeat r times:
 *   root  = policy 0 (degree): the unmarked non-isolated vertex with the
 *           highest degree, ties by smaller id;
 *           policy 1 (random, BASELINE.json configs 1 and 4): draw
 *           v_t = bounded(rand(seed, 1, t), n), t = 0,1,2,... (counter kept
 *           across clusters), until v_t is unmarked and non-isolated;
 *   members = up to k-1 unmarked vertices within floor(d/2) hops of the root
 *           (marked vertices may be passed through), highest
 *           degree first, ties by smaller id;
 *   cluster = [root, members...]; mark all of them.
 * Stops early when no unmarked non-isolated vertex is left.
 * `rand_fn` is the shared counter-based generator (cbfs_inputs).
 * out_sources [r][64] padded with 0xFFFFFFFF, out_sizes [r]; returns the
 * number of clusters produced (<= r) or -1.
 * ------------------------------------------------------------------- */
typedef uint64_t (*or_rand_fn)(uint64_t, uint64_t, uint64_t);

static const uint32_t* g_sel_deg;
static int by_deg_desc_id_asc(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  if (g_sel_deg[x] != g_sel_deg[y]) return g_sel_deg[x] > g_sel_deg[y] ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* clusters of up to k <= stride sources (stride = 64 words of 64 sources
 * each for k > 64, the paper's general k); sizes as uint8 (k <= 64)
 * or uint16 */
static int64_t select_clusters_any(uint32_t n, const uint64_t* off, const uint32_t* cols, uint32_t r, uint32_t k,
                                   uint32_t d, uint32_t policy, uint64_t seed, or_rand_fn rand_fn, uint32_t stride,
                                   uint32_t* out_sources, uint8_t* out_sizes8, uint16_t* out_sizes16) {
  if (k == 0 || k > stride || (policy == 1 && !rand_fn)) return -1;
  uint32_t* deg = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) deg[v] = (uint32_t)(off[v + 1] - off[v]);
  uint8_t* marked = (uint8_t*)calloc(n ? n : 1, 1);
  uint32_t* hop = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) hop[v] = OR_INF32;
  uint32_t* ball = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* cand = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint32_t v = 0; v < n; ++v) order[v] = v;
  g_sel_deg = deg;
  qsort(order, n, sizeof(uint32_t), by_deg_desc_id_asc);
  uint64_t avail = 0;
  for (uint32_t v = 0; v < n; ++v) avail += deg[v] > 0;
  uint64_t cursor = 0, t_draw = 0;
  const uint32_t h = d / 2;
  int64_t produced = 0;
  for (uint32_t c = 0; c < r; ++c) {
    if (avail == 0) break;
    uint32_t root = OR_INF32;
    if (policy == 0) {
      while (cursor < n && (marked[order[cursor]] || deg[order[cursor]] == 0)) ++cursor;
      if (cursor >= n) break;
      root = order[cursor];
    } else {
      for (;;) {
        uint32_t v = (uint32_t)(((unsigned __int128)rand_fn(seed, 1, t_draw++) * n) >> 64);
        if (!marked[v] && deg[v] > 0) { root = v; break; }
      }
    }
    /* floor(d/2)-hop ball around root, through all vertices */
    uint64_t nb = 0, head = 0;
    hop[root] = 0; ball[nb++] = root;
    while (head < nb) {
      uint32_t u = ball[head++];
      if (hop[u] >= h) continue;
      for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
        uint32_t v = cols[e];
        if (hop[v] == OR_INF32) { hop[v] = hop[u] + 1; ball[nb++] = v; }
      }
    }
    uint64_t nc = 0;
    for (uint64_t t = 1; t < nb; ++t) if (!marked[ball[t]]) cand[nc++] = ball[t];
    for (uint64_t t = 0; t < nb; ++t) hop[ball[t]] = OR_INF32;
    qsort(cand, nc, sizeof(uint32_t), by_deg_desc_id_asc);
    uint32_t sz = 0;
    uint32_t* outS = out_sources + (size_t)c * stride;
    for (uint32_t j = 0; j < stride; ++j) outS[j] = OR_INF32;
    outS[sz++] = root;
    for (uint64_t t = 0; t < nc && sz < k; ++t) outS[sz++] = cand[t];
    for (uint32_t j = 0; j < sz; ++j) { marked[outS[j]] = 1; avail -= deg[outS[j]] > 0; }
    if (out_sizes8) out_sizes8[c] = (uint8_t)sz;
    if (out_sizes16) out_sizes16[c] = (uint16_t)sz;
    produced++;
  }
  free(deg); free(marked); free(hop); free(ball); free(cand); free(order);
  return produced;
}

int64_t or_select_clusters(uint32_t n, const uint64_t* off, const uint32_t* cols, uint32_t r, uint32_t k,
                           uint32_t d, uint32_t policy, uint64_t seed, or_rand_fn rand_fn,
                           uint32_t* out_sources, uint8_t* out_sizes) {
  if (k > 64) return -1;
  return select_clusters_any(n, off, cols, r, k, d, policy, seed, rand_fn, 64, out_sources, out_sizes, NULL);
}

/* the same rule for k up to 64 * words sources: out_sources [r][64 words], sizes uint16 */
int64_t or_select_clusters_wide(uint32_t n, const uint64_t* off, const uint32_t* cols, uint32_t r, uint32_t k,
                                uint32_t d, uint32_t policy, uint64_t seed, or_rand_fn rand_fn, uint32_t words,
                                uint32_t* out_sources, uint16_t* out_sizes) {
  if (words == 0 || words > 64) return -1;
  return select_clusters_any(n, off, cols, r, k, d, policy, seed, rand_fn, 64 * words, out_sources, NULL, out_sizes);
}

/* ---------------------------------------------------------------------
 * Landmark query with clustered landmarks (R14-R16):
 * per cluster c with both Delta_u, Delta_v finite:
 *   value_c = Delta_u + Delta_v + min{ i + j : S_u[i] & S_v[j] != 0 },
 * scanning i + j = 0, 1, ..., 2d; answer = min over clusters,
 * INT32_MAX if no cluster reaches both endpoints.  Labels are given
 * cluster-major: dist [C][n], sub [C][d+1][n] (all d+1 subsets).
 * ------------------------------------------------------------------- */
static int32_t query_one_cluster(uint32_t n, uint32_t d, const uint16_t* dist, const uint64_t* sub, uint32_t u,
                                 uint32_t v) {
  if (dist[u] == OR_INF16 || dist[v] == OR_INF16) return INT32_MAX;
  for (uint32_t t = 0; t <= 2 * d; ++t)
    for (uint32_t i = 0; i <= d; ++i) {
      if (t < i || t - i > d) continue;
      uint32_t j = t - i;
      if (sub[(size_t)i * n + u] & sub[(size_t)j * n + v]) return (int32_t)dist[u] + (int32_t)dist[v] + (int32_t)t;
    }
  return INT32_MAX; /* unreachable from this cluster's sources on one side */
}

int or_query(uint32_t n, uint32_t d, uint32_t C, const uint16_t* dist, const uint64_t* sub, uint64_t q,
             const uint32_t* s, const uint32_t* t, int32_t* out) {
  for (uint64_t j = 0; j < q; ++j) {
    if (s[j] >= n || t[j] >= n) return -1;
    int32_t best = INT32_MAX;
    for (uint32_t c = 0; c < C; ++c) {
      int32_t x = query_one_cluster(n, d, dist + (size_t)c * n, sub + (size_t)c * (d + 1) * n, s[j], t[j]);
      if (x < best) best = x;
    }
    out[j] = best;
  }
  return 0;
}

/* Streaming build+query (Alg. 2 Construct_Index with BFS replaced by C-BFS,
 * P:1004-1005, then Query P:1013-1021) without keeping the index: clusters are
 * spread over threads, each runs Alg. 1 and min-merges its per-cluster values
 * into a thread-local answer array; answers are then min-merged. */
typedef struct {
  uint32_t n; const uint64_t* off; const uint32_t* cols; const uint32_t* sources; const uint8_t* sizes;
  uint32_t C, d; uint64_t q; const uint32_t* s; const uint32_t* t; int32_t* best;
  uint32_t* next_c; pthread_mutex_t* mu; int status;
  uint64_t* stats; uint64_t* digest;
} stream_job;

static void* stream_worker(void* p) {
  stream_job* J = (stream_job*)p;
  uint16_t* dist = (uint16_t*)malloc(sizeof(uint16_t) * (J->n ? J->n : 1));
  uint64_t* sub = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(J->d + 1) * (J->n ? J->n : 1));
  for (uint64_t j = 0; j < J->q; ++j) J->best[j] = INT32_MAX;
  for (;;) {
    pthread_mutex_lock(J->mu);
    uint32_t c = (*J->next_c)++;
    pthread_mutex_unlock(J->mu);
    if (c >= J->C) break;
    uint64_t st[4];
    if (or_cluster_bfs(J->n, J->off, J->cols, J->sources + (size_t)c * 64, J->sizes[c], J->d, dist, sub, st, NULL,
                       NULL, 0)) { J->status = -1; continue; }
    if (J->stats) memcpy(J->stats + 4 * (size_t)c, st, sizeof st);
    if (J->digest) J->digest[c] = or_digest_cluster(J->n, J->d + 1, dist, sub);
    for (uint64_t j = 0; j < J->q; ++j) {
      int32_t x = query_one_cluster(J->n, J->d, dist, sub, J->s[j], J->t[j]);
      if (x < J->best[j]) J->best[j] = x;
    }
  }
  free(dist); free(sub);
  return NULL;
}

int or_query_stream_ex(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* sources,
                       const uint8_t* sizes, uint32_t C, uint32_t d, uint64_t q, const uint32_t* s, const uint32_t* t,
                       int threads, int32_t* out, uint64_t* stats, uint64_t* digest) {
  for (uint64_t j = 0; j < q; ++j) if (s[j] >= n || t[j] >= n) return -1;
  if (threads < 1) threads = 1;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  uint32_t next_c = 0;
  stream_job* jobs = (stream_job*)calloc((size_t)threads, sizeof(stream_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int i = 0; i < threads; ++i) {
    jobs[i] = (stream_job){n, off, cols, sources, sizes, C, d, q, s, t, NULL, &next_c, &mu, 0, stats, digest};
    jobs[i].best = (int32_t*)malloc(sizeof(int32_t) * (q ? q : 1));
    pthread_create(&th[i], NULL, stream_worker, &jobs[i]);
  }
  int rc = 0;
  for (uint64_t j = 0; j < q; ++j) out[j] = INT32_MAX;
  for (int i = 0; i < threads; ++i) {
    pthread_join(th[i], NULL);
    if (jobs[i].status) rc = -1;
    for (uint64_t j = 0; j < q; ++j) if (jobs[i].best[j] < out[j]) out[j] = jobs[i].best[j];
    free(jobs[i].best);
  }
  free(jobs); free(th);
  return rc;
}

int or_query_stream(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* sources,
                    const uint8_t* sizes, uint32_t C, uint32_t d, uint64_t q, const uint32_t* s, const uint32_t* t,
                    int threads, int32_t* out) {
  return or_query_stream_ex(n, off, cols, sources, sizes, C, d, q, s, t, threads, out, NULL, NULL);
}

/* ---------------------------------------------------------------------
 * Index budget: a cluster record costs 1 byte for the distance
 * plus d bit-subsets of w/8 bytes; r = floor(t / (1 + d*w/8)).
 * ------------------------------------------------------------------- */
int64_t or_record_bytes(uint32_t w, uint32_t d) { return 1 + (int64_t)d * (int64_t)((w + 7) / 8); }
int64_t or_budget_to_clusters(uint64_t t, uint32_t w, uint32_t d) {
  int64_t rb = or_record_bytes(w, d);
  if ((int64_t)t < rb) return -1;
  return (int64_t)t / rb;
}

/* ---------------------------------------------------------------------
 * csr_build — graph normalisation (R17) for edge lists too large
 * for numpy's unique: every pair {u,v} with u != v becomes arcs u->v and
 * v->u, each row is sorted and its duplicates dropped.  Same result as
 * csr_from_edges in oracle/__init__.py (pinned against scipy there).
 *   work : [2 * P] uint32 scratch; on return work[0..m) holds the columns
 *   off  : [n+1] uint64 row offsets.  Returns m, or -1 on an id >= n.
 * Rows are sorted by `threads` threads (qsort per row).
 * ------------------------------------------------------------------- */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

typedef struct { uint32_t lo, hi; uint64_t* start; uint32_t* work; uint64_t* kept; } csr_job;

static void* csr_sort_rows(void* p) {
  csr_job* J = (csr_job*)p;
  for (uint32_t v = J->lo; v < J->hi; ++v) {
    uint32_t* row = J->work + J->start[v];
    uint64_t len = J->start[v + 1] - J->start[v];
    qsort(row, len, sizeof(uint32_t), cmp_u32);
    uint64_t k = 0;
    for (uint64_t e = 0; e < len; ++e)
      if (k == 0 || row[e] != row[k - 1]) row[k++] = row[e];
    J->kept[v] = k;
  }
  return NULL;
}

int64_t or_csr_build(uint32_t n, uint64_t P, const uint32_t* src, const uint32_t* dst, int threads, uint32_t* work,
                     uint64_t* off) {
  uint64_t* start = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t* kept = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  for (uint64_t e = 0; e < P; ++e) {
    if (src[e] >= n || dst[e] >= n) { free(start); free(kept); return -1; }
    if (src[e] == dst[e]) continue;  /* self loops dropped */
    start[src[e] + 1]++;
    start[dst[e] + 1]++;
  }
  for (uint32_t v = 0; v < n; ++v) start[v + 1] += start[v];
  uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  memcpy(fill, start, sizeof(uint64_t) * ((size_t)n + 1));
  for (uint64_t e = 0; e < P; ++e) {
    uint32_t u = src[e], v = dst[e];
    if (u == v) continue;
    work[fill[u]++] = v;
    work[fill[v]++] = u;
  }
  free(fill);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  csr_job* jobs = (csr_job*)calloc((size_t)threads, sizeof(csr_job));
  for (int t = 0; t < threads; ++t) {
    jobs[t].lo = (uint32_t)((uint64_t)n * t / threads);
    jobs[t].hi = (uint32_t)((uint64_t)n * (t + 1) / threads);
    jobs[t].start = start; jobs[t].work = work; jobs[t].kept = kept;
    pthread_create(&th[t], NULL, csr_sort_rows, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th); free(jobs);
  /* compact the deduplicated rows to the front of work */
  off[0] = 0;
  for (uint32_t v = 0; v < n; ++v) {
    memmove(work + off[v], work + start[v], sizeof(uint32_t) * kept[v]);
    off[v + 1] = off[v] + kept[v];
  }
  int64_t m = (int64_t)off[n];
  free(start); free(kept);
  return m;
}

/* ---------------------------------------------------------------------
 * bidir_refine — the fixed-size bi-directional search of Appendix B
 * (P:1790-1800): "search tau vertices from each side by a BFS order, and take
 * an intersection to find the minimum distance among them".  Reading R27
 * (DESIGN.md §2): from each endpoint a queue BFS over the sorted CSR visits
 * vertices in discovery order (the endpoint first) and stops once tau
 * vertices are visited; the answer is min over x visited by both sides of
 * dist_s(x) + dist_t(x), INT32_MAX when the two visited sets are disjoint
 * (tau = 0: nothing visited).  Sequential, one pair at a time.
 * ------------------------------------------------------------------- */
static uint32_t bidir_side(uint32_t n, const uint64_t* off, const uint32_t* cols, uint32_t src, uint32_t tau,
                           uint32_t* mark, uint32_t stamp, uint32_t* dist, uint32_t* order) {
  if (tau == 0) return 0;
  uint32_t cnt = 0, head = 0;
  mark[src] = stamp; dist[src] = 0; order[cnt++] = src;
  while (head < cnt && cnt < tau) {
    uint32_t x = order[head++];
    for (uint64_t e = off[x]; e < off[x + 1] && cnt < tau; ++e) {
      uint32_t u = cols[e];
      if (mark[u] != stamp) { mark[u] = stamp; dist[u] = dist[x] + 1; order[cnt++] = u; }
    }
  }
  (void)n;
  return cnt;
}

int or_bidir_refine(uint32_t n, const uint64_t* off, const uint32_t* cols, uint64_t q, const uint32_t* s,
                    const uint32_t* t, uint32_t tau, int32_t* out) {
  for (uint64_t j = 0; j < q; ++j) if (s[j] >= n || t[j] >= n) return -1;
  uint32_t* mark_s = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  uint32_t* dist_s = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* ord_s = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* mark_t = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  uint32_t* dist_t = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  uint32_t* ord_t = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  for (uint64_t j = 0; j < q; ++j) {
    const uint32_t stamp = (uint32_t)(j + 1);  /* fresh marks per pair */
    uint32_t cs = bidir_side(n, off, cols, s[j], tau, mark_s, stamp, dist_s, ord_s);
    uint32_t ct = bidir_side(n, off, cols, t[j], tau, mark_t, stamp, dist_t, ord_t);
    int64_t best = INT32_MAX;
    for (uint32_t a = 0; a < cs; ++a) {
      uint32_t x = ord_s[a];
      if (mark_t[x] == stamp && (int64_t)dist_s[x] + dist_t[x] < best) best = (int64_t)dist_s[x] + dist_t[x];
    }
    (void)ct;
    out[j] = (int32_t)best;
  }
  free(mark_s); free(dist_s); free(ord_s); free(mark_t); free(dist_t); free(ord_t);
  return 0;
}

/* ---------------------------------------------------------------------
 * Exact 2-hop distance oracle: PLL with a C-BFS first phase,
 * reading R29.
 *   vertex order: degree desc, id asc (pos[v] = position);
 *   phase 1: the C given clusters (diameter <= d); their labels are the
 *     cluster distance vectors of every vertex (dist16 [C][n], sub
 *     [C][d+1][n], from Alg. 1); every source of a cluster is "covered";
 *   phase 2: the uncovered vertices in order, in batches b_0 = first,
 *     b_{i+1} = min(bmax, floor(3 b_i / 2)) (200 x 1.5^i up to
 *     1000); each root r of a batch runs a BFS pruned against the index as it
 *     was when the batch started (R29): at a visited u at distance delta, if
 *     query(r, u) <= delta then u is pruned (no label, not expanded),
 *     otherwise (pos[r], delta) is appended to L(u) and u is expanded
 *     (P:1883-1887).
 *   query(s, t) = min(min over clusters of the R15 scan value, min over hubs
 *     h in L(s) and L(t) of d_s(h) + d_t(h)).
 * Labels: counts [n], entries [n][cap] = pos << 8 | dist, each list ascending
 * (roots run in increasing pos, one entry per root per vertex).
 * Returns the number of phase-2 labels, -1 bad arguments, -2 a list would
 * exceed cap, -3 a label distance > 254.
 * ------------------------------------------------------------------- */
static int32_t pll_cluster_part(uint32_t n, uint32_t C, uint32_t d, const uint16_t* dist, const uint64_t* sub,
                                uint32_t u, uint32_t v) {
  int32_t best = INT32_MAX;
  for (uint32_t c = 0; c < C; ++c) {
    int32_t x = query_one_cluster(n, d, dist + (size_t)c * n, sub + (size_t)c * (d + 1) * n, u, v);
    if (x < best) best = x;
  }
  return best;
}

static int pll_cmp_pos(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  const uint32_t* deg = g_sel_deg;
  if (deg[x] != deg[y]) return deg[x] > deg[y] ? -1 : 1;
  return x < y ? -1 : (x > y);
}

int64_t or_pll_build(uint32_t n, const uint64_t* off, const uint32_t* cols, const uint32_t* sources,
                     const uint8_t* sizes, uint32_t C, uint32_t d, const uint16_t* cdist, const uint64_t* csub,
                     uint32_t first, uint32_t bmax, uint32_t cap, uint32_t* counts, uint32_t* entries) {
  if (first == 0 || bmax == 0 || cap == 0) return -1;
  const size_t N = n ? n : 1;
  uint32_t* deg = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint8_t* covered = (uint8_t*)calloc(N, 1);
  uint32_t* snap = (uint32_t*)malloc(sizeof(uint32_t) * N);
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * N);   /* hub pos -> d(r, hub) of the root's snapshot label */
  uint32_t* mark = (uint32_t*)calloc(N, sizeof(uint32_t));
  uint32_t* qv = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* qd = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* roots = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (uint32_t v = 0; v < n; ++v) { deg[v] = (uint32_t)(off[v + 1] - off[v]); order[v] = v; counts[v] = 0; tmp[v] = -1; }
  g_sel_deg = deg;
  qsort(order, n, sizeof(uint32_t), pll_cmp_pos);
  for (uint32_t p = 0; p < n; ++p) pos[order[p]] = p;
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t j = 0; j < sizes[c]; ++j) covered[sources[(size_t)c * 64 + j]] = 1;
  uint32_t nroots = 0;
  for (uint32_t p = 0; p < n; ++p) if (!covered[order[p]]) roots[nroots++] = order[p];
  int64_t total = 0, rc = 0;
  uint32_t b = first, stamp = 0;
  for (uint32_t r0 = 0; r0 < nroots && rc == 0; r0 += b, b = (b * 3 / 2 < bmax ? b * 3 / 2 : bmax)) {
    if (b > bmax) b = bmax;
    const uint32_t r1 = r0 + b < nroots ? r0 + b : nroots;
    memcpy(snap, counts, sizeof(uint32_t) * n);  /* the index as of the batch start */
    for (uint32_t ri = r0; ri < r1 && rc == 0; ++ri) {
      const uint32_t r = roots[ri];
      for (uint32_t a = 0; a < snap[r]; ++a) tmp[entries[(size_t)r * cap + a] >> 8] = (int32_t)(entries[(size_t)r * cap + a] & 255u);
      ++stamp;
      uint64_t head = 0, tail = 0;
      qv[tail] = r; qd[tail++] = 0; mark[r] = stamp;
      while (head < tail) {
        const uint32_t u = qv[head], du = qd[head]; ++head;
        int64_t q = pll_cluster_part(n, C, d, cdist, csub, r, u);
        for (uint32_t a = 0; a < snap[u]; ++a) {
          const uint32_t e = entries[(size_t)u * cap + a];
          if (tmp[e >> 8] >= 0 && (int64_t)tmp[e >> 8] + (e & 255u) < q) q = (int64_t)tmp[e >> 8] + (e & 255u);
        }
        if (q <= (int64_t)du) continue;  /* pruned */
        if (counts[u] >= cap) { rc = -2; break; }
        if (du > 254) { rc = -3; break; }
        entries[(size_t)u * cap + counts[u]++] = (pos[r] << 8) | du;
        ++total;
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
          const uint32_t x = cols[e];
          if (mark[x] != stamp) { mark[x] = stamp; qv[tail] = x; qd[tail++] = du + 1; }
        }
      }
      for (uint32_t a = 0; a < snap[r]; ++a) tmp[entries[(size_t)r * cap + a] >> 8] = -1;
    }
  }
  free(deg); free(order); free(pos); free(covered); free(snap); free(tmp); free(mark); free(qv); free(qd); free(roots);
  return rc ? rc : total;
}

int or_pll_query(uint32_t n, uint32_t C, uint32_t d, const uint16_t* cdist, const uint64_t* csub, uint32_t cap,
                 const uint32_t* counts, const uint32_t* entries, uint64_t q, const uint32_t* s, const uint32_t* t,
                 int32_t* out) {
  for (uint64_t j = 0; j < q; ++j) {
    if (s[j] >= n || t[j] >= n) return -1;
    int64_t best = pll_cluster_part(n, C, d, cdist, csub, s[j], t[j]);
    const uint32_t* A = entries + (size_t)s[j] * cap;
    const uint32_t* B = entries + (size_t)t[j] * cap;
    uint32_t a = 0, bb = 0;
    while (a < counts[s[j]] && bb < counts[t[j]]) {  /* merge of two ascending hub lists */
      const uint32_t ha = A[a] >> 8, hb = B[bb] >> 8;
      if (ha == hb) {
        const int64_t x = (int64_t)(A[a] & 255u) + (B[bb] & 255u);
        if (x < best) best = x;
        ++a; ++bb;
      } else if (ha < hb) {
        ++a;
      } else {
        ++bb;
      }
    }
    out[j] = (int32_t)best;
  }
  return 0;
}
