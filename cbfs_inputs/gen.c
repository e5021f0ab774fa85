/*
 * gen.c — seeded synthetic input generators, see include/cbfs_gen.h.
 * Shared by the product tests/bench and the oracle; contains none of the
 * method's arithmetic (BASELINE.json configs).
 */
#include "../include/cbfs_gen.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

uint64_t cg_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t cg_rand(uint64_t seed, uint64_t stream, uint64_t index) {
  uint64_t key = cg_mix64(seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL);
  return cg_mix64(key + (index + 1) * 0x9E3779B97F4A7C15ULL);
}

uint64_t cg_bounded(uint64_t x, uint64_t n) {
  return (uint64_t)(((unsigned __int128)x * (unsigned __int128)n) >> 64);
}

static double unit_double(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

static int default_threads(int threads) {
  if (threads > 0) return threads;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)(c > 64 ? 64 : c) : 1;
}

/* ------------------------------------------------------------------ ER */
int64_t cg_erdos_renyi(uint32_t n, uint64_t pairs, uint64_t seed, uint32_t* src, uint32_t* dst) {
  if (!n || (pairs && (!src || !dst))) return -1;
  for (uint64_t t = 0; t < pairs; ++t) {
    src[t] = (uint32_t)cg_bounded(cg_rand(seed, 0, 2 * t), n);
    dst[t] = (uint32_t)cg_bounded(cg_rand(seed, 0, 2 * t + 1), n);
  }
  return (int64_t)pairs;
}

/* ---------------------------------------------------------------- RMAT */
static uint64_t scramble_id(uint64_t x, int scale, uint64_t seed) {
  const uint64_t mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1);
  const int sh1 = scale / 2 > 0 ? scale / 2 : 1;
  const int sh2 = (scale + 1) / 2 > 0 ? (scale + 1) / 2 : 1;
  const uint64_t k1 = cg_rand(seed, 7, 0), k2 = cg_rand(seed, 7, 1);
  x = (x ^ k1) & mask;
  x = (x * 0x9E3779B97F4A7C15ULL) & mask;      /* odd multiplier: bijective mod 2^s */
  x ^= x >> sh1;                               /* xorshift: bijective */
  x = (x * 0xBF58476D1CE4E5B9ULL) & mask;
  x ^= x >> sh2;
  return (x ^ k2) & mask;
}

typedef struct {
  int scale; uint64_t lo, hi; double a, ab, abc; uint64_t seed; int scramble;
  uint32_t *src, *dst;
} rmat_job;

static void* rmat_worker(void* p) {
  rmat_job* j = (rmat_job*)p;
  for (uint64_t t = j->lo; t < j->hi; ++t) {
    uint64_t u = 0, v = 0;
    for (int l = 0; l < j->scale; ++l) {
      double x = unit_double(cg_rand(j->seed, 0, t * (uint64_t)j->scale + (uint64_t)l));
      uint64_t bu, bv;
      if (x < j->a) { bu = 0; bv = 0; }
      else if (x < j->ab) { bu = 0; bv = 1; }
      else if (x < j->abc) { bu = 1; bv = 0; }
      else { bu = 1; bv = 1; }
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    if (j->scramble) { u = scramble_id(u, j->scale, j->seed); v = scramble_id(v, j->scale, j->seed); }
    j->src[t] = (uint32_t)u;
    j->dst[t] = (uint32_t)v;
  }
  return NULL;
}

int64_t cg_rmat(int scale, uint64_t edges, double a, double b, double c, uint64_t seed, int scramble,
                int threads, uint32_t* src, uint32_t* dst) {
  if (scale < 1 || scale > 32 || (edges && (!src || !dst))) return -1;
  int T = default_threads(threads);
  if ((uint64_t)T > edges) T = edges ? (int)edges : 1;
  pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
  rmat_job* jobs = (rmat_job*)calloc((size_t)T, sizeof(rmat_job));
  for (int i = 0; i < T; ++i) {
    jobs[i] = (rmat_job){scale, edges * (uint64_t)i / (uint64_t)T, edges * (uint64_t)(i + 1) / (uint64_t)T,
                         a, a + b, a + b + c, seed, scramble, src, dst};
    pthread_create(&th[i], NULL, rmat_worker, &jobs[i]);
  }
  for (int i = 0; i < T; ++i) pthread_join(th[i], NULL);
  free(th); free(jobs);
  return (int64_t)edges;
}

/* ---------------------------------------------------------------- grid */
uint64_t cg_grid_capacity(uint32_t side, double p_diag) {
  uint64_t ge = 2ULL * side * (side > 0 ? side - 1 : 0);
  return ge + (uint64_t)llround(p_diag * (double)ge);
}

int64_t cg_grid(uint32_t side, double p_delete, double p_diag, uint64_t seed, uint64_t capacity,
                uint32_t* src, uint32_t* dst) {
  if (side < 2 || !src || !dst || capacity < cg_grid_capacity(side, p_diag)) return -1;
  const uint64_t S = side, H = S * (S - 1);
  uint64_t w = 0;
  for (uint64_t e = 0; e < H; ++e) { /* horizontal (x,y)-(x+1,y) */
    if (unit_double(cg_rand(seed, 0, e)) < p_delete) continue;
    uint64_t y = e / (S - 1), x = e % (S - 1);
    src[w] = (uint32_t)(y * S + x); dst[w] = (uint32_t)(y * S + x + 1); ++w;
  }
  for (uint64_t e = 0; e < H; ++e) { /* vertical (x,y)-(x,y+1) */
    if (unit_double(cg_rand(seed, 0, H + e)) < p_delete) continue;
    uint64_t x = e / (S - 1), y = e % (S - 1);
    src[w] = (uint32_t)(y * S + x); dst[w] = (uint32_t)((y + 1) * S + x); ++w;
  }
  uint64_t nd = (uint64_t)llround(p_diag * (double)(2 * H));
  for (uint64_t t = 0; t < nd; ++t) { /* diagonal shortcut (x,y)-(x+1,y+1) */
    uint64_t pos = cg_bounded(cg_rand(seed, 1, t), (S - 1) * (S - 1));
    uint64_t x = pos % (S - 1), y = pos / (S - 1);
    src[w] = (uint32_t)(y * S + x); dst[w] = (uint32_t)((y + 1) * S + x + 1); ++w;
  }
  return (int64_t)w;
}

/* ----------------------------------------------------------------- kNN */
typedef struct {
  uint32_t n, k, G; uint64_t cellw;
  const uint32_t* xyz;      /* [n][3] 24-bit ints */
  const uint32_t* cell_start; /* [G^3 + 1] */
  const uint32_t* cell_pts;   /* points sorted by cell */
  uint32_t lo, hi; uint32_t *src, *dst;
} knn_job;

static inline uint32_t cell_of(uint32_t c, uint64_t cellw, uint32_t G) {
  uint64_t q = c / cellw; return (uint32_t)(q >= G ? G - 1 : q);
}

static void* knn_worker(void* p) {
  knn_job* J = (knn_job*)p;
  const uint32_t k = J->k, G = J->G;
  uint64_t* bd = (uint64_t*)malloc(sizeof(uint64_t) * k);
  uint32_t* bi = (uint32_t*)malloc(sizeof(uint32_t) * k);
  for (uint32_t i = J->lo; i < J->hi; ++i) {
    const uint32_t* P = J->xyz + 3ULL * i;
    int cx = (int)cell_of(P[0], J->cellw, G), cy = (int)cell_of(P[1], J->cellw, G), cz = (int)cell_of(P[2], J->cellw, G);
    uint32_t have = 0;
    for (int r = 0; r <= (int)G; ++r) {
      /* every point in Chebyshev ring >= r+1 is at least r*cellw away on some axis */
      if (have == k && r >= 1) {
        uint64_t lb = (uint64_t)(r - 1) * J->cellw;  /* rings < r done; next ring r is >= (r-1)*w away */
        if (bd[k - 1] < lb * lb) break;
      }
      for (int dz = -r; dz <= r; ++dz) for (int dy = -r; dy <= r; ++dy) for (int dx = -r; dx <= r; ++dx) {
        if (abs(dx) != r && abs(dy) != r && abs(dz) != r) continue; /* shell only */
        int X = cx + dx, Y = cy + dy, Z = cz + dz;
        if (X < 0 || Y < 0 || Z < 0 || X >= (int)G || Y >= (int)G || Z >= (int)G) continue;
        uint64_t cidx = ((uint64_t)Z * G + (uint64_t)Y) * G + (uint64_t)X;
        for (uint32_t t = J->cell_start[cidx]; t < J->cell_start[cidx + 1]; ++t) {
          uint32_t j = J->cell_pts[t];
          if (j == i) continue;
          const uint32_t* Q = J->xyz + 3ULL * j;
          int64_t ex = (int64_t)P[0] - Q[0], ey = (int64_t)P[1] - Q[1], ez = (int64_t)P[2] - Q[2];
          uint64_t d2 = (uint64_t)(ex * ex) + (uint64_t)(ey * ey) + (uint64_t)(ez * ez);
          /* insert (d2, j) into the sorted top-k list, order (dist, index) */
          if (have == k && (d2 > bd[k - 1] || (d2 == bd[k - 1] && j > bi[k - 1]))) continue;
          uint32_t pos = have < k ? have++ : k - 1;
          while (pos > 0 && (bd[pos - 1] > d2 || (bd[pos - 1] == d2 && bi[pos - 1] > j))) {
            bd[pos] = bd[pos - 1]; bi[pos] = bi[pos - 1]; --pos;
          }
          bd[pos] = d2; bi[pos] = j;
        }
      }
    }
    for (uint32_t t = 0; t < have; ++t) { J->src[(uint64_t)i * k + t] = i; J->dst[(uint64_t)i * k + t] = bi[t]; }
    for (uint32_t t = have; t < k; ++t) { J->src[(uint64_t)i * k + t] = i; J->dst[(uint64_t)i * k + t] = i; } /* n <= k: self loop pad */
  }
  free(bd); free(bi);
  return NULL;
}

int64_t cg_knn3d(uint32_t n, uint32_t k, uint64_t seed, int threads, uint32_t* src, uint32_t* dst, uint32_t* coords) {
  if (!n || !k || !src || !dst) return -1;
  uint32_t* xyz = coords ? coords : (uint32_t*)malloc(sizeof(uint32_t) * 3ULL * n);
  for (uint64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) xyz[3 * i + a] = (uint32_t)(cg_rand(seed, 0, 3 * i + (uint64_t)a) >> 40);
  uint32_t G = (uint32_t)cbrt((double)n / 2.0);
  if (G < 1) G = 1;
  if (G > 1024) G = 1024;
  uint64_t cellw = ((1ULL << 24) + G - 1) / G;
  uint64_t NC = (uint64_t)G * G * G;
  uint32_t* cs = (uint32_t*)calloc(NC + 1, sizeof(uint32_t));
  uint32_t* cp = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  uint32_t* cid = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t c = ((uint64_t)cell_of(xyz[3ULL * i + 2], cellw, G) * G + cell_of(xyz[3ULL * i + 1], cellw, G)) * G +
                 cell_of(xyz[3ULL * i], cellw, G);
    cid[i] = (uint32_t)c; cs[c + 1]++;
  }
  for (uint64_t c = 0; c < NC; ++c) cs[c + 1] += cs[c];
  uint32_t* fill = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)NC);
  memcpy(fill, cs, sizeof(uint32_t) * (size_t)NC);
  for (uint32_t i = 0; i < n; ++i) cp[fill[cid[i]]++] = i;
  free(fill); free(cid);
  int T = default_threads(threads);
  if ((uint32_t)T > n) T = (int)n;
  pthread_t* th = (pthread_t*)calloc((size_t)T, sizeof(pthread_t));
  knn_job* jobs = (knn_job*)calloc((size_t)T, sizeof(knn_job));
  for (int t = 0; t < T; ++t) {
    jobs[t] = (knn_job){n, k, G, cellw, xyz, cs, cp, (uint32_t)((uint64_t)n * t / T), (uint32_t)((uint64_t)n * (t + 1) / T), src, dst};
    pthread_create(&th[t], NULL, knn_worker, &jobs[t]);
  }
  for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
  free(th); free(jobs); free(cs); free(cp);
  if (!coords) free(xyz);
  return (int64_t)n * k;
}

/* ------------------------------------------------------------- queries */
int64_t cg_query_pairs(uint32_t n, uint64_t q, uint64_t seed, uint64_t stream, uint32_t* s, uint32_t* t) {
  if (!n || (q && (!s || !t))) return -1;
  for (uint64_t j = 0; j < q; ++j) {
    s[j] = (uint32_t)cg_bounded(cg_rand(seed, stream, 2 * j), n);
    t[j] = (uint32_t)cg_bounded(cg_rand(seed, stream, 2 * j + 1), n);
  }
  return (int64_t)q;
}
