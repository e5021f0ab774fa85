/*
 * cbfs_gen.h — seeded synthetic input generators (libcbfsgen.so).
 *
 * This module is the ONLY code shared by the CUDA product path and the CPU
 * oracle.  It holds none of the method's arithmetic (no CSR normalisation, no
 * traversal, no selection): it emits raw, possibly duplicated / self-looped,
 * undirected edge lists as COO pairs and random query pairs.  Both sides then
 * normalise (symmetrise, dedup, drop self loops, sort) on their own.
 *
 * Workload shapes follow BASELINE.json `configs` (ER n=4096 / RMAT-20 ef16 /
 * RMAT-24 ef32 / 4096^2 grid / 10M-point 3-D k-NN) and the generator readings
 * R21-R24 of SURVEY.md §8(c) (recorded in DESIGN.md §3).
 *
 * Random numbers: a counter-based SplitMix64, cg_rand(seed, stream, index),
 * so every draw is a pure function of its coordinates (thread-count
 * independent, reproducible on any host).  The product's random-root
 * cluster selection implements the same counter-based function on its own
 * (paper_2410_17226_b200/csrc) — that is the only RNG either side draws.
 *
 * Ownership: all output arrays are caller-allocated host memory.
 * Errors: functions return the number of pairs written (>=0) or -1 on a bad
 * argument (null pointer, n == 0, capacity too small).
 */
#ifndef CBFS_GEN_H
#define CBFS_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64 finaliser and the counter-based draw used everywhere. */
uint64_t cg_mix64(uint64_t z);
uint64_t cg_rand(uint64_t seed, uint64_t stream, uint64_t index);
/* floor(x * n / 2^64): unbiased-enough bounded draw, exact integer arithmetic. */
uint64_t cg_bounded(uint64_t x, uint64_t n);

/* Erdos-Renyi G(n, pairs): `pairs` endpoint pairs drawn with replacement
 * (u = bounded(rand(seed,0,2t)), v = bounded(rand(seed,0,2t+1))).  Writes
 * exactly `pairs` pairs into src/dst[pairs]. */
int64_t cg_erdos_renyi(uint32_t n, uint64_t pairs, uint64_t seed,
                       uint32_t* src, uint32_t* dst);

/* R-MAT (Chakrabarti et al.) with 2^scale vertices and `edges` pairs.
 * Level l of edge t draws u = rand(seed, 0, t*scale + l) as a dyadic double
 * in [0,1) and picks quadrant a / b / c / d by comparison with the cumulative
 * a, a+b, a+b+c.  If `scramble` != 0 the ids are passed through a seeded
 * bijection of [0, 2^scale) (Graph500-style, so hubs are not at low ids). */
int64_t cg_rmat(int scale, uint64_t edges, double a, double b, double c,
                uint64_t seed, int scramble, int threads,
                uint32_t* src, uint32_t* dst);

/* side x side 4-neighbour grid, id = y*side + x.  Each of the 2*side*(side-1)
 * grid edges is deleted iff its uniform draw < p_delete; then
 * llround(p_diag * 2*side*(side-1)) diagonal shortcuts (x,y)-(x+1,y+1) at
 * uniform positions.  Capacity must be >= cg_grid_capacity(side, p_diag). */
uint64_t cg_grid_capacity(uint32_t side, double p_diag);
int64_t cg_grid(uint32_t side, double p_delete, double p_diag, uint64_t seed,
                uint64_t capacity, uint32_t* src, uint32_t* dst);

/* n points uniform in [0,1)^3 with coordinates (rand >> 40) * 2^-24 (exact
 * float32 values); each point emits its k nearest other points (squared
 * Euclidean distance computed exactly in integers, ties -> smaller index) as
 * k directed pairs (i, j).  Writes n*k pairs.  coords (optional, may be NULL)
 * receives the 24-bit integer coordinates [n][3]. */
int64_t cg_knn3d(uint32_t n, uint32_t k, uint64_t seed, int threads,
                 uint32_t* src, uint32_t* dst, uint32_t* coords);

/* q query pairs, s = bounded(rand(seed, stream, 2j), n),
 * t = bounded(rand(seed, stream, 2j+1), n); s == t allowed (R24). */
int64_t cg_query_pairs(uint32_t n, uint64_t q, uint64_t seed, uint64_t stream,
                       uint32_t* s, uint32_t* t);

#ifdef __cplusplus
}
#endif
#endif
