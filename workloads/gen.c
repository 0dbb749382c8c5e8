/* Seeded synthetic hypergraph generator shared by the oracle and the CUDA path.
 *
 * This file holds NO STTSV arithmetic: it only draws edge sizes, member
 * vertices, weights and the input vector x for the BASELINE.json configs,
 * under the readings A9-A13 recorded in DESIGN.md.
 *
 * Randomness is counter-based: every draw is a function of
 * (seed, stream, index), so results do not depend on the thread count.
 *   stream 1: edge sizes        (index = candidate edge)
 *   stream 2: member vertices   (index = candidate edge)
 *   stream 3: weights           (index = edge)
 *   stream 4: x                 (index = vertex)
 *   stream 5: rank -> id permutation (one sequential stream)
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC gen.c -o libgen.so -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- RNG ---- */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;

static inline rng_t rng_at(uint64_t seed, uint64_t stream, uint64_t index) {
  rng_t r;
  r.s = mix64(mix64(seed ^ (stream * 0xd1b54a32d192ed03ULL)) ^ mix64(index + 0x632be59bd9b4e019ULL));
  return r;
}

static inline uint64_t rng_next(rng_t* r) {
  r->s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = r->s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* uniform in [0,1) with 53 random bits */
static inline double rng_u01(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
/* uniform in (0,1]  (reading A12: "(0,1]" draws are 1 - U[0,1)) */
static inline double rng_u01_open0(rng_t* r) { return 1.0 - rng_u01(r); }

/* ------------------------------------------ Zipf over {1..n}, exponent s -- */
/* P(k) proportional to k^-s on {1..n}, s > 1 (every config draws members with
 * s = 2.0 or 2.2).  The rejection method for the Zipf law in L. Devroye,
 * "Non-Uniform Random Variate Generation" (Springer 1986), ch. X §6.1:
 * propose X = floor(U^(-1/(s-1))) (a discretised Pareto variable), accept
 * when V X (T - 1) / (b - 1) <= T / b with T = (1 + 1/X)^(s-1) and
 * b = 2^(s-1).  That samples the unbounded law on {1, 2, ...}; proposals
 * above n are rejected too, which conditions it on {1..n} (reading A9). */
typedef struct {
  double n;         /* upper end of the support */
  double inv_sm1;   /* 1/(s-1) */
  double sm1;       /* s-1 */
  double b;         /* 2^(s-1) */
} zipf_law;

static void zipf_law_init(zipf_law* z, int64_t n, double s) {
  z->n = (double)n;
  z->sm1 = s - 1.0;
  z->inv_sm1 = 1.0 / (s - 1.0);
  z->b = pow(2.0, s - 1.0);
}

static inline int64_t zipf_law_draw(const zipf_law* z, rng_t* r) {
  for (;;) {
    const double u = rng_u01_open0(r); /* (0,1]: the power below stays finite */
    const double v = rng_u01(r);
    const double x = floor(z->sm1 == 1.0 ? 1.0 / u : pow(u, -z->inv_sm1));
    if (x > z->n) continue;           /* outside {1..n}: condition by rejection */
    const double t = z->sm1 == 1.0 ? 1.0 + 1.0 / x : pow(1.0 + 1.0 / x, z->sm1);
    if (v * x * (t - 1.0) / (z->b - 1.0) <= t / z->b) return (int64_t)x;
  }
}

/* ------------------------------------------------------------- exports --- */
int gen_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* sizes[i] for candidate edges i in [first, first+count): inverse CDF on a
 * table cdf[0..nk-1] over sizes kmin..kmin+nk-1 (cdf[nk-1] == 1). */
void gen_sizes(uint64_t seed, int64_t first, int64_t count, int32_t kmin, int32_t nk,
               const double* cdf, int32_t* sizes) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    rng_t r = rng_at(seed, 1, (uint64_t)(first + i));
    double u = rng_u01(&r);
    int32_t j = 0;
    while (j < nk - 1 && u >= cdf[j]) ++j;
    sizes[i] = kmin + j;
  }
}

/* Random permutation perm[rank-1] = vertex id, Fisher-Yates on stream 5. */
void gen_permutation(uint64_t seed, int64_t n, int32_t* perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  rng_t r = rng_at(seed, 5, 0);
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)(rng_u01(&r) * (double)(i + 1));
    if (j > i) j = i;
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Members of candidate edges [first, first+count).  offsets[i] is the start of
 * edge i in idx (relative to idx).  kind 0: uniform without replacement over
 * {0..n-1}; kind 1: Zipf(s) popularity over ranks, successive sampling
 * without replacement (draw with replacement, discard repeats), rank -> id
 * via perm.  Each edge's ids are written sorted ascending (IOU form).
 * Returns the total number of draws (for statistics). */
int64_t gen_members(uint64_t seed, int64_t n, int64_t first, int64_t count,
                    const int32_t* sizes, const int64_t* offsets, int32_t kind,
                    double s, const int32_t* perm, int32_t* idx) {
  zipf_law z;
  if (kind == 1) zipf_law_init(&z, n, s);
  int64_t draws_total = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : draws_total)
  for (int64_t i = 0; i < count; ++i) {
    rng_t r = rng_at(seed, 2, (uint64_t)(first + i));
    int32_t k = sizes[i];
    int32_t* e = idx + offsets[i];
    int32_t have = 0;
    while (have < k) {
      int32_t v;
      if (kind == 1) {
        v = perm[zipf_law_draw(&z, &r) - 1];
      } else {
        int64_t j = (int64_t)(rng_u01(&r) * (double)n);
        if (j >= n) j = n - 1;
        v = (int32_t)j;
      }
      ++draws_total;
      int dup = 0;
      for (int32_t q = 0; q < have; ++q) if (e[q] == v) { dup = 1; break; }
      if (!dup) e[have++] = v;
    }
    qsort(e, (size_t)k, sizeof(int32_t), cmp_i32);
  }
  return draws_total;
}

/* Weights: kind 0 uniform (0,1]; kind 1 lognormal(mu, sigma) = exp(N(mu,sigma));
 * kind 2 constant a. */
void gen_weights(uint64_t seed, int64_t m, int32_t kind, double a, double b, double* w) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    rng_t r = rng_at(seed, 3, (uint64_t)i);
    if (kind == 0) {
      w[i] = rng_u01_open0(&r);
    } else if (kind == 1) {
      double u1 = rng_u01_open0(&r), u2 = rng_u01(&r);
      double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
      w[i] = exp(a + b * g);
    } else {
      w[i] = a;
    }
  }
}

/* x uniform (0,1] on stream 4 */
void gen_x(uint64_t seed, int64_t n, double* x) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    rng_t r = rng_at(seed, 4, (uint64_t)i);
    x[i] = rng_u01_open0(&r);
  }
}

/* raw uniform [0,1) draws on an arbitrary stream (tests of the generator) */
void gen_uniform(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) {
    rng_t r = rng_at(seed, stream, (uint64_t)i);
    out[i] = rng_u01(&r);
  }
}

/* raw Zipf draws (tests of the generator) */
void gen_zipf(uint64_t seed, int64_t n, double s, int64_t count, int64_t* out) {
  zipf_law z;
  zipf_law_init(&z, n, s);
  rng_t r = rng_at(seed, 6, 0);
  for (int64_t i = 0; i < count; ++i) out[i] = zipf_law_draw(&z, &r);
}
