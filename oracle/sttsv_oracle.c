/* ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2311_08595_b200/csrc) and never forms E_N, never convolves and
 * never uses the per-edge DP of the CUDA path.
 *
 * What it computes is the plain definition of STTSV on the blowup tensor:
 *
 *   PAPER.md:335-337 (§II, Eq. 2):
 *       s_{i1} = sum_{i2..iN} B_{i1..iN} * prod_{k=2..N} b_{ik}
 *   PAPER.md:341-343 (§II, blowup tensor): for each edge e and each ordered
 *       N-tuple i in beta(e) (tuples over e whose support is exactly e),
 *       B_i = w(e) / |beta(e)|;
 *   PAPER.md:342 footnote: |beta(e)| = |e|! * S(N, |e|)  (Stirling 2nd kind).
 *   PAPER.md:29 (draft §II): the unordered blowups kappa(e) = size-N
 *       multisets with support e.
 *
 * Main mode ("kappa"): the ordered tuples of beta(e) are grouped by their
 * multiset m = (m_u)_{u in e} in kappa(e) (m_u >= 1, sum m_u = N).  Of the
 * N!/prod m_u! ordered tuples with that multiset, (N-1)!/((m_v-1)! prod_{u!=v} m_u!)
 * start with v, and each contributes w/|beta| * x_v^{m_v-1} prod_{u!=v} x_u^{m_u}
 * to s_v (Eq. 2).  Literal mode enumerates all |e|^N maps positions -> e,
 * keeps the surjective ones (the tuples of beta(e)) and adds
 * w/|beta| * prod_{j>=2} x_{i_j} to s_{i_1} — Eq. (2) tuple by tuple.
 *
 * Arithmetic: long double (x86 80-bit) accumulation; |beta| as an exact
 * integer (unsigned __int128) for N <= 26.  Edges are split over OpenMP
 * threads in fixed static chunks with per-thread partial sums reduced in
 * thread order, so a given thread count is deterministic.
 *
 * Parity pins (tests/test_oracle.py): Fig. 1 degree identity,
 * exact-rational brute force on tiny random hypergraphs, closed forms for
 * k=1, 2, N-1, N and N=2 (graph SpMV), homogeneity, linearity in w,
 * relabel-equivariance, Euler's identity x.s = B x^N computed without the
 * per-vertex split, and sum_k C(N,k) |beta(k)| = N^N.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC sttsv_oracle.c -o liboracle.so -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MAX_RANK 64

typedef unsigned __int128 u128;

/* Stirling numbers of the second kind by the textbook recurrence
 * S(n,k) = k S(n-1,k) + S(n-1,k-1), S(0,0) = 1 (PAPER.md:342 footnote). */
static int stirling2_u128(int N, int k, u128* out) {
  if (N < 0 || k < 0 || N > ORACLE_MAX_RANK || k > N) return -1;
  u128 S[ORACLE_MAX_RANK + 1][ORACLE_MAX_RANK + 1];
  memset(S, 0, sizeof(S));
  S[0][0] = 1;
  for (int a = 1; a <= N; ++a)
    for (int b = 1; b <= a; ++b) S[a][b] = (u128)b * S[a - 1][b] + S[a - 1][b - 1];
  *out = S[N][k];
  return 0;
}

/* |beta(e)| = k! S(N,k) as long double.  Exact (one rounding) while k!S(N,k)
 * fits in 128 bits (N <= 26); beyond that the long double recurrence is used. */
long double oracle_beta_ld(int N, int k) {
  if (k < 1 || k > N || N > ORACLE_MAX_RANK) return 0.0L;
  if (N <= 26) {
    u128 s;
    stirling2_u128(N, k, &s);
    u128 f = 1;
    for (int i = 2; i <= k; ++i) f *= (u128)i;
    return (long double)(s * f);
  }
  long double S[ORACLE_MAX_RANK + 1][ORACLE_MAX_RANK + 1];
  memset(S, 0, sizeof(S));
  S[0][0] = 1.0L;
  for (int a = 1; a <= N; ++a)
    for (int b = 1; b <= a; ++b) S[a][b] = (long double)b * S[a - 1][b] + S[a - 1][b - 1];
  long double f = 1.0L;
  for (int i = 2; i <= k; ++i) f *= (long double)i;
  return S[N][k] * f;
}

double oracle_beta(int N, int k) { return (double)oracle_beta_ld(N, k); }

/* S(N,k) exported for tests (as double). */
double oracle_stirling2(int N, int k) {
  u128 s;
  if (N > 26 || stirling2_u128(N, k, &s) != 0) return -1.0;
  return (double)s;
}

static long double factorial_ld(int a) {
  long double f = 1.0L;
  for (int i = 2; i <= a; ++i) f *= (long double)i;
  return f;
}

/* ------------------------------------------------------------------------ */
/* kappa mode: contributions of ONE edge to s_v for every member v.          */
/* out[i] receives the contribution to member i (long double).               */
/* ------------------------------------------------------------------------ */
typedef struct {
  int N, k;
  const double* xv;           /* x of the k members */
  long double invx[ORACLE_MAX_RANK];  /* 1 / x_u (x_u != 0) */
  long double val;            /* w / |beta| */
  long double fact[ORACLE_MAX_RANK + 1];
  long double pf[ORACLE_MAX_RANK][ORACLE_MAX_RANK + 1];   /* pf[u][t] = x_u^t / t! */
  int m[ORACLE_MAX_RANK];     /* current multiplicities */
  long double* out;
  long double* euler;         /* optional: accumulates sum over tuples of B_i prod x (all N factors) */
} kappa_ctx;

/* One multiset m in kappa(e), with T = prod_u x_u^{m_u} / m_u!: add the Eq. (2)
 * terms of the ordered tuples it groups.  Of its N!/prod m_u! tuples,
 * (N-1)!/((m_v-1)! prod_{u!=v} m_u!) start with v, and each adds
 * w/|beta| * x_v^{m_v-1} prod_{u!=v} x_u^{m_u} to s_v; together that is
 *     w/|beta| * (N-1)! * x_v^{m_v-1}/(m_v-1)! * prod_{u!=v} x_u^{m_u}/m_u!
 *   = w/|beta| * (N-1)! * T * m_v / x_v                       (x_v != 0),
 * the form written out in SURVEY.md §8(c).  For x_v = 0 only m_v = 1 survives
 * (x_v^0 = 1) and the product over u != v is formed directly.  The factor
 * w/|beta| * (N-1)!, common to every term of the edge, is applied once in
 * kappa_edge (out[v] here accumulates T * m_v / x_v). */
static void kappa_visit(kappa_ctx* c, long double T) {
  const int k = c->k;
  for (int v = 0; v < k; ++v) {
    long double term;
    if (c->xv[v] != 0.0) {
      term = T * (long double)c->m[v] * c->invx[v];
    } else if (c->m[v] == 1) {
      long double prod = 1.0L;
      for (int u = 0; u < k; ++u)
        if (u != v) prod *= c->pf[u][c->m[u]];
      term = prod;
    } else {
      term = 0.0L;
    }
    c->out[v] += term;
  }
  /* Euler form: all N!/prod m_u! tuples, each val * prod_u x_u^{m_u} = N T per
   * (N-1)! (the common factor applied in kappa_edge) */
  if (c->euler) *c->euler += (long double)c->N * T;
}

/* enumerate compositions m_0..m_{k-1} >= 1 with sum N; `part` carries
 * prod_{u < pos} x_u^{m_u}/m_u! down the enumeration */
static void kappa_rec(kappa_ctx* c, int pos, int remaining, long double part) {
  if (pos == c->k - 1) {
    c->m[pos] = remaining;
    kappa_visit(c, part * c->pf[pos][remaining]);
    return;
  }
  int slots_after = c->k - 1 - pos;
  for (int mv = 1; mv <= remaining - slots_after; ++mv) {
    c->m[pos] = mv;
    kappa_rec(c, pos + 1, remaining - mv, part * c->pf[pos][mv]);
  }
}

static void kappa_edge(int N, int k, const double* xv, long double val, long double* out,
                       long double* euler) {
  kappa_ctx c;
  c.N = N;
  c.k = k;
  c.xv = xv;
  c.val = val;
  c.out = out;
  c.euler = euler;
  for (int i = 0; i <= N; ++i) c.fact[i] = factorial_ld(i);
  for (int u = 0; u < k; ++u) {
    long double pw = 1.0L;
    c.invx[u] = xv[u] != 0.0 ? 1.0L / (long double)xv[u] : 0.0L;
    c.pf[u][0] = 1.0L;
    for (int t = 1; t <= N; ++t) {
      pw *= (long double)xv[u];
      c.pf[u][t] = pw / c.fact[t];
    }
  }
  for (int i = 0; i < k; ++i) out[i] = 0.0L;
  long double eu = 0.0L;
  if (euler) c.euler = &eu;
  kappa_rec(&c, 0, N, 1.0L);
  const long double common = val * c.fact[N - 1];   /* w/|beta| * (N-1)! */
  for (int i = 0; i < k; ++i) out[i] *= common;
  if (euler) *euler += common * eu;
}

/* literal mode for one edge: all k^N maps positions -> members, surjective only */
static void literal_edge(int N, int k, const double* xv, long double val, long double* out) {
  int pos[ORACLE_MAX_RANK];
  int hit[ORACLE_MAX_RANK];
  for (int i = 0; i < k; ++i) out[i] = 0.0L;
  for (int j = 0; j < N; ++j) pos[j] = 0;
  for (;;) {
    for (int i = 0; i < k; ++i) hit[i] = 0;
    for (int j = 0; j < N; ++j) hit[pos[j]] = 1;
    int surj = 1;
    for (int i = 0; i < k; ++i) surj &= hit[i];
    if (surj) {
      long double prod = 1.0L;
      for (int j = 1; j < N; ++j) prod *= (long double)xv[pos[j]];
      out[pos[0]] += val * prod;
    }
    int j = N - 1;
    while (j >= 0 && ++pos[j] == k) { pos[j] = 0; --j; }
    if (j < 0) break;
  }
}

static int validate(int64_t n, int N, int64_t m, const int32_t* sizes, const int64_t* offsets,
                    const int32_t* idx) {
  if (N < 1 || N > ORACLE_MAX_RANK || n < 0 || m < 0) return -1;
  for (int64_t e = 0; e < m; ++e) {
    int k = sizes[e];
    if (k < 1 || k > N || offsets[e + 1] - offsets[e] != k) return -2;
    for (int i = 0; i < k; ++i) {
      int32_t v = idx[offsets[e] + i];
      if (v < 0 || v >= n) return -3;
    }
  }
  return 0;
}

/* s = B x^{N-1}.  mode 0: kappa grouping, mode 1: literal tuples.
 * y has length n and is overwritten.  Returns 0 or a negative error. */
int oracle_sttsv(int64_t n, int N, int64_t m, const int32_t* sizes, const int64_t* offsets,
                 const int32_t* idx, const double* w, const double* x, double* y, int mode,
                 int nthreads) {
  int rc = validate(n, N, m, sizes, offsets, idx);
  if (rc) return rc;
  long double beta[ORACLE_MAX_RANK + 1];
  for (int k = 1; k <= N; ++k) beta[k] = oracle_beta_ld(N, k);
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
  nthreads = 1;
#endif
  /* per-thread partial sums, reduced in thread order */
  long double* part = (long double*)calloc((size_t)n * (size_t)nthreads, sizeof(long double));
  if (!part && n) return -4;
#pragma omp parallel num_threads(nthreads)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    long double* my = part + (size_t)t * (size_t)n;
    double xv[ORACLE_MAX_RANK];
    long double out[ORACLE_MAX_RANK];
#pragma omp for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
      int k = sizes[e];
      const int32_t* ev = idx + offsets[e];
      for (int i = 0; i < k; ++i) xv[i] = x[ev[i]];
      long double val = (long double)w[e] / beta[k];
      if (mode == 1) literal_edge(N, k, xv, val, out);
      else kappa_edge(N, k, xv, val, out, NULL);
      for (int i = 0; i < k; ++i) my[ev[i]] += out[i];
    }
  }
  for (int64_t v = 0; v < n; ++v) {
    long double s = 0.0L;
    for (int t = 0; t < nthreads; ++t) s += part[(size_t)t * (size_t)n + (size_t)v];
    y[v] = (double)s;
  }
  free(part);
  return 0;
}

/* s_v for a list of vertices, one by one: each sums the kappa contributions
 * of the edges that contain it (sampled-output parity at full size). */
int oracle_sttsv_vertices(int64_t n, int N, int64_t m, const int32_t* sizes, const int64_t* offsets,
                          const int32_t* idx, const double* w, const double* x, int64_t nv,
                          const int64_t* verts, double* out_y, int nthreads) {
  int rc = validate(n, N, m, sizes, offsets, idx);
  if (rc) return rc;
  long double beta[ORACLE_MAX_RANK + 1];
  for (int k = 1; k <= N; ++k) beta[k] = oracle_beta_ld(N, k);
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#endif
  for (int64_t q = 0; q < nv; ++q) {
    int64_t v = verts[q];
    long double acc = 0.0L;
#pragma omp parallel for schedule(static) reduction(+ : acc) num_threads(nthreads)
    for (int64_t e = 0; e < m; ++e) {
      int k = sizes[e];
      const int32_t* ev = idx + offsets[e];
      int pos = -1;
      for (int i = 0; i < k; ++i) if (ev[i] == v) pos = i;
      if (pos < 0) continue;
      double xv[ORACLE_MAX_RANK];
      long double out[ORACLE_MAX_RANK];
      for (int i = 0; i < k; ++i) xv[i] = x[ev[i]];
      kappa_edge(N, k, xv, (long double)w[e] / beta[k], out, NULL);
      acc += out[pos];
    }
    out_y[q] = (double)acc;
  }
  return 0;
}

/* Euler form B x^N = sum over all tuples of B_i prod_{j=1..N} x_{ij}, grouped by
 * kappa(e) (N!/prod m_u! tuples per multiset) — no per-vertex split. */
int oracle_full_contraction(int64_t n, int N, int64_t m, const int32_t* sizes, const int64_t* offsets,
                            const int32_t* idx, const double* w, const double* x, double* out) {
  int rc = validate(n, N, m, sizes, offsets, idx);
  if (rc) return rc;
  long double beta[ORACLE_MAX_RANK + 1];
  for (int k = 1; k <= N; ++k) beta[k] = oracle_beta_ld(N, k);
  long double total = 0.0L;
  double xv[ORACLE_MAX_RANK];
  long double tmp[ORACLE_MAX_RANK];
  for (int64_t e = 0; e < m; ++e) {
    int k = sizes[e];
    const int32_t* ev = idx + offsets[e];
    for (int i = 0; i < k; ++i) xv[i] = x[ev[i]];
    long double euler = 0.0L;
    kappa_edge(N, k, xv, (long double)w[e] / beta[k], tmp, &euler);
    total += euler;
  }
  *out = (double)total;
  return 0;
}

/* number of kappa terms (compositions) an apply enumerates: sum_e C(N-1, k-1) */
double oracle_kappa_terms(int N, int64_t m, const int32_t* sizes) {
  double tot = 0.0;
  for (int64_t e = 0; e < m; ++e) {
    int k = sizes[e];
    double c = 1.0;
    for (int i = 1; i <= k - 1; ++i) c = c * (double)(N - 1 - (k - 1) + i) / (double)i;
    tot += c;
  }
  return tot;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
