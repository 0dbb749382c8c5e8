// dp.cuh — per-edge coefficient DP of the blowup STTSV (row a3 of SURVEY.md §8(a)).
//
// For an edge e = {u_0..u_{K-1}} and global rank N, Alg. 2
// gives member v the coefficient
//     (N-1)! [t^{N-1}]  e^{x_v t} prod_{u in e\v} (e^{x_u t} - 1)
// (E_N / Ebar_N are the truncated EGFs of e^{ct} and e^{ct}-1),
// to be scaled by w(e)/|beta(e)|.  Write
//     e^{x t} - 1 = t g(t),   g[j] = x^{j+1}/(j+1)!   (j >= 0)
// and e^{x_v t} = 1 + t g_v(t).  Then, with D = N - K,
//     [t^{N-1}] e^{x_v t} prod_{u!=v} (e^{x_u t}-1) = [t^D] prod_{u!=v} g_u  +  [t^{D-1}] prod_u g_u
//                                                   =        Q_v[D]          +       F[D-1].
// Only coefficients 0..D of each g are ever needed (L = D + 1 of them), and
// every term is a product of positive numbers when x > 0 (no cancellation).
// Q_v = P_{i-1} S_{i+1} with prefix products P_i = g_0..g_i and suffix products
// S_i = g_i..g_{K-1}; [t^D] of a product is a length-L dot product.
//
// The series g of every active vertex is tabulated once per apply (gather /
// normalize kernels, `series_row`), so the edge kernel loads g rows instead of
// recomputing powers per incidence.  dp_core<K, L> returns q_i = Q_{u_i}[D] and
// F = F[D-1], so c_i = q_i + F (WITHOUT the (N-1)!/|beta| factor: the planner
// folds (N-1)!/|beta(K)| into the stored weight w'; the kernel forms
// w' c_i = fma(w', q_i, w' F)).  All loops are over compile-time bounds, so the
// arrays live in registers.
#pragma once

namespace sttsv {


// The table writer.  norm = 0: g[j] = x^{j+1}/(j+1)!, j = 0..GS-1.
// norm = 1 (large-rank path): g[0] = x and g[j] = h[j] = x^j/(j+1)! for j >= 1,
// the series normalised to a leading 1 (g_full = x * h, h[0] = 1 implicit).
__device__ __forceinline__ void series_row(double x, double* __restrict__ g, int GS, int norm = 0) {
  if (norm) {
    double pw = 1.0, f = 1.0;
    g[0] = x;
    for (int j = 1; j < GS; ++j) {
      pw *= x;
      f *= double(j + 1);
      g[j] = pw * (1.0 / f);
    }
  } else {
    double pw = x, f = 1.0;
    g[0] = pw;
    for (int j = 1; j < GS; ++j) {
      pw *= x;
      f *= double(j + 1);
      g[j] = pw * (1.0 / f);
    }
  }
}

// load coefficients 0..L-1 of one table row with 128-bit loads (rows are 32-B
// aligned with a stride that is a multiple of 4 and >= L, so an odd L reads one
// unused coefficient inside the row).  (256-bit LDG.E.ENL2.256 loads measured
// 1.4x slower on the edge kernel.)
template <int L>
__device__ __forceinline__ void load_series(const double* __restrict__ row, double (&g)[L]) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int j = 0; j < L; j += 2) {
    const double2 v = __ldg(r2 + j / 2);
    g[j] = v.x;
    if (j + 1 < L) g[j + 1] = v.y;
  }
}

// truncated product r = (a*b) mod t^L
template <int L>
__device__ __forceinline__ void trunc_mul(const double (&a)[L], const double (&b)[L], double (&r)[L]) {
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s = a[0] * b[j];
#pragma unroll
    for (int i = 1; i <= j; ++i) s = fma(a[i], b[j - i], s);
    r[j] = s;
  }
}

// [t^D] (a*b) over the first D+1 coefficients
template <int D, int L>
__device__ __forceinline__ double coef(const double (&a)[L], const double (&b)[L]) {
  static_assert(D < L, "coef degree");
  double s = a[0] * b[D];
#pragma unroll
  for (int j = 1; j <= D; ++j) s = fma(a[j], b[D - j], s);
  return s;
}

// K >= 2 members with series g[i][0..L-1]; prefix products P[i] = g_0 * ... * g_i
// (i = 0..K-3) and a running suffix S.
template <int K, int L>
__device__ __forceinline__ void dp_core(const double (&g)[K][L], double (&q)[K], double& F) {
  static_assert(K >= 2, "dp_core needs K >= 2");
  constexpr int D = L - 1;
  F = 0.0;
  if constexpr (K == 2) {
    if constexpr (D >= 1) F = coef<D - 1, L>(g[0], g[1]);
    q[0] = g[1][D];
    q[1] = g[0][D];
  } else {
    double P[K - 2][L];
#pragma unroll
    for (int j = 0; j < L; ++j) P[0][j] = g[0][j];
#pragma unroll
    for (int i = 1; i <= K - 3; ++i) trunc_mul<L>(P[i - 1], g[i], P[i]);
    // last two members
    q[K - 1] = coef<D, L>(P[K - 3], g[K - 2]);   // [t^D] P_{K-2}
    q[K - 2] = coef<D, L>(P[K - 3], g[K - 1]);   // [t^D] P_{K-3} S_{K-1}
    double S[L];
    trunc_mul<L>(g[K - 2], g[K - 1], S);          // S_{K-2}
    if constexpr (D >= 1) F = coef<D - 1, L>(P[K - 3], S);   // [t^{D-1}] P_{K-3} S_{K-2}
#pragma unroll
    for (int i = K - 3; i >= 1; --i) {
      q[i] = coef<D, L>(P[i - 1], S);            // [t^D] P_{i-1} S_{i+1}
      if (i > 1) {
        double T[L];
        trunc_mul<L>(g[i], S, T);                 // S_i
#pragma unroll
        for (int j = 0; j < L; ++j) S[j] = T[j];
      } else {
        q[0] = coef<D, L>(g[1], S);               // [t^D] S_1 = [t^D] g_1 S_2
      }
    }
    if constexpr (K == 3) q[0] = S[D];           // S = S_1
  }
}

// One edge from the series table: rows[i] = table row of member i.
template <int K, int L>
__device__ __forceinline__ void dp_edge_table(const double* const (&rows)[K], double (&q)[K], double& F) {
  constexpr int D = L - 1;
  if constexpr (K == 1) {
    // singleton: Q = 1 (empty product), F = g_0:  q = [D == 0],  F[D-1] = x^D / D!
    q[0] = D == 0 ? 1.0 : 0.0;
    F = D >= 1 ? __ldg(rows[0] + (D >= 1 ? D - 1 : 0)) : 0.0;
  } else {
    double g[K][L];
#pragma unroll
    for (int i = 0; i < K; ++i) load_series<L>(rows[i], g[i]);
    dp_core<K, L>(g, q, F);
  }
}

// ---- the same DP on series normalised to a leading 1 (table rows: slot 0 = x,
// h[j] = x^j/(j+1)! for j >= 1; g_u = x_u h_u).  Truncated products of
// normalised series skip the multiplications by the leading 1 (L(L-1)/2
// operations instead of L(L+1)/2); the scalar prefix / suffix products of the
// x_u are carried separately.  Used for ranks N >= 11 (L up to N-1).

// r = (a*b) mod t^L with a[0] = b[0] = r[0] = 1: slot 0 of a normalised series
// is never read or written (the leading 1 stays implicit, no register moves)
template <int L>
__device__ __forceinline__ void trunc_mul_norm(const double (&a)[L], const double (&b)[L], double (&r)[L]) {
#pragma unroll
  for (int j = 1; j < L; ++j) {
    double s = a[j] + b[j];
#pragma unroll
    for (int i = 1; i < j; ++i) s = fma(a[i], b[j - i], s);
    r[j] = s;
  }
}

// [t^D] (a*b) with a[0] = b[0] = 1
template <int D, int L>
__device__ __forceinline__ double coef_n(const double (&a)[L], const double (&b)[L]) {
  static_assert(D < L, "coef degree");
  if constexpr (D == 0) {
    return 1.0;
  } else {
    double s = a[D] + b[D];
#pragma unroll
    for (int j = 1; j < D; ++j) s = fma(a[j], b[D - j], s);
    return s;
  }
}

template <int K, int L>
__device__ __forceinline__ void dp_edge_table_norm(const double* const (&rows)[K], double (&q)[K], double& F) {
  constexpr int D = L - 1;
  F = 0.0;
  if constexpr (K == 1) {
    // singleton: q = [D == 0], F = g_0[D-1] = x h[D-1]
    const double x = __ldg(rows[0]);
    q[0] = D == 0 ? 1.0 : 0.0;
    if constexpr (D == 1) F = x;
    if constexpr (D >= 2) F = x * __ldg(rows[0] + (D - 1));
  } else {
    double h[K][L], x[K];  // h[i][0] holds x_i (slot 0 of a normalised series is implicit 1)
#pragma unroll
    for (int i = 0; i < K; ++i) {
      load_series<L>(rows[i], h[i]);
      x[i] = h[i][0];
    }
    if constexpr (K == 2) {
      if constexpr (D >= 1) F = x[0] * x[1] * coef_n<D - 1, L>(h[0], h[1]);
      q[0] = D == 0 ? x[1] : x[1] * h[1][D];
      q[1] = D == 0 ? x[0] : x[0] * h[0][D];
    } else {
      double P[K - 2][L], Xp[K - 2];
#pragma unroll
      for (int j = 0; j < L; ++j) P[0][j] = h[0][j];
      Xp[0] = x[0];
#pragma unroll
      for (int i = 1; i <= K - 3; ++i) {
        trunc_mul_norm<L>(P[i - 1], h[i], P[i]);
        Xp[i] = Xp[i - 1] * x[i];
      }
      q[K - 1] = Xp[K - 3] * x[K - 2] * coef_n<D, L>(P[K - 3], h[K - 2]);
      q[K - 2] = Xp[K - 3] * x[K - 1] * coef_n<D, L>(P[K - 3], h[K - 1]);
      double S[L];
      trunc_mul_norm<L>(h[K - 2], h[K - 1], S);
      double Xs = x[K - 2] * x[K - 1];
      if constexpr (D >= 1) F = Xp[K - 3] * Xs * coef_n<D - 1, L>(P[K - 3], S);
#pragma unroll
      for (int i = K - 3; i >= 1; --i) {
        q[i] = Xp[i - 1] * Xs * coef_n<D, L>(P[i - 1], S);
        if (i > 1) {
          double T[L];
          trunc_mul_norm<L>(h[i], S, T);
#pragma unroll
          for (int j = 0; j < L; ++j) S[j] = T[j];
          Xs *= x[i];
        } else {
          q[0] = x[1] * Xs * coef_n<D, L>(h[1], S);
        }
      }
      if constexpr (K == 3) q[0] = D == 0 ? Xs : Xs * S[D];
    }
  }
}

}  // namespace sttsv
