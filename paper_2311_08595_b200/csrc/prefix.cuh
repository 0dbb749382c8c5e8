// prefix.cuh — shared-prefix memoisation of the per-edge DP (
// the idea of the paper's CCSS storage and Alg. 4 memoisation, PAPER.md:404-429,
// 616-689: edges that share a sorted prefix share its partial products).
//
// The plan sorts every cardinality bucket lexicographically (degree-relabelled
// ids, hot vertices first) and records, per tile, U = the length of the member
// prefix (u_0 .. u_{U-1}) that ALL edges of the tile share (the common prefix
// of the tile's first and last edge).  Under the configs' Zipf popularity most
// tiles share long prefixes (large: 91% of the incidences lie in a shared
// prefix; two thirds of its tiles are runs of one repeated vertex set).
//
// For such a tile write A = prod_{j<U} g_j (the shared part, a tile constant)
// and B_e = prod_{j>=U} g_j (the edge's own members), with g the shifted
// series of dp.cuh, D = N-K.  Then for every edge
//     F = [t^{D-1}] A B_e,
//     member i >= U:  q_i = [t^D] A prod_{j>=U, j!=i} g_j     (per edge: the DP
//                     of dp.cuh over the M = K-U own members with A in front),
//     member i <  U:  w'(q_i + F) = w' ([t^D] A_{\i} B_e + [t^{D-1}] A B_e),
// with A_{\i} = prod_{j<U, j!=i} g_j.  The prefix members' contributions are
// LINEAR in B_e, so over all edges e of a prefix group
//     sum_e w'_e (q_i + F) = [t^D] A_{\i} SB + [t^{D-1}] A SB,   SB = sum_e w'_e B_e.
// A lane therefore only accumulates the L-term series SB over its edges of the
// tile; per tile the warp sums SB and the prefix members' totals are the dot
// products  sum_j C_i[j] SB[j]  with
//     C_i[j] = A_{\i}[D-j] + A[D-1-j]   (the second term for j <= D-1),
// rows that depend only on x and the prefix, so they are formed ONCE per apply
// per prefix group (group_kernel, kernels.cu) — consecutive tiles with the same
// bucket, U and prefix ids form a group (plan.cpp).  Per edge the DP shrinks
// from K members to the M own members (+ the front A), the U shared id columns
// are not streamed at all, and a tile whose edges are all the same set (M = 0)
// costs one addition per edge.
//
// Exact in real arithmetic (it regroups the same products); every product is
// still of positive terms for x > 0.
//
// Group table (doubles, one record per group at goff[g]):
//     [ A in row format: L ][ C_0 .. C_{U-1}: U x L ][ prefix ids: U, int64 bit patterns ]
// The ids are written by the planner, A and C by group_kernel every apply.
#pragma once

#include "dp.cuh"

namespace sttsv {

// Per-edge DP with a front series: members 0 = A (row format: a[0] = X_A, a[1..L-1]
// the normalised coefficients, implicit leading 1) and the M own members
// (h[i] row format: h[i][0] = x_i).  Returns q[i] = [t^D] A prod_{j!=i} g_j for
// the own members, F = [t^{D-1}] A B, and B = prod g_i in row format (bh[0] = X_B).
template <int M, int L>
__device__ __forceinline__ void dp_front_norm(const double (&a)[L], const double (&h)[M][L], double (&q)[M],
                                              double& F, double (&bh)[L]) {
  static_assert(M >= 1, "dp_front_norm needs an own member");
  constexpr int D = L - 1;
  const double Xa = a[0];
  F = 0.0;
  if constexpr (M == 1) {
    const double x = h[0][0];
    if constexpr (D >= 1) F = Xa * x * coef_n<D - 1, L>(a, h[0]);
    q[0] = D == 0 ? Xa : Xa * a[D];  // [t^D] A
#pragma unroll
    for (int j = 0; j < L; ++j) bh[j] = h[0][j];
  } else {
    // K' = M + 1 members g'_0 = A, g'_i = h[i-1]; prefix chain P'_0 .. P'_{M-2}
    constexpr int KP = M + 1;
    double P[KP - 2][L], Xp[KP - 2];
#pragma unroll
    for (int j = 1; j < L; ++j) P[0][j] = a[j];
    Xp[0] = Xa;
#pragma unroll
    for (int i = 1; i <= KP - 3; ++i) {
      trunc_mul_norm<L>(P[i - 1], h[i - 1], P[i]);
      Xp[i] = Xp[i - 1] * h[i - 1][0];
    }
    const double xa = h[KP - 3][0], xb = h[KP - 2][0];  // g'_{K'-2}, g'_{K'-1}
    q[KP - 2] = Xp[KP - 3] * xa * coef_n<D, L>(P[KP - 3], h[KP - 3]);  // own member M-1
    q[KP - 3] = Xp[KP - 3] * xb * coef_n<D, L>(P[KP - 3], h[KP - 2]);  // own member M-2
    double S[L];
    trunc_mul_norm<L>(h[KP - 3], h[KP - 2], S);
    double Xs = xa * xb;
    if constexpr (D >= 1) F = Xp[KP - 3] * Xs * coef_n<D - 1, L>(P[KP - 3], S);
#pragma unroll
    for (int i = KP - 3; i >= 1; --i) {
      q[i - 1] = Xp[i - 1] * Xs * coef_n<D, L>(P[i - 1], S);  // own member i-1
      double T[L];
      trunc_mul_norm<L>(h[i - 1], S, T);  // S'_i = g'_i S'_{i+1}
#pragma unroll
      for (int j = 1; j < L; ++j) S[j] = T[j];
      Xs *= h[i - 1][0];
    }
    bh[0] = Xs;  // S'_1 = B
#pragma unroll
    for (int j = 1; j < L; ++j) bh[j] = S[j];
  }
}

}  // namespace sttsv
