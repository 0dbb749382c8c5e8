// edge_kernel.cuh — the hot kernel of one STTSV apply.
//
// Work decomposition.  The plan stores each cardinality bucket k as SoA int32
// id columns + fp64 weights w' = w (N-1)!/|beta(k)| (PAPER.md:342 footnote and
// Alg. 2's factor), edges sorted lexicographically by their
// (degree-relabelled, ascending) member ids.  A tile is TILE = 32*NCW
// consecutive edges of one bucket; tiles are ordered most-expensive bucket
// first and dealt to the persistent CTAs round-robin.
//
// Warp specialisation.  Per CTA, one producer warp streams tiles into an
// STAGES-deep shared-memory ring with 1-D TMA bulk copies (cp.async.bulk ->
// SASS UBLKCP, completion on a `full` mbarrier with expect_tx); NCW consumer
// warps each take 32 edges of the tile (one edge per lane), run the fully
// unrolled register DP of dp.cuh for (k, L = N-k+1), and release the stage on
// an `empty` mbarrier.  No CTA-wide barrier sits on the tile loop.
//
// Scatter.  Because edges are sorted, the 32 lanes of a warp mostly hold the
// SAME vertex in a given slot (the hottest vertices sit in the low slots).
// For each slot the warp reduces its 32 contributions over runs of equal
// adjacent ids (a shuffle butterfly when the whole warp is one run, else a
// segmented suffix scan), and only each run's head lane deposits:
//   slot i holds vertex i (i < kDiag)  -> register accumulator racc[i]
//   id < H                             -> CTA shared accumulator sacc (atomicAdd)
//   id >= H                            -> red.global.add.f64 into y_a
// Each CTA flushes racc and sacc into y_a once, after its last tile.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dp.cuh"
#include "internal.h"

namespace sttsv {

constexpr int kDiag = 8;
constexpr unsigned kFull = 0xffffffffu;

template <int N>
struct EdgeCfg {
  static constexpr int NCW = (N >= 1 && N <= 16) ? 8 : 4;  // consumer warps
  static constexpr int TILE = 32 * NCW;                    // edges per tile
  static constexpr int THREADS = TILE + 32;                // + one producer warp
  static constexpr int KMAX = N < 1 ? STTSV_MAX_RANK : N;
  static constexpr int STAGES = 4;
  static constexpr int MIN_BLOCKS = 2;
  static constexpr int STAGE_BYTES = TILE * (4 * KMAX + 8);
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------ scatter
__device__ __forceinline__ void deposit_run(int slot, int v, double d, double (&racc)[kDiag],
                                            double* __restrict__ sacc, double* __restrict__ ya, int H) {
  if (slot < kDiag && v == slot) {
#pragma unroll
    for (int q = 0; q < kDiag; ++q)
      if (q == slot) racc[q] += d;
  } else if (v < H) {
    atomicAdd(&sacc[v], d);
  } else {
    atomicAdd(&ya[v], d);
  }
}

// Reduce (v, d) over the warp's runs of equal adjacent v; each run's first
// lane deposits the run total.  v < 0 marks an empty lane (ragged tail).
__device__ __forceinline__ void warp_deposit(int slot, int v, double d, int lane, double (&racc)[kDiag],
                                             double* __restrict__ sacc, double* __restrict__ ya, int H) {
  const int v0 = __shfl_sync(kFull, v, 0);
  if (__all_sync(kFull, v == v0)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(kFull, d, o);
    if (lane == 0 && v >= 0) deposit_run(slot, v, d, racc, sacc, ya, H);
    return;
  }
  // segmented suffix scan: after the loop a lane holds the sum from itself to
  // the end of its run (f = "my run ends inside the span summed so far")
  const int vn = __shfl_down_sync(kFull, v, 1);
  int f = (lane == 31) || (vn != v);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double dn = __shfl_down_sync(kFull, d, o);
    const int fn = __shfl_down_sync(kFull, f, o);
    if (!f && lane + o < 32) {
      d += dn;
      f = fn;
    }
  }
  const int vp = __shfl_up_sync(kFull, v, 1);
  if ((lane == 0 || vp != v) && v >= 0) deposit_run(slot, v, d, racc, sacc, ya, H);
}

// 32 edges of a size-K bucket, one per lane, from the shared stage
template <int N, int K, int TILE>
__device__ __forceinline__ void warp_edges(const int32_t* __restrict__ sids, const double* __restrict__ sw,
                                           int col, bool valid, const double* __restrict__ xa,
                                           double (&racc)[kDiag], double* sacc, double* ya, int H, int lane) {
  constexpr int L = N - K + 1;
  int id[K];
  double x[K], c[K];
#pragma unroll
  for (int i = 0; i < K; ++i) id[i] = valid ? sids[i * TILE + col] : -1;
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = valid ? __ldg(xa + id[i]) : 0.0;
  const double w = valid ? sw[col] : 0.0;
  dp_edge<K, L>(x, c);
#pragma unroll
  for (int i = 0; i < K; ++i) warp_deposit(i, id[i], w * c[i], lane, racc, sacc, ya, H);
}

template <int N, int K, int TILE>
__device__ __forceinline__ void dispatch_k(int k, const int32_t* sids, const double* sw, int col, bool valid,
                                           const double* xa, double (&racc)[kDiag], double* sacc, double* ya,
                                           int H, int lane) {
  if constexpr (K <= N) {
    if (k == K) {
      warp_edges<N, K, TILE>(sids, sw, col, valid, xa, racc, sacc, ya, H, lane);
      return;
    }
    dispatch_k<N, K + 1, TILE>(k, sids, sw, col, valid, xa, racc, sacc, ya, H, lane);
  }
}

// ---------------------------------------------------------------- generic
// Runtime (K, L) DP for ranks without a compiled specialisation: same
// recurrence as dp_edge, arrays in local memory.
static __device__ __noinline__ void dp_edge_generic(int K, int L, const double* x, double* c) {
  const int D = L - 1;
  double g[STTSV_MAX_RANK][STTSV_MAX_RANK];
  for (int i = 0; i < K; ++i) {
    double pw = x[i], f = 1.0;
    g[i][0] = pw;
    for (int j = 1; j < L; ++j) {
      pw *= x[i];
      f *= double(j + 1);
      g[i][j] = pw / f;
    }
  }
  if (K == 1) {
    if (D == 0) {
      c[0] = 1.0;
    } else {
      double pw = x[0], f = 1.0;
      for (int j = 1; j < D; ++j) pw *= x[0];
      for (int j = 2; j <= D; ++j) f *= double(j);
      c[0] = pw / f;
    }
    return;
  }
  auto coefD = [&](const double* a, const double* b, int deg) {
    double s = a[0] * b[deg];
    for (int j = 1; j <= deg; ++j) s = fma(a[j], b[deg - j], s);
    return s;
  };
  auto tmul = [&](const double* a, const double* b, double* r) {
    for (int j = 0; j < L; ++j) {
      double s = a[0] * b[j];
      for (int i = 1; i <= j; ++i) s = fma(a[i], b[j - i], s);
      r[j] = s;
    }
  };
  if (K == 2) {
    double F = D >= 1 ? coefD(g[0], g[1], D - 1) : 0.0;
    c[0] = g[1][D] + F;
    c[1] = g[0][D] + F;
    return;
  }
  double P[STTSV_MAX_RANK][STTSV_MAX_RANK];
  for (int j = 0; j < L; ++j) P[0][j] = g[0][j];
  for (int i = 1; i <= K - 3; ++i) tmul(P[i - 1], g[i], P[i]);
  c[K - 1] = coefD(P[K - 3], g[K - 2], D);
  c[K - 2] = coefD(P[K - 3], g[K - 1], D);
  double S[STTSV_MAX_RANK], T[STTSV_MAX_RANK];
  tmul(g[K - 2], g[K - 1], S);
  double F = D >= 1 ? coefD(P[K - 3], S, D - 1) : 0.0;
  for (int i = K - 3; i >= 1; --i) {
    c[i] = coefD(P[i - 1], S, D);
    if (i > 1) {
      tmul(g[i], S, T);
      for (int j = 0; j < L; ++j) S[j] = T[j];
    } else {
      c[0] = coefD(g[1], S, D);
    }
  }
  if (K == 3) c[0] = S[D];
  for (int i = 0; i < K; ++i) c[i] += F;
}


template <int TILE>
__device__ __forceinline__ void warp_edges_generic(int N, int k, const int32_t* sids, const double* sw, int col,
                                                   bool valid, const double* xa, double (&racc)[kDiag],
                                                   double* sacc, double* ya, int H, int lane) {
  int id[STTSV_MAX_RANK];
  double x[STTSV_MAX_RANK], c[STTSV_MAX_RANK];
  for (int i = 0; i < k; ++i) {
    id[i] = valid ? sids[i * TILE + col] : -1;
    x[i] = valid ? __ldg(xa + id[i]) : 0.0;
  }
  dp_edge_generic(k, N - k + 1, x, c);
  const double w = valid ? sw[col] : 0.0;
  for (int i = 0; i < k; ++i) warp_deposit(i, id[i], w * c[i], lane, racc, sacc, ya, H);
}

// ------------------------------------------------------------- the kernel
// N == 0 is the generic instantiation (any rank <= STTSV_MAX_RANK).
template <int N>
__global__ void __launch_bounds__(EdgeCfg<N>::THREADS, EdgeCfg<N>::MIN_BLOCKS)
    edge_kernel(const __grid_constant__ EdgeKernelParams p) {
  using Cfg = EdgeCfg<N>;
  constexpr int TILE = Cfg::TILE, STAGES = Cfg::STAGES, KMAX = Cfg::KMAX, NCW = Cfg::NCW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // layout: [STAGES][ ids KMAX*TILE int32 | w TILE f64 ] | sacc [H] f64
  unsigned char* ring = smem_raw;
  double* sacc = reinterpret_cast<double*>(smem_raw + STAGES * Cfg::STAGE_BYTES);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t G = gridDim.x;

  for (int j = tid; j < p.H; j += Cfg::THREADS) sacc[j] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_proxy_async();
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------- producer warp: TMA bulk copies of tile t into stage it % STAGES
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += G, ++it) {
        const int s = (int)(it % STAGES);
        if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
        int b = 0;
        while (b + 1 < p.nb && t >= p.b[b + 1].tile_begin) ++b;
        const BucketDesc& bd = p.b[b];
        const int64_t e0 = (t - bd.tile_begin) * TILE;
        const int64_t cnt = bd.m - e0 < TILE ? bd.m - e0 : TILE;
        const uint32_t id_bytes = (uint32_t)(((cnt + 3) & ~3LL) * 4);
        const uint32_t w_bytes = (uint32_t)(((cnt + 1) & ~1LL) * 8);
        unsigned char* st = ring + s * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], id_bytes * bd.k + w_bytes);
        for (int i = 0; i < bd.k; ++i)
          bulk_g2s(st + i * TILE * 4, p.ids + bd.ids_off + i * bd.stride + e0, id_bytes, &full[s]);
        bulk_g2s(st + KMAX * TILE * 4, p.w + bd.w_off + e0, w_bytes, &full[s]);
      }
    }
  } else {
    // ---------------- consumer warps
    double racc[kDiag];
#pragma unroll
    for (int i = 0; i < kDiag; ++i) racc[i] = 0.0;
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += G, ++it) {
      const int s = (int)(it % STAGES);
      int b = 0;
      while (b + 1 < p.nb && t >= p.b[b + 1].tile_begin) ++b;
      const BucketDesc& bd = p.b[b];
      const int64_t e0 = (t - bd.tile_begin) * TILE + warp * 32;
      mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
      if (e0 < bd.m) {
        const unsigned char* st = ring + s * Cfg::STAGE_BYTES;
        const int32_t* sids = reinterpret_cast<const int32_t*>(st);
        const double* sw = reinterpret_cast<const double*>(st + KMAX * TILE * 4);
        const bool valid = e0 + lane < bd.m;
        const int col = warp * 32 + lane;
        if constexpr (N > 0) {
          dispatch_k<N, 1, TILE>(bd.k, sids, sw, col, valid, p.xa, racc, sacc, p.ya, p.H, lane);
        } else {
          warp_edges_generic<TILE>(p.N, bd.k, sids, sw, col, valid, p.xa, racc, sacc, p.ya, p.H, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // fold the register accumulators (vertex i < kDiag exists whenever racc[i] != 0, and H >= min(n_a, kDiag))
#pragma unroll
    for (int i = 0; i < kDiag; ++i) {
      double v = racc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      if (lane == 0 && v != 0.0) atomicAdd(&sacc[i], v);
    }
  }
  __syncthreads();
  for (int j = tid; j < p.H; j += Cfg::THREADS)
    if (sacc[j] != 0.0) atomicAdd(&p.ya[j], sacc[j]);
}

}  // namespace sttsv
