// edge_kernel.cuh — the hot kernel of one STTSV apply.
//
// Persistent CTAs claim tiles of TILE edges from a device counter.  A tile
// lies in one cardinality bucket (size k), so the switch on k is uniform over
// the CTA and every (k, L = N-k+1) runs the fully unrolled register DP of
// dp.cuh, one edge per thread.  The tile's SoA id columns and weights are
// staged into shared memory by 1-D TMA bulk copies (cp.async.bulk, SASS
// UBLKCP) on an STAGES-deep mbarrier ring, so the HBM stream runs ahead of the
// FP64 work independently of occupancy.
//
// Each contribution delta = w' c (w' = w (N-1)!/|beta(k)| folded at plan time,
// PAPER.md:391) is reduced through four tiers keyed on the relabelled vertex
// id (ids are ordered by descending degree, so hot vertices are small):
//   0. edge slot i holds vertex i (i < kDiag)  -> register accumulator racc[i]
//   1. id < T                                   -> this thread's private shared
//      column pc[id][tid] (plain read-modify-write: no atomics, no conflicts)
//   2. T <= id < H                              -> CTA shared accumulator (atomicAdd)
//   3. id >= H                                  -> red.global.add.f64 into y_a
// Each CTA flushes tiers 0-2 into y_a once, after its last tile.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dp.cuh"
#include "internal.h"

namespace sttsv {

constexpr int kDiag = 8;

template <int N>
struct EdgeCfg {
  static constexpr int BLOCK = (N >= 1 && N <= 16) ? 256 : 128;  // = TILE (one edge per thread)
  static constexpr int KMAX = N < 1 ? STTSV_MAX_RANK : N;
  static constexpr int STAGES = N <= 8 ? 4 : 3;
  static constexpr int MIN_BLOCKS = 2;
  static constexpr int STAGE_BYTES = BLOCK * (4 * KMAX + 8);
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
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------ scatter tiers
template <int BLOCK>
__device__ __forceinline__ void deposit(int i, int v, double d, double (&racc)[kDiag], double* __restrict__ pc,
                                        double* __restrict__ sacc, double* __restrict__ ya, int T, int H,
                                        int tid) {
  if (i < kDiag && v == i) {
#pragma unroll
    for (int q = 0; q < kDiag; ++q)
      if (q == i) racc[q] += d;
  } else if (v < T) {
    pc[v * BLOCK + tid] += d;
  } else if (v < H) {
    atomicAdd(&sacc[v], d);
  } else {
    atomicAdd(&ya[v], d);
  }
}

// one edge of a size-K bucket, ids/w from the shared stage
template <int N, int K, int BLOCK>
__device__ __forceinline__ void edge_from_stage(const int32_t* __restrict__ sids, const double* __restrict__ sw,
                                                const double* __restrict__ xa, double (&racc)[kDiag],
                                                double* pc, double* sacc, double* ya, int T, int H, int tid) {
  constexpr int L = N - K + 1;
  int id[K];
  double x[K], c[K];
#pragma unroll
  for (int i = 0; i < K; ++i) id[i] = sids[i * BLOCK + tid];
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = __ldg(xa + id[i]);
  const double w = sw[tid];
  dp_edge<K, L>(x, c);
#pragma unroll
  for (int i = 0; i < K; ++i) deposit<BLOCK>(i, id[i], w * c[i], racc, pc, sacc, ya, T, H, tid);
}

template <int N, int K, int BLOCK>
__device__ __forceinline__ void dispatch_k(int k, const int32_t* sids, const double* sw, const double* xa,
                                           double (&racc)[kDiag], double* pc, double* sacc, double* ya, int T,
                                           int H, int tid) {
  if constexpr (K <= N) {
    if (k == K) {
      edge_from_stage<N, K, BLOCK>(sids, sw, xa, racc, pc, sacc, ya, T, H, tid);
      return;
    }
    dispatch_k<N, K + 1, BLOCK>(k, sids, sw, xa, racc, pc, sacc, ya, T, H, tid);
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


template <int BLOCK>
__device__ __forceinline__ void edge_generic_from_stage(int N, int k, const int32_t* sids, const double* sw,
                                                        const double* xa, double (&racc)[kDiag], double* pc,
                                                        double* sacc, double* ya, int T, int H, int tid) {
  double x[STTSV_MAX_RANK], c[STTSV_MAX_RANK];
  for (int i = 0; i < k; ++i) x[i] = __ldg(xa + sids[i * BLOCK + tid]);
  dp_edge_generic(k, N - k + 1, x, c);
  const double w = sw[tid];
  for (int i = 0; i < k; ++i) deposit<BLOCK>(i, sids[i * BLOCK + tid], w * c[i], racc, pc, sacc, ya, T, H, tid);
}

// ------------------------------------------------------------- the kernel
// N == 0 is the generic instantiation (any rank <= STTSV_MAX_RANK).
template <int N>
__global__ void __launch_bounds__(EdgeCfg<N>::BLOCK, EdgeCfg<N>::MIN_BLOCKS)
    edge_kernel(const __grid_constant__ EdgeKernelParams p) {
  using Cfg = EdgeCfg<N>;
  constexpr int BLOCK = Cfg::BLOCK, STAGES = Cfg::STAGES, KMAX = Cfg::KMAX;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // layout: [STAGES][ ids KMAX*BLOCK int32 | w BLOCK f64 ] | pc [T][BLOCK] f64 | sacc [H] f64
  unsigned char* ring = smem_raw;
  double* pc = reinterpret_cast<double*>(smem_raw + STAGES * Cfg::STAGE_BYTES);
  double* sacc = pc + p.T * BLOCK;
  __shared__ uint64_t full[STAGES];
  __shared__ int64_t s_tile[STAGES];
  __shared__ int s_bucket[STAGES];
  const int tid = threadIdx.x;

  for (int j = tid; j < p.T * BLOCK + p.H; j += BLOCK) pc[j] = 0.0;
  double racc[kDiag];
#pragma unroll
  for (int i = 0; i < kDiag; ++i) racc[i] = 0.0;

  // producer: claim the next tile and start its copies into stage s
  auto produce = [&](int s) {
    const int64_t tile = atomicAdd(p.tile_counter, 1);
    s_tile[s] = tile;
    if (tile >= p.num_tiles) return;
    int b = 0;
    while (b + 1 < p.nb && tile >= p.b[b + 1].tile_begin) ++b;
    s_bucket[s] = b;
    const BucketDesc& bd = p.b[b];
    const int64_t e0 = (tile - bd.tile_begin) * BLOCK;
    const int64_t cnt = bd.m - e0 < BLOCK ? bd.m - e0 : BLOCK;
    const uint32_t id_bytes = (uint32_t)(((cnt + 3) & ~3LL) * 4);
    const uint32_t w_bytes = (uint32_t)(((cnt + 1) & ~1LL) * 8);
    unsigned char* st = ring + s * Cfg::STAGE_BYTES;
    mbar_arrive_expect_tx(&full[s], id_bytes * bd.k + w_bytes);
    for (int i = 0; i < bd.k; ++i)
      bulk_g2s(st + i * BLOCK * 4, p.ids + bd.ids_off + i * bd.stride + e0, id_bytes, &full[s]);
    bulk_g2s(st + KMAX * BLOCK * 4, p.w + bd.w_off + e0, w_bytes, &full[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_proxy_async();
    for (int s = 0; s < STAGES; ++s) produce(s);
  }
  __syncthreads();

  for (int it = 0;; ++it) {
    const int s = it % STAGES;
    const int64_t tile = s_tile[s];
    if (tile >= p.num_tiles) break;
    const BucketDesc& bd = p.b[s_bucket[s]];
    mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
    const unsigned char* st = ring + s * Cfg::STAGE_BYTES;
    const int32_t* sids = reinterpret_cast<const int32_t*>(st);
    const double* sw = reinterpret_cast<const double*>(st + KMAX * BLOCK * 4);
    const int64_t e = (tile - bd.tile_begin) * BLOCK + tid;
    if (e < bd.m) {
      if constexpr (N > 0) {
        dispatch_k<N, 1, BLOCK>(bd.k, sids, sw, p.xa, racc, pc, sacc, p.ya, p.T, p.H, tid);
      } else {
        edge_generic_from_stage<BLOCK>(p.N, bd.k, sids, sw, p.xa, racc, pc, sacc, p.ya, p.T, p.H, tid);
      }
    }
    __syncthreads();  // stage s fully consumed
    if (tid == 0) {
      fence_proxy_async();
      produce(s);
    }
  }

  // flush tier 0 into the private columns (racc[i] != 0 only if vertex i exists, and i < kDiag <= T then)
#pragma unroll
  for (int i = 0; i < kDiag; ++i)
    if (racc[i] != 0.0) pc[i * BLOCK + tid] += racc[i];
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  for (int t = warp; t < p.T; t += BLOCK / 32) {
    double sum = 0.0;
    for (int j = lane; j < BLOCK; j += 32) sum += pc[t * BLOCK + j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum != 0.0) atomicAdd(&p.ya[t], sum);
  }
  for (int j = p.T + tid; j < p.H; j += BLOCK)
    if (sacc[j] != 0.0) atomicAdd(&p.ya[j], sacc[j]);
}

template <int N>
constexpr size_t edge_kernel_smem(int T, int H) {
  return (size_t)EdgeCfg<N>::STAGES * EdgeCfg<N>::STAGE_BYTES + (size_t)(T * EdgeCfg<N>::BLOCK + H) * 8;
}

}  // namespace sttsv
