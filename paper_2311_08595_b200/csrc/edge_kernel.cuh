// edge_kernel.cuh — the hot kernel of one STTSV apply.
//
// Work decomposition.  The plan stores each cardinality bucket k as SoA int32
// id columns + fp64 weights w' = w (N-1)!/|beta(k)| (PAPER.md:342 footnote and
// Alg. 2's factor), edges sorted lexicographically by their
// (degree-relabelled, ascending) member ids.  A tile is TILE = 32*NCW*EPL
// consecutive edges of one bucket; tiles are ordered most-expensive bucket
// first and dealt to the persistent CTAs round-robin (CTA b takes tiles
// b, b+G, b+2G, ... so its bucket index only moves forward).
//
// Warp specialisation.  Per CTA, one producer warp streams tiles into an
// STAGES-deep shared-memory ring with 1-D TMA bulk copies (cp.async.bulk ->
// SASS UBLKCP, completion on a `full` mbarrier with expect_tx); NCW consumer
// warps each take a contiguous block of 32*EPL edges of the tile (one edge per
// lane per step, EPL steps), run the fully unrolled register DP of dp.cuh for
// (k, L = N-k+1), and release the stage on an `empty` mbarrier.  No CTA-wide
// barrier sits on the tile loop; bucket dispatch is once per tile.
//
// Scatter (row a5).  Contribution d_i = w' c_i goes to vertex id[i] of slot i.
// Because edges are sorted, a lane sees long runs of the same vertex in the low
// slots.  Each lane keeps, per slot i < RMAX, a register run accumulator
// (rid[i], run[i]); a contribution to the same vertex is one DADD.  Only when a
// run ends (or for slots >= RMAX) is a value flushed: the warp (if any lane
// flushes) reduces the flushed values over lanes holding the same vertex
// (adjacent lanes hold adjacent sorted edges, so equal ids are contiguous:
// segmented suffix scan with shuffles), and each segment head deposits once —
// into the CTA shared accumulator sacc[v] for v < H (hot, degree-relabelled
// ids), else with red.global.add.f64 into y_a.  Each CTA flushes sacc once.
// SASS note: shared fp64 atomicAdd is a CAS loop on sm_100a (ATOMS.CAST.SPIN.64),
// global is native (REDG.E.ADD.F64); the warp pre-reduction keeps same-address
// collisions in the CAS loop rare.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dp.cuh"
#include "internal.h"

namespace sttsv {

constexpr unsigned kFull = 0xffffffffu;

template <int N>
struct EdgeCfg {
  static constexpr int KMAX = N < 1 ? STTSV_MAX_RANK : N;
  static constexpr int NCW = (N >= 1 && N <= 10) ? 15 : 7;  // consumer warps (+1 producer: 4 or 2 warps per SMSP)
  static constexpr int EPL = 2;                             // edges per lane per tile
  static constexpr int TILE = 32 * NCW * EPL;               // edges per tile
  static constexpr int THREADS = 32 * NCW + 32;             // + one producer warp
  static constexpr int STAGE_BYTES = TILE * (4 * KMAX + 8);
  static constexpr int RING_BUDGET = 190 * 1024;
  static constexpr int STAGES_FIT = RING_BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT < 2 ? 2 : (STAGES_FIT > 6 ? 6 : STAGES_FIT);
  static constexpr int RMAX = KMAX < 8 ? KMAX : 8;          // slots with a register run accumulator
  static constexpr int MIN_BLOCKS = 1;
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
__device__ __forceinline__ void deposit(int v, double d, double* __restrict__ sacc, double* __restrict__ ya, int H) {
  if (v < H) atomicAdd(&sacc[v], d);
  else atomicAdd(&ya[v], d);
}

// Warp-cooperative flush: lanes with v >= 0 hold a value d for vertex v.
// Reduce over runs of equal adjacent v (v < 0 breaks runs); each run's first
// lane deposits the run total.  Must be called by the whole warp.
__device__ __forceinline__ void warp_flush(int v, double d, int lane, double* __restrict__ sacc,
                                           double* __restrict__ ya, int H) {
  const int v0 = __shfl_sync(kFull, v, 0);
  if (__all_sync(kFull, v == v0)) {
    if (v0 < 0) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(kFull, d, o);
    if (lane == 0) deposit(v0, d, sacc, ya, H);
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
  if ((lane == 0 || vp != v) && v >= 0) deposit(v, d, sacc, ya, H);
}

template <int RMAX>
struct RunAcc {
  int rid[RMAX];
  double run[RMAX];
};

// Slots of the current edge: (id[i], dv[i]); `valid` false for an empty lane
// (dv = 0).  Slot i < RMAX feeds its run accumulator and yields a flush
// (old id, old run) when the id changes; slots >= RMAX flush every value.
// One REDUX gives the warp-uniform set of slots with any flush.
template <int K, int RMAX>
__device__ __forceinline__ void slots_deposit(const int (&id)[K], const double (&dv)[K], bool valid,
                                              RunAcc<RMAX>& ra, int lane, double* sacc, double* ya, int H) {
  int fv[K];
  double fd[K];
  unsigned lm = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (i < RMAX) {
      constexpr int R1 = RMAX - 1;
      const int j = i < RMAX ? i : R1;  // compile-time after unrolling
      const bool same = (id[i] == ra.rid[j]) | !valid;
      fv[i] = same ? -1 : ra.rid[j];
      fd[i] = ra.run[j];
      ra.run[j] = same ? ra.run[j] + dv[i] : dv[i];
      ra.rid[j] = same ? ra.rid[j] : id[i];
    } else {
      fv[i] = valid ? id[i] : -1;
      fd[i] = dv[i];
    }
    lm |= (fv[i] >= 0 ? 1u : 0u) << i;
  }
  const unsigned um = __reduce_or_sync(kFull, lm);
  if (um) {
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (um & (1u << i)) warp_flush(fv[i], fd[i], lane, sacc, ya, H);
  }
}

// EPL*32 edges of a size-K bucket: this warp's block of the staged tile,
// one edge per lane per step.  Empty lanes read member ids of column col0
// (valid table rows) and carry w = 0.
template <int N, int K, int TILE, int EPL, int RMAX>
__device__ __forceinline__ void warp_edges(const int32_t* __restrict__ sids, const double* __restrict__ sw,
                                           int col0, int nvalid, const double* __restrict__ xg, int gs,
                                           RunAcc<RMAX>& ra, double* sacc, double* ya, int H, int lane) {
  constexpr int L = N - K + 1;
#pragma unroll 1
  for (int r = 0; r < EPL; ++r) {
    if (r * 32 >= nvalid) break;
    const bool valid = r * 32 + lane < nvalid;
    const int col = valid ? col0 + r * 32 + lane : col0;
    int id[K];
    const double* rows[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      id[i] = sids[i * TILE + col];
      rows[i] = xg + (size_t)id[i] * gs;
    }
    const double w = valid ? sw[col] : 0.0;
    double q[K], F;
    dp_edge_table<K, L>(rows, q, F);
    const double wF = w * F;
    double dv[K];
#pragma unroll
    for (int i = 0; i < K; ++i) dv[i] = fma(w, q[i], wF);
    slots_deposit<K, RMAX>(id, dv, valid, ra, lane, sacc, ya, H);
  }
}

template <int N, int K, int TILE, int EPL, int RMAX>
__device__ __forceinline__ void dispatch_k(int k, const int32_t* sids, const double* sw, int col0, int nvalid,
                                           const double* xg, int gs, RunAcc<RMAX>& ra, double* sacc, double* ya,
                                           int H, int lane) {
  if constexpr (K <= N) {
    if (k == K) {
      warp_edges<N, K, TILE, EPL, RMAX>(sids, sw, col0, nvalid, xg, gs, ra, sacc, ya, H, lane);
      return;
    }
    dispatch_k<N, K + 1, TILE, EPL, RMAX>(k, sids, sw, col0, nvalid, xg, gs, ra, sacc, ya, H, lane);
  }
}

// ---------------------------------------------------------------- generic
// Runtime (K, L) DP for ranks without a compiled specialisation: same
// recurrence as dp_edge, arrays in local memory.  Returns q_i = Q_i[D] and F = F[D-1].
static __device__ __noinline__ void dp_edge_generic(int K, int L, const double* x, double* q, double* Fout) {
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
    // q = [t^D] (empty product) = [D == 0];  F = [t^{D-1}] g_0 = x^D / D!
    q[0] = D == 0 ? 1.0 : 0.0;
    *Fout = D >= 1 ? g[0][D - 1] : 0.0;
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
    *Fout = D >= 1 ? coefD(g[0], g[1], D - 1) : 0.0;
    q[0] = g[1][D];
    q[1] = g[0][D];
    return;
  }
  double P[STTSV_MAX_RANK][STTSV_MAX_RANK];
  for (int j = 0; j < L; ++j) P[0][j] = g[0][j];
  for (int i = 1; i <= K - 3; ++i) tmul(P[i - 1], g[i], P[i]);
  q[K - 1] = coefD(P[K - 3], g[K - 2], D);
  q[K - 2] = coefD(P[K - 3], g[K - 1], D);
  double S[STTSV_MAX_RANK], T[STTSV_MAX_RANK];
  tmul(g[K - 2], g[K - 1], S);
  *Fout = D >= 1 ? coefD(P[K - 3], S, D - 1) : 0.0;
  for (int i = K - 3; i >= 1; --i) {
    q[i] = coefD(P[i - 1], S, D);
    if (i > 1) {
      tmul(g[i], S, T);
      for (int j = 0; j < L; ++j) S[j] = T[j];
    } else {
      q[0] = coefD(g[1], S, D);
    }
  }
  if (K == 3) q[0] = S[D];
}

template <int TILE, int EPL>
__device__ __forceinline__ void warp_edges_generic(int N, int k, const int32_t* sids, const double* sw, int col0,
                                                   int nvalid, const double* xa, double* sacc, double* ya, int H,
                                                   int lane) {
  for (int r = 0; r < EPL; ++r) {
    const int col = col0 + r * 32 + lane;
    const bool valid = r * 32 + lane < nvalid;
    if (!__any_sync(kFull, valid)) break;
    int id[STTSV_MAX_RANK];
    double x[STTSV_MAX_RANK], q[STTSV_MAX_RANK];
    for (int i = 0; i < k; ++i) {
      id[i] = valid ? sids[i * TILE + col] : -1;
      x[i] = valid ? __ldg(xa + id[i]) : 0.0;
    }
    double F = 0.0;
    dp_edge_generic(k, N - k + 1, x, q, &F);
    const double w = valid ? sw[col] : 0.0;
    const double wF = w * F;
    for (int i = 0; i < k; ++i) warp_flush(id[i], fma(w, q[i], wF), lane, sacc, ya, H);
  }
}

// ------------------------------------------------------------- the kernel
// N == 0 is the generic instantiation (any rank <= STTSV_MAX_RANK).
template <int N>
__global__ void __launch_bounds__(EdgeCfg<N>::THREADS, EdgeCfg<N>::MIN_BLOCKS)
    edge_kernel(const __grid_constant__ EdgeKernelParams p) {
  using Cfg = EdgeCfg<N>;
  constexpr int TILE = Cfg::TILE, STAGES = Cfg::STAGES, KMAX = Cfg::KMAX, NCW = Cfg::NCW, EPL = Cfg::EPL;
  constexpr int RMAX = Cfg::RMAX;
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
      int b = 0;
      for (int64_t t = blockIdx.x; t < p.num_tiles; t += G, ++it) {
        const int s = (int)(it % STAGES);
        if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
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
    RunAcc<RMAX> ra;
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      ra.rid[i] = -1;
      ra.run[i] = 0.0;
    }
    int64_t it = 0;
    int b = 0;
    for (int64_t t = blockIdx.x; t < p.num_tiles; t += G, ++it) {
      const int s = (int)(it % STAGES);
      while (b + 1 < p.nb && t >= p.b[b + 1].tile_begin) ++b;
      const int64_t m = p.b[b].m;
      const int k = p.b[b].k;
      const int64_t e0 = (t - p.b[b].tile_begin) * TILE + warp * 32 * EPL;
      mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
      if (e0 < m) {
        const unsigned char* st = ring + s * Cfg::STAGE_BYTES;
        const int32_t* sids = reinterpret_cast<const int32_t*>(st);
        const double* sw = reinterpret_cast<const double*>(st + KMAX * TILE * 4);
        const int nvalid = m - e0 < 32 * EPL ? (int)(m - e0) : 32 * EPL;
        const int col0 = warp * 32 * EPL;
        if constexpr (N > 0) {
          dispatch_k<N, 1, TILE, EPL, RMAX>(k, sids, sw, col0, nvalid, p.xg, p.gs, ra, sacc, p.ya, p.H, lane);
        } else {
          warp_edges_generic<TILE, EPL>(p.N, k, sids, sw, col0, nvalid, p.xa, sacc, p.ya, p.H, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // flush the run accumulators
#pragma unroll
    for (int i = 0; i < RMAX; ++i) warp_flush(ra.rid[i], ra.run[i], lane, sacc, p.ya, p.H);
  }
  __syncthreads();
  for (int j = tid; j < p.H; j += Cfg::THREADS)
    if (sacc[j] != 0.0) atomicAdd(&p.ya[j], sacc[j]);
}

}  // namespace sttsv
