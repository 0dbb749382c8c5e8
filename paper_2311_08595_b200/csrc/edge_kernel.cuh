// edge_kernel.cuh — the hot kernel of one STTSV apply.
//
// Work decomposition.  The plan stores each cardinality bucket k as SoA int32
// id columns + fp64 weights w' = w (N-1)!/|beta(k)| (PAPER.md:342 footnote and
// Alg. 2's factor), edges sorted lexicographically by their
// (degree-relabelled, ascending) member ids.  A tile is TILE = 32*NCW*EPL
// consecutive edges of one bucket.  One persistent CTA per SM takes a
// CONTIGUOUS, cost-balanced range of tiles [cta_tiles[b], cta_tiles[b+1])
// (plan.cpp), so consecutive tiles of a CTA are neighbours in the sort order.
//
// Warp specialisation.  Per CTA, one producer warp streams tiles into an
// STAGES-deep shared-memory ring with 1-D TMA bulk copies (cp.async.bulk ->
// SASS UBLKCP, completion on a `full` mbarrier with expect_tx); NCW consumer
// warps each take a block of 32*EPL edges of the tile, lane l the EPL
// CONSECUTIVE edges l*EPL .. l*EPL+EPL-1 (EPL odd: the strided shared-memory
// reads are bank-conflict free), run the fully unrolled register DP of dp.cuh
// for (k, L = N-k+1), and release the stage on an `empty` mbarrier.  No
// CTA-wide barrier sits on the tile loop; bucket dispatch is once per tile.
//
// Scatter (row a5).  Contribution d_i = w' c_i goes to vertex id[i] of slot i.
// Because edges are sorted and a lane walks consecutive edges, it sees long
// runs of the same vertex in each slot.  Per slot i < RMAX a lane keeps a
// register run accumulator (rid[i], run[i]): the same vertex again is one DADD;
// a different vertex flushes the run.  Flushes inside a tile are per lane (few
// lanes, distinct vertices); at a tile's first step many lanes can end a run
// of the same long-run vertex at once.  A flush is ONE predicated, fire-and-
// forget red.global.add.f64 (SASS REDG.E.ADD.F64; the warp does not wait):
// for v < H (hot, degree-relabelled ids) into this CTA's private slice
// priv[cta][v] (L2-resident, contention only inside the CTA), else straight
// into y_a.  Each CTA adds its slice into y_a once at the end.  (Shared-memory
// fp64 atomicAdd is a CAS loop on sm_100a — ATOMS.CAST.SPIN.64 — whose latency
// stalled the warps; there is no native shared fp64 red.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dp.cuh"
#include "internal.h"

namespace sttsv {

constexpr unsigned kFull = 0xffffffffu;

// Debug instrumentation (compile with -DSTTSV_WAITPROF=1): consumer warps add the
// cycles they spend waiting on `full` barriers and their total cycles.
#ifndef STTSV_WAITPROF
#define STTSV_WAITPROF 0
#endif
#if STTSV_WAITPROF
__device__ unsigned long long g_wait_cycles[4];
#endif

// Prefix memoisation along a lane's consecutive edges (dp.cuh dp_core, h > 0);
// compile-time switch for A/B timing (0 = recompute every prefix).
#ifndef STTSV_MEMO
#define STTSV_MEMO 0
#endif
// Register-lean DP (dp.cuh dp_edge_lean): rows re-read in the suffix pass.
#ifndef STTSV_LEAN
#define STTSV_LEAN 0
#endif

template <int N>
struct EdgeCfg {
  static constexpr int KMAX = N < 1 ? STTSV_MAX_RANK : N;
#ifndef STTSV_EPL
#define STTSV_EPL 5
#endif
#ifndef STTSV_RING_KB
#define STTSV_RING_KB 220
#endif
  static constexpr int EPL = STTSV_EPL;                     // consecutive edges per lane per tile (odd)
  static constexpr int EDGE_BYTES = 4 * KMAX + 8;           // staged bytes per edge (ids + w')
  static constexpr int RING_BUDGET = STTSV_RING_KB * 1024;  // dynamic shared memory (<= 227 KB)
  // consumer warps: 15 (+1 producer = 4 warps per SMSP) for small ranks; fewer
  // when two stages of the largest bucket would not fit the ring budget
  static constexpr int NCW_FIT = RING_BUDGET / (2 * 32 * EPL * EDGE_BYTES);
#ifndef STTSV_NCW_SMALL
#define STTSV_NCW_SMALL 15
#endif
  static constexpr int NCW_PREF = (N >= 1 && N <= 10) ? STTSV_NCW_SMALL : 7;
  static constexpr int NCW = NCW_FIT < NCW_PREF ? (NCW_FIT < 1 ? 1 : NCW_FIT) : NCW_PREF;
  static constexpr int TILE = 32 * NCW * EPL;               // edges per tile
  static constexpr int THREADS = 32 * NCW + 32;             // + one producer warp
  static constexpr int STAGE_BYTES = TILE * EDGE_BYTES;
  static constexpr int STAGES_FIT = RING_BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT < 2 ? 2 : (STAGES_FIT > 6 ? 6 : STAGES_FIT);
  static constexpr int RMAX = KMAX < 8 ? KMAX : 8;          // slots with a register run accumulator
  static constexpr int MIN_BLOCKS = 1;
#ifndef STTSV_PF
#define STTSV_PF 2
#endif
  static constexpr int PF = STTSV_PF;                       // L2 prefetch distance (tiles)
  static_assert(STAGES * STAGE_BYTES <= RING_BUDGET, "ring does not fit");
  static_assert(TILE % 4 == 0, "tile must keep 16-byte aligned id columns");
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

// L2 prefetch of a global range (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ------------------------------------------------------------ scatter
struct Sink {
  double* priv;  // this CTA's private slice for ids < H
  double* ya;    // y on active vertices
  int H;
  __device__ __forceinline__ double* at(int v) const { return v < H ? priv + v : ya + v; }
};

__device__ __forceinline__ void red_add(double* a, double d) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(a), "d"(d) : "memory");
}
template <int RMAX>
struct RunAcc {
  int rid[RMAX];
  double run[RMAX];
};

// One step of a lane: slots (id[i], dv[i]) of its current edge.  Slot i <
// RMAX: same vertex as the run -> add; else flush the run (one red) and start
// a new one.  Slots >= RMAX: one red.
template <int K, int RMAX>
__device__ __forceinline__ void slots_deposit(const int (&id)[K], const double (&dv)[K], RunAcc<RMAX>& ra,
                                              const Sink& sk) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (i < RMAX) {
      constexpr int R1 = RMAX - 1;
      const int j = i < RMAX ? i : R1;  // compile-time after unrolling
      const bool fl = id[i] != ra.rid[j];
      if (fl) {  // rare: a branch (computing the address every step costs more)
        red_add(sk.at(ra.rid[j]), ra.run[j]);
        ra.rid[j] = id[i];
        ra.run[j] = 0.0;
      }
      ra.run[j] += dv[i];
    } else {
      red_add(sk.at(id[i]), dv[i]);
    }
  }
}

// The warp's block of a staged tile (size-K bucket): lane l takes the EPL
// consecutive columns base + l*EPL + r, r = 0..EPL-1.  Buckets are padded to
// whole tiles with weight-0 copies of their last edge, so every column is valid.
template <int N, int K, int TILE, int EPL, int RMAX>
__device__ __forceinline__ void warp_block(const int32_t* __restrict__ sids, const double* __restrict__ sw, int base,
                                           const double* __restrict__ xg, RunAcc<RMAX>& ra, const Sink& sk,
                                           int lane) {
  constexpr int L = N - K + 1;
  constexpr int KP = K > 2 ? K - 2 : 1;
  constexpr int GS = series_stride(N);
  double P[KP][L];  // prefix products, kept between this lane's consecutive edges
#pragma unroll 1
  for (int r = 0; r < EPL; ++r) {
    const int col = base + lane * EPL + r;
    int id[K];
    const double* rows[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      id[i] = sids[i * TILE + col];
      rows[i] = xg + (size_t)(uint32_t)id[i] * GS;  // GS compile-time: one IMAD.WIDE.U32
    }
    // shared leading members with this lane's previous edge (the run ids hold
    // it); warp minimum, 0 on a tile's first step
    int h = 0;
    if constexpr (K > 3 && STTSV_MEMO) {
      if (r > 0) {
        int hl = 0;
#pragma unroll
        for (int i = 0; i < K - 3 && i < RMAX; ++i)
          if (hl == i && id[i] == ra.rid[i]) hl = i + 1;
        h = __reduce_min_sync(kFull, hl);
      }
    }
    const double w = sw[col];
    double q[K], F;
#if STTSV_LEAN
    dp_edge_lean<K, L>(rows, q, F);
#else
    dp_edge_table<K, L>(rows, P, STTSV_MEMO ? h : 0, q, F);
#endif
    const double wF = w * F;
    double dv[K];
#pragma unroll
    for (int i = 0; i < K; ++i) dv[i] = fma(w, q[i], wF);
    slots_deposit<K, RMAX>(id, dv, ra, sk);
  }
}

template <int N, int K, int TILE, int EPL, int RMAX>
__device__ __forceinline__ void dispatch_k(int k, const int32_t* sids, const double* sw, int base,
                                           const double* xg, RunAcc<RMAX>& ra, const Sink& sk, int lane) {
  if constexpr (K <= N) {
    if (k == K) {
      warp_block<N, K, TILE, EPL, RMAX>(sids, sw, base, xg, ra, sk, lane);
      return;
    }
    dispatch_k<N, K + 1, TILE, EPL, RMAX>(k, sids, sw, base, xg, ra, sk, lane);
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
__device__ __forceinline__ void warp_block_generic(int N, int k, const int32_t* sids, const double* sw, int base,
                                                   const double* xa, const Sink& sk, int lane) {
  for (int r = 0; r < EPL; ++r) {
    const int col = base + lane * EPL + r;
    int id[STTSV_MAX_RANK];
    double x[STTSV_MAX_RANK], q[STTSV_MAX_RANK];
    for (int i = 0; i < k; ++i) {
      id[i] = sids[i * TILE + col];
      x[i] = __ldg(xa + id[i]);
    }
    double F = 0.0;
    dp_edge_generic(k, N - k + 1, x, q, &F);
    const double w = sw[col];
    const double wF = w * F;
    for (int i = 0; i < k; ++i) red_add(sk.at(id[i]), fma(w, q[i], wF));
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
  // layout: [STAGES][ ids KMAX*TILE int32 | w TILE f64 ]
  unsigned char* ring = smem_raw;
  const Sink sk{p.priv + (size_t)blockIdx.x * p.H, p.ya, p.H};
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t t_lo = p.cta_tiles[blockIdx.x], t_hi = p.cta_tiles[blockIdx.x + 1];

  for (int j = tid; j < p.H; j += Cfg::THREADS) sk.priv[j] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_proxy_async();
  }
  __syncthreads();

  // first bucket of this CTA's range (buckets in tile order; the index only moves forward)
  int b0 = 0;
  while (b0 + 1 < p.nb && t_lo >= p.b[b0 + 1].tile_begin) ++b0;

  if (warp == NCW) {
    // ---------------- producer warp: TMA bulk copies of tile t into stage it % STAGES,
    // plus an L2 prefetch of tile t + PF (hides HBM latency beyond the ring's depth)
    if (lane == 0) {
      int b = b0, bp = b0;
      int64_t it = 0;
      for (int64_t t = t_lo; t < t_hi; ++t, ++it) {
        const int s = (int)(it % STAGES);
        if constexpr (Cfg::PF > 0) {
          const int64_t tp = t + Cfg::PF;
          if (tp < t_hi) {
            while (bp + 1 < p.nb && tp >= p.b[bp + 1].tile_begin) ++bp;
            const BucketDesc& bd = p.b[bp];
            const int64_t e0 = (tp - bd.tile_begin) * TILE;
            constexpr uint32_t id_bytes = TILE * 4, w_bytes = TILE * 8;
            for (int i = 0; i < bd.k; ++i) bulk_prefetch_l2(p.ids + bd.ids_off + i * bd.stride + e0, id_bytes);
            bulk_prefetch_l2(p.w + bd.w_off + e0, w_bytes);
          }
        }
        if (it >= STAGES) mbar_wait(&empty[s], (uint32_t)(((it / STAGES) - 1) & 1));
        while (b + 1 < p.nb && t >= p.b[b + 1].tile_begin) ++b;
        const BucketDesc& bd = p.b[b];
        const int64_t e0 = (t - bd.tile_begin) * TILE;  // buckets are padded to whole tiles
        constexpr uint32_t id_bytes = TILE * 4, w_bytes = TILE * 8;
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
      ra.rid[i] = 0;  // flushing (0, 0.0) is a no-op deposit
      ra.run[i] = 0.0;
    }
    int b = b0;
    int64_t it = 0;
#if STTSV_WAITPROF
    long long wait_cyc = 0;
    const long long c_start = clock64();
#endif
    for (int64_t t = t_lo; t < t_hi; ++t, ++it) {
      const int s = (int)(it % STAGES);
      while (b + 1 < p.nb && t >= p.b[b + 1].tile_begin) ++b;
      const int k = p.b[b].k;
      const int base = warp * 32 * EPL;
#if STTSV_WAITPROF
      const long long w0 = clock64();
      mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
      wait_cyc += clock64() - w0;
#else
      mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
#endif
      {
        const unsigned char* st = ring + s * Cfg::STAGE_BYTES;
        const int32_t* sids = reinterpret_cast<const int32_t*>(st);
        const double* sw = reinterpret_cast<const double*>(st + KMAX * TILE * 4);
        if constexpr (N > 0) {
          dispatch_k<N, 1, TILE, EPL, RMAX>(k, sids, sw, base, p.xg, ra, sk, lane);
        } else {
          warp_block_generic<TILE, EPL>(p.N, k, sids, sw, base, p.xa, sk, lane);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#if STTSV_WAITPROF
    if (lane == 0) {
      atomicAdd(&g_wait_cycles[0], (unsigned long long)wait_cyc);
      atomicAdd(&g_wait_cycles[1], (unsigned long long)(clock64() - c_start));
      atomicAdd(&g_wait_cycles[2], 1ull);
    }
#endif
    // flush the run accumulators
    if (t_hi > t_lo) {
#pragma unroll
      for (int i = 0; i < RMAX; ++i)
        if (ra.run[i] != 0.0) red_add(sk.at(ra.rid[i]), ra.run[i]);
    }
  }
  // this CTA's reds into priv are ordered before the reads below (fence + barrier);
  // the reads go to L2 (ld.cg), where the reds were performed
  __threadfence();
  __syncthreads();
  for (int j = tid; j < p.H; j += Cfg::THREADS) {
    const double v = __ldcg(sk.priv + j);
    if (v != 0.0) red_add(p.ya + j, v);
  }
}

}  // namespace sttsv
