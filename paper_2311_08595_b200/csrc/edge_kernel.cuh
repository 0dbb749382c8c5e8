// edge_kernel.cuh — the hot kernel of one STTSV apply.
//
// Work decomposition.  The plan stores each cardinality bucket k as SoA int32
// id columns + fp64 weights w' = w (N-1)!/|beta(k)| (PAPER.md:342 footnote and
// Alg. 2's factor), edges sorted lexicographically by their
// (degree-relabelled, ascending) member ids and padded to whole tiles.  A tile
// is TILE = 32*NCW*EPL consecutive edges of one bucket.  Persistent CTAs (one or
// two per SM); each CTA's producer grabs CHUNKS of p.chunk consecutive tiles
// from a device counter (dynamic load balance; tiles are ordered most expensive
// bucket first, so the tail is the cheapest work), so consecutive tiles of a
// CTA are mostly neighbours in the sort order.
//
// Warp specialisation.  Per CTA, one producer warp streams tiles into an
// shared-memory byte ring (each stage sized by its bucket's k) with 1-D TMA bulk copies (cp.async.bulk ->
// SASS UBLKCP, completion on a `full` mbarrier with expect_tx) and publishes the
// tile index in the stage; NCW consumer warps each take a block of 32*EPL edges
// of the tile, lane l the EPL CONSECUTIVE edges l*EPL .. l*EPL+EPL-1 (EPL odd:
// the strided shared-memory reads are bank-conflict free), run the per-edge DP
// of dp.cuh for (k, L = N-k+1) — fully unrolled in registers for N <= 12, a
// runtime member loop with a local-memory prefix stack (edge_big) otherwise —
// and release the stage on an `empty` mbarrier.  No CTA-wide barrier sits on
// the tile loop; bucket dispatch is once per tile.
//
// Scatter (row a5).  Contribution d_i = w' c_i goes to vertex id[i] of slot i.
// Because edges are sorted and a lane walks consecutive edges, it sees long
// runs of the same vertex in each slot.  Per slot i < RMAX a lane keeps a
// register run accumulator (rid[i], run[i]): the same vertex again is one DADD;
// a different vertex flushes the run with ONE fire-and-forget
// red.global.add.f64 (SASS REDG.E.ADD.F64; the warp does not wait): for v < H
// (hot, degree-relabelled ids) into this CTA's private slice priv[cta][v]
// (L2-resident, contention only inside the CTA), else straight into y_a.  Each
// CTA adds its slice into y_a once at the end.  (Shared-memory fp64 atomicAdd
// is a CAS loop on sm_100a — ATOMS.CAST.SPIN.64 — whose latency stalled the
// warps; there is no native shared fp64 red.)
//
// Variants (template flags): BATCH — nvec vectors per staged tile (f4,
// sttsv_apply_batch); DET — each contribution is stored to its plan-time slot
// of a vertex-major buffer instead (f2, STTSV_DETERMINISTIC).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "dp.cuh"
#include "internal.h"
#include "prefix.cuh"

namespace sttsv {

constexpr unsigned kFull = 0xffffffffu;

// Debug instrumentation (compile with -DSTTSV_WAITPROF=1): consumer warps add the
// cycles they spend waiting on `full` barriers and their total cycles.
#ifndef STTSV_WAITPROF
#define STTSV_WAITPROF 0
#endif
#if STTSV_WAITPROF
__device__ unsigned long long g_wait_cycles[4];
__device__ unsigned long long g_k_cycles[2 * (STTSV_MAX_RANK + 1)];  // per bucket k: cycles, tiles
// per CTA: globaltimer at the consumers' start, at the CTA's end, and its tile count
__device__ unsigned long long g_cta_ns[3 * 1024];
#endif
// STTSV_WAITPROF == 3: g_k_cycles is indexed by block class instead of k:
// 0 = M = 0 block, M = 1..8 own members, 20 + k = full DP (no shared prefix)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}


// ---- compile-time tuning (each default was chosen by A/B timing on B200 with
// tools/variants.py + tools/time_apply.py)
// small ranks (N <= 10): two CTAs per SM, each 7 consumer warps + 1 producer (8 spill
// under the two-CTA register cap once the shared-prefix paths are compiled in)
// with a 112 KB ring (two independent TMA pipelines per SM measured 2.7% faster
// than one CTA of 15 consumers on `large`), 5 edges per lane per tile
#ifndef STTSV_EPL
#define STTSV_EPL 5
#endif
// edges per lane per tile with 16-bit member ids (smaller stages: more in flight)
#ifndef STTSV_EPL16
#define STTSV_EPL16 8
#endif
#ifndef STTSV_RING_KB
#define STTSV_RING_KB 108
#endif
#ifndef STTSV_NCW_SMALL
#define STTSV_NCW_SMALL 7
#endif
// N = 9, 10: 7 consumer warps (8 would spill under the two-CTA register cap)
#ifndef STTSV_NCW_SMALL9
#define STTSV_NCW_SMALL9 7
#endif
#ifndef STTSV_MIN_BLOCKS
#define STTSV_MIN_BLOCKS 2
#endif
// N = 11 .. BIG_MIN-1: one CTA per SM with 11 consumer warps (168 registers, no spills)
#ifndef STTSV_MID_BLOCKS
#define STTSV_MID_BLOCKS 1
#endif
// consumer warps take the warp blocks of the staged tiles from a per-CTA counter
// (block g = tile iteration g / NCW, block g % NCW), so a warp held up by an
// expensive block does not hold the others back (0: warp w always takes block w)
#ifndef STTSV_DYN_BLOCKS
#define STTSV_DYN_BLOCKS 1
#endif
// unroll factor of the per-lane edge loop of a full-DP warp block (2 lets the compiler overlap
// one edge's row gathers with the previous edge's DP; costs registers)
#ifndef STTSV_WB_UNROLL
#define STTSV_WB_UNROLL 1
#endif
// software-pipelined queue loop of the shared-prefix blocks for M*L <= PIPE_ML
// (the next entry's rows in flight during the current DP; more costs registers)
#ifndef STTSV_PIPE_ML
#define STTSV_PIPE_ML 8
#endif
// prefix blocks: the flush's C rows are loaded into registers at the start of the
// block for L <= FLUSHPRE_L8 (N <= 8) / FLUSHPRE_L (larger N, where registers are short)
#ifndef STTSV_FLUSHPRE_L8
#define STTSV_FLUSHPRE_L8 32
#endif
#ifndef STTSV_FLUSHPRE_L
#define STTSV_FLUSHPRE_L 3
#endif
#ifndef STTSV_SLOTS
#define STTSV_SLOTS 16
#endif
#ifndef STTSV_RING_KB_MID
#define STTSV_RING_KB_MID 220
#endif
#ifndef STTSV_NCW_MID
#define STTSV_NCW_MID 11
#endif
// N >= BIG_MIN and the generic runtime-N kernel (N = 0): large-rank path with the
// prefix stack in L1-cached local memory (BIG_LOCAL = 1) or shared memory (0)
#ifndef STTSV_BIG_MIN
#define STTSV_BIG_MIN 13
#endif
#ifndef STTSV_BIG_LOCAL
#define STTSV_BIG_LOCAL 1
#endif
#ifndef STTSV_BIG_NCW
#define STTSV_BIG_NCW 11
#endif
// unrolled kernel for N >= NORM_MIN on series normalised to a leading 1
#ifndef STTSV_MID_NORM
#define STTSV_MID_NORM 1
#endif
#ifndef STTSV_NORM_MIN
#define STTSV_NORM_MIN 2
#endif
// large-rank path on series normalised to a leading 1 (fewer FP64 operations)
#ifndef STTSV_BIG_NORM
#define STTSV_BIG_NORM 1
#endif
// shared-prefix memo (prefix.cuh): a tile whose edges share a prefix of U members
// runs the DP over its M = K - U own members, M <= PREFIX_MMAX
#ifndef STTSV_PREFIX_MMAX
#define STTSV_PREFIX_MMAX 6
#endif
#ifndef STTSV_PREFIX_MMAX_BIG
#define STTSV_PREFIX_MMAX_BIG 8
#endif
// suspend-time hint (ns) of the producer's mbarrier waits
#ifndef STTSV_WAIT_HINT_NS
#define STTSV_WAIT_HINT_NS 1000000
#endif

constexpr int kRedStride = 34;  // doubles per row of the prefix reduction area (32 lanes + pad)

// IDB_: bytes per member id in the edge stream (4; or 2 for plans with n_a <=
// 65536 on the unrolled ranks: 36% fewer stream bytes at mean k = 5)
template <int N, int IDB_ = 4>
struct EdgeCfg {
  static constexpr bool BIG = (N == 0) || (N >= STTSV_BIG_MIN);
  static constexpr int KMAX = N < 1 ? STTSV_MAX_RANK : N;
  static constexpr int IDB = BIG ? 4 : IDB_;               // bytes per member id in the stream
  static constexpr int EPL = BIG ? 1 : (IDB == 2 ? STTSV_EPL16 : STTSV_EPL);  // consecutive edges per lane per tile
  static constexpr int EDGE_BYTES = IDB * KMAX + 8;         // staged bytes per edge (ids + w')
  // dynamic shared memory for the TMA ring (<= 227 KB in total; the large-rank
  // path also needs its prefix stack)
  static constexpr int NCW_PREF = BIG ? (N == 0 && !STTSV_BIG_LOCAL ? 2 : STTSV_BIG_NCW)
                                      : (N <= 8 ? STTSV_NCW_SMALL : N <= 10 ? STTSV_NCW_SMALL9 : STTSV_NCW_MID);
  // shared-prefix memo limits (0: off on this path)
  static constexpr int PMAX = BIG ? (STTSV_BIG_NORM ? STTSV_PREFIX_MMAX_BIG : 0)
                                  : ((N < STTSV_NORM_MIN || !STTSV_MID_NORM) ? 0 : STTSV_PREFIX_MMAX);
  // per consumer warp, LRED rows of kRedStride doubles of shared memory for the
  // prefix tiles' transpose-reduction of SB (L <= KMAX - 1 terms when M >= 1)
  static constexpr int LRED = PMAX > 0 && KMAX > 3 ? KMAX - 1 : 0;
  // per-warp scratch: the reduction rows, or (unrolled path) the run queue of a
  // block (32*EPL entries of (sum w', column): 12 bytes each)
  static constexpr int EPL_ = BIG ? 1 : (IDB == 2 ? STTSV_EPL16 : STTSV_EPL);
  static constexpr int QBYTES = (PMAX > 0 && !BIG) ? 32 * EPL_ * 12 : 0;
  static constexpr int SCR_DOUBLES = ((LRED * kRedStride * 8 > QBYTES ? LRED * kRedStride * 8 : QBYTES) + 15) / 16 * 2;
  static constexpr int RED_BYTES = NCW_PREF * SCR_DOUBLES * 8;
  // (the large-rank path runs one CTA per SM: its reduction rows come on top)
  static constexpr int RING_BUDGET = BIG ? (STTSV_BIG_LOCAL ? 96 : 48) * 1024
                                         : (N <= 10 ? STTSV_RING_KB : STTSV_RING_KB_MID / STTSV_MID_BLOCKS) * 1024 - RED_BYTES;
  // consumer warps per CTA (NCW_PREF), fewer when two stages of the largest
  // bucket would not fit the ring budget
  static constexpr int NCW_FIT = RING_BUDGET / (2 * 32 * EPL * EDGE_BYTES);
  static constexpr int NCW = NCW_FIT < NCW_PREF ? (NCW_FIT < 1 ? 1 : NCW_FIT) : NCW_PREF;
  static constexpr int TILE = 32 * NCW * EPL;               // edges per tile
  static constexpr int THREADS = 32 * NCW + 32;             // + one producer warp
  static constexpr int STAGE_BYTES = TILE * EDGE_BYTES;     // largest stage (k = KMAX)
  static constexpr int STAGES_FIT = RING_BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT < 2 ? 2 : (STAGES_FIT > 6 ? 6 : STAGES_FIT);
  // byte ring: a stage takes TILE*(4k+8) bytes of its bucket's k, so small-k
  // tiles are more deep in flight; SLOTS bounds the stages in flight
  static constexpr int RING_BYTES = (STAGES * STAGE_BYTES > RING_BUDGET ? STAGES * STAGE_BYTES : RING_BUDGET) / 128 * 128;
  static constexpr int SLOTS = STTSV_SLOTS;
  static constexpr int RMAX = BIG ? 4 : (KMAX < 8 ? KMAX : 8);  // slots with a register run accumulator
  static constexpr int MIN_BLOCKS = BIG ? 1 : (N <= 10 ? STTSV_MIN_BLOCKS : STTSV_MID_BLOCKS);
  static constexpr bool BIG_PREFIX = BIG && PMAX > 0;
  static constexpr int PLMAX = KMAX;  // (no limit on L)
  static_assert(STAGES * STAGE_BYTES <= RING_BUDGET, "ring does not fit");
  static_assert(RING_BYTES >= 2 * STAGE_BYTES, "ring must hold two of the largest stages");
  static_assert(TILE % 4 == 0, "tile must keep 16-byte aligned id columns");
};

// doubles of prefix stack one consumer thread of the large-rank path needs for
// rank N: rows P_0..P_{K-4} of length L = N-K+1, maximised over K
__host__ __device__ constexpr int big_stack_doubles(int N) {
  int m = 0;
  for (int K = 4; K <= N; ++K) m = (K - 3) * (N - K + 1) > m ? (K - 3) * (N - K + 1) : m;
  return m;
}

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

// consumer-side wait: spin (default) or, with STTSV_CONSUMER_HINT, a suspend-time-hinted
// try_wait like the producer's (the waiting warp stops taking issue slots)
#ifndef STTSV_CONSUMER_HINT
#define STTSV_CONSUMER_HINT 0
#endif
__device__ __forceinline__ void mbar_wait_consumer(uint64_t* bar, uint32_t parity) {
#if STTSV_CONSUMER_HINT
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(STTSV_CONSUMER_HINT)
        : "memory");
    if (ok) return;
  }
#else
  mbar_wait(bar, parity);
#endif
}
// producer-side wait: try_wait with a suspend-time hint, so the waiting thread
// sleeps in hardware until the phase completes (or the hint expires) instead of
// spinning and stealing issue slots from the consumers
#ifndef STTSV_PRODUCER_SPIN
#define STTSV_PRODUCER_SPIN 0
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
#if STTSV_PRODUCER_SPIN
  mbar_wait(bar, parity);
  return;
#endif
  uint32_t ok = 0;
  const uint32_t a = smem_u32(bar);
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(STTSV_WAIT_HINT_NS)
        : "memory");
    if (ok) return;
  }
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
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
struct Sink {
  double* priv;  // this CTA's private slice for ids < H
  double* ya;    // y on active vertices
  int H;
  __device__ __forceinline__ double* at(int v) const { return v < H ? priv + v : ya + v; }
};

// Weight column of a staged tile: the staged fp64 column, or — buckets whose
// w' are all equal (plan.cpp; large has w = 1) — the constant for the tile's
// real edges and 0 for its padding (no weight bytes are streamed).  pos is the
// edge's sorted position in the tile, col its lane-major column.
struct WSrc {
  const double* sw;
  double wc;
  int real;  // real (non-padding) edges of the tile (uniform buckets)
  bool uni;
  __device__ __forceinline__ double at(int col, int pos) const { return uni ? (pos < real ? wc : 0.0) : sw[col]; }
};

__device__ __forceinline__ void red_add(double* a, double d) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(a), "d"(d) : "memory");
}
// Warp-cooperative flush: lanes with v >= 0 hold a value d for vertex v.
// Reduce over runs of equal adjacent v (v < 0 breaks runs); each run's first
// lane deposits the run total with one red.  Whole warp.
__device__ __forceinline__ void warp_flush(int v, double d, int lane, const Sink& sk) {
  const int v0 = __shfl_sync(kFull, v, 0);
  if (__all_sync(kFull, v == v0)) {
    if (v0 < 0) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(kFull, d, o);
    if (lane == 0) red_add(sk.at(v0), d);
    return;
  }
  // segmented suffix scan: a lane ends with the sum from itself to the end of its run
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
  if ((lane == 0 || vp != v) && v >= 0) red_add(sk.at(v), d);
}

template <int RMAX>
struct RunAcc {
  int rid[RMAX];
  double run[RMAX];
};

// Deterministic mode (STTSV_DETERMINISTIC): every incidence's
// contribution is STORED to its plan-time slot of a vertex-major buffer
// (contrib[slot]), no atomics; a second pass (kernels.cu det_reduce) sums each
// vertex's segment in a fixed order.  The slot column of member i of the
// tile's column c is slot[i * sstride + c].
struct DetSink {
  const int32_t* slot;  // this tile's slot columns (bucket slot pool + tile start)
  int64_t sstride;      // column stride of the slot pool (= the bucket's id stride)
  double* contrib;
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
        if (ra.rid[j] >= 0) red_add(sk.at(ra.rid[j]), ra.run[j]);
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
// consecutive sorted edges base + l*EPL + r, r = 0..EPL-1, which the plan
// stores lane-major at columns base + r*32 + l (conflict-free shared reads).
// Buckets are padded to whole tiles with weight-0 copies of their last edge,
// so every column is valid.
template <int N, int K, int TILE, int EPL, int RMAX, bool DET, typename IdT>
__device__ __forceinline__ void warp_block(const IdT* __restrict__ sids, const WSrc& sw, int base,
                                           const double* __restrict__ xg, RunAcc<RMAX>& ra, const Sink& sk,
                                           const DetSink& ds, int lane) {
  constexpr int L = N - K + 1;
  constexpr int GS = series_stride(N);
  constexpr int WBU = STTSV_WB_UNROLL;
#pragma unroll WBU
  for (int r = 0; r < EPL; ++r) {
    const int col = base + r * 32 + lane;  // lane-major tile layout (plan.cpp): sorted edge base + lane*EPL + r
    int id[K];
    const double* rows[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      id[i] = (int)sids[i * TILE + col];
      rows[i] = xg + (size_t)(uint32_t)id[i] * GS;  // GS compile-time: one IMAD.WIDE.U32
    }
    const double w = sw.at(col, base + lane * EPL + r);
    double q[K], F;
    if constexpr (N >= STTSV_NORM_MIN && STTSV_MID_NORM) dp_edge_table_norm<K, L>(rows, q, F);
    else dp_edge_table<K, L>(rows, q, F);
    const double wF = w * F;
    double dv[K];
#pragma unroll
    for (int i = 0; i < K; ++i) dv[i] = fma(w, q[i], wF);
    if constexpr (DET) {
#pragma unroll
      for (int i = 0; i < K; ++i) ds.contrib[__ldg(ds.slot + i * ds.sstride + col)] = dv[i];
    } else {
      slots_deposit<K, RMAX>(id, dv, ra, sk);
    }
  }
}

template <int N, int K, int TILE, int EPL, int RMAX, bool DET, typename IdT>
__device__ __forceinline__ void dispatch_k(int k, const IdT* sids, const WSrc& sw, int base,
                                           const double* xg, RunAcc<RMAX>& ra, const Sink& sk, const DetSink& ds,
                                           int lane) {
  if constexpr (K <= N) {
    if (k == K) {
      warp_block<N, K, TILE, EPL, RMAX, DET, IdT>(sids, sw, base, xg, ra, sk, ds, lane);
      return;
    }
    dispatch_k<N, K + 1, TILE, EPL, RMAX, DET, IdT>(k, sids, sw, base, xg, ra, sk, ds, lane);
  }
}

// Deposit of own members: slot OFF + i gets (id[i], dv[i]) (run accumulators as slots_deposit)
template <int M, int OFF, int RMAX>
__device__ __forceinline__ void slots_deposit_off(const int (&id)[M], const double (&dv)[M], RunAcc<RMAX>& ra,
                                                  const Sink& sk) {
#pragma unroll
  for (int i = 0; i < M; ++i) {
    constexpr int R1 = RMAX - 1;
    const int slot = OFF + i;
    if (slot < RMAX) {
      const int j = slot < RMAX ? slot : R1;
      if (id[i] != ra.rid[j]) {
        if (ra.rid[j] >= 0) red_add(sk.at(ra.rid[j]), ra.run[j]);
        ra.rid[j] = id[i];
        ra.run[j] = 0.0;
      }
      ra.run[j] += dv[i];
    } else {
      red_add(sk.at(id[i]), dv[i]);
    }
  }
}

// End of a shared-prefix tile (prefix.cuh): sum each of the L terms of the
// lanes' SB over the warp and deposit the prefix members' totals
// sum_j C_i[j] T[j] (lane i < U).  L <= 2: shuffle butterfly; else a transpose
// through this warp's shared-memory rows sred (row j = term j of the 32 lanes,
// kRedStride apart: conflict-free 16-byte reads).
template <int L, bool SHFL = false>
__device__ __forceinline__ void prefix_tile_flush(double (&sb)[L], double* sred, const double* __restrict__ G, int U,
                                                  const Sink& sk, int lane) {
  const double* C = G + L;
  const long long* pid = reinterpret_cast<const long long*>(G + L + U * L);
  if constexpr (L <= 2 || SHFL) {
#pragma unroll
    for (int j = 0; j < L; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sb[j] += __shfl_xor_sync(kFull, sb[j], o);
    for (int i = lane; i < U; i += 32) {
      double c = 0.0;
#pragma unroll
      for (int j = 0; j < L; ++j) c = fma(__ldg(C + i * L + j), sb[j], c);
      red_add(sk.at((int)__ldg(pid + i)), c);
    }
  } else {
#pragma unroll
    for (int j = 0; j < L; ++j) sred[j * kRedStride + lane] = sb[j];
    __syncwarp();
    double t = 0.0;
    if (lane < L) {
      const double2* r = reinterpret_cast<const double2*>(sred + lane * kRedStride);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 v = r[q];
        t += v.x;
        t += v.y;
      }
    }
    __syncwarp();
    if (lane < L) sred[lane] = t;
    __syncwarp();
    for (int i = lane; i < U; i += 32) {
      double c = 0.0;
#pragma unroll
      for (int j = 0; j < L; ++j) c = fma(__ldg(C + i * L + j), sred[j], c);
      red_add(sk.at((int)__ldg(pid + i)), c);
    }
    __syncwarp();
  }
}

// prefix_tile_flush with the prefix members' rows prefetched at the start of the
// block (lane i < U holds C_i in c[] and the member's id in v; U <= 31 here): the
// flush does not wait on the group table
template <int L, bool SHFL = false>
__device__ __forceinline__ void prefix_tile_flush_pre(double (&sb)[L], double* sred, const double (&c)[L], int v,
                                                      const Sink& sk, int lane) {
  if constexpr (L <= 2 || SHFL) {
#pragma unroll
    for (int j = 0; j < L; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sb[j] += __shfl_xor_sync(kFull, sb[j], o);
    if (v >= 0) {
      double d = 0.0;
#pragma unroll
      for (int j = 0; j < L; ++j) d = fma(c[j], sb[j], d);
      red_add(sk.at(v), d);
    }
  } else {
#pragma unroll
    for (int j = 0; j < L; ++j) sred[j * kRedStride + lane] = sb[j];
    __syncwarp();
    double t = 0.0;
    if (lane < L) {
      const double2* r = reinterpret_cast<const double2*>(sred + lane * kRedStride);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 u = r[q];
        t += u.x;
        t += u.y;
      }
    }
    __syncwarp();
    if (lane < L) sred[lane] = t;
    __syncwarp();
    if (v >= 0) {
      double d = 0.0;
#pragma unroll
      for (int j = 0; j < L; ++j) d = fma(c[j], sred[j], d);
      red_add(sk.at(v), d);
    }
    __syncwarp();
  }
}

// M = 0 tile or edge block (every edge the same vertex set): the prefix members
// get sum w' times C_i[0]; with uniform weights the sum is wc x (real edges in
// positions [base, base + n)), no loads at all
__device__ __forceinline__ void prefix_tile_flush0(double t0, const double* __restrict__ G, int L, int U,
                                                   const Sink& sk, int lane) {
  const long long* pid = reinterpret_cast<const long long*>(G + L + U * L);
  for (int i = lane; i < U; i += 32) red_add(sk.at((int)__ldg(pid + i)), __ldg(G + L + i * L) * t0);
}

// The warp's block of a staged tile whose edges share their first U = K - M
// members (the stage holds only the M own id columns).  G: the tile's prefix
// group in the per-apply group table (prefix.cuh: front A, the contraction
// rows C_i and the prefix ids).  Each lane accumulates SB = sum_e w'_e B_e over
// its edges; at the end of the block the warp sums SB and lane i < U deposits
// member i's total  sum_j C_i[j] SB[j].
// BATCH (f4, sttsv_apply_batch): called once per vector (vpass = 0, 1, ...) on
// the same staged block; the run queue is built by pass 0 only (its length is
// kept in qn) and read again by the later passes, so the block flush keeps its
// reduction in registers instead of the queue's shared scratch.
template <int N, int K, int M, int TILE, int EPL, int RMAX, typename IdT, bool BATCH = false>
__device__ __forceinline__ void warp_block_prefix(const IdT* __restrict__ sids, const WSrc& sw,
                                                  int base, const double* __restrict__ xg,
                                                  const double* __restrict__ G, RunAcc<RMAX>& ra, const Sink& sk,
                                                  double* sred, int lane, int vpass, int& qn) {
  constexpr int L = N - K + 1;
  constexpr int GS = series_stride(N);
  constexpr int U = K - M;
  if constexpr (M == 0) {
    // every edge of the tile is the same vertex set: SB = (sum w', 0, ...)
    double t0;
    if (sw.uni) {
      int n = sw.real - base;
      n = n < 0 ? 0 : (n > 32 * EPL ? 32 * EPL : n);
      t0 = sw.wc * (double)n;
    } else {
      t0 = 0.0;
#pragma unroll
      for (int r = 0; r < EPL; ++r) t0 += sw.sw[base + r * 32 + lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t0 += __shfl_xor_sync(kFull, t0, o);
    }
    prefix_tile_flush0(t0, G, L, U, sk, lane);
  } else {
    double sb[L];
#pragma unroll
    for (int j = 0; j < L; ++j) sb[j] = 0.0;
    double a[L];
#pragma unroll
    for (int j = 0; j < L; ++j) a[j] = __ldg(G + j);  // front A (row format), the same on every lane
    // the flush's rows: lane i < U takes prefix member i's C_i and id now (U <= 31),
    // where the registers allow it (FLUSHPRE)
    constexpr bool FLUSHPRE = L <= (N <= 8 ? STTSV_FLUSHPRE_L8 : STTSV_FLUSHPRE_L);
    double cpre[FLUSHPRE ? L : 1];
    int vpre = -1;
    if constexpr (FLUSHPRE) {
      if (lane < U) {
#pragma unroll
        for (int j = 0; j < L; ++j) cpre[j] = __ldg(G + L + lane * L + j);
        vpre = (int)__ldg(reinterpret_cast<const long long*>(G + L + U * L) + lane);
      } else {
#pragma unroll
        for (int j = 0; j < L; ++j) cpre[j] = 0.0;
      }
    }
    // Runs of identical consecutive edges among the lane's EPL edges (sorted
    // buckets keep duplicates adjacent) need one DP each, on the run's summed
    // weight: pass 1 counts the lane's runs, a warp scan places them in this
    // warp's queue (scratch sred), pass 2 writes (sum w', column) per run; then
    // the warp works through the queue, lane l taking entries l*c .. l*c+c-1
    // (consecutive distinct edges: the deposit runs carry over).
    double* qw = sred;
    int* qc = reinterpret_cast<int*>(sred + 32 * EPL);
    int Q;
    if (!BATCH || vpass == 0) {
    int prev[M];
    int nrun = 0;
#pragma unroll
    for (int r = 0; r < EPL; ++r) {
      const int col = base + r * 32 + lane;
      bool same = r > 0;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        const int v = (int)sids[i * TILE + col];
        same = same && v == prev[i];
        prev[i] = v;
      }
      nrun += same ? 0 : 1;
    }
    int incl = nrun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    Q = __shfl_sync(kFull, incl, 31);
    {
      int pos = incl - nrun, rc = -1;
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < EPL; ++r) {
        const int col = base + r * 32 + lane;
        bool same = r > 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
          const int v = (int)sids[i * TILE + col];
          same = same && v == prev[i];
          prev[i] = v;
        }
        const double w = sw.at(col, base + lane * EPL + r);
        if (!same) {
          if (rc >= 0) {
            qw[pos] = acc;
            qc[pos] = rc;
            ++pos;
          }
          rc = col;
          acc = w;
        } else {
          acc += w;
        }
      }
      qw[pos] = acc;
      qc[pos] = rc;
    }
    __syncwarp();
    qn = Q;
    } else {
      Q = qn;
    }
    const int c = (Q + 31) >> 5;
    // one queue entry: the DP over the own members with the front A, the
    // deposits of the own members and the entry's SB term
    auto entry = [&](bool live, double w, const int (&id)[M], const double (&h)[M][L]) {
      double q[M], F, bh[L];
      dp_front_norm<M, L>(a, h, q, F, bh);
      const double wF = w * F;
      double dv[M];
#pragma unroll
      for (int i = 0; i < M; ++i) dv[i] = fma(w, q[i], wF);
      if (live) slots_deposit_off<M, U, RMAX>(id, dv, ra, sk);
      const double cw = w * bh[0];
      sb[0] += cw;
#pragma unroll
      for (int j = 1; j < L; ++j) sb[j] = fma(cw, bh[j], sb[j]);
    };
    auto fetch = [&](int e, bool& live, double& w, int (&id)[M], double (&h)[M][L]) {
      live = e < Q;
      const int col = qc[live ? e : 0];
      w = live ? qw[e] : 0.0;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        id[i] = (int)sids[i * TILE + col];
        load_series<L>(xg + (size_t)(uint32_t)id[i] * GS, h[i]);
      }
    };
    if constexpr (M * L <= STTSV_PIPE_ML) {
      // software pipeline: the next entry's ids and table rows are loaded before
      // the current entry's DP (the row loads are a round's latency)
      bool liven;
      double wn;
      int idn[M];
      double hn[M][L];
      fetch(lane * c, liven, wn, idn, hn);
#pragma unroll 1
      for (int e = lane * c; e < lane * c + c; ++e) {
        const bool live = liven;
        const double w = wn;
        int id[M];
        double h[M][L];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          id[i] = idn[i];
#pragma unroll
          for (int j = 0; j < L; ++j) h[i][j] = hn[i][j];
        }
        if (e + 1 < lane * c + c) fetch(e + 1, liven, wn, idn, hn);
        entry(live, w, id, h);
      }
    } else {
#pragma unroll 1
      for (int e = lane * c; e < lane * c + c; ++e) {
        bool live;
        double w;
        int id[M];
        double h[M][L];
        fetch(e, live, w, id, h);
        entry(live, w, id, h);
      }
    }
    __syncwarp();  // the queue is read before the reduction reuses the scratch
    if constexpr (FLUSHPRE) prefix_tile_flush_pre<L, BATCH>(sb, sred, cpre, vpre, sk, lane);
    else prefix_tile_flush<L, BATCH>(sb, sred, G, U, sk, lane);
  }
}

// prefix tiles of bucket K: dispatch on the number of own members M = K - U
template <int N, int K, int M, int MMAX, int TILE, int EPL, int RMAX, typename IdT, bool BATCH>
__device__ __forceinline__ void dispatch_m(int m, const IdT* sids, const WSrc& sw, int base, const double* xg,
                                           const double* G, RunAcc<RMAX>& ra, const Sink& sk, double* sred,
                                           int lane, int vpass, int& qn) {
  if constexpr (M < K && M <= MMAX) {
    if (m == M) {
      warp_block_prefix<N, K, M, TILE, EPL, RMAX, IdT, BATCH>(sids, sw, base, xg, G, ra, sk, sred, lane, vpass, qn);
      return;
    }
    dispatch_m<N, K, M + 1, MMAX, TILE, EPL, RMAX, IdT, BATCH>(m, sids, sw, base, xg, G, ra, sk, sred, lane, vpass,
                                                               qn);
  }
}

template <int N, int K, int MMAX, int TILE, int EPL, int RMAX, typename IdT, bool BATCH>
__device__ __forceinline__ void dispatch_kp(int k, int U, const IdT* sids, const WSrc& sw, int base,
                                            const double* xg, const double* G, RunAcc<RMAX>& ra, const Sink& sk,
                                            double* sred, int lane, int vpass, int& qn) {
  if constexpr (K <= N) {
    if (k == K) {
      dispatch_m<N, K, 0, MMAX, TILE, EPL, RMAX, IdT, BATCH>(K - U, sids, sw, base, xg, G, ra, sk, sred, lane, vpass,
                                                             qn);
      return;
    }
    dispatch_kp<N, K + 1, MMAX, TILE, EPL, RMAX, IdT, BATCH>(k, U, sids, sw, base, xg, G, ra, sk, sred, lane, vpass,
                                                             qn);
  }
}

// ------------------------------------------------------- large-rank path
// For large L = N-K+1 a lane cannot hold K series in registers.  One edge per
// lane; members are walked by a RUNTIME loop; the working rows (current prefix
// P, one member row g, suffix S) are L-long register arrays; the prefix stack
// P_0..P_{K-4} lives in per-thread local memory (STTSV_BIG_LOCAL = 1, L1-cached)
// or thread-interleaved shared memory; each member's series row is loaded from
// the L1/L2-resident table where it is used.  Products are formed in place
// (descending coefficient order).


// a = (a*b) mod t^L, in place
template <int L>
__device__ __forceinline__ void trunc_mul_inplace(double (&a)[L], const double (&b)[L]) {
#pragma unroll
  for (int j = L - 1; j >= 0; --j) {
    double s = a[0] * b[j];
#pragma unroll
    for (int i = 1; i <= j; ++i) s = fma(a[i], b[j - i], s);
    a[j] = s;
  }
}

// deposit of slot i (warp-uniform runtime index): slots < RB use the run
// accumulators (compile-time register index via a uniform compare chain)
template <int RB>
__device__ __forceinline__ void dep_slot(int i, int v, double d, RunAcc<RB>& ra, const Sink& sk) {
  if (i < RB) {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (i == r) {
        if (v != ra.rid[r]) {
          if (ra.rid[r] >= 0) red_add(sk.at(ra.rid[r]), ra.run[r]);
          ra.rid[r] = v;
          ra.run[r] = 0.0;
        }
        ra.run[r] += d;
      }
    }
  } else {
    red_add(sk.at(v), d);
  }
}

// one edge of size K (runtime) with L = N-K+1 (compile time); sid = member 0's
// id in the staged tile (member i at sid[i * TILE]); stk = this thread's stack
// (row r coefficient j at stk[(r * L + j) * NT])
template <int L, int TILE, int NT, int RB, bool DET>
__device__ __forceinline__ void edge_big(int K, const int32_t* __restrict__ sid, double w,
                                         const double* __restrict__ xg, int gs, double* __restrict__ stk,
                                         RunAcc<RB>& ra, const Sink& sk, const DetSink& ds, int col) {
  // NT = 1: stk is a thread-private (local) array; else thread-interleaved shared memory
  constexpr int D = L - 1;
  auto row = [&](int i) { return xg + (size_t)(uint32_t)sid[i * TILE] * gs; };
  // deposit of member i's contribution (runs + reds, or the deterministic store)
  auto dep = [&](int i, int v, double d) {
    if constexpr (DET) ds.contrib[__ldg(ds.slot + i * ds.sstride + col)] = d;
    else dep_slot<RB>(i, v, d, ra, sk);
  };
  if (K == 1) {
    // singleton: Q = 1 (empty product), F = g_0:  q = [D == 0],  F[D-1] = x^D / D!
    const double F = D >= 1 ? __ldg(row(0) + (D >= 1 ? D - 1 : 0)) : 0.0;
    dep(0, sid[0], w * ((D == 0 ? 1.0 : 0.0) + F));
    return;
  }
  if (K == 2) {
    double a[L], b[L];
    load_series<L>(row(0), a);
    load_series<L>(row(1), b);
    double F = 0.0;
    if constexpr (D >= 1) F = coef<D - 1, L>(a, b);
    const double wF = w * F;
    dep(0, sid[0], fma(w, b[D], wF));
    dep(1, sid[TILE], fma(w, a[D], wF));
    return;
  }
  double cur[L], g[L], S[L];
  load_series<L>(row(0), cur);  // P_0
#pragma unroll 1
  for (int i = 1; i <= K - 3; ++i) {
    load_series<L>(row(i), g);  // issued before the pushes: the load latency overlaps them
    if (i > 1) {                // P_0 = g_0 is re-read from the table later, not stacked
#pragma unroll
      for (int j = 0; j < L; ++j) stk[((i - 1) * L + j) * NT] = cur[j];  // push P_{i-1}
    }
    trunc_mul_inplace<L>(cur, g);  // P_i
  }
  // cur = P_{K-3}
  load_series<L>(row(K - 2), g);
  load_series<L>(row(K - 1), S);
  const double qa = coef<D, L>(cur, g);  // [t^D] P_{K-2}             -> member K-1
  const double qb = coef<D, L>(cur, S);  // [t^D] P_{K-3} g_{K-1}     -> member K-2
  trunc_mul_inplace<L>(S, g);            // S_{K-2} = g_{K-2} g_{K-1}
  double F = 0.0;
  if constexpr (D >= 1) F = coef<D - 1, L>(cur, S);
  const double wF = w * F;
  dep(K - 1, sid[(K - 1) * TILE], fma(w, qa, wF));
  dep(K - 2, sid[(K - 2) * TILE], fma(w, qb, wF));
#pragma unroll 1
  for (int i = K - 3; i >= 1; --i) {
    load_series<L>(row(i), g);  // issued first: overlaps the pop and the coefficient below
    if (i > 1) {
#pragma unroll
      for (int j = 0; j < L; ++j) cur[j] = stk[((i - 1) * L + j) * NT];  // pop P_{i-1}
    } else {
      load_series<L>(row(0), cur);  // P_0 = g_0 (the hottest row: L1-resident)
    }
    dep(i, sid[i * TILE], fma(w, coef<D, L>(cur, S), wF));
    if (i > 1) {
      trunc_mul_inplace<L>(S, g);  // S_i = g_i S_{i+1}
    } else {
      dep(0, sid[0], fma(w, coef<D, L>(g, S), wF));  // [t^D] g_1 S_2
    }
  }
  if (K == 3) dep(0, sid[0], fma(w, S[D], wF));  // S = S_1
}

// ---- normalised variant (STTSV_BIG_NORM): table rows hold x in slot 0 and
// h[j] = x^j/(j+1)! (h[0] = 1 implicit), so g_u = x_u h_u.  Products of
// normalised series keep a leading 1: a truncated product costs L(L-1)/2
// operations instead of L(L+1)/2, and the scalar factors prod x_u are carried
// separately (prefix product X on the stack row's slot 0, suffix product Xs).
// Every term is still a product of positive numbers for x > 0.

// a = (a*b) mod t^L for a[0] = b[0] = 1 (slot 0 never read or written), in place
template <int L>
__device__ __forceinline__ void trunc_mul_norm_inplace(double (&a)[L], const double (&b)[L]) {
#pragma unroll
  for (int j = L - 1; j >= 1; --j) {
    double s = a[j] + b[j];
#pragma unroll
    for (int i = 1; i < j; ++i) s = fma(a[i], b[j - i], s);
    a[j] = s;
  }
}

// [t^D] (a*b) for a[0] = b[0] = 1
template <int D, int L>
__device__ __forceinline__ double coef_norm(const double (&a)[L], const double (&b)[L]) {
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

// load a normalised row: returns x (slot 0), fills h[1..L-1]; h[0] is not a
// coefficient (the leading 1 stays implicit)
template <int L>
__device__ __forceinline__ double load_norm(const double* __restrict__ row, double (&h)[L]) {
  load_series<L>(row, h);
  return h[0];
}

template <int L, int TILE, int NT, int RB, bool DET>
__device__ __forceinline__ void edge_big_norm(int K, const int32_t* __restrict__ sid, double w,
                                              const double* __restrict__ xg, int gs, double* __restrict__ stk,
                                              RunAcc<RB>& ra, const Sink& sk, const DetSink& ds, int col) {
  constexpr int D = L - 1;
  auto row = [&](int i) { return xg + (size_t)(uint32_t)sid[i * TILE] * gs; };
  auto dep = [&](int i, int v, double d) {
    if constexpr (DET) ds.contrib[__ldg(ds.slot + i * ds.sstride + col)] = d;
    else dep_slot<RB>(i, v, d, ra, sk);
  };
  if (K == 1) {
    // singleton: q = [D == 0], F = g_0[D-1] = x h[D-1]
    const double* r = row(0);
    const double x = __ldg(r);
    const double F = D >= 1 ? (D == 1 ? x : x * __ldg(r + (D >= 2 ? D - 1 : 0))) : 0.0;
    dep(0, sid[0], w * ((D == 0 ? 1.0 : 0.0) + F));
    return;
  }
  if (K == 2) {
    double a[L], b[L];
    const double xa = load_norm<L>(row(0), a);
    const double xb = load_norm<L>(row(1), b);
    double F = 0.0;
    if constexpr (D >= 1) F = xa * xb * coef_norm<D - 1, L>(a, b);
    const double wF = w * F;
    dep(0, sid[0], fma(w, D == 0 ? xb : xb * b[D], wF));   // g_1[D] = x_1 h_1[D]
    dep(1, sid[TILE], fma(w, D == 0 ? xa : xa * a[D], wF));
    return;
  }
  double cur[L], g[L], S[L];
  double X = load_norm<L>(row(0), cur);  // P_0 = h_0, scalar prefix x_0
#pragma unroll 1
  for (int i = 1; i <= K - 3; ++i) {
    const double xi = load_norm<L>(row(i), g);
    if (i > 1) {  // P_0 = h_0 is re-read from the table later, not stacked
      stk[((i - 1) * L) * NT] = X;
#pragma unroll
      for (int j = 1; j < L; ++j) stk[((i - 1) * L + j) * NT] = cur[j];  // push (X_{i-1}, P_{i-1})
    }
    trunc_mul_norm_inplace<L>(cur, g);  // P_i
    X *= xi;
  }
  // cur = P_{K-3} (normalised), X = x_0 ... x_{K-3}
  const double xa = load_norm<L>(row(K - 2), g);
  const double xb = load_norm<L>(row(K - 1), S);
  const double qa = X * xa * coef_norm<D, L>(cur, g);  // [t^D] P_{K-2}          -> member K-1
  const double qb = X * xb * coef_norm<D, L>(cur, S);  // [t^D] P_{K-3} g_{K-1}  -> member K-2
  trunc_mul_norm_inplace<L>(S, g);                     // S_{K-2} (normalised)
  double Xs = xa * xb;
  double F = 0.0;
  if constexpr (D >= 1) F = X * Xs * coef_norm<D - 1, L>(cur, S);
  const double wF = w * F;
  dep(K - 1, sid[(K - 1) * TILE], fma(w, qa, wF));
  dep(K - 2, sid[(K - 2) * TILE], fma(w, qb, wF));
#pragma unroll 1
  for (int i = K - 3; i >= 1; --i) {
    const double xi = load_norm<L>(row(i), g);
    double Xp;
    if (i > 1) {
      Xp = stk[((i - 1) * L) * NT];
#pragma unroll
      for (int j = 1; j < L; ++j) cur[j] = stk[((i - 1) * L + j) * NT];  // pop (X_{i-1}, P_{i-1})
    } else {
      Xp = load_norm<L>(row(0), cur);  // P_0 = h_0 (the hottest row: L1-resident)
    }
    dep(i, sid[i * TILE], fma(w, Xp * Xs * coef_norm<D, L>(cur, S), wF));
    if (i > 1) {
      trunc_mul_norm_inplace<L>(S, g);  // S_i = g_i S_{i+1}
      Xs *= xi;
    } else {
      dep(0, sid[0], fma(w, xi * Xs * coef_norm<D, L>(g, S), wF));  // [t^D] g_1 S_2
    }
  }
  if (K == 3) dep(0, sid[0], fma(w, D == 0 ? Xs : Xs * S[D], wF));  // S_1 = x_1 x_2 (h_1 h_2)
}

template <int L, int LMAX, int TILE, int NT, int RB, bool DET>
__device__ __forceinline__ void dispatch_big(int L_rt, int K, const int32_t* sid, double w, const double* xg, int gs,
                                             double* stk, RunAcc<RB>& ra, const Sink& sk, const DetSink& ds,
                                             int col) {
  if constexpr (L <= LMAX) {
    if (L_rt == L) {
#if STTSV_BIG_NORM
      edge_big_norm<L, TILE, NT, RB, DET>(K, sid, w, xg, gs, stk, ra, sk, ds, col);
#else
      edge_big<L, TILE, NT, RB, DET>(K, sid, w, xg, gs, stk, ra, sk, ds, col);
#endif
      return;
    }
    dispatch_big<L + 1, LMAX, TILE, NT, RB, DET>(L_rt, K, sid, w, xg, gs, stk, ra, sk, ds, col);
  }
}

// ---- large-rank path with a shared prefix (prefix.cuh): the lane's edge has U
// shared leading members (front A, row format a[], from the group table) and M
// own members (stage columns sid[i * TILE], i < M).  Deposits the own members'
// contributions (slots U + i) and returns the edge's SB term in sb (+= w' B).
template <int L, int TILE, int NT, int RB>
__device__ __forceinline__ void edge_big_front(int M, int U, const int32_t* __restrict__ sid, double w,
                                               const double (&a)[L], const double* __restrict__ xg, int gs,
                                               double* __restrict__ stk, RunAcc<RB>& ra, const Sink& sk,
                                               double (&sb)[L]) {
  constexpr int D = L - 1;
  auto row = [&](int i) { return xg + (size_t)(uint32_t)sid[i * TILE] * gs; };  // own member i
  const double Xa = a[0];
  if (M == 1) {
    double h[L];
    const double x = load_norm<L>(row(0), h);
    double F = 0.0;
    if constexpr (D >= 1) F = Xa * x * coef_norm<D - 1, L>(a, h);
    const double q = D == 0 ? Xa : Xa * a[D];
    dep_slot<RB>(U, sid[0], w * (q + F), ra, sk);
    const double c = w * x;
    sb[0] += c;
#pragma unroll
    for (int j = 1; j < L; ++j) sb[j] = fma(c, h[j], sb[j]);
    return;
  }
  // members g'_0 = A, g'_i = own member i - 1 (K' = M + 1)
  const int KP = M + 1;
  double cur[L], g[L], S[L];
#pragma unroll
  for (int j = 1; j < L; ++j) cur[j] = a[j];
  double X = Xa;
#pragma unroll 1
  for (int i = 1; i <= KP - 3; ++i) {
    const double xi = load_norm<L>(row(i - 1), g);
    if (i > 1) {  // P'_0 = A stays in registers, not stacked
      stk[((i - 1) * L) * NT] = X;
#pragma unroll
      for (int j = 1; j < L; ++j) stk[((i - 1) * L + j) * NT] = cur[j];
    }
    trunc_mul_norm_inplace<L>(cur, g);
    X *= xi;
  }
  const double xa = load_norm<L>(row(KP - 3), g);
  const double xb = load_norm<L>(row(KP - 2), S);
  const double qa = X * xa * coef_norm<D, L>(cur, g);  // own member M-1
  const double qb = X * xb * coef_norm<D, L>(cur, S);  // own member M-2
  trunc_mul_norm_inplace<L>(S, g);
  double Xs = xa * xb;
  double F = 0.0;
  if constexpr (D >= 1) F = X * Xs * coef_norm<D - 1, L>(cur, S);
  const double wF = w * F;
  dep_slot<RB>(U + M - 1, sid[(M - 1) * TILE], fma(w, qa, wF), ra, sk);
  dep_slot<RB>(U + M - 2, sid[(M - 2) * TILE], fma(w, qb, wF), ra, sk);
#pragma unroll 1
  for (int i = KP - 3; i >= 1; --i) {
    const double xi = load_norm<L>(row(i - 1), g);
    double Xp;
    if (i > 1) {
      Xp = stk[((i - 1) * L) * NT];
#pragma unroll
      for (int j = 1; j < L; ++j) cur[j] = stk[((i - 1) * L + j) * NT];
    } else {
      Xp = Xa;
#pragma unroll
      for (int j = 1; j < L; ++j) cur[j] = a[j];
    }
    dep_slot<RB>(U + i - 1, sid[(i - 1) * TILE], fma(w, Xp * Xs * coef_norm<D, L>(cur, S), wF), ra, sk);
    trunc_mul_norm_inplace<L>(S, g);  // S'_i = g'_i S'_{i+1}
    Xs *= xi;
  }
  // S = S'_1 = B
  const double c = w * Xs;
  sb[0] += c;
#pragma unroll
  for (int j = 1; j < L; ++j) sb[j] = fma(c, S[j], sb[j]);
}

// one warp's 32 edges (lane = column) of a shared-prefix tile on the large-rank path
template <int L, int TILE, int NT, int RB>
__device__ __forceinline__ void big_prefix_block(int K, int U, const int32_t* sid, double w, const WSrc& sw, int base,
                                                 const double* G, const double* xg, int gs, double* stk,
                                                 RunAcc<RB>& ra, const Sink& sk, double* sred, int lane) {
  const int M = K - U;
  if (M == 0) {
    double t0;
    if (sw.uni) {
      int n = sw.real - base;
      t0 = sw.wc * (double)(n < 0 ? 0 : (n > 32 ? 32 : n));
    } else {
      t0 = w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t0 += __shfl_xor_sync(kFull, t0, o);
    }
    prefix_tile_flush0(t0, G, L, U, sk, lane);
    return;
  }
  double sb[L];
#pragma unroll
  for (int j = 0; j < L; ++j) sb[j] = 0.0;
  double a[L];
#pragma unroll
  for (int j = 0; j < L; ++j) a[j] = __ldg(G + j);
  edge_big_front<L, TILE, NT, RB>(M, U, sid, w, a, xg, gs, stk, ra, sk, sb);
  prefix_tile_flush<L>(sb, sred, G, U, sk, lane);
}

template <int L, int LMAX, int TILE, int NT, int RB>
__device__ __forceinline__ void dispatch_big_prefix(int L_rt, int K, int U, const int32_t* sid, double w,
                                                    const WSrc& sw, int base, const double* G, const double* xg,
                                                    int gs, double* stk, RunAcc<RB>& ra, const Sink& sk,
                                                    double* sred, int lane) {
  if constexpr (L <= LMAX) {
    if (L_rt == L) {
      big_prefix_block<L, TILE, NT, RB>(K, U, sid, w, sw, base, G, xg, gs, stk, ra, sk, sred, lane);
      return;
    }
    dispatch_big_prefix<L + 1, LMAX, TILE, NT, RB>(L_rt, K, U, sid, w, sw, base, G, xg, gs, stk, ra, sk, sred,
                                                   lane);
  }
}

// ------------------------------------------------------------- the kernel
// N == 0 is the generic instantiation (any rank <= STTSV_MAX_RANK).
// BATCH = false: one vector (sttsv_apply; runs continue across tiles);
// BATCH = true: p.nvec vectors per tile (sttsv_apply_batch, f4).
// DET = true: deterministic stores into the vertex-major buffer (f2; one vector).
// IDB: bytes per member id in the edge stream (EdgeCfg).
template <int N, bool BATCH, bool DET, int IDB = 4>
__global__ void __launch_bounds__(EdgeCfg<N, IDB>::THREADS, EdgeCfg<N, IDB>::MIN_BLOCKS)
    edge_kernel(const __grid_constant__ EdgeKernelParams p) {
  using Cfg = EdgeCfg<N, IDB>;
  constexpr int TILE = Cfg::TILE, KMAX = Cfg::KMAX, NCW = Cfg::NCW, EPL = Cfg::EPL;
  constexpr int RMAX = Cfg::RMAX;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // layout: byte ring of stages [ ids k*TILE int32 | w TILE f64 ] | (large-rank path) prefix
  // stacks [p.stack_doubles][NCW*32] f64, thread-interleaved
  unsigned char* ring = smem_raw;
  double* sred_all = reinterpret_cast<double*>(smem_raw + Cfg::RING_BYTES);  // prefix reduction rows
  double* stack = reinterpret_cast<double*>(smem_raw + Cfg::RING_BYTES + Cfg::RED_BYTES);
  // batch (f4): vector v uses xg + v*xg_vstride, ya + v*ya_vstride, priv slice + v*H
  const int nvec = BATCH ? p.nvec : 1;
  double* const priv_cta = p.priv + (size_t)blockIdx.x * p.H * nvec;
  const Sink sk{priv_cta, p.ya, p.H};
  constexpr int SLOTS = Cfg::SLOTS;
  __shared__ uint64_t full[SLOTS], empty[SLOTS];
  __shared__ uint32_t soff[SLOTS];  // byte offset of each slot's stage in the ring
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ int64_t stile[SLOTS];  // tile index staged in each slot (-1: no more work)
  __shared__ uint8_t su[SLOTS];     // its staged prefix length U_stage (id columns 0..U_stage-1 are not staged)
  __shared__ long long sblk[SLOTS][NCW];  // per warp block: (group record offset << 8) | U (prefix.cuh)
  __shared__ uint8_t sbk[SLOTS];    // its bucket (index into p.b)
  __shared__ int64_t sit[SLOTS];    // the producer iteration staged in each slot (dynamic blocks)
  __shared__ unsigned int s_next;   // next warp block of the CTA's staged sequence (dynamic blocks)

  for (int j = tid; j < p.H * nvec; j += Cfg::THREADS) priv_cta[j] = 0.0;
#if STTSV_WAITPROF > 1
  __shared__ unsigned long long s_kc[2 * (STTSV_MAX_RANK + 1)];  // per-CTA class counters (one global add each at the end)
  for (int j = tid; j < 2 * (STTSV_MAX_RANK + 1); j += Cfg::THREADS) s_kc[j] = 0ull;
#endif
  if (tid == 0) {
    s_next = 0u;
    for (int s = 0; s < SLOTS; ++s) {
      sit[s] = -1;
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_proxy_async();
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------- producer warp: grab chunks of tiles; each tile's stage is
    // TILE*(4k+8) bytes carved FIFO out of the byte ring (wrapping to offset 0
    // when the tail of the ring is too short); slot it % SLOTS carries its
    // offset and tile index (published before the mbarrier's release)
    // The whole warp loads the packed headers (shared-prefix length U and group
    // record offset, prefix.cuh) of up to 32 upcoming tiles of its chunk at once, so
    // lane 0's per-tile path has no dependent global load.
    __shared__ long long shdr[32];
    __shared__ long long shblk[32][NCW];
    int b = 0;
    int64_t ct = 0, ce = 0, hb = 0, he = 0;
    uint64_t head = 0, tail = 0;  // ring positions (monotonic; offset = pos % RING_BYTES), lane 0
    uint64_t endpos[SLOTS];       // ring position just past each in-flight slot's stage, lane 0
    int64_t oldest = 0;           // oldest iteration whose stage may still be in use, lane 0
    for (int64_t it = 0;; ++it) {
      const int s = (int)(it % SLOTS);
      if (ct == ce) {
        // guided: chunks of p.chunk tiles, single tiles once the counter passes
        // p.guided_from (the tail is split finely across the CTAs)
        const int64_t want = ct < p.guided_from ? p.chunk : 1;
        unsigned long long c0 = 0;
        if (lane == 0) c0 = atomicAdd(p.tile_counter, (unsigned long long)want);
        ct = (int64_t)__shfl_sync(kFull, c0, 0);
        ce = ct + want < p.num_tiles ? ct + want : p.num_tiles;
      }
      const int64_t t = ct < p.num_tiles ? ct++ : -1;
      if (t >= 0 && t >= he) {
        hb = t;
        he = ce < t + 32 ? ce : t + 32;
        const bool hv = p.tile_hdr && hb + lane < he;
        const long long* th = p.tile_hdr + (size_t)(hb + lane) * (NCW + 1);
        shdr[lane] = hv ? __ldg(th) : 0ll;
#pragma unroll
        for (int w = 0; w < NCW; ++w) shblk[lane][w] = hv ? __ldg(th + 1 + w) : 0ll;
        __syncwarp();
      }
      if (lane == 0) {
        if (t >= 0)
          while (b + 1 < p.nb && t >= p.b[b + 1].tile_begin) ++b;
        const int k = t >= 0 ? p.b[b].k : 0;
        const long long hdr = t >= 0 ? shdr[t - hb] : 0ll;
        const int tu = (int)(hdr & 255);
        const uint32_t need = t >= 0 ? (uint32_t)(TILE * (Cfg::IDB * (k - tu) + (p.b[b].wuni ? 0 : 8))) : 0u;
        uint64_t start = head;
        if (start % Cfg::RING_BYTES + need > (uint64_t)Cfg::RING_BYTES) start += Cfg::RING_BYTES - start % Cfg::RING_BYTES;
        while (it - oldest >= SLOTS || (oldest < it && start + need - tail > (uint64_t)Cfg::RING_BYTES)) {
          const int so = (int)(oldest % SLOTS);
          mbar_wait_sleep(&empty[so], (uint32_t)((oldest / SLOTS) & 1));
          tail = endpos[so];
          ++oldest;
        }
        endpos[s] = start + need;
        head = start + need;
        const uint32_t off = (uint32_t)(start % Cfg::RING_BYTES);
        soff[s] = off;
        stile[s] = t;
        sit[s] = it;
        su[s] = (uint8_t)tu;
        sbk[s] = (uint8_t)b;
#pragma unroll
        for (int w = 0; w < NCW; ++w) sblk[s][w] = t >= 0 ? shblk[t - hb][w] : 0ll;
        if (t < 0) {
          mbar_arrive_expect_tx(&full[s], 0);
        } else {
          const BucketDesc& bd = p.b[b];
          const int64_t e0 = (t - bd.tile_begin) * TILE;  // buckets are padded to whole tiles
          constexpr uint32_t id_bytes = TILE * Cfg::IDB, w_bytes = TILE * 8;
          unsigned char* st = ring + off;
          const unsigned char* idp = reinterpret_cast<const unsigned char*>(p.ids);
          mbar_arrive_expect_tx(&full[s], need);
          for (int i = tu; i < k; ++i)  // the shared prefix columns 0..U-1 are not staged
            bulk_g2s(st + (i - tu) * id_bytes, idp + (size_t)(bd.ids_off + i * bd.stride + e0) * Cfg::IDB, id_bytes,
                     &full[s]);
          if (!bd.wuni) bulk_g2s(st + (k - tu) * id_bytes, p.w + bd.w_off + e0, w_bytes, &full[s]);
        }
      }
      __syncwarp();
      if (t < 0) break;
    }
  } else {
    // ---------------- consumer warps
#if STTSV_BIG_LOCAL
    double lstk[Cfg::BIG ? big_stack_doubles(KMAX) + 1 : 1];  // large-rank prefix stack (local memory)
#endif
    RunAcc<RMAX> ra;
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      ra.rid[i] = -1;  // empty run
      ra.run[i] = 0.0;
    }
    constexpr bool PREFIX = Cfg::PMAX > 0 && !Cfg::BIG && !DET;
    double* const sred = sred_all + warp * Cfg::SCR_DOUBLES;
    bool any = false;
    // programmatic dependent launch: x_a, the series table and y_a are written
    // by the prologue grid (no-op when launched without the PDL attribute).  Behind
    // the group kernel (p.group_wait) only the group table comes from the preceding
    // grid: the wait is deferred to the first read of the table (gready).
    bool gready = !p.group_wait;
    if (gready) griddep_wait();
    auto need_groups = [&]() {
      if (!gready) {
        griddep_wait();
        gready = true;
      }
    };
    // pending M = 0 prefix group (prefix.cuh): consecutive tiles whose edges are all one
    // vertex set of the same group only add their weights (this lane's share) here;
    // the group's totals are deposited once, when another M = 0 group starts or at the end
    int64_t pend_goff = -1;
    int pend_L = 0, pend_U = 0;
    double pend_w = 0.0;
    auto flush_pending = [&]() {
      need_groups();
      double t0 = pend_w;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t0 += __shfl_xor_sync(kFull, t0, o);
      for (int v = 0; v < nvec; ++v)
        prefix_tile_flush0(t0, p.gtab + (size_t)v * p.gtab_vstride + pend_goff, pend_L, pend_U,
                           Sink{priv_cta + (size_t)v * p.H, p.ya + (size_t)v * p.ya_vstride, p.H}, lane);
    };
#if STTSV_WAITPROF
    long long wait_cyc = 0;
    const long long c_start = clock64();
    if (tid == 0 && blockIdx.x < 1024) g_cta_ns[3 * blockIdx.x] = gtimer();
    unsigned long long ntiles = 0;
#endif
#if !STTSV_DYN_BLOCKS
    const int wb = warp;  // this warp's block of every tile
#endif
    for (int64_t it = 0;; ++it) {
#if STTSV_DYN_BLOCKS
      // the next block of the CTA's sequence.  Its tile may be more than one
      // phase ahead of the slot's barrier (the slot's previous tile not yet
      // staged), where a parity wait would pass on the older phase: the warp
      // first waits until the producer has published this iteration in the slot
      // (then the barrier is in this iteration's phase) and then on the barrier
      unsigned int gblk = 0u;
      if (lane == 0) gblk = atomicAdd(&s_next, 1u);
      gblk = __shfl_sync(kFull, gblk, 0);
      it = (int64_t)(gblk / NCW);
      const int wb = (int)(gblk % NCW);
#endif
      const int s = (int)(it % SLOTS);
      const int base = wb * 32 * EPL;
#if STTSV_WAITPROF
      const long long w0 = clock64();
#endif
#if STTSV_DYN_BLOCKS
      while (*(volatile int64_t*)&sit[s] != it) __nanosleep(32);
      mbar_wait_consumer(&full[s], (uint32_t)((it / SLOTS) & 1));
#else
      mbar_wait_consumer(&full[s], (uint32_t)((it / SLOTS) & 1));
#endif
#if STTSV_WAITPROF
      wait_cyc += clock64() - w0;
#endif
      const int64_t t = stile[s];
      if (t < 0) break;
      any = true;
#if STTSV_WAITPROF
      ++ntiles;
#endif
      const int b = sbk[s];
      const int k = p.b[b].k;
#if STTSV_WAITPROF > 1
      const long long kc0 = clock64();
#endif
      const DetSink ds{DET ? p.slot + p.b[b].ids_off + (t - p.b[b].tile_begin) * TILE : nullptr, p.b[b].stride,
                       p.contrib};
      const int us = su[s];                 // staged from column us
      const long long bh = sblk[s][wb];     // this warp's block: shared prefix length and group
      const int tu = (int)(bh & 255);
      const int64_t goff = bh >> 8;
      {
        const unsigned char* st = ring + soff[s];
        using IdT = typename std::conditional<Cfg::IDB == 2, uint16_t, int32_t>::type;
        // the warp's own id columns (slots tu..k-1) start at stage column tu - us
        const IdT* sids = reinterpret_cast<const IdT*>(st) + (size_t)(tu - us) * TILE;
        const BucketDesc& bdc = p.b[b];
        const int64_t rem = bdc.m - (t - bdc.tile_begin) * TILE;
        const WSrc sw{reinterpret_cast<const double*>(st + (k - us) * TILE * Cfg::IDB), bdc.wc,
                      (int)(rem < TILE ? rem : TILE), bdc.wuni != 0};
        if constexpr (PREFIX || Cfg::BIG_PREFIX) {
          if (tu > 0 && tu == k && !DET) {
            // M = 0: every edge of the warp's block is the same vertex set
            const int nb = Cfg::BIG ? 32 : 32 * EPL;
            const int bb = Cfg::BIG ? wb * 32 : base;
            double part = 0.0;
            if (sw.uni) {
              int n = sw.real - bb;
              n = n < 0 ? 0 : (n > nb ? nb : n);
              part = lane == 0 ? sw.wc * (double)n : 0.0;
            } else {
#pragma unroll
              for (int r = 0; r < (Cfg::BIG ? 1 : EPL); ++r) part += sw.sw[bb + r * 32 + lane];
            }
            const int64_t g = goff;
            if (g != pend_goff) {
              if (pend_goff >= 0) flush_pending();
              pend_goff = g;
              pend_L = p.N - k + 1;
              pend_U = tu;
              pend_w = 0.0;
            }
            pend_w += part;
            __syncwarp();
#if STTSV_WAITPROF == 3
            if (lane == 0) {
              atomicAdd(&s_kc[0], (unsigned long long)(clock64() - kc0));
              atomicAdd(&s_kc[1], 1ull);
            }
#endif
            if (lane == 0) mbar_arrive(&empty[s]);
            continue;
          }
        }
        // one pass per vector; with several vectors the runs of a pass are flushed
        // (warp-aggregated) at its end, with one they continue across tiles
        int qn = 0;  // batch: the block's run-queue length (built by the first vector's pass)
        for (int v = 0; v < nvec; ++v) {
          const Sink skv{priv_cta + (size_t)v * p.H, p.ya + (size_t)v * p.ya_vstride, p.H};
          const double* xgv = p.xg + (size_t)v * p.xg_vstride;
          // shared-prefix tiles (prefix.cuh): the DP over the own members, the
          // prefix members' totals from the vector's group table
          const double* Gv = p.gtab + (size_t)v * p.gtab_vstride + goff;
          bool done = false;
          if constexpr (!Cfg::BIG) {
            if constexpr (PREFIX) {
              if (tu > 0) {
                need_groups();
                dispatch_kp<N, 1, Cfg::PMAX, TILE, EPL, RMAX, IdT, BATCH>(k, tu, sids, sw, base, xgv, Gv, ra, skv,
                                                                          sred, lane, v, qn);
                done = true;
              }
            }
            if (!done) dispatch_k<N, 1, TILE, EPL, RMAX, DET, IdT>(k, sids, sw, base, xgv, ra, skv, ds, lane);
          } else {
            const int col = wb * 32 + lane;  // EPL = 1
            if constexpr (Cfg::BIG_PREFIX && !DET) {
              if (tu > 0) {  // shared-prefix tile (prefix.cuh); warp-uniform
                need_groups();
#if STTSV_BIG_LOCAL
                dispatch_big_prefix<1, KMAX, TILE, 1, RMAX>(p.N - k + 1, k, tu, sids + col, sw.at(col, col), sw,
                                                            wb * 32, Gv, xgv, p.gs, lstk, ra, skv, sred, lane);
#else
                dispatch_big_prefix<1, KMAX, TILE, NCW * 32, RMAX>(p.N - k + 1, k, tu, sids + col, sw.at(col, col),
                                                                   sw, wb * 32, Gv, xgv, p.gs,
                                                                   stack + (warp * 32 + lane), ra, skv, sred, lane);
#endif
                done = true;
              }
            }
            if (!done) {
#if STTSV_BIG_LOCAL
              dispatch_big<1, KMAX, TILE, 1, RMAX, DET>(p.N - k + 1, k, sids + col, sw.at(col, col), xgv, p.gs, lstk,
                                                        ra, skv, ds, col);
#else
              dispatch_big<1, KMAX, TILE, NCW * 32, RMAX, DET>(p.N - k + 1, k, sids + col, sw.at(col, col), xgv,
                                                               p.gs, stack + (warp * 32 + lane), ra, skv, ds, col);
#endif
            }
          }
          if constexpr (BATCH) {
#pragma unroll
            for (int i = 0; i < RMAX; ++i) {
              warp_flush(ra.rid[i], ra.run[i], lane, skv);
              ra.rid[i] = -1;
              ra.run[i] = 0.0;
            }
          }
        }
      }
      __syncwarp();
#if STTSV_WAITPROF > 1
      if (lane == 0) {
        const int cls = STTSV_WAITPROF == 3 ? (tu == 0 ? 20 + (k < 12 ? k : 12) : k - tu) : k;
        atomicAdd(&s_kc[2 * cls], (unsigned long long)(clock64() - kc0));
        atomicAdd(&s_kc[2 * cls + 1], 1ull);
      }
#endif
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#if STTSV_WAITPROF
    if (lane == 0) {
      atomicAdd(&g_wait_cycles[0], (unsigned long long)wait_cyc);
      atomicAdd(&g_wait_cycles[1], (unsigned long long)(clock64() - c_start));
      atomicAdd(&g_wait_cycles[2], 1ull);
      if (warp == 0 && blockIdx.x < 1024) g_cta_ns[3 * blockIdx.x + 2] = ntiles;
    }
#endif
    if (pend_goff >= 0) flush_pending();
    // flush the run accumulators (single-vector mode)
    if (any && !BATCH) {
#pragma unroll
      for (int i = 0; i < RMAX; ++i)
        if (ra.rid[i] >= 0 && ra.run[i] != 0.0) red_add(sk.at(ra.rid[i]), ra.run[i]);
    }
  }
  // this CTA's reds into priv are ordered before the reads below (fence + barrier);
  // the reads go to L2 (ld.cg), where the reds were performed
  if (warp == NCW) griddep_wait();  // the producer warp also adds into y_a below
  __threadfence();
  __syncthreads();
  for (int j = tid; j < p.H * nvec; j += Cfg::THREADS) {
    const double v = __ldcg(priv_cta + j);
    if (v != 0.0) red_add(p.ya + (size_t)(j / p.H) * p.ya_vstride + j % p.H, v);
  }
#if STTSV_WAITPROF
  if (tid == 0 && blockIdx.x < 1024) g_cta_ns[3 * blockIdx.x + 1] = gtimer();
#endif
#if STTSV_WAITPROF > 1
  for (int j = tid; j < 2 * (STTSV_MAX_RANK + 1); j += Cfg::THREADS)
    if (s_kc[j]) atomicAdd(&g_k_cycles[j], s_kc[j]);
#endif
  // the last CTA to finish resets the scheduler counters for the next launch
  // (every producer has stopped taking tiles once all CTAs have counted in)
  if (tid == 0) {
    const unsigned long long done = atomicAdd(p.tile_counter + 1, 1ull);
    if (done == gridDim.x - 1) {
      p.tile_counter[0] = 0ull;
      p.tile_counter[1] = 0ull;
    }
  }
}

}  // namespace sttsv
