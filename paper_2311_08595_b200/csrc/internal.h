// internal.h — structures shared by the host planner (plan.cpp) and the CUDA
// kernels (kernels.cu).  Not part of the public ABI (include/sttsv.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sttsv.h"

namespace sttsv {

// One cardinality bucket of the device hyperedge store:
// edges of size k, SoA: ids[i * stride + e] is member i (relabelled id, members
// ascending) of edge e; w[e] = w(e) (N-1)!/|beta(k)| (Alg. 2 factor).
struct BucketDesc {
  int32_t k;
  int32_t wuni;        // 1: every stored edge has the same w' = wc (no weight column is streamed)
  int64_t m;           // edges in this bucket (this shard)
  int64_t stride;      // column stride of ids: m padded to whole tiles (weight-0 copies of the last edge)
  int64_t tile_begin;  // first tile of this bucket in the kernel's tile order
  int64_t ids_off;     // element offset of column 0 in the ids pool
  int64_t w_off;       // element offset in the weight pool
  double wc;           // the common w' of a uniform-weight bucket
};

constexpr int kMaxBuckets = 2 * STTSV_MAX_RANK;  // per size k: the input edges and (plan.cpp) the M = 0 runs' representatives

// Row stride (doubles) of the per-apply series table x_g (dp.cuh): coefficients
// j = 0..N-2 are used (L - 1 <= N - 2 for k >= 2; the singleton needs j = N - 2),
// padded to a multiple of 4 so rows are 32-byte aligned (256-bit loads).
__host__ __device__ constexpr int series_stride(int N) { return N < 2 ? 4 : ((N - 1 + 3) & ~3); }

struct EdgeKernelParams {
  int32_t N;             // rank
  int32_t nb;            // number of non-empty buckets, in tile order
  BucketDesc b[kMaxBuckets];
  const int32_t* ids;    // ids pool
  const double* w;       // weight pool
  const double* xa;      // x on active vertices (relabelled)
  const double* xg;      // series table: row i = g[j] = x_a[i]^{j+1}/(j+1)!, j < gs (dp.cuh)
  int32_t gs;            // row stride of xg (doubles, even)
  double* ya;            // y on active vertices (accumulated)
  double* priv;          // [grid][nvec][H] per-CTA accumulators of the hot ids (zeroed by the kernel)
  int32_t nvec;          // vectors per apply (f4 batch; 1 = sttsv_apply)
  int64_t xg_vstride;    // doubles between the series tables of consecutive vectors
  int64_t ya_vstride;    // doubles between the y_a of consecutive vectors
  const int32_t* slot;   // deterministic mode: slot pool (layout of ids) -> position in contrib
  double* contrib;       // deterministic mode: vertex-major contributions
  int32_t n_active;
  int32_t T;             // slots with a per-lane register run accumulator (informational)
  int32_t H;             // ids < H accumulate in the CTA's private slice of priv
  int32_t tile_edges;    // edges per tile
  int64_t num_tiles;
  // [0]: chunk counter of the dynamic tile scheduler, [1]: CTAs finished; both
  // zero at launch (zeroed at plan creation; the last CTA of every launch
  // resets them)
  unsigned long long* tile_counter;
  int64_t chunk;         // tiles per grab
  int64_t guided_from;   // tile index after which grabs are single tiles
  // shared-prefix memo (prefix.cuh; nullptr = off): per tile (goff << 8) | U with
  // U the number of leading members all its edges share (their id columns are
  // not streamed) and goff the offset of its prefix group's record in gtab
  const long long* tile_hdr;
  const double* gtab;    // per-apply group table (prefix.cuh)
  int64_t gtab_vstride;  // doubles between the group tables of consecutive vectors (batch)
  int32_t group_wait;    // 1: the preceding grid is group_kernel (consumers wait for it only before their
                         // first group-table read; x_a / the series table come from an earlier, completed grid)
};

// Ranks with a fully unrolled edge kernel (one object file each); every other
// rank <= STTSV_MAX_RANK runs the generic instantiation (N = 0).
#define STTSV_COMPILED_RANKS(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(25)

struct EdgeKernelEntry {
  const void* fn;       // __global__ edge_kernel<N, false> (one vector)
  const void* fn_batch; // __global__ edge_kernel<N, true, false> (sttsv_apply_batch)
  const void* fn_det;   // __global__ edge_kernel<N, false, true> (STTSV_DETERMINISTIC plans)
  int block;           // threads per CTA (consumer warps + one producer warp)
  int tile;            // edges per tile
  size_t ring_bytes;   // shared memory of the TMA ring
  int rank;            // N of the instantiation (0 = generic)
  int run_slots;       // slots with a register run accumulator (EdgeCfg::RMAX)
  int big;             // large-rank path (runtime member loop): 1 prefix stack in shared memory, 2 in local memory
  int consumers;       // consumer threads per CTA
  int table_norm;      // series table rows normalised to a leading 1 (dp.cuh series_row norm = 1)
  int epl;             // consecutive edges per lane per tile (lane l: columns l*epl .. l*epl+epl-1 of its warp block)
  int id_bytes;        // bytes per member id in the edge stream (4, or 2: plans with n_a <= 65536)
  int prefix_mmax;     // shared-prefix memo: tiles with U > 0 are allowed when K - U <= prefix_mmax ...
  int prefix_lmax;     // ... and, for K - U >= 1, when L = N - K + 1 <= prefix_lmax (0 / 0: no memo)
  size_t red_bytes;    // shared memory of the prefix tiles' reduction rows (after the ring)
};
// Ranks that also have a 16-bit-member-id instantiation (unrolled path; used by
// plans with n_a <= 65536).
#define STTSV_ID16_RANKS(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)

#define STTSV_DECLARE_ENTRY(n) EdgeKernelEntry edge_entry_##n();
STTSV_COMPILED_RANKS(STTSV_DECLARE_ENTRY)
#undef STTSV_DECLARE_ENTRY
#define STTSV_DECLARE_ENTRY(n) EdgeKernelEntry edge_entry16_##n();
STTSV_ID16_RANKS(STTSV_DECLARE_ENTRY)
EdgeKernelEntry edge_entry_0();
#undef STTSV_DECLARE_ENTRY

// launchers (kernels.cu)
// id16: prefer the 16-bit-id instantiation (falls back to 32-bit ids where none exists)
EdgeKernelEntry edge_entry(int N, bool id16 = false);
// dynamic shared memory of the edge kernel for rank N (TMA ring + large-rank prefix stacks)
size_t edge_kernel_smem_bytes(const EdgeKernelEntry& e, int N);
// doubles of prefix stack per consumer thread of the large-rank path (edge_kernel.cuh)
int edge_big_stack_doubles(int N);
cudaError_t edge_kernel_config(const EdgeKernelEntry& e, size_t smem, int* max_blocks_per_sm);
// mode: 0 one vector, 1 batch, 2 deterministic; pdl: programmatic dependent
// launch (only directly behind launch_prologue on the same stream)
cudaError_t launch_edge_kernel(const EdgeKernelEntry& e, const EdgeKernelParams& p, int grid, size_t smem,
                               cudaStream_t s, int mode = 0, bool pdl = false);
// deterministic mode, pass 2: chunk sums (chunk c = contrib[cstart[c] .. cstart[c+1])) in a fixed
// tree order, then y_a[v] = sum of v's chunks (vchunk[v] .. vchunk[v+1]) in order
cudaError_t launch_det_reduce(const double* contrib, const int64_t* cstart, int64_t nchunks, double* csum,
                              const int64_t* vchunk, double* ya, int64_t n_active, cudaStream_t s);
constexpr int kDetChunk = 4096;  // contributions per deterministic reduction chunk
// norm: series table format (dp.cuh series_row; EdgeKernelEntry::table_norm)
cudaError_t launch_gather(const double* x, const int32_t* act, double* xa, double* xg, int gs, int norm,
                          int64_t n_active, cudaStream_t s);
cudaError_t launch_prologue(const double* x, const int32_t* act, double* xa, double* xg, int gs, int norm,
                            int64_t n_active, double* ya, cudaStream_t s);
cudaError_t launch_series(const double* xa, double* xg, int gs, int norm, int64_t n_active, cudaStream_t s);
// shared-prefix group table (prefix.cuh): A and the rows C_i of every group from
// the series table; gku[g] = k | U << 8
// items[t] = (group << 8) | i, one per prefix member of every group; gtab_in: the
// plan's table (its prefix ids); gtab_out receives A, C (and the ids when it is a
// batch vector's copy)
cudaError_t launch_groups(const double* xg, int gs, int N, const int32_t* gku, const int64_t* goff,
                          const long long* items, int64_t nitems, int lmax, const double* gtab_in,
                          double* gtab_out, cudaStream_t s);
// M = 0 runs (plan.cpp): each representative's weight = the sum of its run's stored
// weights w0, one warp job per (x, y) pair of job[] (kernels.cu m0sum_kernel): whole
// runs, chunks of split runs (rc0 / wpos per split run, part / cnt: per-job partial sums
// and per-run counters, zero at rest) and packs of short runs (pentry).
cudaError_t launch_m0sum(const double* w0, const long long* job, int64_t njobs, const long long* pentry,
                         const int64_t* rc0, const int64_t* wpos, double* part, unsigned int* cnt, double* w,
                         cudaStream_t s);
cudaError_t launch_expand(const double* ya, const int32_t* act, double* y, int64_t n_active, cudaStream_t s);
constexpr int kNormalizeScratch = 296;  // blocks of the reduction kernels (scratch: 2x doubles + 2)
cudaError_t launch_normalize(const double* z, double* x, double* xg, int gs, int norm, double* partial,
                             int64_t n_active, int N, cudaStream_t s);
cudaError_t launch_lambda(const double* z, const double* x, double* partial, double* out, int64_t n_active, int N,
                          cudaStream_t s);

}  // namespace sttsv
