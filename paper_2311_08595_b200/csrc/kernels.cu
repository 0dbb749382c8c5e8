// kernels.cu — the small kernels of one STTSV apply and the edge-kernel
// registry (the hot rows a3-a5 live in
// edge_kernel.cuh, instantiated per rank by edge_inst.cu).
//
//   a2 gather      x_a[i] = x[act[i]], series table row i        gather_kernel
//   a7 expand      y[act[i]] = y_a[i]                        expand_kernel
//   a8 power step  x_a = z_a^[1/(N-1)] / ||.||_1              normalize_{partial,apply}_kernel
//      (Alg. 1 line 6)
#include <cuda_runtime.h>
#include <stdint.h>

#include "dp.cuh"
#include "edge_kernel.cuh"
#include "internal.h"

namespace sttsv {

// ------------------------------------------------------- small kernels
// x_a[i] = x[act[i]] and the series row g_i[j] = x_a[i]^{j+1}/(j+1)! (dp.cuh)
__global__ void gather_kernel(const double* __restrict__ x, const int32_t* __restrict__ act,
                              double* __restrict__ xa, double* __restrict__ xg, int gs, int norm, int64_t n_active) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_active;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[act[i]];
    xa[i] = v;
    series_row(v, xg + i * gs, gs, norm);
  }
}

// gather + series table + y_a = 0 in one launch (sttsv_apply; sttsv_apply_host
// passes act = nullptr with x = the host-gathered x_a).  The edge kernel that
// follows is a programmatic dependent launch: it may start (barrier setup,
// private-slice zeroing, the first TMA stages of the edge stream) as soon as
// every CTA here has started; its consumers wait (griddepcontrol.wait) for this
// grid's completion before reading x_a / the series table / y_a.
__global__ void prologue_kernel(const double* x, const int32_t* __restrict__ act,
                                double* xa, double* __restrict__ xg, int gs, int norm, int64_t n_active,
                                double* __restrict__ ya) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_active;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = act ? x[act[i]] : x[i];  // act == nullptr: x is already x_a
    xa[i] = v;
    series_row(v, xg + i * gs, gs, norm);
    ya[i] = 0.0;
  }
}

// series table rows from x_a (sttsv_apply_host's host-gathered path)
__global__ void series_kernel(const double* __restrict__ xa, double* __restrict__ xg, int gs, int norm,
                              int64_t n_active) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_active;
       i += (int64_t)gridDim.x * blockDim.x)
    series_row(xa[i], xg + i * gs, gs, norm);
}

// Shared-prefix group table (prefix.cuh), one thread per (group, prefix member i):
// from the normalised series rows of the group's U prefix members it forms, in
// one pass over the rows, A_{\i} and A = prod g_j (compile-time L: register
// arrays) and writes C_i[j] = A_{\i}[D-j] + A[D-1-j] (unnormalised coefficients;
// the second term for j <= D-1); the i = 0 thread also writes the front A (row
// format) and, for a batch vector's copy of the table, the prefix ids.  The edge
// kernel that follows is a programmatic dependent launch (its consumers wait for
// this grid before reading the table).
template <int L>
__device__ __forceinline__ void group_item(const double* __restrict__ xg, int gs, const long long* ids, int U, int i,
                                           double* T, long long* ids_out) {
  constexpr int D = L - 1;
  double ah[L], ai[L];
  double X = 1.0, Xi = 1.0;
  ah[0] = ai[0] = 1.0;
#pragma unroll
  for (int j = 1; j < L; ++j) ah[j] = ai[j] = 0.0;
#pragma unroll 1
  for (int m = 0; m < U; ++m) {
    double h[L];
    load_series<L>(xg + (size_t)ids[m] * gs, h);
    const bool in = m != i;
#pragma unroll
    for (int j = L - 1; j >= 1; --j) {  // truncated products with implicit leading 1 (descending: in place)
      double s = ah[j] + h[j], si = ai[j] + h[j];
#pragma unroll
      for (int q = 1; q < j; ++q) {
        s = fma(ah[q], h[j - q], s);
        si = fma(ai[q], h[j - q], si);
      }
      ah[j] = s;
      ai[j] = in ? si : ai[j];
    }
    X *= h[0];
    Xi = in ? Xi * h[0] : Xi;
  }
  if (i == 0) {
    T[0] = X;
#pragma unroll
    for (int j = 1; j < L; ++j) T[j] = ah[j];
    if (ids_out)
      for (int m = 0; m < U; ++m) ids_out[m] = ids[m];
  }
  double* C = T + L + i * L;
#pragma unroll
  for (int j = 0; j <= D; ++j) C[j] = Xi * ai[D - j] + (j <= D - 1 ? X * ah[D - 1 - j] : 0.0);
}

template <int L, int LMAX>
__device__ __forceinline__ void group_item_dispatch(int L_rt, const double* xg, int gs, const long long* ids, int U,
                                                    int i, double* T, long long* ids_out) {
  if constexpr (L <= LMAX) {
    if (L_rt == L) {
      group_item<L>(xg, gs, ids, U, i, T, ids_out);
      return;
    }
    group_item_dispatch<L + 1, LMAX>(L_rt, xg, gs, ids, U, i, T, ids_out);
  }
}

template <int LMIN, int LMAX>
__global__ void __launch_bounds__(128) group_kernel(const double* __restrict__ xg, int gs, int N,
                                                    const int32_t* __restrict__ gku, const int64_t* __restrict__ goff,
                                                    const long long* __restrict__ items, int64_t nitems,
                                                    const double* gtab_in, double* gtab) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nitems;
       t += (int64_t)gridDim.x * blockDim.x) {
    const long long it = items[t];
    const int64_t g = it >> 8;
    const int i = (int)(it & 255);
    const int k = gku[g] & 255, U = gku[g] >> 8, L = N - k + 1;
    const long long* ids = reinterpret_cast<const long long*>(gtab_in + goff[g] + L + U * L);
    double* T = gtab + goff[g];
    long long* ids_out = gtab_in != gtab ? reinterpret_cast<long long*>(T + L + U * L) : nullptr;
    group_item_dispatch<LMIN, LMAX>(L, xg, gs, ids, U, i, T, ids_out);
  }
}

// Weights of the M = 0 runs' representative edges (plan.cpp): representative r
// stands for a run of one repeated vertex set and takes w' summed over the run's
// stored weights w0[...] (read every apply).  One warp per job; a job is one
// 16-byte record, so its loads of w0 issue right after it (no dependent metadata):
//   x = (a << 24) | n, y >= 0      a whole run w0[a .. a+n) (n <= 2048): w[y] = its sum
//   x = (a << 24) | n, y < 0       a chunk of split run r = -1 - y: the run's chunks (jobs
//                                  rc0[2r] .. rc0[2r+1]) store partial sums; the last to
//                                  finish (a per-run counter, reset by it) adds them, the
//                                  whole warp in a fixed order, into w[wpos[r]]
//   x = 2^62 | (a << 24) | n       a pack of neighbouring short runs in w0[a .. a+n)
//                                  (n <= 256), y = (first entry << 9) | runs; entry
//                                  (wpos << 18) | (offset << 9) | length per run
// The loads of a whole run / chunk keep 8 independent loads in flight per lane.
constexpr int kM0Block = 256, kM0Pack = 256;
__global__ void __launch_bounds__(kM0Block) m0sum_kernel(const double* __restrict__ w0,
                                                         const longlong2* __restrict__ job, int64_t njobs,
                                                         const long long* __restrict__ pentry,
                                                         const int64_t* __restrict__ rc0,
                                                         const int64_t* __restrict__ wpos, double* __restrict__ part,
                                                         unsigned int* __restrict__ cnt, double* __restrict__ w) {
  __shared__ double sbuf[kM0Block / 32][kM0Pack];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < njobs; c += nwarps) {
    const longlong2 jb = job[c];
    const long long x = jb.x, y = jb.y;
    const double* p = w0 + ((x >> 24) & ((1ll << 38) - 1));
    const int len = (int)(x & 0xffffff);
    if (!((x >> 62) & 1)) {
      double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int j = lane;
      for (; j + 7 * 32 < len; j += 8 * 32) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] += __ldcs(p + j + q * 32);
      }
      for (; j < len; j += 32) s[0] += __ldcs(p + j);
      double r = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      if (y >= 0) {
        if (lane == 0) w[y] = r;
        continue;
      }
      const int64_t run = -1 - y;
      unsigned last = 0u;
      if (lane == 0) {
        part[c] = r;
        __threadfence();
        last = atomicAdd(cnt + run, 1u) == (unsigned)(rc0[2 * run + 1] - rc0[2 * run] - 1) ? 1u : 0u;
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        __threadfence();
        const int64_t a = rc0[2 * run], b = rc0[2 * run + 1];
        double t0 = 0.0, t1 = 0.0;
        int64_t q = a + lane;
        for (; q + 32 < b; q += 64) {
          t0 += __ldcg(part + q);
          t1 += __ldcg(part + q + 32);
        }
        if (q < b) t0 += __ldcg(part + q);
        double tot = t0 + t1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (lane == 0) {
          w[wpos[run]] = tot;
          cnt[run] = 0u;
        }
      }
    } else {
      const int64_t e0 = y >> 9;
      const int nr = (int)(y & 511);
      const long long ent = lane < nr ? pentry[e0 + lane] : 0ll;  // runs beyond 32: loaded below
      double* sb = sbuf[wib];
#pragma unroll
      for (int j = 0; j < kM0Pack / 32; ++j)
        if (lane + 32 * j < len) sb[lane + 32 * j] = __ldcs(p + lane + 32 * j);
      __syncwarp();
      for (int i = 0; i < nr; ++i) {  // warp-wide sum of each run
        const long long e = i < 32 ? __shfl_sync(0xffffffffu, ent, i) : pentry[e0 + i];
        const int off = (int)((e >> 9) & 511), n = (int)(e & 511);
        double r = 0.0;
        for (int j = lane; j < n; j += 32) r += sb[off + j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (lane == 0) w[e >> 18] = r;
      }
      __syncwarp();
    }
  }
}

__global__ void expand_kernel(const double* __restrict__ ya, const int32_t* __restrict__ act,
                              double* __restrict__ y, int64_t n_active) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_active;
       i += (int64_t)gridDim.x * blockDim.x)
    y[act[i]] = ya[i];
}


constexpr int kNormBlock = 1024;
constexpr int kNormMaxGrid = kNormalizeScratch;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (warp == 0) {
    s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// r_i = z_i^{1/(N-1)} into x, per-block partial sums of r into partial[blockIdx]
__global__ void __launch_bounds__(kNormBlock) normalize_partial_kernel(const double* __restrict__ z,
                                                                      double* __restrict__ x,
                                                                      double* __restrict__ partial,
                                                                      int64_t n, double inv_root) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = pow(z[i], inv_root);
    x[i] = r;
    s += r;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// every block sums all partials in the same order, then scales its slice
__global__ void __launch_bounds__(kNormBlock) normalize_apply_kernel(double* __restrict__ x,
                                                                    double* __restrict__ xg, int gs, int norm,
                                                                    const double* __restrict__ partial,
                                                                    int nparts, int64_t n) {
  __shared__ double tot;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int j = threadIdx.x; j < nparts; j += 32) s += partial[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) tot = s;
  }
  __syncthreads();
  const double t = tot;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i] / t;
    x[i] = v;
    series_row(v, xg + i * gs, gs, norm);
  }
}

// Alg. 1 lines 8-9: lambda_min/max of z ./ x^[N-1] over the
// vertices with x^[N-1] > 0 (reading A15: isolated vertices, x = 0, and
// underflowed powers are excluded).  Per-block partials,
// then one block combines them.
__global__ void __launch_bounds__(kNormBlock) lambda_partial_kernel(const double* __restrict__ z,
                                                                   const double* __restrict__ x,
                                                                   double* __restrict__ partial, int64_t n,
                                                                   int Nm1) {
  __shared__ double smin[32], smax[32];
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xv = x[i];
    double p = 1.0;
    for (int j = 0; j < Nm1; ++j) p *= xv;
    if (p > 0.0) {  // x_v^[N-1] > 0: x_v > 0 and no underflow (reading A15)
      const double r = z[i] / p;
      lo = fmin(lo, r);
      hi = fmax(hi, r);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smin[warp] = lo;
    smax[warp] = hi;
  }
  __syncthreads();
  if (warp == 0) {
    lo = lane < (int)(blockDim.x >> 5) ? smin[lane] : INFINITY;
    hi = lane < (int)(blockDim.x >> 5) ? smax[lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      partial[2 * blockIdx.x] = lo;
      partial[2 * blockIdx.x + 1] = hi;
    }
  }
}

__global__ void lambda_final_kernel(const double* __restrict__ partial, int nparts, double* __restrict__ out) {
  double lo = INFINITY, hi = -INFINITY;
  for (int j = threadIdx.x; j < nparts; j += 32) {
    lo = fmin(lo, partial[2 * j]);
    hi = fmax(hi, partial[2 * j + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (threadIdx.x == 0) {
    out[0] = lo;
    out[1] = hi;
  }
}

// Deterministic reduction (STTSV_DETERMINISTIC).  Each chunk (<= kDetChunk
// consecutive contributions of ONE vertex) is summed by one CTA of 256 threads:
// thread j adds elements j, j+256, ... in order, then a fixed shuffle/shared
// tree; the result depends only on the data, never on scheduling.
constexpr int kDetBlock = 256;
__global__ void __launch_bounds__(kDetBlock) det_chunk_kernel(const double* __restrict__ contrib,
                                                              const int64_t* __restrict__ cstart,
                                                              double* __restrict__ csum) {
  __shared__ double red[kDetBlock / 32];
  const int64_t c = blockIdx.x;
  const int64_t a = cstart[c], b = cstart[c + 1];
  double s = 0.0;
  for (int64_t i = a + threadIdx.x; i < b; i += kDetBlock) s += contrib[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kDetBlock / 32; ++w) t += red[w];
    csum[c] = t;
  }
}

// one CTA per vertex: thread j sums chunks j, j+256, ... in order, then the same
// fixed tree as det_chunk_kernel (a hot vertex has ~1e4 chunks)
__global__ void __launch_bounds__(kDetBlock) det_vertex_kernel(const double* __restrict__ csum,
                                                               const int64_t* __restrict__ vchunk,
                                                               double* __restrict__ ya) {
  __shared__ double red[kDetBlock / 32];
  const int64_t v = blockIdx.x;
  const int64_t a = vchunk[v], b = vchunk[v + 1];
  double s = 0.0;
  for (int64_t c = a + threadIdx.x; c < b; c += kDetBlock) s += csum[c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kDetBlock / 32; ++w) t += red[w];
    ya[v] = t;
  }
}

// ------------------------------------------------------------- launchers
EdgeKernelEntry edge_entry(int N, bool id16) {
  if (id16) {
    switch (N) {
#define STTSV_CASE(n) \
  case n:             \
    return edge_entry16_##n();
      STTSV_ID16_RANKS(STTSV_CASE)
#undef STTSV_CASE
      default:
        break;
    }
  }
  switch (N) {
#define STTSV_CASE(n) \
  case n:             \
    return edge_entry_##n();
    STTSV_COMPILED_RANKS(STTSV_CASE)
#undef STTSV_CASE
    default:
      return edge_entry_0();
  }
}

int edge_big_stack_doubles(int N) { return big_stack_doubles(N); }

size_t edge_kernel_smem_bytes(const EdgeKernelEntry& e, int N) {
  return e.ring_bytes + e.red_bytes + (e.big == 1 ? (size_t)e.consumers * big_stack_doubles(N) * sizeof(double) : 0);
}

cudaError_t edge_kernel_config(const EdgeKernelEntry& e, size_t smem, int* max_blocks_per_sm) {
  cudaError_t err = cudaFuncSetAttribute(e.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(e.fn_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(e.fn_det, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(max_blocks_per_sm, e.fn, e.block, smem);
}

cudaError_t launch_edge_kernel(const EdgeKernelEntry& e, const EdgeKernelParams& p, int grid, size_t smem,
                               cudaStream_t s, int mode, bool pdl) {
  void* args[] = {const_cast<EdgeKernelParams*>(&p)};
  const void* fn = mode == 1 ? e.fn_batch : (mode == 2 ? e.fn_det : e.fn);
  if (!pdl) return cudaLaunchKernel(fn, dim3(grid), dim3(e.block), args, smem, s);
  // programmatic dependent launch behind the prologue kernel
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(e.block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

static int grid_for(int64_t n, int block, int cap) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

cudaError_t launch_gather(const double* x, const int32_t* act, double* xa, double* xg, int gs, int norm,
                          int64_t n_active, cudaStream_t s) {
  if (n_active <= 0) return cudaSuccess;
  gather_kernel<<<grid_for(n_active, 256, 4096), 256, 0, s>>>(x, act, xa, xg, gs, norm, n_active);
  return cudaGetLastError();
}

cudaError_t launch_prologue(const double* x, const int32_t* act, double* xa, double* xg, int gs, int norm,
                            int64_t n_active, double* ya, cudaStream_t s) {
  prologue_kernel<<<grid_for(n_active, 256, 4096), 256, 0, s>>>(x, act, xa, xg, gs, norm, n_active, ya);
  return cudaGetLastError();
}

cudaError_t launch_series(const double* xa, double* xg, int gs, int norm, int64_t n_active, cudaStream_t s) {
  if (n_active <= 0) return cudaSuccess;
  series_kernel<<<grid_for(n_active, 256, 4096), 256, 0, s>>>(xa, xg, gs, norm, n_active);
  return cudaGetLastError();
}

cudaError_t launch_groups(const double* xg, int gs, int N, const int32_t* gku, const int64_t* goff,
                          const long long* items, int64_t nitems, int lmax, const double* gtab_in,
                          double* gtab_out, cudaStream_t s) {
  // one launch, instantiated up to the plan's largest L (a kernel's register count is
  // the maximum over the L it instantiates: 72 / 134 / 254 for L <= 8 / 16 / 32)
  if (nitems <= 0) return cudaSuccess;
  const int g = grid_for(nitems, 128, 8192);
  if (lmax <= 8)
    group_kernel<1, 8><<<g, 128, 0, s>>>(xg, gs, N, gku, goff, items, nitems, gtab_in, gtab_out);
  else if (lmax <= 16)
    group_kernel<1, 16><<<g, 128, 0, s>>>(xg, gs, N, gku, goff, items, nitems, gtab_in, gtab_out);
  else
    group_kernel<1, STTSV_MAX_RANK><<<g, 128, 0, s>>>(xg, gs, N, gku, goff, items, nitems, gtab_in, gtab_out);
  return cudaGetLastError();
}

cudaError_t launch_m0sum(const double* w0, const long long* job, int64_t njobs, const long long* pentry,
                         const int64_t* rc0, const int64_t* wpos, double* part, unsigned int* cnt, double* w,
                         cudaStream_t s) {
  if (njobs <= 0) return cudaSuccess;
  m0sum_kernel<<<grid_for(32 * njobs, kM0Block, 148 * 8), kM0Block, 0, s>>>(
      w0, reinterpret_cast<const longlong2*>(job), njobs, pentry, rc0, wpos, part, cnt, w);
  return cudaGetLastError();
}

cudaError_t launch_expand(const double* ya, const int32_t* act, double* y, int64_t n_active, cudaStream_t s) {
  if (n_active <= 0) return cudaSuccess;
  expand_kernel<<<grid_for(n_active, 256, 4096), 256, 0, s>>>(ya, act, y, n_active);
  return cudaGetLastError();
}

// out[0..1] = (lambda_min, lambda_max); `partial` holds 2 * kNormalizeScratch doubles
cudaError_t launch_lambda(const double* z, const double* x, double* partial, double* out, int64_t n_active, int N,
                          cudaStream_t s) {
  const int grid = grid_for(n_active, kNormBlock, kNormMaxGrid);
  lambda_partial_kernel<<<grid, kNormBlock, 0, s>>>(z, x, partial, n_active, N - 1);
  lambda_final_kernel<<<1, 32, 0, s>>>(partial, grid, out);
  return cudaGetLastError();
}

cudaError_t launch_det_reduce(const double* contrib, const int64_t* cstart, int64_t nchunks, double* csum,
                              const int64_t* vchunk, double* ya, int64_t n_active, cudaStream_t s) {
  if (nchunks > 0) det_chunk_kernel<<<(unsigned)nchunks, kDetBlock, 0, s>>>(contrib, cstart, csum);
  if (n_active > 0) det_vertex_kernel<<<(unsigned)n_active, kDetBlock, 0, s>>>(csum, vchunk, ya);
  return cudaGetLastError();
}


// x and z are n_active long; `partial` holds kNormalizeScratch doubles.
cudaError_t launch_normalize(const double* z, double* x, double* xg, int gs, int norm, double* partial,
                             int64_t n_active, int N, cudaStream_t s) {
  if (n_active <= 0) return cudaSuccess;
  const int grid = grid_for(n_active, kNormBlock, kNormMaxGrid);
  normalize_partial_kernel<<<grid, kNormBlock, 0, s>>>(z, x, partial, n_active, 1.0 / double(N - 1));
  normalize_apply_kernel<<<grid, kNormBlock, 0, s>>>(x, xg, gs, norm, partial, grid, n_active);
  return cudaGetLastError();
}

}  // namespace sttsv
