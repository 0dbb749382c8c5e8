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

// Shared-prefix group table (prefix.cuh), one warp per group, lane j holding
// coefficient j of a normalised series (lane 0: the scalar x-product, lanes
// 1..L-1: the coefficients under the implicit leading 1).  From the group's U
// prefix rows it forms the prefix products P_m = g_0..g_m and suffix products
// S_m = g_m..g_{U-1}, then A = P_{U-1}, A_{\i} = P_{i-1} S_{i+1}, and writes the
// front A (row format) and C_i[j] = A_{\i}[D-j] + A[D-1-j] (unnormalised; the
// second term for j <= D-1).  The edge kernel that follows is a programmatic
// dependent launch (its consumers wait for this grid before the first table read).
__device__ __forceinline__ double gmul(double a, double h, int lane, int L) {
  // (a*h) mod t^L of two lane-distributed normalised series; lane 0: scalar product
  double s = lane == 0 ? a * h : a + h;
  for (int q = 1; q < L - 1; ++q) {
    const double aq = __shfl_sync(0xffffffffu, a, q);
    const double hq = __shfl_sync(0xffffffffu, h, (lane - q) & 31);
    if (lane > q && lane < L) s = fma(aq, hq, s);
  }
  return lane < L ? s : 0.0;
}

__global__ void group_kernel(const double* __restrict__ xg, int gs, int N, const int32_t* __restrict__ gku,
                             const int64_t* __restrict__ goff, int64_t ngroups, const double* gtab_in,
                             double* gtab) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < ngroups; g += warps) {
    const int k = gku[g] & 255, U = gku[g] >> 8, L = N - k + 1, D = L - 1;
    const long long* ids = reinterpret_cast<const long long*>(gtab_in + goff[g] + L + U * L);
    double* T = gtab + goff[g];
    double hr[STTSV_MAX_RANK], P[STTSV_MAX_RANK], Sf[STTSV_MAX_RANK];  // per-lane values (local memory)
    for (int m = 0; m < U; ++m) hr[m] = (lane < L && lane < gs) ? __ldg(xg + (size_t)ids[m] * gs + lane) : 0.0;
    double acc = hr[0];
    P[0] = acc;
    for (int m = 1; m < U; ++m) P[m] = acc = gmul(acc, hr[m], lane, L);
    acc = hr[U - 1];
    Sf[U - 1] = acc;
    for (int m = U - 2; m >= 0; --m) Sf[m] = acc = gmul(hr[m], acc, lane, L);
    const double A = P[U - 1];
    const double one = lane == 0 ? 1.0 : 0.0;  // the empty product
    if (lane < L) T[lane] = A;
    const double Xa = __shfl_sync(0xffffffffu, A, 0);
    for (int i = 0; i < U; ++i) {
      const double lo = i > 0 ? P[i - 1] : one, hi = i + 1 < U ? Sf[i + 1] : one;
      const double Ai = gmul(lo, hi, lane, L);
      const double Xi = __shfl_sync(0xffffffffu, Ai, 0);
      // lane j: C_i[j] = X_i ah_i[D-j] + X_A ah[D-1-j]  (ah[0] = 1)
      const double ai = __shfl_sync(0xffffffffu, Ai, (D - lane) & 31);
      const double aa = __shfl_sync(0xffffffffu, A, (D - 1 - lane) & 31);
      if (lane <= D) {
        const double t1 = Xi * (lane == D ? 1.0 : ai);
        const double t2 = lane <= D - 1 ? Xa * (lane == D - 1 ? 1.0 : aa) : 0.0;
        T[L + i * L + lane] = t1 + t2;
      }
    }
    if (gtab_in != gtab && lane < U) reinterpret_cast<long long*>(T + L + U * L)[lane] = ids[lane];
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
                          int64_t ngroups, const double* gtab_in, double* gtab_out, cudaStream_t s) {
  if (ngroups <= 0) return cudaSuccess;
  group_kernel<<<grid_for(ngroups * 32, 128, 8192), 128, 0, s>>>(xg, gs, N, gku, goff, ngroups, gtab_in, gtab_out);
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
