// Microbenchmarks that fix the B200 roofline denominators this repo needs but
// MEASURED_PEAKS.json does not carry: FP64 FMA throughput (the a3 DP is FP64
// ALU work), shared-memory and global fp64 atomics (the a5 scatter), and the
// clocks seen meanwhile.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void smem_atomic_kernel(double* out, int iters, int spread) {
  __shared__ double acc[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  int slot = spread ? (threadIdx.x & 1023) : 0;
  for (int it = 0; it < iters; ++it) atomicAdd(&acc[slot], 1.0);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acc[0];
}

__global__ void smem_rmw_kernel(double* out, int iters) {
  // private-column read-modify-write (no atomics): acc[t][tid]
  __shared__ double acc[8][256];
  for (int t = 0; t < 8; ++t) acc[t][threadIdx.x] = 0;
  for (int it = 0; it < iters; ++it) {
    int t = (it * 7 + threadIdx.x) & 7;
    acc[t][threadIdx.x] += 1.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = acc[0][0];
}

__global__ void gmem_red_kernel(double* tgt, int iters, int spread_mask) {
  int slot = (blockIdx.x * blockDim.x + threadIdx.x) & spread_mask;
  for (int it = 0; it < iters; ++it) atomicAdd(&tgt[slot], 1.0);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms %d l2 %d smem/blk optin %zu clock(kHz) %d\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);
  double* d; CK(cudaMalloc(&d, 1 << 26)); CK(cudaMemset(d, 0, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DFMA
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 8, threads = 256, iters = 20000;
    dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e0));
    dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * blocks * threads * (double)iters * 8;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)  => %.1f DFMA/clk/SM at %d MHz nominal\n", fl / ms / 1e9, ms,
           fl / 2 / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  // smem atomics
  for (int spread = 0; spread < 2; ++spread) {
    int blocks = sms * 4, threads = 256, iters = 2000;
    smem_atomic_kernel<<<blocks, threads>>>(d, iters, spread);
    CK(cudaEventRecord(e0));
    smem_atomic_kernel<<<blocks, threads>>>(d, iters, spread);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters;
    printf("smem fp64 atomicAdd spread=%d: %.3f Gops/s => %.2f lane-ops/clk/SM\n", spread, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (p.clockRate * 1e3));
  }
  {
    int blocks = sms * 4, threads = 256, iters = 2000;
    smem_rmw_kernel<<<blocks, threads>>>(d, iters);
    CK(cudaEventRecord(e0));
    smem_rmw_kernel<<<blocks, threads>>>(d, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters;
    printf("smem private RMW fp64: %.3f Gops/s => %.2f lane-ops/clk/SM\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / (p.clockRate * 1e3));
  }
  int masks[4] = {0, 31, 4095, (1 << 22) - 1};
  for (int mi = 0; mi < 4; ++mi) {
    int blocks = sms * 8, threads = 256, iters = mi == 0 ? 20 : 200;
    gmem_red_kernel<<<blocks, threads>>>(d, iters, masks[mi]);
    CK(cudaEventRecord(e0));
    gmem_red_kernel<<<blocks, threads>>>(d, iters, masks[mi]);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters;
    printf("gmem fp64 red addrs=%d: %.3f Gops/s\n", masks[mi] + 1, ops / ms / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
