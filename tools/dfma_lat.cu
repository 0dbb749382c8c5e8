// DFMA dependent-issue latency and per-SMSP throughput vs independent chains
// (one CTA of W warps on one SM).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dfma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  const int iters = 4096;
  chain<CH><<<1, 32 * warps>>>(out, cyc, iters, 0.999, 1e-3);
  chain<CH><<<1, 32 * warps>>>(out, cyc, iters, 0.999, 1e-3);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double per = (double)c / iters;  // cycles per iteration (CH dependent-chain steps)
  printf("chains=%2d warps=%2d: %.2f cyc/iter  -> %.2f cyc per dependent DFMA, %.2f warp-DFMA/cyc/SM\n", CH, warps,
         per, per, (double)CH * warps / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1);
  run<2>(1);
  run<4>(1);
  run<8>(1);
  run<1>(4);
  run<4>(4);
  run<1>(16);
  run<2>(16);
  run<4>(16);
  run<8>(16);
  run<1>(32);
  run<4>(32);
  return 0;
}
