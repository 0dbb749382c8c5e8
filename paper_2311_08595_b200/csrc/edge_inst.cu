// edge_inst.cu — one instantiation of edge_kernel<N> per object file (compiled
// once per rank in STTSV_COMPILED_RANKS with -DSTTSV_INST_N=<N>, and once with
// N = 0 for the generic kernel), so the build parallelises over ranks.
#include "edge_kernel.cuh"

#ifndef STTSV_INST_N
#error "compile with -DSTTSV_INST_N=<rank>"
#endif

#define STTSV_CAT2(a, b) a##b
#define STTSV_CAT(a, b) STTSV_CAT2(a, b)

namespace sttsv {
EdgeKernelEntry STTSV_CAT(edge_entry_, STTSV_INST_N)() {
  EdgeKernelEntry e;
  e.fn = (const void*)edge_kernel<STTSV_INST_N, false, false>;
  e.fn_batch = (const void*)edge_kernel<STTSV_INST_N, true, false>;
  e.fn_det = (const void*)edge_kernel<STTSV_INST_N, false, true>;
  e.block = EdgeCfg<STTSV_INST_N>::THREADS;
  e.tile = EdgeCfg<STTSV_INST_N>::TILE;
  e.ring_bytes = (size_t)EdgeCfg<STTSV_INST_N>::RING_BYTES;
  e.rank = STTSV_INST_N;
  e.run_slots = EdgeCfg<STTSV_INST_N>::RMAX;
  e.big = EdgeCfg<STTSV_INST_N>::BIG ? (STTSV_BIG_LOCAL ? 2 : 1) : 0;
  e.consumers = 32 * EdgeCfg<STTSV_INST_N>::NCW;
  e.epl = EdgeCfg<STTSV_INST_N>::EPL;
  e.table_norm = ((EdgeCfg<STTSV_INST_N>::BIG && STTSV_BIG_NORM) ||
                  (!EdgeCfg<STTSV_INST_N>::BIG && STTSV_INST_N >= STTSV_NORM_MIN && STTSV_MID_NORM)) ? 1 : 0;
  return e;
}
}  // namespace sttsv

#if STTSV_WAITPROF
extern "C" int sttsv_debug_wait(unsigned long long out[4], int reset) {
  cudaMemcpyFromSymbol(out, sttsv::g_wait_cycles, sizeof(unsigned long long) * 4);
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(sttsv::g_wait_cycles, z, sizeof(z));
  }
  return 0;
}
extern "C" int sttsv_debug_kcycles(unsigned long long out[2 * (STTSV_MAX_RANK + 1)], int reset) {
  cudaMemcpyFromSymbol(out, sttsv::g_k_cycles, sizeof(unsigned long long) * 2 * (STTSV_MAX_RANK + 1));
  if (reset) {
    unsigned long long z[2 * (STTSV_MAX_RANK + 1)] = {0};
    cudaMemcpyToSymbol(sttsv::g_k_cycles, z, sizeof(z));
  }
  return 0;
}
#endif
