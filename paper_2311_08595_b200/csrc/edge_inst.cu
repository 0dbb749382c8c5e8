// edge_inst.cu — one instantiation of edge_kernel<N> per object file (compiled
// once per rank in STTSV_COMPILED_RANKS with -DSTTSV_INST_N=<N>, and once with
// N = 0 for the generic kernel), so the build parallelises over ranks.
#include "edge_kernel.cuh"

#ifndef STTSV_INST_N
#error "compile with -DSTTSV_INST_N=<rank>"
#endif

#define STTSV_CAT2(a, b) a##b
#define STTSV_CAT(a, b) STTSV_CAT2(a, b)

// -DSTTSV_INST_ID16=1: the 16-bit-id instantiation (edge_entry16_<N>, STTSV_ID16_RANKS)
#ifndef STTSV_INST_ID16
#define STTSV_INST_ID16 0
#endif

namespace sttsv {
#if STTSV_INST_ID16
EdgeKernelEntry STTSV_CAT(edge_entry16_, STTSV_INST_N)() {
  constexpr int IDB = 2;
#else
EdgeKernelEntry STTSV_CAT(edge_entry_, STTSV_INST_N)() {
  constexpr int IDB = 4;
#endif
  using C = EdgeCfg<STTSV_INST_N, IDB>;
  EdgeKernelEntry e;
  e.fn = (const void*)edge_kernel<STTSV_INST_N, false, false, IDB>;
  e.fn_batch = (const void*)edge_kernel<STTSV_INST_N, true, false, IDB>;
  e.fn_det = (const void*)edge_kernel<STTSV_INST_N, false, true, IDB>;
  e.block = C::THREADS;
  e.tile = C::TILE;
  e.ring_bytes = (size_t)C::RING_BYTES;
  e.rank = STTSV_INST_N;
  e.run_slots = C::RMAX;
  e.big = C::BIG ? (STTSV_BIG_LOCAL ? 2 : 1) : 0;
  e.consumers = 32 * C::NCW;
  e.epl = C::EPL;
  e.id_bytes = C::IDB;
  e.prefix_mmax = C::PMAX;
  e.prefix_lmax = C::PLMAX;
  e.red_bytes = (size_t)C::RED_BYTES;
  e.table_norm = ((C::BIG && STTSV_BIG_NORM) || (!C::BIG && STTSV_INST_N >= STTSV_NORM_MIN && STTSV_MID_NORM)) ? 1 : 0;
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
extern "C" int sttsv_debug_cta(unsigned long long out[3 * 1024], int reset) {
  cudaMemcpyFromSymbol(out, sttsv::g_cta_ns, sizeof(unsigned long long) * 3 * 1024);
  if (reset) {
    static unsigned long long z[3 * 1024] = {0};
    cudaMemcpyToSymbol(sttsv::g_cta_ns, z, sizeof(z));
  }
  return 0;
}
#endif
