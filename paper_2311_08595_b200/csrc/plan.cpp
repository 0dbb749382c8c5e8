// plan.cpp — host planner and C ABI of libsttsv.so (include/sttsv.h).
//
// sttsv_plan_create validates the IOU hyperedges,
// computes global degrees, relabels active vertices by descending degree
// (hot vertices get small ids: the kernel's per-CTA hot slices key on them),
// buckets the edges of this shard by cardinality into SoA int32 id columns
// sorted lexicographically and padded to whole tiles, folds the per-size
// constant (N-1)!/|beta(k)| = (N-1)!/(k! S(N,k)) (PAPER.md:342 footnote,
// Alg. 2 factor PAPER.md:391) into the fp64 weights, optionally merges
// duplicate edges or builds the deterministic slot map, and uploads
// everything once.  sttsv_apply is then gather -> edge kernel -> (NCCL
// allreduce) -> expand, all on the caller's stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <omp.h>

#include <parallel/algorithm>

#include <algorithm>
#include <numeric>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

using namespace sttsv;

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

static sttsv_status_t fail(sttsv_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

static sttsv_status_t cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return fail(STTSV_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
  return fail(STTSV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(expr, what)                         \
  do {                                               \
    cudaError_t e_ = (expr);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

extern "C" const char* sttsv_status_string(sttsv_status_t s) {
  switch (s) {
    case STTSV_OK: return "STTSV_OK";
    case STTSV_ERR_INVALID_ARGUMENT: return "STTSV_ERR_INVALID_ARGUMENT";
    case STTSV_ERR_EDGE_SIZE: return "STTSV_ERR_EDGE_SIZE";
    case STTSV_ERR_VERTEX_RANGE: return "STTSV_ERR_VERTEX_RANGE";
    case STTSV_ERR_UNSORTED: return "STTSV_ERR_UNSORTED";
    case STTSV_ERR_REPEATED_VERTEX: return "STTSV_ERR_REPEATED_VERTEX";
    case STTSV_ERR_NONFINITE: return "STTSV_ERR_NONFINITE";
    case STTSV_ERR_ALIAS: return "STTSV_ERR_ALIAS";
    case STTSV_ERR_CUDA: return "STTSV_ERR_CUDA";
    case STTSV_ERR_NCCL: return "STTSV_ERR_NCCL";
    case STTSV_ERR_OUT_OF_MEMORY: return "STTSV_ERR_OUT_OF_MEMORY";
    case STTSV_ERR_UNSUPPORTED: return "STTSV_ERR_UNSUPPORTED";
  }
  return "STTSV_ERR_UNKNOWN";
}

extern "C" const char* sttsv_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* sttsv_version(void) { return "sttsv-b200 0.1 (sm_100a)"; }

// -------------------------------------------------------------------- NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    if (api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString) api.h = h;
  });
  return api.h ? &api : nullptr;
}

struct sttsv_comm_s {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
};

extern "C" sttsv_status_t sttsv_comm_unique_id(unsigned char id[128]) {
  if (!id) return fail(STTSV_ERR_INVALID_ARGUMENT, "id is NULL");
  NcclApi* api = nccl_api();
  if (!api) return fail(STTSV_ERR_NCCL, "could not load libnccl.so.2");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId uid;
  ncclResult_t r = api->GetUniqueId(&uid);
  if (r != ncclSuccess) return fail(STTSV_ERR_NCCL, "ncclGetUniqueId: %s", api->GetErrorString(r));
  memcpy(id, &uid, 128);
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_comm_create(sttsv_comm_t* out, const unsigned char id[128], int world, int rank,
                                            int device) {
  if (!out || !id) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(STTSV_ERR_INVALID_ARGUMENT, "bad world/rank");
  NcclApi* api = nccl_api();
  if (!api) return fail(STTSV_ERR_NCCL, "could not load libnccl.so.2");
  CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  auto* c = new sttsv_comm_s();
  ncclResult_t r = api->CommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(STTSV_ERR_NCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
  }
  c->world = world;
  c->rank = rank;
  c->device = device;
  *out = c;
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_comm_destroy(sttsv_comm_t c) {
  if (!c) return STTSV_OK;
  NcclApi* api = nccl_api();
  if (api && c->comm) api->CommDestroy(c->comm);
  delete c;
  return STTSV_OK;
}

// ------------------------------------------------------------ combinatorics
// (N-1)!/(k! S(N,k)) in long double.  S(N,k) by the explicit alternating sum
// S(N,k) = (1/k!) sum_j (-1)^j C(k,j) (k-j)^N is exact in 128-bit integers for
// N <= 26; beyond that the recurrence S(n,k) = k S(n-1,k) + S(n-1,k-1) in long
// double.  |beta(k)| = k! S(N,k) = sum_j (-1)^j C(k,j) (k-j)^N  (surjections).
static long double surjections_ld(int N, int k) {
  if (N <= 26) {
    __int128 tot = 0, binom = 1;
    for (int j = 0; j <= k; ++j) {
      __int128 p = 1;
      for (int t = 0; t < N; ++t) p *= (k - j);
      tot += (j & 1) ? -binom * p : binom * p;
      binom = binom * (k - j) / (j + 1);
    }
    return (long double)tot;
  }
  std::vector<std::vector<long double>> S(N + 1, std::vector<long double>(N + 1, 0.0L));
  S[0][0] = 1.0L;
  for (int a = 1; a <= N; ++a)
    for (int b = 1; b <= a; ++b) S[a][b] = (long double)b * S[a - 1][b] + S[a - 1][b - 1];
  long double f = 1.0L;
  for (int i = 2; i <= k; ++i) f *= i;
  return S[N][k] * f;
}

static long double scale_constant(int N, int k) {
  long double f = 1.0L;
  for (int i = 2; i <= N - 1; ++i) f *= i;
  return f / surjections_ld(N, k);
}

// FP64 operations (FMA or MUL) of the per-edge DP for an edge of size k
// (SURVEY.md Appendix A closed form) plus the k scalings w'(q_i + F); the
// series table is built once per apply per active vertex, not per edge.  Used
// for the tile cost balance and plan info (roofline flops = 2 x this).
static double dp_fma(int N, int k) {
  const double D = N - k, L = D + 1;
  double f;
  if (k == 1) f = 0;
  else if (k == 2) f = D;
  else if (k == 3) f = L * (L + 1) / 2 + 4 * L - 1;
  else f = (k - 3) * L * (L + 1) + (k + 1) * L - 1;
  return f + k + 1;
}

// FP64 operations per edge with the shared-prefix memo (prefix.cuh) for a tile
// whose edges share U leading members: M = K - U own members; mirrors
// dp_front_norm + the SB update + the scalings.  U = 0: dp_fma.
static double dp_fma_prefix(int N, int k, int U) {
  if (U == 0) return dp_fma(N, k);
  const int M = k - U;
  if (M == 0) return 1.0;  // SB[0] += w'
  const double L = N - k + 1, D = L - 1, T = L * (L - 1) / 2;
  double f;
  if (M == 1) f = (D >= 1 ? D - 1 + 2 : 0) + 1;
  else f = (M - 2) * (T + 1) + 2 * D + 4 + T + 1 + (D >= 1 ? D - 1 + 2 : 0) + (M - 2) * (D + 3 + T);
  return f + (L + 1) + 1 + M;
}

constexpr int64_t kMemoMinEdges = (int64_t)1 << 22;  // shared-prefix memo for plans of >= 4.2 M edges

// ------------------------------------------------------------------- plans
struct sttsv_plan_s {
  int device = 0;
  int64_t n = 0;
  int32_t N = 0;
  int world = 1, rank = 0;
  sttsv_comm_t comm = nullptr;
  int64_t total_edges = 0, total_inc = 0, local_edges = 0, local_inc = 0;
  int64_t stored_edges = 0, stored_inc = 0;  // after STTSV_MERGE_DUPLICATES
  int64_t n_active = 0;
  int64_t edges_per_size[STTSV_MAX_RANK + 1] = {0};
  // device memory
  void* dmem = nullptr;
  size_t dbytes = 0;
  int32_t* d_act = nullptr;
  double* d_xa = nullptr;
  double* d_ya = nullptr;
  double* d_scratch = nullptr;
  double* d_xg = nullptr;   // series table (n_active x gs)
  int gs = 2;
  // e2e staging (sttsv_apply_host)
  double* d_xhost = nullptr;
  double* d_yhost = nullptr;
  cudaStream_t host_stream = nullptr;
  double* h_lambda = nullptr;  // pinned (lambda_min, lambda_max) of sttsv_hec
  // side stream: zero-fills the dense output concurrently with the edge kernel
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::vector<int32_t> h_act;  // host copy of act[] (sttsv_apply_host gathers x on the host)
  double* h_xa = nullptr;      // pinned staging of x on the active vertices
  // deterministic mode (STTSV_DETERMINISTIC): slot pool, vertex-major buffer, chunks
  bool det = false;
  bool batch_fused = false;  // STTSV_BATCH_FUSED: sttsv_apply_batch as one pass over the edge stream
  void* det_mem = nullptr;
  int64_t det_chunks = 0;
  double *d_contrib = nullptr, *d_csum = nullptr;
  int64_t *d_cstart = nullptr, *d_vchunk = nullptr;
  // batch (f4) workspace, grown on demand by sttsv_apply_batch
  int batch_cap = 0;
  void* batch_mem = nullptr;
  double *b_xa = nullptr, *b_xg = nullptr, *b_ya = nullptr, *b_priv = nullptr, *b_gtab = nullptr;
  int64_t gtab_doubles = 0;  // size of the group table (prefix.cuh)
  // kernel
  EdgeKernelEntry ent{};
  EdgeKernelParams kp{};
  int grid = 0, block = 0;
  size_t smem = 0;
  int64_t stream_bytes = 0;
  double fma = 0;
  int64_t allreduces = 0;  // ncclAllReduce calls issued (sttsv_plan_info)
  double fma_exec = 0;      // FP64 operations the kernel executes per apply (shared-prefix memo counted)
  const int32_t* d_gku = nullptr;  // per prefix group: k | U << 8 (group_kernel)
  const int64_t* d_goff = nullptr;  // per prefix group: offset of its record in the group table
  const long long* d_items = nullptr;  // group_kernel work items
  int group_lmax = 0;                    // largest L among the prefix groups
  int64_t nitems = 0;
  int64_t prefix_tiles = 0, prefix_groups = 0, prefix_inc = 0;
  // M = 0 runs (plan_create): edges whose warp block is one vertex set leave the tile
  // stream; each run is one representative edge whose weight is the run's summed w'
  // (plan-time for uniform-weight buckets, m0sum_kernel every apply otherwise)
  int64_t m0_edges = 0, m0_groups = 0, m0_chunks = 0;
  const long long* d_m0job = nullptr;    // m0sum_kernel jobs (x, y) pairs (kernels.cu)
  const long long* d_pentry = nullptr;   // per short run of a pack: (wpos << 18) | (offset << 9) | length
  const int64_t* d_rc0 = nullptr;        // per split run: its chunk jobs rc0[2r] .. rc0[2r+1]
  const int64_t* d_wpos = nullptr;       // per split run: its representative's weight slot
  const double* d_w0 = nullptr;          // the runs' stored weights
  double* d_m0part = nullptr;            // per chunk: partial sum (runs of several chunks)
  unsigned int* d_m0cnt = nullptr;       // per run: chunks done (reset by the last)
  double* d_wpool = nullptr;             // the plan's weight pool (the representatives' slots)
  // edge-kernel timing (sttsv_plan_profile)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  size_t events_used = 0;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static inline int64_t bucket_lo(int64_t mk, int world, int rank) {
  return (int64_t)((__int128)mk * rank / world);
}

// shared by the planner and sttsv_shard_edges: per edge its position in its
// size bucket; per bucket its global count
static void bucket_positions(int64_t m, const int32_t* sizes, int N, std::vector<int64_t>& pos,
                             std::vector<int64_t>& count) {
  count.assign(N + 1, 0);
  pos.resize(m);
  for (int64_t e = 0; e < m; ++e) pos[e] = count[sizes[e]]++;
}

extern "C" sttsv_status_t sttsv_shard_edges(int64_t m, const int32_t* sizes, int32_t N, int world, int rank,
                                            int64_t* out_edges, int64_t* out_count) {
  if (!out_count || (m > 0 && (!sizes || !out_edges))) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  if (m < 0 || N < 1 || N > STTSV_MAX_RANK || world < 1 || rank < 0 || rank >= world)
    return fail(STTSV_ERR_INVALID_ARGUMENT, "bad m/N/world/rank");
  for (int64_t e = 0; e < m; ++e)
    if (sizes[e] < 1 || sizes[e] > N) return fail(STTSV_ERR_EDGE_SIZE, "edge %lld has size %d", (long long)e, sizes[e]);
  std::vector<int64_t> pos, count;
  bucket_positions(m, sizes, N, pos, count);
  int64_t c = 0;
  for (int k = 1; k <= N; ++k) {
    const int64_t lo = bucket_lo(count[k], world, rank), hi = bucket_lo(count[k], world, rank + 1);
    for (int64_t e = 0; e < m; ++e)
      if (sizes[e] == k && pos[e] >= lo && pos[e] < hi) out_edges[c++] = e;
  }
  *out_count = c;
  return STTSV_OK;
}

static void free_plan(sttsv_plan_s* p) {
  if (!p) return;
  DeviceGuard g(p->device);
  if (p->host_stream) cudaStreamSynchronize(p->host_stream);
  cudaDeviceSynchronize();
  for (auto& ev : p->events) {
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  if (p->dmem) cudaFree(p->dmem);
  if (p->d_xhost) cudaFree(p->d_xhost);
  if (p->host_stream) cudaStreamDestroy(p->host_stream);
  if (p->h_lambda) cudaFreeHost(p->h_lambda);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->h_xa) cudaFreeHost(p->h_xa);
  if (p->batch_mem) cudaFree(p->batch_mem);
  if (p->det_mem) cudaFree(p->det_mem);
  delete p;
}

extern "C" sttsv_status_t sttsv_destroy(sttsv_plan_t p) {
  free_plan(p);
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_plan_destroy(sttsv_plan_t p) { return sttsv_destroy(p); }

extern "C" sttsv_status_t sttsv_plan_create(sttsv_plan_t* out, int64_t n, int32_t N, int64_t m,
                                            const int32_t* sizes, const int32_t* indices, const double* weights,
                                            int device, int world, int rank, sttsv_comm_t comm, uint32_t flags) {
  if (!out) return fail(STTSV_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > INT32_MAX) return fail(STTSV_ERR_INVALID_ARGUMENT, "n must be in [1, 2^31-1], got %lld", (long long)n);
  if (N < 1 || N > STTSV_MAX_RANK)
    return fail(STTSV_ERR_INVALID_ARGUMENT, "rank_Nk must be in [1, %d], got %d", STTSV_MAX_RANK, N);
  if (m < 0) return fail(STTSV_ERR_INVALID_ARGUMENT, "num_edges < 0");
  if (m > 0 && (!sizes || !indices)) return fail(STTSV_ERR_INVALID_ARGUMENT, "sizes/indices NULL");
  if (world < 1 || rank < 0 || rank >= world) return fail(STTSV_ERR_INVALID_ARGUMENT, "bad world/rank");
  if (comm && (comm->world != world || comm->rank != rank || comm->device != device))
    return fail(STTSV_ERR_INVALID_ARGUMENT, "comm world/rank/device differ from the plan's");
  const uint32_t known =
      STTSV_CANONICALIZE | STTSV_MERGE_DUPLICATES | STTSV_DETERMINISTIC | STTSV_BATCH_FUSED | STTSV_NO_PREFIX_MEMO;
  if (flags & ~known) return fail(STTSV_ERR_UNSUPPORTED, "flags 0x%x not implemented in this build", flags & ~known);

  // ---- validate; offsets
  std::vector<int64_t> off(m + 1, 0);
  for (int64_t e = 0; e < m; ++e) {
    if (sizes[e] < 1 || sizes[e] > N)
      return fail(STTSV_ERR_EDGE_SIZE, "edge %lld has size %d (rank %d)", (long long)e, sizes[e], N);
    off[e + 1] = off[e] + sizes[e];
  }
  const int64_t total_inc = off[m];
  std::vector<int32_t> canon;
  const int32_t* idx = indices;
  if (flags & STTSV_CANONICALIZE) {
    canon.assign(indices, indices + total_inc);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) std::sort(canon.begin() + off[e], canon.begin() + off[e + 1]);
    idx = canon.data();
  }
  int64_t bad_e = -1;
  int bad_kind = 0;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int kind = 0;
    for (int64_t j = off[e]; j < off[e + 1]; ++j) {
      if (idx[j] < 0 || idx[j] >= n) { kind = 1; break; }
      if (j > off[e] && idx[j] <= idx[j - 1]) { kind = idx[j] == idx[j - 1] ? 3 : 2; break; }
    }
    if (kind == 0 && weights && !std::isfinite(weights[e])) kind = 4;
    if (kind) {
#pragma omp critical
      if (bad_e < 0 || e < bad_e) { bad_e = e; bad_kind = kind; }
    }
  }
  if (bad_e >= 0) {
    switch (bad_kind) {
      case 1: return fail(STTSV_ERR_VERTEX_RANGE, "edge %lld has an id outside [0, %lld)", (long long)bad_e, (long long)n);
      case 2: return fail(STTSV_ERR_UNSORTED, "edge %lld is not strictly increasing", (long long)bad_e);
      case 3: return fail(STTSV_ERR_REPEATED_VERTEX, "edge %lld repeats a vertex", (long long)bad_e);
      default: return fail(STTSV_ERR_NONFINITE, "weight of edge %lld is not finite", (long long)bad_e);
    }
  }

  auto* p = new sttsv_plan_s();
  p->device = device;
  p->n = n;
  p->N = N;
  p->world = world;
  p->rank = rank;
  p->comm = comm;
  p->total_edges = m;
  p->total_inc = total_inc;

  // ---- degrees over ALL edges (identical relabel on every rank)
  std::vector<int64_t> deg(n, 0);
  for (int64_t j = 0; j < total_inc; ++j) deg[idx[j]]++;
  std::vector<int32_t> act;
  act.reserve(1024);
  for (int64_t v = 0; v < n; ++v)
    if (deg[v] > 0) act.push_back((int32_t)v);
  std::stable_sort(act.begin(), act.end(), [&](int32_t a, int32_t b) { return deg[a] > deg[b]; });
  const int64_t na = (int64_t)act.size();
  p->n_active = na;
  std::vector<int32_t> newid(n, -1);
  for (int64_t i = 0; i < na; ++i) newid[act[i]] = (int32_t)i;
  std::vector<int64_t>().swap(deg);

  // ---- buckets and this shard's slices
  std::vector<int64_t> pos, count;
  bucket_positions(m, sizes, N, pos, count);
  // 16-bit member ids in the edge stream when every relabelled id fits
  // (STTSV_ID32=1 forces 32-bit ids, for experiments)
  p->ent = edge_entry(N, na <= 65536 && !getenv("STTSV_ID32"));
  const int tile = p->ent.tile;
  const int idb = p->ent.id_bytes;  // 2: 16-bit member ids in the edge stream
  // bucket index bi: 1..N the input edges of size bi, N + k the representatives of the
  // size-k M = 0 runs (below)
  const int NB = 2 * N;
  auto ksz = [N](int bi) { return bi <= N ? bi : bi - N; };
  std::vector<int64_t> lo(N + 1), mk(NB + 1, 0), stride(NB + 1, 0);
  for (int k = 1; k <= N; ++k) {
    lo[k] = bucket_lo(count[k], world, rank);
    mk[k] = bucket_lo(count[k], world, rank + 1) - lo[k];
    stride[k] = (mk[k] + tile - 1) / tile * tile;  // padded to whole tiles (see below)
    p->edges_per_size[k] = mk[k];
    p->local_edges += mk[k];
    p->local_inc += mk[k] * k;
  }
  // pools: ids [sum_k k*stride_k] int32, w [sum_k stride_k] f64
  std::vector<int64_t> ids_off(NB + 1, 0), w_off(NB + 1, 0);
  int64_t ids_total = 0, w_total = 0;
  for (int k = 1; k <= N; ++k) {
    ids_off[k] = ids_total;
    w_off[k] = w_total;
    ids_total += (int64_t)k * stride[k];
    w_total += stride[k];
  }
  std::vector<int32_t> h_ids((size_t)ids_total, 0);
  std::vector<double> h_w((size_t)w_total, 0.0);
  std::vector<long double> Ckl(N + 1, 0.0L);
  for (int k = 1; k <= N; ++k) Ckl[k] = scale_constant(N, k);
  // rows: this shard's edges, row-major per bucket, members relabelled and ascending
  std::vector<int64_t> row_off(N + 1, 0);
  int64_t rows_total = 0;
  for (int k = 1; k <= N; ++k) {
    row_off[k] = rows_total;
    rows_total += (int64_t)k * mk[k];
  }
  std::vector<int32_t> rows((size_t)rows_total);
  std::vector<int64_t> stored(NB + 1, 0);  // edges stored per bucket (after optional merging)
  std::vector<double> wrow((size_t)w_total);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    const int k = sizes[e];
    const int64_t le = pos[e] - lo[k];
    if (le < 0 || le >= mk[k]) continue;
    int32_t* v = rows.data() + row_off[k] + le * k;
    for (int i = 0; i < k; ++i) v[i] = newid[idx[off[e] + i]];
    for (int i = 1; i < k; ++i) {  // members ascending by relabelled id
      int32_t t = v[i];
      int j = i - 1;
      while (j >= 0 && v[j] > t) { v[j + 1] = v[j]; --j; }
      v[j + 1] = t;
    }
    const long double w = weights ? (long double)weights[e] : (long double)k;
    wrow[w_off[k] + le] = (double)(w * Ckl[k]);
  }
  // shared-prefix memo: per warp block (the NCW blocks of 32*epl consecutive sorted
  // edges of a tile, one per consumer warp) the shared prefix length U
  std::vector<std::vector<uint8_t>> tile_u(NB + 1);
  const int nblk = p->ent.consumers / 32, wblk = tile / nblk;
  std::vector<int> wuni(NB + 1, 0);
  std::vector<double> wconst(NB + 1, 0.0);
  // The memo pays once the stream is long enough to amortise its group-table kernel and
  // per-block control work: measured on B200, mid (1e6 edges) runs faster without it and
  // high-rank (5e6) faster with it; below kMemoMinEdges a plan uses the plain per-edge path
  // (STTSV_MEMO_MIN_EDGES overrides, for experiments).
  int64_t memo_min = kMemoMinEdges;
  if (const char* env = getenv("STTSV_MEMO_MIN_EDGES")) memo_min = atoll(env);
  const bool memo = p->ent.prefix_mmax > 0 && !(flags & (STTSV_DETERMINISTIC | STTSV_NO_PREFIX_MEMO)) &&
                    !getenv("STTSV_NO_PREFIX") && p->local_edges >= memo_min;
  // shared-prefix memo: per warp block of wblk consecutive sorted edges, the length U of
  // the member prefix all its edges share (0: none usable, the block runs the full DP)
  auto block_u = [&](int k, const int32_t* col, int64_t st, std::vector<uint8_t>& tu) {
    const int L = N - k + 1;
    for (int64_t bl = 0; bl < (int64_t)tu.size(); ++bl) {
      const int64_t j0 = bl * wblk, j1 = j0 + wblk - 1;
      int u = 0;
      while (u < k && col[(int64_t)u * st + j0] == col[(int64_t)u * st + j1]) ++u;
      const int M = k - u;
      const bool ok = u >= 1 && (M == 0 || (M <= p->ent.prefix_mmax && L <= p->ent.prefix_lmax));
      tu[bl] = (uint8_t)(ok ? u : 0);
    }
  };
  struct M0Run {
    int k;
    int64_t ids;     // offset of its vertex set in m0ids
    int64_t cnt;     // edges
    int64_t w0, w1;  // its weights in h_w0 (non-uniform buckets)
  };
  std::vector<M0Run> m0runs;
  std::vector<int32_t> m0ids;
  std::vector<double> h_w0;
  std::vector<int64_t> m0cnt(N + 1, 0);
  // Sort each bucket lexicographically (stable: the plan is deterministic).
  // Consecutive edges then share their hot low slots, which the kernel's
  // per-lane run accumulators turn into one deposit per run.
  for (int k = 1; k <= N; ++k) {
    if (mk[k] == 0) continue;
    const int32_t* R = rows.data() + row_off[k];
    std::vector<int64_t> perm(mk[k]);
    std::iota(perm.begin(), perm.end(), (int64_t)0);
    __gnu_parallel::stable_sort(perm.begin(), perm.end(), [R, k](int64_t a, int64_t b) {
      const int32_t* x = R + a * k;
      const int32_t* y = R + b * k;
      for (int i = 0; i < k; ++i)
        if (x[i] != y[i]) return x[i] < y[i];
      return false;
    });
    int32_t* col = h_ids.data() + ids_off[k];
    const int64_t st = stride[k];
    int64_t kept = mk[k];
    if (flags & STTSV_MERGE_DUPLICATES) {
      // identical vertex sets are adjacent after the sort: keep the first of each
      // run with the run's summed weight (B is linear in w)
      kept = 0;
      for (int64_t j = 0; j < mk[k];) {
        const int32_t* src = R + perm[j] * k;
        long double wsum = 0.0L;
        int64_t j2 = j;
        while (j2 < mk[k] && std::equal(src, src + k, R + perm[j2] * k)) wsum += (long double)wrow[w_off[k] + perm[j2++]];
        for (int i = 0; i < k; ++i) col[(int64_t)i * st + kept] = src[i];
        h_w[w_off[k] + kept] = (double)wsum;
        ++kept;
        j = j2;
      }
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t j = 0; j < mk[k]; ++j) {
        const int32_t* src = R + perm[j] * k;
        for (int i = 0; i < k; ++i) col[(int64_t)i * st + j] = src[i];
        h_w[w_off[k] + j] = wrow[w_off[k] + perm[j]];
      }
    }
    stored[k] = kept;
    // pad the bucket to whole tiles with copies of its last edge at weight 0:
    // the kernel then never meets a partial tile (no per-lane validity tests),
    // a padded edge contributes exactly 0 and continues the last edge's runs
    const int64_t padded = (kept + tile - 1) / tile * tile;
    for (int64_t j = kept; j < padded; ++j) {
      for (int i = 0; i < k; ++i) col[(int64_t)i * st + j] = col[(int64_t)i * st + kept - 1];
      h_w[w_off[k] + j] = 0.0;
    }
    // uniform weights (e.g. the configs' w = 1): no weight column is streamed; the
    // kernel uses the constant for real edges and 0 for padding (edge_kernel.cuh WSrc)
    wuni[k] = memo && kept > 0;
    for (int64_t j = 1; j < kept && wuni[k]; ++j)
      if (h_w[w_off[k] + j] != h_w[w_off[k]]) wuni[k] = 0;
    wconst[k] = kept > 0 ? h_w[w_off[k]] : 0.0;
    // shared-prefix memo (prefix.cuh): per tile, the number U of leading members
    // all its edges share = the common prefix of its first and last (sorted) edge
    const int64_t ntl = padded / tile;
    tile_u[k].assign(ntl * nblk, 0);
    if (memo) {
      block_u(k, col, st, tile_u[k]);
      // M = 0 blocks (U = k: every edge of the block is the same vertex set) leave the
      // tile stream.  B is linear in w, so a run of such blocks (one set;
      // the sort makes it one contiguous run per set) contributes exactly what ONE edge
      // of that set with w' summed over the run does: the run is replaced by a
      // representative edge in the bucket N + k below.  Uniform-weight buckets give it
      // w' x (edges of the run); otherwise the run's weights move to the M = 0 weight
      // column, which m0sum_kernel sums into the representative's weight every apply.
      // The kept blocks are compacted in order and the bucket is re-padded to whole tiles.
      std::vector<uint8_t> nu;
      nu.reserve(tile_u[k].size());
      int64_t nkept = 0, kreal = 0;
      for (int64_t bl = 0; bl < ntl * nblk; ++bl) {
        const int64_t j0 = bl * wblk;
        const int64_t real = std::max<int64_t>(0, std::min<int64_t>(wblk, kept - j0));
        if (real == 0) break;  // only padding from here on
        if (tile_u[k][bl] == k) {
          M0Run* r = m0runs.empty() ? nullptr : &m0runs.back();
          bool same = r && r->k == k;
          for (int q = 0; q < k && same; ++q) same = m0ids[r->ids + q] == col[(int64_t)q * st + j0];
          if (!same) {
            m0runs.push_back(M0Run{k, (int64_t)m0ids.size(), 0, (int64_t)h_w0.size(), (int64_t)h_w0.size()});
            for (int q = 0; q < k; ++q) m0ids.push_back(col[(int64_t)q * st + j0]);
            r = &m0runs.back();
          }
          r->cnt += real;
          if (!wuni[k]) {
            h_w0.insert(h_w0.end(), h_w.begin() + w_off[k] + j0, h_w.begin() + w_off[k] + j0 + real);
            r->w1 = (int64_t)h_w0.size();
          }
          m0cnt[k] += real;
          continue;
        }
        if (nkept != bl) {
          for (int q = 0; q < k; ++q)
            std::copy(col + (int64_t)q * st + j0, col + (int64_t)q * st + j0 + wblk, col + (int64_t)q * st + nkept * wblk);
          std::copy(h_w.begin() + w_off[k] + j0, h_w.begin() + w_off[k] + j0 + wblk,
                    h_w.begin() + w_off[k] + nkept * wblk);
        }
        nu.push_back(tile_u[k][bl]);
        kreal = nkept * wblk + real;
        ++nkept;
      }
      if (nkept < ntl * nblk) {
        // re-pad: weight-0 copies of the last kept edge, full-DP blocks (U = 0)
        const int64_t npad = (nkept + nblk - 1) / nblk * nblk * wblk;
        for (int64_t j = kreal; j < npad; ++j) {
          for (int q = 0; q < k; ++q) col[(int64_t)q * st + j] = col[(int64_t)q * st + kreal - 1];
          h_w[w_off[k] + j] = 0.0;
        }
        while ((int64_t)nu.size() < npad / wblk) nu.push_back(0);
        tile_u[k].swap(nu);
        stored[k] = kreal;
      }
    }
  }
  std::vector<int32_t>().swap(rows);
  std::vector<double>().swap(wrow);
  std::vector<int32_t>().swap(newid);

  // ---- representatives of the M = 0 runs: bucket N + k holds one edge per size-k run
  // (distinct sets, already in sorted order); weight slot wpos of each non-uniform one
  // is written by m0sum_kernel every apply from its run's chunks of h_w0
  std::vector<long long> h_m0job;    // m0sum_kernel jobs: (x, y) pairs (kernels.cu)
  std::vector<long long> h_pentry;   // per short run of a pack: (wpos << 18) | (offset << 9) | length
  std::vector<int64_t> h_rc0;        // per split run (several chunk jobs): its first and end job
  std::vector<int64_t> h_wpos;       // per split run: its representative's weight slot
  struct WRun { int64_t a, b, wpos; };
  std::vector<WRun> wruns;
  if (!m0runs.empty()) {
    // m0sum_kernel jobs: a run of > kShort weights is cut into chunks of <= kChunk, one
    // warp each; a shorter run is one thread's job
    constexpr int64_t kChunk = 2048, kShort = 256;
    const int epl = p->ent.epl, wblock = 32 * epl;
    for (int k = 1; k <= N; ++k) {
      const int bi = N + k;
      int64_t nrep = 0;
      for (const M0Run& r : m0runs) nrep += r.k == k;
      if (nrep == 0) continue;
      mk[bi] = nrep;
      stride[bi] = (nrep + tile - 1) / tile * tile;
      ids_off[bi] = ids_total;
      w_off[bi] = w_total;
      ids_total += (int64_t)k * stride[bi];
      w_total += stride[bi];
      h_ids.resize((size_t)ids_total, 0);
      h_w.resize((size_t)w_total, 0.0);
      int32_t* col = h_ids.data() + ids_off[bi];
      const int64_t st = stride[bi];
      int64_t j = 0;
      for (const M0Run& r : m0runs) {
        if (r.k != k) continue;
        for (int q = 0; q < k; ++q) col[(int64_t)q * st + j] = m0ids[r.ids + q];
        if (wuni[k]) {
          h_w[w_off[bi] + j] = (double)((long double)wconst[k] * (long double)r.cnt);
        } else {
          // the lane-major layout (below) moves sorted position j of a warp block
          const int64_t b0 = j / wblock * wblock, in = j % wblock;
          wruns.push_back(WRun{r.w0, r.w1, w_off[bi] + b0 + (in % epl) * 32 + in / epl});
        }
        ++j;
      }
      for (; j < st; ++j) {  // padding: weight-0 copies of the last representative
        for (int q = 0; q < k; ++q) col[(int64_t)q * st + j] = col[(int64_t)q * st + nrep - 1];
        h_w[w_off[bi] + j] = 0.0;
      }
      stored[bi] = nrep;
      wuni[bi] = 0;
      tile_u[bi].assign(st / tile * nblk, 0);
      block_u(k, col, st, tile_u[bi]);
      p->m0_groups += nrep;
    }
    // one warp job each: a run of <= kChunk weights (y = its weight slot); a chunk of a
    // longer run (y = -1 - run: partial sum + fold); a pack of neighbouring short runs
    // (<= kShort weights each, adjacent in h_w0, <= kShort in all; y = (first entry << 9) | runs)
    constexpr long long kPack = 1ll << 62;
    auto job = [&](long long x, long long y) { h_m0job.push_back(x); h_m0job.push_back(y); };
    for (size_t q = 0; q < wruns.size();) {
      const WRun& wr = wruns[q];
      const int64_t n = wr.b - wr.a;
      if (n > kShort) {
        if (n <= kChunk) {
          job(((long long)wr.a << 24) | n, wr.wpos);
        } else {
          const long long run = (long long)h_wpos.size();
          h_rc0.push_back((int64_t)(h_m0job.size() / 2));
          for (int64_t a = wr.a; a < wr.b; a += kChunk) job(((long long)a << 24) | std::min<int64_t>(kChunk, wr.b - a), -1 - run);
          h_rc0.push_back((int64_t)(h_m0job.size() / 2));
          h_wpos.push_back(wr.wpos);
        }
        ++q;
        continue;
      }
      size_t q1 = q + 1;
      while (q1 < wruns.size() && wruns[q1].a == wruns[q1 - 1].b && wruns[q1].b - wr.a <= kShort) ++q1;
      job(kPack | ((long long)wr.a << 24) | (wruns[q1 - 1].b - wr.a), ((long long)h_pentry.size() << 9) | (long long)(q1 - q));
      for (size_t i = q; i < q1; ++i)
        h_pentry.push_back(((long long)wruns[i].wpos << 18) | ((wruns[i].a - wr.a) << 9) | (wruns[i].b - wruns[i].a));
      q = q1;
    }
    p->m0_chunks = (int64_t)(h_m0job.size() / 2);
  }

  // ---- tile order: buckets most expensive first (the dynamic scheduler's tail is the cheapest work)
  int occ = 0;
  int hot = 256;  // ids below H accumulate in per-CTA L2 slices (STTSV_HOT overrides, for experiments;
                  // 256-512 measured best: smaller slices are cheaper to zero and fold, 64 contends)
  if (const char* env = getenv("STTSV_HOT")) hot = std::max(0, atoi(env));
  const int H = (int)std::min<int64_t>(na, hot);
  const int T = p->ent.run_slots;
  {
    DeviceGuard g(device);
    cudaError_t e0 = cudaSetDevice(device);
    if (e0 != cudaSuccess) { free_plan(p); return cuda_fail(e0, "cudaSetDevice"); }
    p->smem = edge_kernel_smem_bytes(p->ent, N);
    e0 = edge_kernel_config(p->ent, p->smem, &occ);
    if (e0 != cudaSuccess) { free_plan(p); return cuda_fail(e0, "edge kernel configuration"); }
    if (occ < 1) { free_plan(p); return fail(STTSV_ERR_CUDA, "edge kernel cannot be resident (smem %zu)", p->smem); }
  }
  std::vector<int> order;  // bucket indices in kernel order
  for (int bi = 1; bi <= NB; ++bi)
    if (stored[bi] > 0) order.push_back(bi);
  // per-edge cost of a bucket as the kernel will execute it (the shared-prefix memo
  // makes most of a bucket cheap; its unshared blocks cost the full DP)
  std::vector<double> ecost(NB + 1, 0.0);
  for (int bi : order) {
    const int k = ksz(bi);
    double c = 0;
    for (size_t bl = 0; bl < tile_u[bi].size(); ++bl) c += dp_fma_prefix(N, k, tile_u[bi][bl]);
    ecost[bi] = tile_u[bi].empty() ? dp_fma(N, k) : c / (double)tile_u[bi].size();
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ecost[a] > ecost[b]; });
  EdgeKernelParams& kp = p->kp;
  kp.N = N;
  kp.nb = (int)order.size();
  int64_t tiles = 0;
  double fma = 0;
  for (int k = 1; k <= N; ++k) {  // input edges: in the stream or in an M = 0 run
    fma += dp_fma(N, k) * (double)(stored[k] + m0cnt[k]);
    p->stored_edges += stored[k] + m0cnt[k];
    p->stored_inc += (stored[k] + m0cnt[k]) * k;
    p->m0_edges += m0cnt[k];
    if (!wuni[k]) p->stream_bytes += m0cnt[k] * 8;  // the M = 0 weights m0sum_kernel reads
  }
  for (int i = 0; i < kp.nb; ++i) {
    const int bi = order[i], k = ksz(bi);
    BucketDesc& b = kp.b[i];
    b.k = k;
    b.m = stored[bi];
    b.stride = stride[bi];
    b.tile_begin = tiles;
    b.ids_off = ids_off[bi];
    b.w_off = w_off[bi];
    b.wuni = wuni[bi];
    b.wc = wconst[bi];
    tiles += (stored[bi] + tile - 1) / tile;
    const int64_t ntl = (stored[bi] + tile - 1) / tile;
    for (int64_t tl = 0; tl < ntl; ++tl) {
      int us = k;  // staged columns: from the smallest prefix of the tile's blocks
      for (int w = 0; w < nblk; ++w) us = std::min<int>(us, tile_u[bi][tl * nblk + w]);
      p->stream_bytes += (int64_t)tile * (idb * (k - us) + (wuni[bi] ? 0 : 8));
      for (int w = 0; w < nblk; ++w) {
        const int u = tile_u[bi][tl * nblk + w];
        const int64_t first = tl * tile + (int64_t)w * wblk;
        const int64_t real = std::max<int64_t>(0, std::min<int64_t>(wblk, stored[bi] - first));  // not padding
        p->fma_exec += dp_fma_prefix(N, k, u) * (double)real;
        if (u > 0) {
          p->prefix_tiles += 1;
          if (bi <= N) p->prefix_inc += (int64_t)u * real;
        }
      }
    }
  }
  for (int k = 1; k <= N; ++k) p->prefix_inc += m0cnt[k] * k;  // M = 0 runs: every member is shared
  kp.num_tiles = tiles;
  // shared-prefix groups: consecutive tiles (kernel order) with the same bucket, U and
  // prefix ids share a group id; U = 0 tiles have none (-1)
  std::vector<long long> h_hdr;  // per tile: U_stage; then per warp block (goff << 8) | U
  std::vector<int32_t> h_gku;
  std::vector<int64_t> h_goff;
  std::vector<double> h_gtab;  // group records (prefix.cuh): [A: L][C: U x L][ids: U]; ids filled here
  std::vector<long long> h_items;  // group_kernel work items: (group << 8) | prefix member
  std::map<std::vector<int32_t>, int32_t> gmap;
  if (memo && p->prefix_tiles > 0) {
    h_hdr.assign((size_t)tiles * (1 + nblk), 0);
    int32_t gid = -1;
    int pk = -1, pu = -1;
    std::vector<int32_t> pref, cur;
    for (int i = 0; i < kp.nb; ++i) {
      const int bi = order[i], k = kp.b[i].k;
      const int32_t* col = h_ids.data() + ids_off[bi];
      const int64_t ntl = (stored[bi] + tile - 1) / tile;
      for (int64_t tl = 0; tl < ntl; ++tl) {
        const int64_t t = kp.b[i].tile_begin + tl;
        int us = k;
        for (int w = 0; w < nblk; ++w) us = std::min<int>(us, tile_u[bi][tl * nblk + w]);
        h_hdr[(size_t)t * (1 + nblk)] = us;
        for (int w = 0; w < nblk; ++w) {
          const int u = tile_u[bi][tl * nblk + w];
          if (u == 0) {
            pk = -1;
            continue;
          }
          const int64_t j0 = tl * tile + (int64_t)w * wblk;
          cur.assign(u, 0);
          for (int q = 0; q < u; ++q) cur[q] = col[(int64_t)q * stride[bi] + j0];
          if (!(k == pk && u == pu && cur == pref)) {
            pk = k;
            pu = u;
            pref = cur;
            // one record per distinct (k, U, prefix) over the whole plan
            std::vector<int32_t> key(cur);
            key.push_back(k);
            key.push_back(u);
            auto f = gmap.find(key);
            if (f != gmap.end()) {
              gid = f->second;
            } else {
              gid = (int32_t)h_gku.size();
              gmap.emplace(std::move(key), gid);
              const int L = N - k + 1;
              h_gku.push_back(k | (u << 8));
              h_goff.push_back((int64_t)h_gtab.size());
              h_gtab.resize(h_gtab.size() + L + (size_t)u * L + u, 0.0);
              long long* ids = reinterpret_cast<long long*>(h_gtab.data() + h_gtab.size() - u);
              for (int q = 0; q < u; ++q) ids[q] = cur[q];
              for (int q = 0; q < u; ++q) h_items.push_back(((long long)gid << 8) | q);
            }
          }
          h_hdr[(size_t)t * (1 + nblk) + 1 + w] = ((long long)h_goff[gid] << 8) | u;
        }
      }
    }
    p->prefix_groups = (int64_t)h_gku.size();
    // the group kernel is instantiated up to the largest L of the plan's groups (kernels.cu)
    for (int32_t gk : h_gku) p->group_lmax = std::max(p->group_lmax, N - (gk & 255) + 1);
  }
  kp.n_active = (int32_t)na;
  kp.T = T;
  kp.H = H;
  kp.tile_edges = tile;
  p->fma = fma;

  // ---- persistent grid: one CTA per SM (x occupancy); tiles are grabbed in chunks
  // from a device counter (edge_kernel.cuh), which balances the load dynamically
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int64_t grid = (int64_t)sms * std::max(occ, 1);
  if (grid > tiles) grid = std::max<int64_t>(tiles, 1);
  // chunk: long enough for run continuity, short enough that the tail (the
  // cheapest bucket) balances: about 1/16 of a CTA's fair share
  kp.chunk = std::max<int64_t>(1, tiles / (grid * 16));
  if (const char* env = getenv("STTSV_CHUNK")) kp.chunk = std::max(1, atoi(env));
  // the last ~2 chunks' worth per CTA is handed out one tile at a time
  kp.guided_from = std::max<int64_t>(0, tiles - grid * kp.chunk * 2);
  if (const char* env = getenv("STTSV_GUIDED")) kp.guided_from = std::max<int64_t>(0, tiles - grid * kp.chunk * atoi(env));

  // ---- deterministic mode: every stored incidence gets a slot in a vertex-major
  // buffer (vertex v's incidences in bucket / edge / member order), and each
  // vertex's segment is cut into chunks of <= kDetChunk for the fixed-order sum
  std::vector<int32_t> h_slot;
  std::vector<int64_t> h_cstart, h_vchunk;
  int64_t det_total = 0;
  p->batch_fused = (flags & STTSV_BATCH_FUSED) != 0;
  if (flags & STTSV_DETERMINISTIC) {
    p->det = true;
    std::vector<int64_t> voff(na + 1, 0);
    for (int i = 0; i < kp.nb; ++i) {
      const BucketDesc& bd = kp.b[i];
      const int32_t* col = h_ids.data() + bd.ids_off;
      for (int r = 0; r < bd.k; ++r)
        for (int64_t j = 0; j < bd.m; ++j) voff[col[r * bd.stride + j] + 1]++;
    }
    for (int64_t v = 0; v < na; ++v) voff[v + 1] += voff[v];
    det_total = voff[na];
    if (det_total >= INT32_MAX) { free_plan(p); return fail(STTSV_ERR_UNSUPPORTED, "deterministic mode needs < 2^31 incidences per shard"); }
    h_slot.assign(h_ids.size(), (int32_t)det_total);  // padding -> trash slot det_total
    // order of a vertex's incidences = the order the kernel issues their stores:
    // tile, warp block, step r, lane (lane l of a warp block owns columns
    // l*epl .. l*epl+epl-1), so one warp-wide store of a hot vertex's
    // contributions hits consecutive slots
    std::vector<int64_t> cur(voff.begin(), voff.end() - 1);
    const int epl = p->ent.epl, wblock = 32 * epl;
    for (int i = 0; i < kp.nb; ++i) {
      const BucketDesc& bd = kp.b[i];
      const int32_t* col = h_ids.data() + bd.ids_off;
      int32_t* sc = h_slot.data() + bd.ids_off;
      for (int64_t wb = 0; wb * wblock < bd.m; ++wb)
        for (int r = 0; r < epl; ++r)
          for (int l = 0; l < 32; ++l) {
            const int64_t j = wb * wblock + (int64_t)l * epl + r;
            if (j >= bd.m) continue;
            for (int q = 0; q < bd.k; ++q) sc[q * bd.stride + j] = (int32_t)cur[col[q * bd.stride + j]]++;
          }
    }
    h_vchunk.resize(na + 1);
    for (int64_t v = 0; v < na; ++v) {
      h_vchunk[v] = (int64_t)h_cstart.size();
      for (int64_t a = voff[v]; a < voff[v + 1]; a += kDetChunk) h_cstart.push_back(a);
    }
    h_vchunk[na] = (int64_t)h_cstart.size();
    p->det_chunks = (int64_t)h_cstart.size();
    h_cstart.push_back(det_total);
  }

  // ---- lane-major tile layout: within each warp block of 32*epl columns, lane l
  // walks the epl CONSECUTIVE sorted edges l*epl + r (its register runs follow
  // the sort order), stored at column r*32 + l so that a warp's read of one
  // member slot at step r touches 32 consecutive ids (bank-conflict-free for
  // 2- and 4-byte ids).  Ids, weights and the deterministic slot pool move alike.
  if (p->ent.epl > 1) {
    const int epl = p->ent.epl, wblock = 32 * epl;
    for (int i = 0; i < kp.nb; ++i) {
      const BucketDesc& bd = kp.b[i];
      const int64_t cols = (bd.m + tile - 1) / tile * tile;  // whole tiles (a tile is whole warp blocks)
      auto permute = [&](auto* base) {
        using T = std::remove_reference_t<decltype(*base)>;
#pragma omp parallel
        {
          std::vector<T> tmp(wblock);
#pragma omp for schedule(static)
          for (int64_t b0 = 0; b0 < cols; b0 += wblock) {
            for (int l = 0; l < 32; ++l)
              for (int r = 0; r < epl; ++r) tmp[r * 32 + l] = base[b0 + l * epl + r];
            std::copy(tmp.begin(), tmp.end(), base + b0);
          }
        }
      };
      for (int q = 0; q < bd.k; ++q) {
        permute(h_ids.data() + bd.ids_off + q * bd.stride);
        if (p->det) permute(h_slot.data() + bd.ids_off + q * bd.stride);
      }
      permute(h_w.data() + bd.w_off);
    }
  }

  // ---- device memory: one allocation
  DeviceGuard g(device);
  auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t b_ids = align(ids_total * idb), b_w = align(w_total * 8), b_act = align(na * 4 + 4),
               b_xa = align(na * 8 + 8), b_ya = align(na * 8 + 8), b_scr = align((2 * kNormalizeScratch + 4) * 8);
  const int gs = series_stride(N);
  const size_t b_xg = align((size_t)na * gs * 8 + 16);
  const size_t b_cta = align(8);
  const size_t b_priv = align((size_t)grid * H * 8 + 8);
  const size_t b_tu = align(h_hdr.size() * 8 + 8), b_tg = 0;
  const size_t b_gku = align(h_gku.size() * 4 + 4), b_goff = align(h_goff.size() * 8 + 8),
               b_gtab = align(h_gtab.size() * 8 + 8), b_items = align(h_items.size() * 8 + 8);
  const size_t b_m0chunk = align(h_m0job.size() * 8 + 16), b_crun = align(h_pentry.size() * 8 + 8),
               b_rc0 = align(h_rc0.size() * 8 + 8), b_wpos = align(h_wpos.size() * 8 + 8),
               b_w0 = align(h_w0.size() * 8 + 8), b_part = align(h_m0job.size() / 2 * 8 + 8),
               b_rcnt = align(h_wpos.size() * 4 + 4);
  const size_t b_m0 = b_m0chunk + b_crun + b_rc0 + b_wpos + b_w0 + b_part + b_rcnt;
  p->dbytes = b_ids + b_w + b_act + b_xa + b_ya + b_scr + b_xg + b_cta + b_priv + b_tu + b_tg + b_gku + b_goff + b_gtab +
              b_items + b_m0;
  cudaError_t ce = cudaMalloc(&p->dmem, p->dbytes);
  if (ce != cudaSuccess) { free_plan(p); return cuda_fail(ce, "cudaMalloc plan"); }
  char* base = (char*)p->dmem;
  int32_t* d_ids = (int32_t*)base;
  double* d_w = (double*)(base + b_ids);
  p->d_act = (int32_t*)(base + b_ids + b_w);
  p->d_xa = (double*)(base + b_ids + b_w + b_act);
  p->d_ya = (double*)(base + b_ids + b_w + b_act + b_xa);
  p->d_scratch = (double*)(base + b_ids + b_w + b_act + b_xa + b_ya);
  p->d_xg = (double*)(base + b_ids + b_w + b_act + b_xa + b_ya + b_scr);
  unsigned long long* d_cnt = (unsigned long long*)(base + b_ids + b_w + b_act + b_xa + b_ya + b_scr + b_xg);
  double* d_priv = (double*)(base + b_ids + b_w + b_act + b_xa + b_ya + b_scr + b_xg + b_cta);
  long long* d_hdr = (long long*)(base + b_ids + b_w + b_act + b_xa + b_ya + b_scr + b_xg + b_cta + b_priv);
  char* gbase = base + b_ids + b_w + b_act + b_xa + b_ya + b_scr + b_xg + b_cta + b_priv + b_tu + b_tg;
  int32_t* d_gku = (int32_t*)gbase;
  int64_t* d_goff = (int64_t*)(gbase + b_gku);
  double* d_gtab = (double*)(gbase + b_gku + b_goff);
  long long* d_items = (long long*)(gbase + b_gku + b_goff + b_gtab);
  char* mbase = gbase + b_gku + b_goff + b_gtab + b_items;
  long long* d_m0job = (long long*)mbase;
  long long* d_pentry = (long long*)(mbase + b_m0chunk);
  int64_t* d_rc0 = (int64_t*)(mbase + b_m0chunk + b_crun);
  int64_t* d_wpos = (int64_t*)(mbase + b_m0chunk + b_crun + b_rc0);
  double* d_w0 = (double*)(mbase + b_m0chunk + b_crun + b_rc0 + b_wpos);
  p->d_m0part = (double*)(mbase + b_m0chunk + b_crun + b_rc0 + b_wpos + b_w0);
  p->d_m0cnt = (unsigned int*)(mbase + b_m0chunk + b_crun + b_rc0 + b_wpos + b_w0 + b_part);
  p->gs = gs;
  if (ids_total && idb == 4) ce = cudaMemcpy(d_ids, h_ids.data(), ids_total * 4, cudaMemcpyHostToDevice);
  if (ids_total && idb == 2) {
    std::vector<uint16_t> h16((size_t)ids_total);
    for (int64_t i = 0; i < ids_total; ++i) h16[i] = (uint16_t)h_ids[i];
    ce = cudaMemcpy(d_ids, h16.data(), ids_total * 2, cudaMemcpyHostToDevice);
  }
  if (ce == cudaSuccess && w_total) ce = cudaMemcpy(d_w, h_w.data(), w_total * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && na) ce = cudaMemcpy(p->d_act, act.data(), na * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !h_hdr.empty()) ce = cudaMemcpy(d_hdr, h_hdr.data(), h_hdr.size() * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !h_gku.empty()) ce = cudaMemcpy(d_gku, h_gku.data(), h_gku.size() * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !h_goff.empty()) ce = cudaMemcpy(d_goff, h_goff.data(), h_goff.size() * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !h_gtab.empty()) ce = cudaMemcpy(d_gtab, h_gtab.data(), h_gtab.size() * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !h_items.empty())
    ce = cudaMemcpy(d_items, h_items.data(), h_items.size() * 8, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess && !h_m0job.empty()) {
    ce = cudaMemcpy(d_m0job, h_m0job.data(), h_m0job.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess && !h_pentry.empty())
      ce = cudaMemcpy(d_pentry, h_pentry.data(), h_pentry.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(d_rc0, h_rc0.data(), h_rc0.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess && !h_wpos.empty())
      ce = cudaMemcpy(d_wpos, h_wpos.data(), h_wpos.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(d_w0, h_w0.data(), h_w0.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess && !h_wpos.empty()) ce = cudaMemset(p->d_m0cnt, 0, h_wpos.size() * 4);
  }
  p->d_m0job = d_m0job;
  p->d_pentry = d_pentry;
  p->d_rc0 = d_rc0;
  p->d_wpos = d_wpos;
  p->d_w0 = d_w0;
  p->d_items = d_items;
  p->nitems = (int64_t)h_items.size();
  kp.tile_hdr = h_hdr.empty() ? nullptr : d_hdr;
  kp.gtab = h_gtab.empty() ? nullptr : d_gtab;
  kp.gtab_vstride = 0;
  kp.group_wait = kp.gtab != nullptr;  // every launch of a plan with groups follows the group kernel
  p->gtab_doubles = (int64_t)h_gtab.size();
  p->d_gku = d_gku;
  p->d_goff = d_goff;
  p->h_act = act;
  if (ce != cudaSuccess) { free_plan(p); return cuda_fail(ce, "plan upload"); }
  kp.ids = d_ids;
  kp.w = d_w;
  p->d_wpool = d_w;
  kp.xa = p->d_xa;
  kp.xg = p->d_xg;
  kp.gs = gs;
  kp.ya = p->d_ya;
  kp.tile_counter = d_cnt;
  if (ce == cudaSuccess) ce = cudaMemset(d_cnt, 0, 2 * sizeof(unsigned long long));
  if (ce != cudaSuccess) { free_plan(p); return cuda_fail(ce, "plan counters"); }
  if (p->det) {
    const size_t a_slot = align(h_slot.size() * 4), a_con = align((det_total + 1) * 8),
                 a_cs = align(h_cstart.size() * 8), a_sum = align(p->det_chunks * 8 + 8), a_vc = align(h_vchunk.size() * 8);
    ce = cudaMalloc(&p->det_mem, a_slot + a_con + a_cs + a_sum + a_vc);
    if (ce != cudaSuccess) { free_plan(p); return cuda_fail(ce, "cudaMalloc deterministic buffers"); }
    char* db = (char*)p->det_mem;
    int32_t* d_slot = (int32_t*)db;
    p->d_contrib = (double*)(db + a_slot);
    p->d_cstart = (int64_t*)(db + a_slot + a_con);
    p->d_csum = (double*)(db + a_slot + a_con + a_cs);
    p->d_vchunk = (int64_t*)(db + a_slot + a_con + a_cs + a_sum);
    ce = cudaMemcpy(d_slot, h_slot.data(), h_slot.size() * 4, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(p->d_cstart, h_cstart.data(), h_cstart.size() * 8, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(p->d_vchunk, h_vchunk.data(), h_vchunk.size() * 8, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) { free_plan(p); return cuda_fail(ce, "deterministic upload"); }
    kp.slot = d_slot;
    kp.contrib = p->d_contrib;
    p->dbytes += a_slot + a_con + a_cs + a_sum + a_vc;
  }
  kp.nvec = 1;
  kp.xg_vstride = (int64_t)na * gs;
  kp.ya_vstride = na;
  kp.priv = d_priv;

  p->grid = (int)grid;
  p->block = p->ent.block;
  *out = p;
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_plan_info(sttsv_plan_t p, sttsv_plan_info_t* info) {
  if (!p || !info) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  memset(info, 0, sizeof(*info));
  info->n = p->n;
  info->rank_Nk = p->N;
  info->world = p->world;
  info->rank = p->rank;
  info->num_edges = p->local_edges;
  info->incidences = p->local_inc;
  info->stored_edges = p->stored_edges;
  info->stored_incidences = p->stored_inc;
  info->total_edges = p->total_edges;
  info->total_incidences = p->total_inc;
  info->n_active = p->n_active;
  for (int k = 0; k <= STTSV_MAX_RANK; ++k) info->edges_per_size[k] = p->edges_per_size[k];
  info->device_bytes = (int64_t)p->dbytes;
  info->stream_bytes = p->stream_bytes;
  info->fma_per_apply = p->fma;
  info->hot_private = p->kp.T;
  info->hot_shared = p->kp.H;
  info->kernel_grid = p->grid;
  info->kernel_block = p->block;
  info->id_bytes = p->ent.id_bytes;
  info->allreduces = p->allreduces;
  info->fma_executed = p->fma_exec;
  info->prefix_tiles = p->prefix_tiles;
  info->prefix_groups = p->prefix_groups;
  info->prefix_incidences = p->prefix_inc;
  info->num_tiles = p->kp.num_tiles;
  info->m0_edges = p->m0_edges;
  info->m0_groups = p->m0_groups;
  info->m0_chunks = p->m0_chunks;
  return STTSV_OK;
}

extern "C" int sttsv_apply_launches(sttsv_plan_t p) {
  if (!p) return 0;
  int l = 0;
  if (p->n_active > 0) l += 2;          // gather + expand
  if (p->kp.num_tiles > 0) l += 1;      // edge kernel
  if (p->kp.gtab) l += 1;               // shared-prefix group table
  if (p->m0_chunks > 0) l += 1;         // M = 0 weight sums
  if (p->det) l += 2;                   // deterministic chunk + vertex sums
  return l;
}

extern "C" sttsv_status_t sttsv_plan_profile(sttsv_plan_t p, int enable) {
  if (!p) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL plan");
  if (enable) p->events_used = 0;
  p->profiling = enable != 0;
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_plan_profile_read(sttsv_plan_t p, double* total_ms, int64_t* launches) {
  if (!p || !total_ms || !launches) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard g(p->device);
  double tot = 0.0;
  for (size_t i = 0; i < p->events_used; ++i) {
    CUDA_TRY(cudaEventSynchronize(p->events[i].second), "cudaEventSynchronize");
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, p->events[i].first, p->events[i].second), "cudaEventElapsedTime");
    tot += ms;
  }
  *total_ms = tot;
  *launches = (int64_t)p->events_used;
  return STTSV_OK;
}

static sttsv_status_t check_async(sttsv_plan_s* p) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error");
  if (p->comm) {
    NcclApi* api = nccl_api();
    ncclResult_t r = ncclSuccess;
    if (api && api->CommGetAsyncError && api->CommGetAsyncError(p->comm->comm, &r) == ncclSuccess && r != ncclSuccess)
      return fail(STTSV_ERR_NCCL, "NCCL async error: %s", api->GetErrorString(r));
  }
  return STTSV_OK;
}

// the M = 0 runs' representative weights (x-independent; a no-op for plans without runs
// of non-uniform weights)
static cudaError_t launch_m0(sttsv_plan_s* p, cudaStream_t s) {
  return launch_m0sum(p->d_w0, p->d_m0job, p->m0_chunks, p->d_pentry, p->d_rc0, p->d_wpos, p->d_m0part, p->d_m0cnt,
                      p->d_wpool, s);
}

// y_a = (B x_a^{N-1}) on the active vertices (x_a already gathered)
// zeroed: the prologue kernel, launched just before on `s`, cleared y_a; the
// edge kernel is then a programmatic dependent launch (kernels.cu)
static sttsv_status_t apply_active(sttsv_plan_s* p, cudaStream_t s, bool zeroed = false) {
  if (p->n_active == 0) return STTSV_OK;
  if (!p->det && !zeroed) CUDA_TRY(cudaMemsetAsync(p->d_ya, 0, p->n_active * sizeof(double), s), "memset y_a");
  const bool groups = p->kp.gtab != nullptr;
  if (p->kp.num_tiles > 0) {
    std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
    if (p->profiling) {
      if (p->events_used == p->events.size()) {
        std::pair<cudaEvent_t, cudaEvent_t> e2;
        CUDA_TRY(cudaEventCreate(&e2.first), "cudaEventCreate");
        CUDA_TRY(cudaEventCreate(&e2.second), "cudaEventCreate");
        p->events.push_back(e2);
      }
      ev = &p->events[p->events_used++];
      CUDA_TRY(cudaEventRecord(ev->first, s), "cudaEventRecord");
    }
    // the M = 0 runs' weight sums (x-independent; prefix.cuh), then the per-apply
    // shared-prefix group table with the M = 0 deposits (prefix.cuh)
    if (p->m0_chunks > 0) CUDA_TRY(launch_m0(p, s), "m0sum launch");
    if (groups)
      CUDA_TRY(launch_groups(p->d_xg, p->gs, p->N, p->d_gku, p->d_goff, p->d_items, p->nitems, p->group_lmax,
                             p->kp.gtab, const_cast<double*>(p->kp.gtab), s), "group kernel launch");
    CUDA_TRY(launch_edge_kernel(p->ent, p->kp, p->grid, p->smem, s, p->det ? 2 : 0,
                                groups || (zeroed && p->m0_chunks == 0)), "edge kernel launch");
    if (ev) CUDA_TRY(cudaEventRecord(ev->second, s), "cudaEventRecord");
  }
  if (p->det)  // fixed-order sums of the vertex-major buffer (every active vertex written)
    CUDA_TRY(launch_det_reduce(p->d_contrib, p->d_cstart, p->det_chunks, p->d_csum, p->d_vchunk, p->d_ya,
                               p->n_active, s), "deterministic reduce launch");
  // a6: the one exchange step, whenever a communicator is
  // attached (also at world = 1, where NCCL reduces over a single rank)
  if (p->comm) {
    NcclApi* api = nccl_api();
    ncclResult_t r = api->AllReduce(p->d_ya, p->d_ya, (size_t)p->n_active, ncclFloat64, ncclSum, p->comm->comm, s);
    if (r != ncclSuccess) return fail(STTSV_ERR_NCCL, "ncclAllReduce: %s", api->GetErrorString(r));
    ++p->allreduces;
  }
  return STTSV_OK;
}

static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

// gather -> edge kernel (+ allreduce) -> expand into a dense y.  For a large y
// the zero-fill of y (8n bytes of HBM writes) runs on a side stream, forked
// from and joined back into `s`, so it overlaps the edge kernel.
static sttsv_status_t apply_dense(sttsv_plan_s* p, const double* x, double* y, cudaStream_t s) {
  const size_t bytes = (size_t)p->n * sizeof(double);
  const bool fork = bytes >= ((size_t)8 << 20) && p->kp.num_tiles > 0;
  if (fork) {
    if (!p->side) {
      CUDA_TRY(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking), "side stream");
      CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "event");
      CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming), "event");
    }
    CUDA_TRY(cudaEventRecord(p->ev_fork, s), "fork record");
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0), "fork wait");
    CUDA_TRY(cudaMemsetAsync(y, 0, bytes, p->side), "memset y");
    CUDA_TRY(cudaEventRecord(p->ev_join, p->side), "join record");
  }
  // one prologue launch: gather x_a, series table, y_a = 0
  CUDA_TRY(launch_prologue(x, p->d_act, p->d_xa, p->d_xg, p->gs, p->ent.table_norm, p->n_active, p->d_ya, s),
           "prologue launch");
  sttsv_status_t st = apply_active(p, s, true);
  if (st != STTSV_OK) return st;
  if (fork) CUDA_TRY(cudaStreamWaitEvent(s, p->ev_join, 0), "join wait");
  else CUDA_TRY(cudaMemsetAsync(y, 0, bytes, s), "memset y");
  CUDA_TRY(launch_expand(p->d_ya, p->d_act, y, p->n_active, s), "expand launch");
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_apply(sttsv_plan_t p, const double* x, double* y, void* stream) {
  if (!p || !x || !y) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  const size_t bytes = (size_t)p->n * sizeof(double);
  if (overlap(x, bytes, y, bytes)) return fail(STTSV_ERR_ALIAS, "x and y overlap");
  DeviceGuard g(p->device);
  sttsv_status_t st = check_async(p);
  if (st != STTSV_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  return apply_dense(p, x, y, s);
}

extern "C" sttsv_status_t sttsv_apply_host(sttsv_plan_t p, const double* x_host, double* y_host) {
  if (!p || !x_host || !y_host) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  const size_t bytes = (size_t)p->n * sizeof(double);
  if (overlap(x_host, bytes, y_host, bytes)) return fail(STTSV_ERR_ALIAS, "x and y overlap");
  DeviceGuard g(p->device);
  if (!p->host_stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->host_stream, cudaStreamNonBlocking), "stream");
  cudaStream_t s = p->host_stream;
  const int64_t na = p->n_active;
  if (na > 0 && na * 8 <= p->n) {
    // sparse active set: only the active parts of x and y cross PCIe.  Gather x
    // on the host (OpenMP) into a pinned buffer, copy n_a doubles in, build the
    // series table, apply, copy y_a out; the host zero-fills y while the GPU
    // computes, then scatters y_a (y is 0 off the active set: a
    // vertex in no hyperedge gets no tensor entry).
    if (!p->h_xa) CUDA_TRY(cudaMallocHost(&p->h_xa, 2 * (size_t)na * sizeof(double)), "cudaMallocHost x_a/y_a");
    const int32_t* act = p->h_act.data();
    double* xa = p->h_xa;
    double* ya = p->h_xa + na;
#pragma omp parallel for schedule(dynamic, 2048) if (na > 16384)
    for (int64_t i = 0; i < na; ++i) xa[i] = x_host[act[i]];
    sttsv_status_t st0 = check_async(p);
    if (st0 != STTSV_OK) return st0;
    CUDA_TRY(cudaMemcpyAsync(p->d_xa, xa, (size_t)na * sizeof(double), cudaMemcpyHostToDevice, s), "H2D x_a");
    CUDA_TRY(launch_prologue(p->d_xa, nullptr, p->d_xa, p->d_xg, p->gs, p->ent.table_norm, na, p->d_ya, s),
             "prologue launch");
    sttsv_status_t st = apply_active(p, s, true);
    if (st != STTSV_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(ya, p->d_ya, (size_t)na * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H y_a");
    const int64_t n = p->n;
    // dynamic: a descheduled thread must not hold its share of the 8n bytes back (static
    // scheduling showed 1-5 ms outliers on a 0.32 ms call, tools/e2e_diag.py)
#pragma omp parallel for schedule(dynamic, 1) if (n > (1 << 20))
    for (int64_t c = 0; c < (n + 65535) / 65536; ++c) {
      const int64_t a = c * 65536, b = std::min<int64_t>(n, a + 65536);
      memset(y_host + a, 0, (size_t)(b - a) * sizeof(double));
    }
    CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
#pragma omp parallel for schedule(dynamic, 2048) if (na > 16384)
    for (int64_t i = 0; i < na; ++i) y_host[act[i]] = ya[i];
    return STTSV_OK;
  }
  if (!p->d_xhost) {
    CUDA_TRY(cudaMalloc(&p->d_xhost, 2 * bytes), "cudaMalloc e2e staging");
    p->d_yhost = p->d_xhost + p->n;
  }
  {
    CUDA_TRY(cudaMemcpyAsync(p->d_xhost, x_host, bytes, cudaMemcpyHostToDevice, s), "H2D x");
    sttsv_status_t st = sttsv_apply(p, p->d_xhost, p->d_yhost, s);
    if (st != STTSV_OK) return st;
  }
  CUDA_TRY(cudaMemcpyAsync(y_host, p->d_yhost, bytes, cudaMemcpyDeviceToHost, s), "D2H y");
  CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_power_iterate(sttsv_plan_t p, double* x, double* z, int iters, void* stream) {
  if (!p || !x) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  if (iters < 0) return fail(STTSV_ERR_INVALID_ARGUMENT, "iters < 0");
  if (p->N < 2) return fail(STTSV_ERR_INVALID_ARGUMENT, "power iteration needs rank >= 2");
  const size_t bytes = (size_t)p->n * sizeof(double);
  if (z && overlap(x, bytes, z, bytes)) return fail(STTSV_ERR_ALIAS, "x and z overlap");
  if (iters == 0) return STTSV_OK;
  DeviceGuard g(p->device);
  sttsv_status_t st = check_async(p);
  if (st != STTSV_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(launch_gather(x, p->d_act, p->d_xa, p->d_xg, p->gs, p->ent.table_norm, p->n_active, s), "gather launch");
  for (int it = 0; it < iters; ++it) {
    st = apply_active(p, s);
    if (st != STTSV_OK) return st;
    CUDA_TRY(launch_normalize(p->d_ya, p->d_xa, p->d_xg, p->gs, p->ent.table_norm, p->d_scratch, p->n_active, p->N, s), "normalize launch");
  }
  CUDA_TRY(cudaMemsetAsync(x, 0, bytes, s), "memset x");
  CUDA_TRY(launch_expand(p->d_xa, p->d_act, x, p->n_active, s), "expand x");
  if (z) {
    CUDA_TRY(cudaMemsetAsync(z, 0, bytes, s), "memset z");
    CUDA_TRY(launch_expand(p->d_ya, p->d_act, z, p->n_active, s), "expand z");
  }
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_hec(sttsv_plan_t p, double* x, double* z, double tau, int max_iters,
                                    double* lambda_min, double* lambda_max, int* iters_done, void* stream) {
  if (!p || !x || !lambda_min || !lambda_max || !iters_done) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  if (max_iters < 1) return fail(STTSV_ERR_INVALID_ARGUMENT, "max_iters < 1");
  if (!(tau >= 0.0)) return fail(STTSV_ERR_INVALID_ARGUMENT, "tau must be >= 0");
  if (p->N < 2) return fail(STTSV_ERR_INVALID_ARGUMENT, "HEC needs rank >= 2");
  const size_t bytes = (size_t)p->n * sizeof(double);
  if (z && overlap(x, bytes, z, bytes)) return fail(STTSV_ERR_ALIAS, "x and z overlap");
  DeviceGuard g(p->device);
  sttsv_status_t st = check_async(p);
  if (st != STTSV_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (!p->h_lambda) CUDA_TRY(cudaMallocHost(&p->h_lambda, 2 * sizeof(double)), "cudaMallocHost");
  double* d_lam = p->d_scratch + 2 * kNormalizeScratch;
  // Alg. 1: y = x0 (caller's, e.g. (1/n) 1); z = TTSV1(y)
  CUDA_TRY(launch_gather(x, p->d_act, p->d_xa, p->d_xg, p->gs, p->ent.table_norm, p->n_active, s), "gather launch");
  st = apply_active(p, s);
  if (st != STTSV_OK) return st;
  double lo = 0.0, hi = 0.0;
  int it = 0;
  while (it < max_iters) {
    // x = z^[1/(N-1)] / ||z^[1/(N-1)]||_1 ; z = TTSV1(x) ; lambda bracket of z ./ x^[N-1]
    CUDA_TRY(launch_normalize(p->d_ya, p->d_xa, p->d_xg, p->gs, p->ent.table_norm, p->d_scratch, p->n_active, p->N, s),
             "normalize launch");
    st = apply_active(p, s);
    if (st != STTSV_OK) return st;
    CUDA_TRY(launch_lambda(p->d_ya, p->d_xa, p->d_scratch, d_lam, p->n_active, p->N, s), "lambda launch");
    CUDA_TRY(cudaMemcpyAsync(p->h_lambda, d_lam, 2 * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H lambda");
    CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
    ++it;
    lo = p->h_lambda[0];
    hi = p->h_lambda[1];
    if ((hi - lo) / lo < tau) break;  // until (lambda_max - lambda_min) / lambda_min < tau
  }
  CUDA_TRY(cudaMemsetAsync(x, 0, bytes, s), "memset x");
  CUDA_TRY(launch_expand(p->d_xa, p->d_act, x, p->n_active, s), "expand x");
  if (z) {
    CUDA_TRY(cudaMemsetAsync(z, 0, bytes, s), "memset z");
    CUDA_TRY(launch_expand(p->d_ya, p->d_act, z, p->n_active, s), "expand z");
  }
  CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
  *lambda_min = lo;
  *lambda_max = hi;
  *iters_done = it;
  return STTSV_OK;
}

extern "C" sttsv_status_t sttsv_apply_batch(sttsv_plan_t p, const double* X, double* Y, int nvec, int64_t ld,
                                            void* stream) {
  if (!p || !X || !Y) return fail(STTSV_ERR_INVALID_ARGUMENT, "NULL argument");
  if (nvec < 1 || nvec > STTSV_MAX_BATCH) return fail(STTSV_ERR_INVALID_ARGUMENT, "nvec must be in [1, %d]", STTSV_MAX_BATCH);
  if (ld < p->n) return fail(STTSV_ERR_INVALID_ARGUMENT, "ld < n");
  if (p->batch_fused && p->det && nvec > 1)
    return fail(STTSV_ERR_UNSUPPORTED, "fused batched apply of a STTSV_DETERMINISTIC plan");
  const size_t span = ((size_t)(nvec - 1) * (size_t)ld + (size_t)p->n) * sizeof(double);
  if (overlap(X, span, Y, span)) return fail(STTSV_ERR_ALIAS, "X and Y overlap");
  DeviceGuard g(p->device);
  sttsv_status_t st = check_async(p);
  if (st != STTSV_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (!p->batch_fused) {
    // one single-vector pass per vector (faster on B200 while the single pass is
    // issue-bound; X and Y do not overlap)
    for (int v = 0; v < nvec; ++v) {
      st = apply_dense(p, X + (size_t)v * ld, Y + (size_t)v * ld, s);
      if (st != STTSV_OK) return st;
    }
    return STTSV_OK;
  }
  const int64_t na = p->n_active;
  if (p->batch_cap < nvec) {
    CUDA_TRY(cudaStreamSynchronize(s), "synchronize");
    if (p->batch_mem) CUDA_TRY(cudaFree(p->batch_mem), "cudaFree batch");
    p->batch_mem = nullptr;
    p->batch_cap = 0;
    const size_t a = ((size_t)nvec * na * 8 + 255) & ~(size_t)255;
    const size_t gbytes = ((size_t)nvec * na * p->gs * 8 + 255) & ~(size_t)255;
    const size_t pr = ((size_t)p->grid * p->kp.H * nvec * 8 + 8 + 255) & ~(size_t)255;
    const size_t gt = (size_t)nvec * p->gtab_doubles * 8 + 8;  // per-vector group tables (prefix.cuh)
    CUDA_TRY(cudaMalloc(&p->batch_mem, 2 * a + gbytes + pr + gt), "cudaMalloc batch workspace");
    char* b = (char*)p->batch_mem;
    p->b_xa = (double*)b;
    p->b_ya = (double*)(b + a);
    p->b_xg = (double*)(b + 2 * a);
    p->b_priv = (double*)(b + 2 * a + gbytes);
    p->b_gtab = (double*)(b + 2 * a + gbytes + pr);
    p->batch_cap = nvec;
  }
  // the zero-fill of the dense outputs (8n bytes per vector) on the side stream,
  // overlapping the edge kernel (as apply_dense)
  const bool fork = p->kp.num_tiles > 0;
  if (fork) {
    if (!p->side) {
      CUDA_TRY(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking), "side stream");
      CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "event");
      CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming), "event");
    }
    CUDA_TRY(cudaEventRecord(p->ev_fork, s), "fork record");
    CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0), "fork wait");
  }
  CUDA_TRY(cudaMemset2DAsync(Y, (size_t)ld * sizeof(double), 0, (size_t)p->n * sizeof(double), (size_t)nvec,
                             fork ? p->side : s), "memset Y");
  if (fork) CUDA_TRY(cudaEventRecord(p->ev_join, p->side), "join record");
  for (int v = 0; v < nvec; ++v)
    CUDA_TRY(launch_gather(X + (size_t)v * ld, p->d_act, p->b_xa + (size_t)v * na, p->b_xg + (size_t)v * na * p->gs,
                           p->gs, p->ent.table_norm, na, s), "gather launch");
  if (na > 0) {
    CUDA_TRY(cudaMemsetAsync(p->b_ya, 0, (size_t)nvec * na * sizeof(double), s), "memset y_a");
    if (p->m0_chunks > 0) CUDA_TRY(launch_m0(p, s), "m0sum launch");
    if (p->kp.num_tiles > 0) {
      EdgeKernelParams kp = p->kp;
      kp.nvec = nvec;
      kp.xa = p->b_xa;
      kp.xg = p->b_xg;
      kp.xg_vstride = na * p->gs;
      kp.ya = p->b_ya;
      kp.ya_vstride = na;
      kp.priv = p->b_priv;
      // shared-prefix memo: one group table per vector (prefix.cuh)
      const bool groups = p->kp.gtab != nullptr;
      if (groups) {
        for (int v = 0; v < nvec; ++v)
          CUDA_TRY(launch_groups(p->b_xg + (size_t)v * na * p->gs, p->gs, p->N, p->d_gku, p->d_goff, p->d_items,
                                 p->nitems, p->group_lmax, p->kp.gtab, p->b_gtab + (size_t)v * p->gtab_doubles, s),
                   "group kernel launch");
        kp.gtab = p->b_gtab;
        kp.gtab_vstride = p->gtab_doubles;
      }
      kp.group_wait = groups;
      CUDA_TRY(launch_edge_kernel(p->ent, kp, p->grid, p->smem, s, nvec > 1 ? 1 : (p->det ? 2 : 0), groups),
               "edge kernel launch");
      if (p->det) CUDA_TRY(launch_det_reduce(p->d_contrib, p->d_cstart, p->det_chunks, p->d_csum, p->d_vchunk,
                                             p->b_ya, na, s), "deterministic reduce launch");
    }
    if (p->comm) {
      NcclApi* api = nccl_api();
      ncclResult_t r = api->AllReduce(p->b_ya, p->b_ya, (size_t)nvec * na, ncclFloat64, ncclSum, p->comm->comm, s);
      if (r != ncclSuccess) return fail(STTSV_ERR_NCCL, "ncclAllReduce: %s", api->GetErrorString(r));
      ++p->allreduces;
    }
  }
  if (fork) CUDA_TRY(cudaStreamWaitEvent(s, p->ev_join, 0), "join wait");
  for (int v = 0; v < nvec; ++v) {
    CUDA_TRY(launch_expand(p->b_ya + (size_t)v * na, p->d_act, Y + (size_t)v * ld, na, s), "expand launch");
  }
  return STTSV_OK;
}
