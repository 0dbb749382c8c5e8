/* sttsv.h — C ABI of the B200 STTSV library (libsttsv.so).
 *
 * STTSV on the blowup tensor of a weighted non-uniform hypergraph
 * (arXiv 2311.08595; PAPER.md = /root/reference/PAPER.md of the build):
 *
 *   s = B x^{N-1},   s_{i1} = sum_{i2..iN} B_{i1..iN} prod_{k=2..N} x_{ik}
 *        PAPER.md:335-337 (§II, Eq. (2)); PAPER.md:326-333 (Eq. (1)).
 *   B, the order-N blowup tensor: for each hyperedge e and each ordered
 *        N-tuple i in beta(e) (tuples over e whose support is exactly e),
 *        B_i = w(e)/|beta(e)|;  PAPER.md:341-343 (§II).
 *   |beta(e)| = |e|! S(N,|e|), the footnote at PAPER.md:342.
 *
 * Only the IOU (sorted-index) hyperedges are stored (PAPER.md:406 footnote).
 * The library evaluates, per edge e and member v, Alg. 2's coefficient
 * (line "c += w(e)/|beta(e)| (N-1)! E_N(b_v) * (*_{u in e\v} Ebar_N(b_u))[N-1]")
 * with a per-edge DP on shifted series, then reduces the
 * contributions into s.  Everything after sttsv_plan_create runs in CUDA
 * kernels on the plan's device; there is no CPU fallback.
 *
 * Conventions for every call:
 *  - Return value: STTSV_OK or an sttsv_status_t error; no exception or
 *    abort crosses the ABI.  On error sttsv_last_error() returns a
 *    thread-local, human-readable detail string (valid until the next call
 *    from the same thread).
 *  - Vertex ids are 0-based int32 in [0, n).  Vectors x, y, z are fp64,
 *    length n, dense.
 *  - "device pointer" means memory on the plan's CUDA device (e.g. a torch
 *    CUDA tensor's data_ptr); "host pointer" means CPU memory (pinned or
 *    pageable).  The caller owns every pointer it passes.
 *  - Streams are passed as void* holding a cudaStream_t (NULL = the legacy
 *    default stream).  Calls taking a stream are stream-ordered and return
 *    before the GPU work finishes; asynchronous CUDA/NCCL faults surface as
 *    STTSV_ERR_CUDA / STTSV_ERR_NCCL on a later call.
 */
#ifndef STTSV_H
#define STTSV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Largest supported rank N_k (tensor order).  The paper's datasets reach
 * 26 (R6); its synthetic S4 reaches 60. */
#define STTSV_MAX_RANK 32

typedef struct sttsv_plan_s* sttsv_plan_t;
typedef struct sttsv_comm_s* sttsv_comm_t;

typedef enum {
  STTSV_OK = 0,
  STTSV_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, n < 1, num_edges < 0, rank_Nk out of [1, STTSV_MAX_RANK],
                                     world/rank inconsistent, iters < 0                              */
  STTSV_ERR_EDGE_SIZE = 2,        /* sizes[e] < 1 or sizes[e] > rank_Nk                                */
  STTSV_ERR_VERTEX_RANGE = 3,     /* an index < 0 or >= n                                              */
  STTSV_ERR_UNSORTED = 4,         /* an edge's ids not strictly increasing (IOU form)
                                     and STTSV_CANONICALIZE not set                                    */
  STTSV_ERR_REPEATED_VERTEX = 5,  /* the same id twice in one edge (a hyperedge is a set)             */
  STTSV_ERR_NONFINITE = 6,        /* a weight is NaN or infinite                                       */
  STTSV_ERR_ALIAS = 7,            /* input and output vectors overlap                                 */
  STTSV_ERR_CUDA = 8,             /* a CUDA runtime error (detail in sttsv_last_error)               */
  STTSV_ERR_NCCL = 9,             /* an NCCL error, or NCCL could not be loaded                       */
  STTSV_ERR_OUT_OF_MEMORY = 10,   /* host or device allocation failed                                  */
  STTSV_ERR_UNSUPPORTED = 11      /* a flag or mode this build does not implement                     */
} sttsv_status_t;

/* plan flags */
enum {
  STTSV_CANONICALIZE = 1u << 0,     /* sort each edge's ids instead of rejecting unsorted edges;
                                       repeated ids are still an error                             */
  STTSV_MERGE_DUPLICATES = 1u << 1, /* merge identical vertex sets of a shard, summing their weights
                                       (B is linear in w); the plan stores fewer edges */
  STTSV_DETERMINISTIC = 1u << 2,    /* bit-reproducible y: each contribution is stored to a
                                       plan-time slot of a vertex-major buffer and summed in a fixed order
                                       (no atomics); costs ~12 B more per incidence per apply, needs
                                       < 2^31 incidences per shard; not with STTSV_BATCH_FUSED nvec > 1 */
  STTSV_BATCH_FUSED = 1u << 3,      /* sttsv_apply_batch runs ONE pass over the hyperedge stream for all
                                       vectors (the fused batch kernel) instead of one sttsv_apply pass
                                       per vector; see sttsv_apply_batch for when each is faster       */
  STTSV_NO_PREFIX_MEMO = 1u << 4    /* turn off the shared-prefix memo: every
                                       edge runs its full per-edge DP and streams all its ids (for A/B
                                       measurements; the memo is on by default)                        */
};

/* ------------------------------------------------------------------ plans */

/* sttsv_plan_create — build the device hyperedge store for B.
 *
 *  out       [out] receives the plan handle; *out is NULL on error.
 *  n         number of vertices (>= 1); x, y have length n.
 *  rank_Nk   tensor order N (global for every edge, reading A3 of DESIGN.md);
 *            must be >= max |e| and <= STTSV_MAX_RANK.
 *  num_edges number of hyperedges m (>= 0).
 *  sizes     host int32[m]: |e| of each edge, 1 <= |e| <= rank_Nk.
 *  indices   host int32[sum sizes]: member ids of each edge, concatenated in
 *            edge order, each edge strictly increasing (IOU) unless
 *            STTSV_CANONICALIZE.
 *  weights   host fp64[m]: w(e), finite; NULL means w(e) = |e|
 *            (which makes B 1^{N-1} the degree vector).
 *  device    CUDA device ordinal the plan lives on.
 *  world     number of edge shards (>= 1); rank in [0, world).  The plan keeps
 *            shard `rank`: slice [m_k*rank/world, m_k*(rank+1)/world) of every
 *            cardinality bucket k, in input order.  Every rank must pass the
 *            same full edge list.
 *  comm      NULL, or a communicator from sttsv_comm_create with the same
 *            world/rank: every sttsv_apply (and every power / HEC step) then
 *            all-reduces the active part of y over NCCL (one ncclAllReduce,
 *            also at world = 1) so every rank returns the full s.  With
 *            world > 1 and comm == NULL, sttsv_apply returns only this
 *            shard's partial sum.
 *  flags     STTSV_CANONICALIZE, STTSV_MERGE_DUPLICATES, STTSV_DETERMINISTIC.
 *
 * The host arrays are copied; the caller may free them on return.  The plan
 * owns all its device memory until sttsv_plan_destroy.  A plan is immutable
 * after creation but holds apply workspaces: do not run two applies on the
 * same plan concurrently.  Errors: INVALID_ARGUMENT, EDGE_SIZE, VERTEX_RANGE,
 * UNSORTED, REPEATED_VERTEX, NONFINITE, UNSUPPORTED, CUDA, OUT_OF_MEMORY. */
sttsv_status_t sttsv_plan_create(sttsv_plan_t* out, int64_t n, int32_t rank_Nk, int64_t num_edges,
                                 const int32_t* sizes, const int32_t* indices, const double* weights,
                                 int device, int world, int rank, sttsv_comm_t comm, uint32_t flags);

/* sttsv_destroy — release the plan and its device memory (waits for its
 * pending work).  NULL is accepted and ignored.  (north_star's name;
 * sttsv_plan_destroy is the same call under its round-1 name.) */
sttsv_status_t sttsv_destroy(sttsv_plan_t plan);
sttsv_status_t sttsv_plan_destroy(sttsv_plan_t plan);

/* sttsv_apply — y = B x^{N-1} (Eq. (2)).
 *  x_dev  device fp64[n], read only.
 *  y_dev  device fp64[n], overwritten (vertices in no local edge get exact 0
 *         on a single shard).  Must not overlap x_dev (STTSV_ERR_ALIAS).
 *  stream cudaStream_t as void*.
 * With a comm the result is identical on all ranks (allreduce semantics). */
sttsv_status_t sttsv_apply(sttsv_plan_t plan, const double* x_dev, double* y_dev, void* stream);

/* sttsv_apply_batch — Y_v = B X_v^{N-1} for nvec vectors.
 *  X_dev  device fp64, vector v at X_dev + v*ld (length n), read only.
 *  Y_dev  device fp64, same layout, overwritten; must not overlap X_dev.
 *  nvec   1 .. STTSV_MAX_BATCH;  ld >= n.
 * Two strategies, chosen by the plan's STTSV_BATCH_FUSED flag:
 *  - default: one sttsv_apply pass per vector (the edge stream is re-read per
 *    vector).  On B200 the single-vector edge kernel is issue/FP64-bound, not
 *    HBM-bound, so this is the faster one on every measured
 *    configuration; any plan, including STTSV_DETERMINISTIC.
 *  - STTSV_BATCH_FUSED: the hyperedge stream is read ONCE for all vectors; each
 *    vector's DP and scatter run in turn on the staged tile (per-tile run
 *    flushes).  Pays only where the single pass is HBM-bound.  The first call
 *    with a larger nvec allocates a workspace (and synchronises the stream);
 *    with a comm, one allreduce of all vectors' active parts; not with
 *    STTSV_DETERMINISTIC and nvec > 1 (UNSUPPORTED).
 * Stream-ordered like sttsv_apply.  Errors: INVALID_ARGUMENT, ALIAS, UNSUPPORTED,
 * CUDA, NCCL, OUT_OF_MEMORY. */
#define STTSV_MAX_BATCH 16
sttsv_status_t sttsv_apply_batch(sttsv_plan_t plan, const double* X_dev, double* Y_dev, int nvec, int64_t ld,
                                 void* stream);

/* sttsv_apply_host — the same product from HOST vectors, synchronous.  When the
 * active set is sparse (n_active <= n/8) only the active parts cross PCIe: x is
 * gathered on the host into a pinned buffer (n_active doubles in), y_a comes
 * back (n_active doubles out) and the host zero-fills y (overlapping the GPU
 * work) and scatters y_a into it.  Otherwise x and y (fp64[n]) are copied in
 * full.  Host buffers may be pageable. */
sttsv_status_t sttsv_apply_host(sttsv_plan_t plan, const double* x_host, double* y_host);

/* sttsv_power_iterate — the x-update of Alg. 1 (NQZ, PAPER.md:351-355 lines 3-6),
 * reading A14 of DESIGN.md: starting from x = x_dev (device fp64[n], e.g. (1/n)1),
 * repeat `iters` times { z = B x^{N-1};  x = z^[1/(N-1)] / ||z^[1/(N-1)]||_1 }.
 * On return x_dev holds x_iters and z_dev (device fp64[n], may be NULL) holds
 * z_iters.  Vertices in no edge get x = z = 0.  With a comm each step costs one
 * allreduce of the active part of z.  Requires N >= 2 and iters >= 0. */
sttsv_status_t sttsv_power_iterate(sttsv_plan_t plan, double* x_dev, double* z_dev, int iters, void* stream);

/* sttsv_hec — H-eigenvector centrality by the NQZ iteration, Alg. 1 of the
 * paper, with the lambda bracket of lines 8-9:
 *   y = x_dev (on entry: x_0, e.g. (1/n) 1, line 3);  z = B y^{N-1} (line 4);
 *   repeat:  x = z^[1/(N-1)] / ||z^[1/(N-1)]||_1   (line 6)
 *            z = B x^{N-1}                          (line 7)
 *            lambda_min = min(z ./ x^[N-1]),  lambda_max = max(z ./ x^[N-1])   (lines 8-9)
 *   until (lambda_max - lambda_min) / lambda_min < tau  or  max_iters repetitions.
 * Min/max run over vertices with x_v^(N-1) > 0 (reading A15 of DESIGN.md:
 * isolated vertices have x_v = 0; powers that underflow are excluded).  On return x_dev (device fp64[n]) holds x, z_dev
 * (device fp64[n] or NULL) the last z, *lambda_min / *lambda_max the last
 * bracket and *iters_done the repetitions run.  Synchronous: the host reads the
 * bracket after every repetition.  tau >= 0 (0 runs exactly max_iters);
 * max_iters >= 1; N >= 2.  With a comm each STTSV costs one allreduce. */
sttsv_status_t sttsv_hec(sttsv_plan_t plan, double* x_dev, double* z_dev, double tau, int max_iters,
                         double* lambda_min, double* lambda_max, int* iters_done, void* stream);

/* Plan introspection (host values; no device work). */
typedef struct {
  int64_t n;               /* vertex count                                               */
  int32_t rank_Nk;         /* tensor order N                                             */
  int32_t world, rank;     /* shard of this plan                                         */
  int64_t num_edges;       /* input edges of this shard                                  */
  int64_t incidences;      /* sum of |e| over this shard's input edges                   */
  int64_t stored_edges;    /* edges the plan stores (< num_edges with MERGE_DUPLICATES)  */
  int64_t stored_incidences; /* sum of |e| over the stored edges                         */
  int64_t total_edges;     /* edges in the full input                                    */
  int64_t total_incidences;/* sum of |e| over the full input                             */
  int64_t n_active;        /* vertices of degree >= 1 in the full input                  */
  int64_t edges_per_size[STTSV_MAX_RANK + 1]; /* this shard's input edges of each size     */
  int64_t device_bytes;    /* device memory owned by the plan                            */
  int64_t stream_bytes;    /* bytes of the edge stream one apply reads (ids + weights, incl. tile padding) */
  double  fma_per_apply;   /* FP64 fused multiply-adds of the per-edge DP per apply      */
  int32_t hot_private;     /* slots 0..T-1 of every edge accumulate in per-lane register runs */
  int32_t hot_shared;      /* H: ids below H accumulate in per-CTA L2 slices            */
  int32_t kernel_grid;     /* CTAs of the edge kernel                                    */
  int32_t kernel_block;    /* threads per CTA of the edge kernel                         */
  int32_t id_bytes;        /* bytes per member id in the edge stream: 2 when n_active <= 65536
                              on ranks <= 12, else 4                                      */
  int64_t allreduces;      /* ncclAllReduce calls this plan has issued (0 without a comm) */
  double  fma_executed;    /* FP64 operations the edge kernel executes per apply: fma_per_apply minus
                              what the shared-prefix memo saves                 */
  int64_t prefix_tiles;    /* warp blocks (num_tiles x consumer warps in all) whose edges share a member
                              prefix; the columns every block of a tile shares are not streamed    */
  int64_t prefix_groups;   /* runs of consecutive such blocks with the same prefix                 */
  int64_t prefix_incidences; /* incidences that lie in a shared prefix                            */
  int64_t num_tiles;       /* tiles of the edge stream                                            */
  int64_t m0_edges;        /* edges in warp blocks of one repeated vertex set (M = 0): not in the tile
                              stream; their prefix members get C_i[0] x (sum of w') per apply     */
  int64_t m0_groups;       /* distinct vertex sets of those blocks                                */
  int64_t m0_chunks;       /* chunks of their stored weights summed per apply (non-uniform weights) */
} sttsv_plan_info_t;

sttsv_status_t sttsv_plan_info(sttsv_plan_t plan, sttsv_plan_info_t* info);

/* Number of launches of the library's own kernels one sttsv_apply issues
 * (memsets and NCCL calls excluded). */
int sttsv_apply_launches(sttsv_plan_t plan);

/* Edge-kernel timing for roofline reports.  sttsv_plan_profile(plan, 1)
 * clears previous samples and makes every later apply / power-iteration step
 * record a CUDA event pair around its edge kernel on the launching stream;
 * (plan, 0) stops recording.  sttsv_plan_profile_read synchronises on the
 * recorded events and returns the summed edge-kernel time (ms) and the number
 * of timed launches. */
sttsv_status_t sttsv_plan_profile(sttsv_plan_t plan, int enable);
sttsv_status_t sttsv_plan_profile_read(sttsv_plan_t plan, double* total_ms, int64_t* launches);

/* Host-only helper: which edges shard `rank` of `world` owns under the rule of
 * sttsv_plan_create.  out_edges (host int64[num_edges]) receives the owned
 * input edge indices, bucket by bucket (k ascending) in input order; *out_count
 * their number.  sizes as in sttsv_plan_create (validated only for range). */
sttsv_status_t sttsv_shard_edges(int64_t num_edges, const int32_t* sizes, int32_t rank_Nk, int world,
                                 int rank, int64_t* out_edges, int64_t* out_count);

/* ------------------------------------------------------- communicators
 * NCCL is loaded at run time (libnccl.so.2).  Rank 0 calls
 * sttsv_comm_unique_id, the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed), then every rank calls sttsv_comm_create. */
sttsv_status_t sttsv_comm_unique_id(unsigned char id[128]);
sttsv_status_t sttsv_comm_create(sttsv_comm_t* out, const unsigned char id[128], int world, int rank,
                                 int device);
sttsv_status_t sttsv_comm_destroy(sttsv_comm_t comm);

/* ------------------------------------------------------------ errors */
const char* sttsv_status_string(sttsv_status_t status);
const char* sttsv_last_error(void);

/* Library version string and the CUDA architecture it was built for. */
const char* sttsv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STTSV_H */
