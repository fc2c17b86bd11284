/*
 * sg2v.h — C ABI of libsg2v.so: the B200 colour-coding hot path of
 * SubGraph2Vec (arXiv:2009.11665).
 *
 * Citations: P:n = PAPER.md line n (section / algorithm in brackets),
 * S:n = SPEC.md line n, SURVEY §x = SURVEY.md section.
 *
 * Problem (P:119-126 [§II-B]): count the non-induced embeddings emb(T,G) of
 * a k-vertex tree template T in a simple undirected graph G by colour coding.
 * For each colouring j = 0..N-1 the library computes the exact number of
 * colourful injective homomorphisms of T into G,
 *     colorful_j = Σ_i Σ_C M_0(i, I_C)                 (P:154, P:461 [Alg. 1, 5])
 * by the two-stage DP of Alg. 3/5: per sub-template
 * split, B = A_G·M_p (SpMM) and M_s(:,I_s) += M_a(:,I_a) ⊙ B(:,I_p)
 * (eMA), and the estimate
 *     estimate = mean_j colorful_j / (P·α),  P = k!/k^k, α = |Aut(T)|
 *
 * Conventions for every entry point:
 *  - Return value: SG2V_OK or an error code; on error sg2v_last_error()
 *    returns a thread-local, human-readable message.  No C++ exception ever
 *    crosses this boundary.
 *  - Ownership: the caller owns every array it passes; the library copies what
 *    it keeps before returning.  Opaque handles are owned by the library and
 *    released with the matching *_free.  Output arrays are caller-allocated.
 *  - Device: every GPU call runs on options.device (default: the current
 *    device) and options.stream (default: the legacy default stream).  There is
 *    no CPU fallback: without a usable sm_100 device GPU calls return SG2V_ECUDA.
 */
#ifndef SG2V_H
#define SG2V_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sg2v_graph sg2v_graph;       /* device CSR + processing order       */
typedef struct sg2v_template sg2v_template; /* validated tree, α, P, cached plans   */

typedef enum {
    SG2V_OK = 0,
    SG2V_EINVAL = 1,    /* bad argument / malformed CSR / k out of range          */
    SG2V_ENOTTREE = 2,  /* template is not a tree on vertices 0..k-1             */
    SG2V_ENOMEM = 3,    /* workspace would exceed the memory budget (no alloc)   */
    SG2V_ECUDA = 4,     /* CUDA runtime / launch failure, or no sm_100 device    */
    SG2V_ENCCL = 5,     /* NCCL / all-gather transport failure (mode 1)          */
    SG2V_EOVERFLOW = 6  /* F32 result not finite (values are still written)      */
} sg2v_status;

/* Arithmetic of the count tables (P:815-818 uses fp32; SURVEY §8(c) "Precision").
 *  F32: tables in binary32, per-vertex top values and the Σ_i reduction in fp64.
 *  F64: binary64 throughout; bit-exact while every intermediate < 2^53.
 *  U64: exact residues mod 2^64 (a ring homomorphism of the integer DP).      */
typedef enum { SG2V_F32 = 0, SG2V_F64 = 1, SG2V_U64 = 2 } sg2v_precision;

/* Flags for sg2v_graph_load_csr. */
#define SG2V_GRAPH_VALIDATE 1u    /* check sorted rows, no self-loops, symmetric   */
#define SG2V_GRAPH_DEVICE_PTRS 2u /* row_offsets / col_indices are device pointers */

/*
 * sg2v_graph_load_csr — A_G of P:357 [§V-A] ("A_G(i,j) = 1 iff V_j ∈ N(V_i)").
 *   n            number of vertices (0 <= n < 2^31).
 *   row_offsets  int64[n+1], row_offsets[0] = 0, non-decreasing, [n] = nnz.
 *   col_indices  int32[nnz], neighbours of row i in [row_offsets[i], row_offsets[i+1]),
 *                sorted ascending, no self-loops, symmetric (undirected).
 *   flags        SG2V_GRAPH_VALIDATE checks the CSR invariants on the device
 *                (EINVAL on violation); SG2V_GRAPH_DEVICE_PTRS means both
 *                arrays are device pointers on the options device (copied
 *                device-to-device), otherwise they are host pointers.
 *   out          receives the handle (free with sg2v_graph_free).
 * The library uploads the CSR and builds a degree-descending processing order
 * for its row-owner kernels (heavy rows first).
 */
sg2v_status sg2v_graph_load_csr(int64_t n, const int64_t *row_offsets,
                                const int32_t *col_indices, int64_t nnz,
                                uint32_t flags, sg2v_graph **out);
void sg2v_graph_free(sg2v_graph *g);

/*
 * sg2v_template_build — the template T (P:162-170 [§II-C-2]).
 *   k          number of template vertices, 1 <= k <= 31; the number of
 *              colours equals k ("we consider k=|V_T|").
 *   edges      int32[2*(k-1)], (u,v) pairs over vertex ids 0..k-1 (NULL if k=1).
 *   root_hint  -1: the planner chooses the root ρ and cut order (the count is
 *              independent of both, SURVEY finding 1); otherwise forces ρ.
 * Errors: EINVAL (k out of range, bad root_hint), ENOTTREE (ids out of range,
 * self-loop, duplicate edge, cycle or disconnected).
 */
sg2v_status sg2v_template_build(int32_t k, const int32_t *edges, int32_t root_hint,
                                sg2v_template **out);
void sg2v_template_free(sg2v_template *t);

/* α = |Aut(T)| of the unrooted tree (reading in SURVEY §8(c)), P = k!/k^k. */
sg2v_status sg2v_template_info(const sg2v_template *t, int32_t *k, double *alpha,
                               double *colorful_probability);

typedef struct {
    sg2v_precision precision; /* default SG2V_F32                                   */
    int64_t iter_offset;      /* colouring index of the first colouring (default 0) */
    int64_t iter_stride;      /* colouring t of the call is j = iter_offset +
                                 t*iter_stride (default 1; replica sharding)        */
    int32_t mode;             /* 0 = replicas / single GPU, 1 = vertex partition       */
    void *nccl_comm;          /* mode 1: the sg2v_comm of this rank                  */
    int32_t device;           /* CUDA ordinal; -1 = current device                   */
    uint64_t mem_budget_bytes;/* planning budget: the planner picks the fastest plan
                                 whose workspace fits; 0 = device memory minus 6 GiB
                                 (unlimited for host-only planning).  sg2v_count also
                                 refuses (ENOMEM) a library-allocated workspace larger
                                 than the free device memory                         */
    int32_t col_tile;         /* mode 1: column tile width in elements (0 = auto)    */
    void *stream;             /* cudaStream_t (e.g. torch's current stream); NULL =
                                 legacy default stream                               */
    void *workspace;          /* caller-owned device buffer (>= sg2v_workspace_bytes)
                                 or NULL: the library allocates and frees its own    */
    uint64_t workspace_bytes;
    void *row_values;         /* optional device array[n]: per-vertex Σ_C M_0(i,I_C)
                                 of the LAST colouring of the call (double for
                                 F32/F64, uint64 for U64)                            */
    int32_t layout;           /* count-table layout: 0 = root-colour anchored
                                 (default; rows hold only colour sets containing
                                 c(i), C(k-1,s-1) columns), where
                                 the planner may store a table read only as a
                                 passive child as k-1 per-consumer-colour segments
                                 of C(k-2,s-1) sets ("exclusion-projected", more
                                 memory, fewer gathered bytes),
                                 1 = dense n x C(k,s) as in P:227,
                                 2 = anchored without projected tables,
                                 3 = anchored with every eligible table projected
                                     (as far as the budget allows; tests).
                                 Same results in every layout. */
} sg2v_options;

void sg2v_options_default(sg2v_options *o);
/* Thread-local defaults used by sg2v_count. */
sg2v_status sg2v_set_options(const sg2v_options *o);

/* Device bytes sg2v_count needs for (g, t, precision): all count tables live
 * at the peak of the planned schedule + colours + histogram + row values.
 * sg2v_workspace_bytes and sg2v_plan_describe* plan for the layout of the
 * thread-local options (sg2v_set_options). */
sg2v_status sg2v_workspace_bytes(const sg2v_graph *g, const sg2v_template *t,
                                 sg2v_precision precision, uint64_t *bytes);

/*
 * sg2v_count — the colour-coding estimator (Alg. 1 / Alg. 5).
 *   k                 must equal the template's k (EINVAL otherwise).
 *   n_iter            number of colourings N >= 1 (EINVAL otherwise).
 *   seed              colouring j colours vertex v with COLOR(seed, j, v, k)
 *                     (counter hash of SURVEY §8(c) step 1; a pure function of
 *                     (seed, j, v), so shards reproduce 1-GPU values exactly).
 *   estimate_out      mean_t colorful_t/(P·α); NaN in U64 mode.  May be NULL.
 *   colorful_out      double[n_iter] (F32/F64) or NULL.
 *   colorful_u64_out  uint64[n_iter], residues mod 2^64 (U64 mode) or NULL.
 * Uses the thread-local options of sg2v_set_options.  Synchronises the stream
 * before returning.  EOVERFLOW: some F32 colourful count is not finite.
 * ENOMEM: the planned peak exceeds the budget (required bytes in last_error),
 * detected before any allocation.
 */
sg2v_status sg2v_count(const sg2v_graph *g, const sg2v_template *t, int32_t k,
                       int64_t n_iter, uint64_t seed, double *estimate_out,
                       double *colorful_out, uint64_t *colorful_u64_out);
/* As sg2v_count with explicit options (NULL = thread-local defaults). */
sg2v_status sg2v_count_ex(const sg2v_graph *g, const sg2v_template *t, int32_t k,
                          int64_t n_iter, uint64_t seed, const sg2v_options *o,
                          double *estimate_out, double *colorful_out,
                          uint64_t *colorful_u64_out);

/*
 * sg2v_estimate — a7 for colourful counts gathered elsewhere (replica shards,
 * SURVEY §8(e) R): estimate_out = (Σ_q colorful[q]) / n_iter / (P·α), summed in
 * index order (deterministic), P = k!/k^k, α = |Aut(T)| of t (Alg. 1
 * last line).  colorful: host double[n_iter] (F32/F64 counts).  EINVAL for NULL
 * pointers or n_iter < 1; EOVERFLOW if a count is not finite (estimate written).
 */
sg2v_status sg2v_estimate(const sg2v_template *t, int64_t n_iter, const double *colorful,
                          double *estimate_out);

/*
 * sg2v_count_batch — m templates of the same size k on the SAME colourings
 * (treelet distributions, Fig. 1): the colouring and the
 * colour buckets / histogram are computed once per colouring and shared, then
 * each template's DP runs in turn in one workspace (tables of consecutive
 * templates reuse the same arena).
 *   templates      array of m template handles, all with k vertices (EINVAL otherwise)
 *   estimates_out  double[m] or NULL;  colorful_out / colorful_u64_out:
 *                  [m * n_iter], template-major (entry t*n_iter + q), or NULL.
 * Values are identical to m separate sg2v_count calls with the same options.
 */
sg2v_status sg2v_count_batch(const sg2v_graph *g, const sg2v_template *const *templates, int32_t m,
                             int32_t k, int64_t n_iter, uint64_t seed, const sg2v_options *o,
                             double *estimates_out, double *colorful_out,
                             uint64_t *colorful_u64_out);
/* Workspace bytes of sg2v_count_batch (thread-local layout / budget options). */
sg2v_status sg2v_workspace_bytes_batch(const sg2v_graph *g, const sg2v_template *const *templates,
                                       int32_t m, sg2v_precision precision, uint64_t *bytes);

/*
 * Vertex-partitioned mode (SURVEY §8(e) "V": capacity for tables larger than one
 * GPU).  Rank r of W owns rows [r*nl, r*nl + n_local) of G and of every count
 * table, nl = ceil(n_global / W).  Each SpMM step all-gathers the passive table
 * in column tiles (options.col_tile elements; 0 = ~2 GB staging) and every rank
 * pushes its own rows' colour-bucket sums; the eMA and the top step are row-local;
 * the per-rank Σ_i are all-gathered and summed in rank order.  Select it with
 * options.mode = 1 and options.nccl_comm = an sg2v_comm (anchored layout, one
 * template per call).  Values equal the single-GPU ones (exact in U64).
 */
typedef struct sg2v_comm sg2v_comm;
/* host all-gather: recv[r*bytes .. (r+1)*bytes) = rank r's send (returns 0 on success) */
typedef int32_t (*sg2v_allgather_fn)(const void *send, void *recv, uint64_t bytes, void *user);
/* NCCL transport (one process per GPU): rank 0 creates the id, the caller
 * broadcasts its 128 bytes (e.g. torch.distributed), every rank calls init. */
sg2v_status sg2v_comm_unique_id(uint8_t id_out[128]);
sg2v_status sg2v_comm_init_nccl(const uint8_t id[128], int32_t rank, int32_t world, sg2v_comm **out);
/* Host-callback transport (tests: gloo, several processes on one GPU). */
sg2v_status sg2v_comm_init_callback(int32_t rank, int32_t world, sg2v_allgather_fn fn, void *user,
                                    sg2v_comm **out);
void sg2v_comm_free(sg2v_comm *c);
/* Rows [row_begin, row_begin + n_local) of an n_global-vertex graph: row_offsets
 * int64[n_local+1] starting at 0, col_indices int32[nnz] GLOBAL ids (sorted per
 * row, no self-loops, symmetric as a whole graph).  Host or device pointers as in
 * sg2v_graph_load_csr (VALIDATE is not available per partition). */
sg2v_status sg2v_graph_load_partition(int64_t n_global, int64_t row_begin, int64_t n_local,
                                      const int64_t *row_offsets, const int32_t *col_indices,
                                      int64_t nnz, uint32_t flags, sg2v_graph **out);

/*
 * Balanced relabelling for the vertex-partitioned mode ("blocks balanced
 * by nnz + n·c_max weight, after a random relabel; colours stay keyed by the input id").
 * Blocks keep the contract above (rank r owns new ids [r·nl, r·nl + n_local)); the
 * vertices are dealt to the blocks by degree, heaviest first, in snake order, so every
 * block holds ~nnz/world edges (the n·c_max table term is equal by construction).
 *   n, row_offsets[n+1], col_indices[nnz]  the input CSR (host)
 *   old_of_new[n]   out: input id of new vertex u
 *   ro_out[n+1], ci_out[nnz]  out: the relabelled CSR (rows sorted)
 * Pass old_of_new (the slice-independent map) to sg2v_graph_set_vertex_ids of every
 * rank's partition so colours, hence every count, equal the input graph's.
 */
sg2v_status sg2v_partition_relabel(int64_t n, const int64_t *row_offsets, const int32_t *col_indices, int32_t world,
                                   int32_t *old_of_new, int64_t *ro_out, int32_t *ci_out);

/*
 * Vertex ids for colouring (P:150 leaves the RNG open; SURVEY §8(c) "RNG": colours are
 * keyed by the INPUT vertex id, so a relabelled graph must carry the original ids):
 * vertex v of g is coloured COLOR(seed, j, orig_ids[v], k).  count = n, or n_global
 * for a partition (host array, copied).  count = 0 clears the map.
 */
sg2v_status sg2v_graph_set_vertex_ids(sg2v_graph *g, const int32_t *orig_ids, int64_t count);

/*
 * sg2v_colorize — kernel a1 alone: writes
 * COLOR(seed, j, v, k) for v in [0,n) to the DEVICE array colors_out (uint8[n])
 * on `stream` (cudaStream_t or NULL).  For parity tests of the colouring.
 */
sg2v_status sg2v_colorize(uint64_t seed, int64_t j, int64_t n, int32_t k,
                          uint8_t *colors_out, void *stream);

/*
 * sg2v_plan_describe — JSON text of the plan chosen for (g, t, precision):
 * root, schedule, per-step sizes (s, a, p), kernel kind, column counts and
 * the algorithmic bytes / eMA terms of each step.
 * Writes at most buf_len bytes (NUL-terminated); *needed = full length + 1.
 */
sg2v_status sg2v_plan_describe(const sg2v_graph *g, const sg2v_template *t,
                               sg2v_precision precision, char *buf, uint64_t buf_len,
                               uint64_t *needed);

/* As sg2v_plan_describe for a graph of n vertices and nnz CSR entries, without
 * a graph handle or a GPU (the planner is host code). */
sg2v_status sg2v_plan_describe_n(int64_t n, int64_t nnz, const sg2v_template *t,
                                 sg2v_precision precision, char *buf, uint64_t buf_len,
                                 uint64_t *needed);

/*
 * Live per-kernel timing with CUDA events recorded around every launch on the
 * launching stream (used by bench.py for the roofline of the dominant kernel).
 * sg2v_profile_enable(1) clears and starts collection; sg2v_profile_read
 * synchronises the recorded events and returns, for kernel class c in
 * 0=colour, 1=hist, 2=step (fused SpMM+eMA), 3=top, 4=reduce:
 * launches[c], total milliseconds ms[c], and algorithmic bytes bytes[c].
 */
sg2v_status sg2v_profile_enable(int32_t on);
sg2v_status sg2v_profile_read(int64_t launches[5], double ms[5], double bytes[5]);
/* Per-launch records of the same profile, in launch order (q < min(cap, *n_out)):
 * class (0..4 as above), CUDA-event ms on the launching stream, the launch's
 * algorithmic bytes (the method's useful gather + CSR + M_a + output at
 * plain width — independent of the table layout the planner chose), its impl bytes
 * (the implemented layout: plain-width gathers of plain sources, projected-copy
 * writes) and its eMA split terms (GENERAL steps).  *n_out = number of records. */
sg2v_status sg2v_profile_read_launches(int64_t cap, int32_t *cls, double *ms, double *alg_bytes,
                                       double *impl_bytes, double *ema_terms, int64_t *n_out);

/* Kernels of this library launched (on any stream, by any thread) since the last
 * sg2v_profile_enable(1), counted at every launch site — a step may run several
 * kernels (heavy rows, hub rows of the bucket pass), so this can exceed the
 * records of sg2v_profile_read_launches.  Counted only while profiling is on;
 * *n_out must not be NULL (SG2V_EINVAL). */
sg2v_status sg2v_profile_kernel_count(uint64_t *n_out);

const char *sg2v_last_error(void);
const char *sg2v_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SG2V_H */
