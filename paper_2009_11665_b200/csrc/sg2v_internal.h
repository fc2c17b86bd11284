// sg2v_internal.h — host-side structures shared by the C ABI, the planner and
// the kernel launchers of libsg2v.so.  Nothing here is visible through the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sg2v.h"

namespace sg2v {

void set_error(const std::string &msg);

// ---------------------------------------------------------------------------
// Graph: device CSR + degree-descending processing order.
// ---------------------------------------------------------------------------
struct Graph {
    int64_t n = 0, nnz = 0;
    int device = 0;
    int64_t *d_rowptr = nullptr;
    int32_t *d_col = nullptr;
    int32_t *d_order = nullptr;  // rows sorted by degree, descending
    uint8_t *d_vclass = nullptr; // floor(log2(1 + rank in degree order)) per vertex (L2 hints)
    int64_t max_deg = 0;
    int64_t n_deg_ge[32] = {0};  // rows with degree >= 2^q (a prefix of d_order)
    // vertex-partitioned mode: this handle holds rows
    // [row_begin, row_begin + n) of a graph with n_global vertices; col ids are global
    bool partitioned = false;
    int64_t n_global = 0, row_begin = 0;
    // optional relabelling (sg2v_graph_set_vertex_ids): vertex v of this graph is vertex
    // d_orig[v] of the caller's input graph; colours are keyed by that id (SURVEY §8(c)
    // "RNG": reordering must carry original ids).  n_global entries when partitioned.
    int32_t *d_orig = nullptr;
};

// Column tile / combine descriptor of a vertex-partitioned step.
struct VpArgs {
    int mode = 0;               // 1 = tile gather into bg, 2 = combine from bg,
                                // 3 = fused step gathering whole rows from `stage`,
                                // 4/5 = split eMA pipeline: gather -> bg / eMA from bg (by position)
    const char *stage = nullptr;  // [n_global][stage_ld] all-gathered column tile
    int64_t stage_ld = 0, u0 = 0, cnt = 0;
    char *bg = nullptr;         // [n_local][ldb]
    int64_t row_begin = 0;      // mode 3: first global row of this rank
};

// ---------------------------------------------------------------------------
// Plan of one colouring (P:162-170 partition, Alg. 5 schedule P:443-457).
// ---------------------------------------------------------------------------
enum StepSrc { SRC_GATHER = 0, SRC_HIST = 1 };        // B = A·M_p  |  B = H (leaf passive)
enum StepComb { COMB_ACTIVE_LEAF = 0, COMB_GENERAL = 1 };

struct Node {            // sub-template T_s: vertex r with children[r][j..] + subtrees
    int r = 0, j = 0;
    int size = 1;
    int active = -1, passive = -1;  // node ids, -1 for a leaf
};

struct Step {
    int node = 0;
    int s = 0, a = 0, p = 0;
    bool top = false;
    StepSrc src = SRC_GATHER;
    StepComb comb = COMB_ACTIVE_LEAF;
    int64_t cs = 0, ca = 0, cp = 0;        // row widths of M_s, M_a, M_p (dense: C(k,·);
                                           //   anchored: C(k-1,·-1))
    int64_t cb = 0;                        // width of B(i,·) (dense: = cp; anchored: C(k-1,p))
    int64_t lds = 0, lda = 0, ldp = 0, ldb = 0;  // padded row strides (elements)
    int64_t map_off = -1;                  // anchored gather: push map [x][c(i)][u] (int32 offset)
    int buf_out = -1, buf_a = -1, buf_p = -1;  // workspace buffers (-1: none / leaf / H)
    int64_t idx_off = 0;                   // int32 offset into the plan's index blob
    int64_t nterms = 0;                    // splits per output (GENERAL)
    int packed = 0;                        // anchored GENERAL: pairs packed ia | ip << 16, term-major
    bool self_a = false;                   // anchored: T_s = root + 2 copies of X, M_a(i,·) = B(i,·)
    // exclusion-projected tables (anchored): a row holds, for every consumer colour
    // y ≠ c(i), the segment of its sets avoiding y (C(k-2,·-1) entries, stride ldseg)
    bool proj_out = false, proj_p = false;
    bool plain_out = false;                // the plain table is written (someone reads it)
    int64_t ldseg_out = 0, ldseg_p = 0, ldsx = 0;   // ldsx: projected row stride (k-1)·ldseg_out
    int buf_outx = -1;                     // projected output buffer
    int64_t omap_off = -1;                 // projected output: write map (int32 offset)
    std::string canon_out, canon_a, canon_p;  // rooted classes of T_s, T_a, T_p (table sharing)
    int gt = 32;                           // threads per row group (step kernel)
    bool split_ema = false;                // eMA-heavy GENERAL step: gather and eMA as a two-stream pipeline
    double alg_bytes = 0.0;                // algorithmic HBM bytes of the METHOD:
                                           //   useful gather + CSR + M_a + plain-width output (layout-independent)
    double impl_bytes = 0.0;               // compulsory bytes of the implemented layout (plain-width gathers
                                           //   from plain sources, projected-copy writes)
    double ema_terms = 0.0;
};

struct Buffer {
    int64_t offset = 0, bytes = 0;
};

enum Layout { LAYOUT_ANCHORED = 0, LAYOUT_DENSE = 1 };

struct Plan {
    int k = 0, root = 0;
    Layout layout = LAYOUT_ANCHORED;
    int elem = 4;                 // sizeof element
    sg2v_precision prec = SG2V_F32;
    std::vector<Node> nodes;
    std::vector<Step> steps;      // children-first order
    bool need_hist = false;
    int64_t ldh = 0;              // histogram row stride (elements)
    std::vector<Buffer> bufs;     // count tables (offsets inside the workspace)
    int64_t tables_bytes = 0;     // peak of the table arena
    int64_t kp = 0;               // anchored: hcnt row stride (int32 colour counts)
    int64_t off_colors = 0, off_hist = 0, off_rowval = 0, off_partial = 0, off_results = 0, off_flag = 0;
    int64_t off_hcnt = 0, off_bcol = 0;   // anchored: colour counts + colour-bucketed CSR
    // vertex-partitioned mode: rows are local (n = n_local), colours/staging are global
    bool vp = false;
    bool vp_full = false;                  // whole passive rows exchanged (no column tiles)
    int64_t n_global = 0, tile_w = 0;      // tile width in elements (multiple of 16 B)
    int64_t off_stage = 0, off_send = 0, off_bg = 0, off_colors_g = 0, off_part = 0;
    int64_t ws_bytes = 0;
    int64_t n_rows = 0;                    // rows the plan was made for (n)
    int64_t split_rows = 0, split_bytes = 0, off_split = 0;  // split eMA pipeline: chunk rows, 2 B buffers
    std::vector<int32_t> index;   // concatenated index tables (host copy)
    int32_t *d_index = nullptr;   // device copy (owned by the template's cache)
    int top_leaf_col_off = -1;    // idx offset of topcol[k] when the top step is leaf-active
    double model_time = 0.0;
    double alg_bytes_total = 0.0, impl_bytes_total = 0.0;
    int64_t hist_bytes = 0;
    bool allow_proj = true;       // planner may choose exclusion-projected tables
    std::vector<std::string> proj_cands;  // classes that could be projected (planning)
    std::set<std::string> proj;   // classes stored projected
    std::string describe() const;
};

static constexpr int kResultsRing = 4096;
static constexpr int kReduceBlocks = 512;

// ---------------------------------------------------------------------------
// Template: validated tree, α, P, cached plans per (precision, n, nnz, device).
// ---------------------------------------------------------------------------
struct Template {
    int k = 0;
    int root_hint = -1;
    std::vector<std::pair<int, int>> edges;
    std::vector<std::vector<int>> adj;
    double alpha = 1.0;
    double P = 1.0;
    // (precision, n, nnz, device | vertex-mode tag, layout, budget | col_tile, vertex-mode staging rows)
    std::map<std::tuple<int, int64_t, int64_t, int, int, uint64_t, int64_t>, std::unique_ptr<Plan>> plans;
    std::mutex mu;  // guards plans and the lazy index upload (handles may be shared by threads)
    ~Template();
};

// planner.cpp
sg2v_status validate_template(int k, const int32_t *edges, Template &t);
double automorphisms(const Template &t);
sg2v_status make_plan(const Template &t, int64_t n, int64_t nnz, sg2v_precision prec, Layout layout,
                      uint64_t budget, std::unique_ptr<Plan> &out, int64_t vp_n_global = 0, int64_t vp_tile = 0,
                      int proj_mode = 1);  // exclusion-projected tables: 0 off, 1 model, 2 all that fit
int64_t binom(int n, int r);

// kernels.cu — launchers; all return cudaError_t as int (0 = success)
struct Profiler;
int launch_colorize(uint64_t seed, int64_t j, int64_t n, int k, uint8_t *out, void *stream,
                    const int32_t *ids = nullptr);
int launch_hist(const Graph &g, const Plan &pl, const uint8_t *colors, void *H, void *stream);
int launch_bucket(const Graph &g, const Plan &pl, const uint8_t *colors, int32_t *hcnt, int32_t *bcol,
                  void *stream);
int launch_astep(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const int32_t *hcnt,
                 const int32_t *bcol, char *tables, void *rowval, int *ovf, void *stream);
int launch_astep_vp(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const int32_t *hcnt,
                    const int32_t *bcol, char *tables, void *rowval, int *ovf, void *stream, const VpArgs *vp);
// F32 overflow flag of one sg2v_count call: a device int inside its workspace
int ovf_reset(int *dflag, void *stream);
int ovf_read(const int *dflag, int *flag, void *stream);
// split eMA pipeline context (count_core): aux stream, events, the two B-row buffers
struct SplitCtx {
    void *aux = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
    char *bg = nullptr;
    int64_t rows = 0;
};
int launch_astep_split(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const int32_t *hcnt,
                       const int32_t *bcol, char *tables, void *rowval, int *ovf, void *stream, const SplitCtx &sp);
int launch_pack_tile(int64_t n, const char *src, int64_t ld_bytes, int64_t u0_bytes, int64_t w_bytes, char *dst,
                     int64_t dst_ld_bytes, void *stream);
int launch_bg_rowval(const Plan &pl, int64_t n, const char *bg, int64_t ldb, void *rowval, void *stream);
int launch_step(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors,
                const void *H, char *tables, void *rowval, int *ovf, void *stream);
int launch_reduce(const Plan &pl, int64_t n, const void *rowval, void *partial, void *result,
                  void *stream);
int graph_build_order(Graph &g, void *stream);
size_t colour_order_tmp_bytes(int64_t n);
int launch_colour_order(const Graph &g, const uint8_t *colors, int32_t *order_out, uint8_t *keys, void *tmp,
                        size_t tmp_bytes, void *stream);
int graph_validate(const Graph &g, int *bad, void *stream);

// profiling (api.cpp)
void prof_begin(int cls, void *stream);
// alg: SURVEY §8(d) bytes of the launch; impl: the implemented layout's bytes; terms: eMA terms
void prof_end(int cls, double alg, void *stream, double impl = -1.0, double terms = 0.0);
void note_launch();  // one kernel of this library launched (sg2v_profile_kernel_count)

}  // namespace sg2v
