// api.cpp — the C ABI of libsg2v.so (include/sg2v.h).  Argument checking,
// handle ownership, plan cache, workspace, the per-colouring launch sequence of
// Alg. 5 and the estimate of Alg. 1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "sg2v_internal.h"

// NCCL is resolved at first use (dlopen, preferring the copy torch already loaded)
// instead of at link time: linking the system libnccl.so.2 would shadow torch's
// newer one for any process that loads libsg2v.so first.
namespace {
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};
const NcclApi &nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy && api.getErrorString;
    return api;
}
}  // namespace

// Communicator of the vertex-partitioned mode: NCCL over NVLink (one process per
// GPU), or a host all-gather callback (tests: gloo, several processes per GPU).
struct sg2v_comm {
    int rank = 0, world = 1;
    ncclComm_t nccl = nullptr;
    sg2v_allgather_fn cb = nullptr;
    void *user = nullptr;
    char *hsend = nullptr, *hrecv = nullptr;  // pinned staging of the callback transport
    size_t hcap = 0;
};

namespace sg2v {

static thread_local std::string g_err;
static thread_local sg2v_options g_opts;
static thread_local bool g_opts_init = false;

void set_error(const std::string &msg) { g_err = msg; }

static sg2v_status cuda_fail(const char *what, int code) {
    set_error(std::string(what) + ": " + cudaGetErrorString((cudaError_t)code));
    return SG2V_ECUDA;
}

#define SG2V_CK(call)                                                   \
    do {                                                                \
        cudaError_t _e = (call);                                        \
        if (_e != cudaSuccess) return cuda_fail(#call, (int)_e);        \
    } while (0)

Template::~Template() {
    for (auto &kv : plans)
        if (kv.second && kv.second->d_index) cudaFree(kv.second->d_index);
}

// ----------------------------------------------------------------- profiling
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
    double bytes, impl, terms;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_ev_pool;
static thread_local cudaEvent_t g_pending = nullptr;
static std::atomic<uint64_t> g_kernels{0};

void note_launch() {
    if (g_prof_on) g_kernels.fetch_add(1, std::memory_order_relaxed);
}

static cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(int, void *stream) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_pending = ev_get();
    cudaEventRecord(g_pending, (cudaStream_t)stream);
}

void prof_end(int cls, double bytes, void *stream, double impl, double terms) {
    if (!g_prof_on || !g_pending) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = ev_get();
    cudaEventRecord(b, (cudaStream_t)stream);
    g_prof.push_back({cls, g_pending, b, bytes, impl < 0 ? bytes : impl, terms});
    g_pending = nullptr;
}

// ------------------------------------------------------------------- helpers
static int resolve_device(int dev) {
    if (dev >= 0) return dev;
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

static sg2v_status ensure_device(int dev) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error("no CUDA device available (libsg2v has no CPU fallback)");
        return SG2V_ECUDA;
    }
    if (dev >= count) { set_error("device ordinal out of range"); return SG2V_EINVAL; }
    SG2V_CK(cudaSetDevice(dev));
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) {
        set_error("libsg2v is built for sm_100a (B200) only");
        return SG2V_ECUDA;
    }
    return SG2V_OK;
}

// Plans are cached per (precision, n, nnz, device); the index tables are
// uploaded lazily, so planning itself needs no GPU (host-only tests use it).
static Layout current_layout(int32_t lay) { return lay == 1 ? LAYOUT_DENSE : LAYOUT_ANCHORED; }

static int32_t tls_layout() { return g_opts_init ? g_opts.layout : 0; }

// Planning budget: the explicit mem_budget_bytes, else the device's total memory
// minus a 6 GiB reserve (graph, context, allocator slack) — total, not free, so that
// sg2v_workspace_bytes and sg2v_count agree on the plan — else unlimited (no device).
static uint64_t plan_budget(uint64_t explicit_budget, int device) {
    if (explicit_budget) return explicit_budget;
    if (device < 0) return 0;
    size_t fr = 0, tot = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    cudaError_t e = cudaMemGetInfo(&fr, &tot);
    if (cur != device) cudaSetDevice(cur);
    if (e != cudaSuccess || tot == 0) return 0;
    const uint64_t reserve = 6ull << 30;
    return tot > reserve ? tot - reserve : tot;
}

static void keep_pool(int dev) {
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

static uint64_t tls_budget() { return g_opts_init ? g_opts.mem_budget_bytes : 0; }

static sg2v_status get_plan(int64_t n, int64_t nnz, int device, const Template &t, sg2v_precision prec,
                            int32_t layout, bool upload, Plan **out, uint64_t explicit_budget = 0) {
    if (layout < 0 || layout > 3) {
        set_error("layout must be 0 (anchored), 1 (dense), 2 (anchored, no projected tables) or 3 (anchored, "
                  "every eligible table projected)");
        return SG2V_EINVAL;
    }
    const uint64_t budget = plan_budget(explicit_budget, device);
    auto key = std::make_tuple((int)prec, n, nnz, device, (int)layout, budget, (int64_t)0);
    Template &tm = const_cast<Template &>(t);
    std::lock_guard<std::mutex> plan_lock(tm.mu);  // plan cache + lazy index upload
    auto &slot = tm.plans[key];
    if (!slot) {
        std::unique_ptr<Plan> pl;
        sg2v_status st = make_plan(t, n, nnz, prec, current_layout(layout), budget, pl, 0, 0,
                                   layout == 0 ? 1 : layout == 3 ? 2 : 0);
        if (st != SG2V_OK) return st;
        slot = std::move(pl);
    }
    if (upload && !slot->d_index) {
        SG2V_CK(cudaMalloc(&slot->d_index, slot->index.size() * sizeof(int32_t)));
        SG2V_CK(cudaMemcpy(slot->d_index, slot->index.data(), slot->index.size() * sizeof(int32_t),
                           cudaMemcpyHostToDevice));
    }
    *out = slot.get();
    return SG2V_OK;
}

}  // namespace sg2v

using namespace sg2v;

struct sg2v_graph : public sg2v::Graph {};
struct sg2v_template : public sg2v::Template {};

extern "C" {

const char *sg2v_last_error(void) { return g_err.c_str(); }
const char *sg2v_version(void) { return "sg2v 0.1 (sm_100a)"; }

void sg2v_options_default(sg2v_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->precision = SG2V_F32;
    o->iter_offset = 0;
    o->iter_stride = 1;
    o->mode = 0;
    o->device = -1;
}

sg2v_status sg2v_set_options(const sg2v_options *o) {
    if (!o) { set_error("options is NULL"); return SG2V_EINVAL; }
    if (o->mode < 0 || o->mode > 1) { set_error("mode must be 0 (replicas) or 1 (vertex partition)"); return SG2V_EINVAL; }
    g_opts = *o;
    g_opts_init = true;
    return SG2V_OK;
}

sg2v_status sg2v_graph_load_csr(int64_t n, const int64_t *row_offsets, const int32_t *col_indices, int64_t nnz,
                                uint32_t flags, sg2v_graph **out) {
    if (!out) { set_error("out is NULL"); return SG2V_EINVAL; }
    *out = nullptr;
    if (n < 0 || n >= (int64_t(1) << 31) || nnz < 0) { set_error("n or nnz out of range"); return SG2V_EINVAL; }
    if (!row_offsets || (nnz > 0 && !col_indices)) { set_error("CSR arrays are NULL"); return SG2V_EINVAL; }
    const bool dev_ptrs = flags & SG2V_GRAPH_DEVICE_PTRS;
    if (!dev_ptrs) {
        if (row_offsets[0] != 0 || row_offsets[n] != nnz) { set_error("row_offsets[0] != 0 or row_offsets[n] != nnz"); return SG2V_EINVAL; }
    }
    sg2v_options o;
    if (g_opts_init) o = g_opts; else sg2v_options_default(&o);
    int dev = resolve_device(o.device);
    sg2v_status st = ensure_device(dev);
    if (st != SG2V_OK) return st;
    auto *g = new sg2v_graph();
    g->n = n;
    g->nnz = nnz;
    g->device = dev;
    cudaStream_t s = (cudaStream_t)o.stream;
    auto fail = [&](sg2v_status code) { sg2v_graph_free(g); return code; };
    cudaError_t e;
    // stream-ordered allocations from the device's default pool, which keeps freed
    // memory mapped (release threshold = max): repeated load/free cycles cost no
    // page-table work (the e2e path of bench.py)
    keep_pool(dev);
    if ((e = cudaMallocAsync((void **)&g->d_rowptr, (n + 1) * sizeof(int64_t), s)) != cudaSuccess) return fail(cuda_fail("cudaMallocAsync rowptr", e));
    if ((e = cudaMallocAsync((void **)&g->d_col, std::max<int64_t>(nnz, 1) * sizeof(int32_t), s)) != cudaSuccess) return fail(cuda_fail("cudaMallocAsync col", e));
    if ((e = cudaMallocAsync((void **)&g->d_order, std::max<int64_t>(n, 1) * sizeof(int32_t), s)) != cudaSuccess) return fail(cuda_fail("cudaMallocAsync order", e));
    if ((e = cudaMallocAsync((void **)&g->d_vclass, std::max<int64_t>(n, 1), s)) != cudaSuccess) return fail(cuda_fail("cudaMallocAsync vclass", e));
    cudaMemcpyKind kind = dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if ((e = cudaMemcpyAsync(g->d_rowptr, row_offsets, (n + 1) * sizeof(int64_t), kind, s)) != cudaSuccess) return fail(cuda_fail("copy rowptr", e));
    if (nnz > 0 && (e = cudaMemcpyAsync(g->d_col, col_indices, nnz * sizeof(int32_t), kind, s)) != cudaSuccess) return fail(cuda_fail("copy col", e));
    if (dev_ptrs) {
        int64_t ends[2];
        cudaMemcpyAsync(&ends[0], g->d_rowptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&ends[1], g->d_rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_fail("sync", e));
        if (ends[0] != 0 || ends[1] != nnz) { set_error("row_offsets[0] != 0 or row_offsets[n] != nnz"); return fail(SG2V_EINVAL); }
    }
    if (flags & SG2V_GRAPH_VALIDATE) {
        int bad = 0;
        int rc = graph_validate(*g, &bad, s);
        if (rc) return fail(cuda_fail("validate", rc));
        if (bad) {
            std::string m = "invalid CSR:";
            if (bad & 1) m += " bad row_offsets;";
            if (bad & 2) m += " column id out of range;";
            if (bad & 4) m += " self-loop;";
            if (bad & 8) m += " row not strictly sorted (unsorted or duplicate);";
            if (bad & 16) m += " not symmetric;";
            set_error(m);
            return fail(SG2V_EINVAL);
        }
    }
    int rc = graph_build_order(*g, s);
    if (rc) return fail(cuda_fail("degree order", rc));
    *out = g;
    return SG2V_OK;
}

void sg2v_graph_free(sg2v_graph *g) {
    if (!g) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    // stream-ordered on the legacy default stream (ordered after work on blocking streams)
    if (g->d_rowptr) cudaFreeAsync(g->d_rowptr, 0);
    if (g->d_col) cudaFreeAsync(g->d_col, 0);
    if (g->d_order) cudaFreeAsync(g->d_order, 0);
    if (g->d_vclass) cudaFreeAsync(g->d_vclass, 0);
    if (g->d_orig) cudaFreeAsync(g->d_orig, 0);
    cudaSetDevice(cur);
    delete g;
}

sg2v_status sg2v_template_build(int32_t k, const int32_t *edges, int32_t root_hint, sg2v_template **out) {
    if (!out) { set_error("out is NULL"); return SG2V_EINVAL; }
    *out = nullptr;
    if (k < 1 || k > 31) { set_error("k must be in [1, 31]"); return SG2V_EINVAL; }
    if (root_hint < -1 || root_hint >= k) { set_error("root_hint out of range"); return SG2V_EINVAL; }
    auto *t = new sg2v_template();
    sg2v_status st = validate_template(k, edges, *t);
    if (st != SG2V_OK) { delete t; return st; }
    t->root_hint = root_hint;
    t->alpha = automorphisms(*t);
    double P = 1.0;
    for (int i = 1; i <= k; ++i) P *= (double)i / (double)k;   // k!/k^k
    t->P = P;
    *out = t;
    return SG2V_OK;
}

void sg2v_template_free(sg2v_template *t) { delete t; }

sg2v_status sg2v_template_info(const sg2v_template *t, int32_t *k, double *alpha, double *P) {
    if (!t) { set_error("template is NULL"); return SG2V_EINVAL; }
    if (k) *k = t->k;
    if (alpha) *alpha = t->alpha;
    if (P) *P = t->P;
    return SG2V_OK;
}

sg2v_status sg2v_workspace_bytes(const sg2v_graph *g, const sg2v_template *t, sg2v_precision prec, uint64_t *bytes) {
    if (!g || !t || !bytes) { set_error("NULL argument"); return SG2V_EINVAL; }
    if (prec < SG2V_F32 || prec > SG2V_U64) { set_error("bad precision"); return SG2V_EINVAL; }
    if (t->k == 1 || g->n == 0) { *bytes = 0; return SG2V_OK; }
    Plan *pl = nullptr;
    sg2v_status st = get_plan(g->n, g->nnz, g->device, *t, prec, tls_layout(), false, &pl, tls_budget());
    if (st != SG2V_OK) return st;
    *bytes = (uint64_t)pl->ws_bytes;
    return SG2V_OK;
}

static sg2v_status plan_describe_dev(int64_t n, int64_t nnz, int device, const sg2v_template *t,
                                     sg2v_precision prec, char *buf, uint64_t buf_len, uint64_t *needed);

sg2v_status sg2v_plan_describe(const sg2v_graph *g, const sg2v_template *t, sg2v_precision prec, char *buf,
                               uint64_t buf_len, uint64_t *needed) {
    if (!g) { set_error("NULL argument"); return SG2V_EINVAL; }
    // the plan sg2v_count will use on g's device (its memory budget)
    return plan_describe_dev(g->n, g->nnz, g->device, t, prec, buf, buf_len, needed);
}

sg2v_status sg2v_plan_describe_n(int64_t n, int64_t nnz, const sg2v_template *t, sg2v_precision prec, char *buf,
                                 uint64_t buf_len, uint64_t *needed) {
    return plan_describe_dev(n, nnz, -1, t, prec, buf, buf_len, needed);
}

static sg2v_status plan_describe_dev(int64_t n, int64_t nnz, int device, const sg2v_template *t,
                                     sg2v_precision prec, char *buf, uint64_t buf_len, uint64_t *needed) {
    if (!t || n < 0 || nnz < 0) { set_error("bad argument"); return SG2V_EINVAL; }
    if (prec < SG2V_F32 || prec > SG2V_U64) { set_error("bad precision"); return SG2V_EINVAL; }
    std::string s;
    if (t->k == 1 || n == 0) {
        s = "{\"k\":" + std::to_string(t->k) + ",\"steps\":[],\"workspace_bytes\":0,\"alg_bytes\":0}";
    } else {
        Plan *pl = nullptr;
        sg2v_status st = get_plan(n, nnz, device, *t, prec, tls_layout(), false, &pl, tls_budget());
        if (st != SG2V_OK) return st;
        s = pl->describe();
    }
    if (needed) *needed = s.size() + 1;
    if (buf && buf_len > 0) {
        size_t m = std::min<size_t>(s.size(), buf_len - 1);
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
    }
    return SG2V_OK;
}

sg2v_status sg2v_colorize(uint64_t seed, int64_t j, int64_t n, int32_t k, uint8_t *colors_out, void *stream) {
    if (n < 0 || k < 1 || k > 31 || (n > 0 && !colors_out)) { set_error("bad argument"); return SG2V_EINVAL; }
    int rc = launch_colorize(seed, j, n, k, colors_out, stream);
    if (rc) return cuda_fail("colorize", rc);
    return SG2V_OK;
}

}  // extern "C"

namespace sg2v {

// Workspace of a batch of m same-k templates run on every colouring: the table
// arenas overlap (templates run one after another), the per-colouring buffers
// (colours, histogram / colour buckets, row values) are shared.  For m = 1 this
// is exactly the plan's own layout (Plan::ws_bytes).
struct BatchLayout {
    int64_t off_colors = 0, off_hist = 0, off_hcnt = 0, off_bcol = 0, off_rowval = 0, off_partial = 0,
            off_results = 0, off_flag = 0, off_split = 0, bytes = 0;
};

static int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static BatchLayout batch_layout(const std::vector<Plan *> &pls, int64_t n, int64_t nnz, int64_t joint_tables = -1) {
    BatchLayout L;
    int64_t tables = 0, hist = 0;
    bool anch = false;
    for (Plan *p : pls) {
        tables = std::max(tables, joint_tables >= 0 ? joint_tables : p->tables_bytes);
        hist = std::max(hist, p->hist_bytes);
        anch = anch || p->layout == LAYOUT_ANCHORED;
    }
    const int64_t kp = pls.empty() ? 0 : pls[0]->kp;
    int64_t off = rup(tables, 256);
    L.off_colors = off;  off = rup(off + std::max<int64_t>(n, 1) + 16, 256);
    L.off_hist = off;    off = rup(off + hist, 256);
    L.off_hcnt = off;    off = rup(off + (anch ? n * kp * 4 : 0), 256);
    L.off_bcol = off;    off = rup(off + (anch ? nnz * 4 : 0), 256);
    L.off_rowval = off;  off = rup(off + std::max<int64_t>(n, 1) * 8, 256);
    L.off_partial = off; off = rup(off + kReduceBlocks * 8, 256);
    L.off_results = off; off = rup(off + (int64_t)kResultsRing * 8 * (int64_t)std::max<size_t>(pls.size(), 1), 256);
    L.off_flag = off;    off = rup(off + 16, 256);
    int64_t split = 0;
    for (Plan *p : pls) split = std::max(split, p->split_bytes);
    L.off_split = off;   off = rup(off + split, 256);
    L.bytes = off;
    return L;
}

// Joint schedule of a batch: the templates' plans run in turn, and a rooted
// sub-template class already computed for an earlier template (same canonical
// string, e.g. the short paths and stars every treelet shares) is not recomputed
// — its table stays live until its last consumer in any template.  The result is
// one view Plan per template whose steps/buffers index a joint table arena.
struct JointPlan {
    std::vector<Plan> views;       // per template: steps to run + the joint buffer table
    int64_t tables_bytes = 0;
};

static void joint_schedule(const std::vector<Plan *> &pls, JointPlan &J) {
    std::vector<Buffer> bufs;
    std::map<std::string, int> class_buf, uses;
    for (Plan *p : pls)
        for (const Step &st : p->steps) {
            if (!st.self_a) uses[st.canon_a]++;
            uses[st.canon_p]++;
        }
    std::vector<std::pair<int64_t, int64_t>> live;
    int64_t arena = 0;
    auto alloc = [&](int64_t bytes) -> int64_t {
        int64_t pos = 0;
        std::sort(live.begin(), live.end());
        for (auto &iv : live) {
            if (iv.first - pos >= bytes) break;
            pos = std::max(pos, rup(iv.first + iv.second, 256));
        }
        live.push_back({pos, bytes});
        arena = std::max(arena, pos + bytes);
        return pos;
    };
    auto release = [&](int b) {
        if (b < 0) return;
        for (size_t q = 0; q < live.size(); ++q)
            if (live[q].first == bufs[b].offset) { live.erase(live.begin() + q); break; }
    };
    J.views.clear();
    for (Plan *p : pls) {
        Plan v = *p;  // copies index offsets; d_index stays owned by p
        v.steps.clear();
        for (const Step &st0 : p->steps) {
            Step st = st0;
            const bool have = !st.top && class_buf.count(st.canon_out);
            if (have) {  // computed by an earlier template: only release bookkeeping
                if (!st.self_a && --uses[st.canon_a] == 0) release(class_buf[st.canon_a]);
                if (--uses[st.canon_p] == 0) release(class_buf[st.canon_p]);
                continue;
            }
            st.buf_a = (!st.self_a && class_buf.count(st.canon_a)) ? class_buf[st.canon_a] : -1;
            st.buf_p = class_buf.count(st.canon_p) ? class_buf[st.canon_p] : -1;
            if (!st.top) {
                Buffer b;
                b.bytes = st0.buf_out >= 0 ? p->bufs[st0.buf_out].bytes : 0;
                b.offset = alloc(b.bytes);
                bufs.push_back(b);
                st.buf_out = (int)bufs.size() - 1;
                class_buf[st.canon_out] = st.buf_out;
            }
            if (!st.self_a && --uses[st.canon_a] == 0) release(st.buf_a);
            if (--uses[st.canon_p] == 0) release(st.buf_p);
            v.steps.push_back(st);
        }
        J.views.push_back(std::move(v));
    }
    for (Plan &v : J.views) v.bufs = bufs;
    J.tables_bytes = rup(arena, 256);
}

static sg2v_status batch_plans(const sg2v_graph *g, const sg2v_template *const *ts, int32_t m, sg2v_precision prec,
                               int32_t layout, bool upload, uint64_t budget, std::vector<Plan *> &pls) {
    pls.clear();
    for (int32_t q = 0; q < m; ++q) {
        if (ts[q]->k == 1 || g->n == 0) continue;
        Plan *pl = nullptr;
        // a joint schedule of several templates shares tables across them: plain
        // anchored rows only (a single template may use exclusion-projected tables)
        sg2v_status st = get_plan(g->n, g->nnz, g->device, *ts[q], prec, (layout == 0 || layout == 3) && m > 1 ? 2 : layout, upload,
                                  &pl, budget);
        if (st != SG2V_OK) return st;
        pls.push_back(pl);
    }
    return SG2V_OK;
}

// ----------------------------------------------------------- vertex partition
static sg2v_status comm_allgather(sg2v_comm *c, const void *send, void *recv, size_t bytes, cudaStream_t s) {
    if (c->nccl) {
        ncclResult_t r = nccl_api().allGather(send, recv, bytes, ncclUint8, c->nccl, s);
        if (r != ncclSuccess) {
            set_error(std::string("ncclAllGather: ") + nccl_api().getErrorString(r));
            return SG2V_ENCCL;
        }
        return SG2V_OK;
    }
    if (!c->cb) { set_error("communicator has no transport"); return SG2V_EINVAL; }
    const size_t need = bytes * (size_t)c->world;
    if (c->hcap < need) {
        if (c->hsend) cudaFreeHost(c->hsend);
        if (c->hrecv) cudaFreeHost(c->hrecv);
        SG2V_CK(cudaMallocHost((void **)&c->hsend, std::max<size_t>(bytes, 1)));
        SG2V_CK(cudaMallocHost((void **)&c->hrecv, std::max<size_t>(need, 1)));
        c->hcap = need;
    }
    SG2V_CK(cudaMemcpyAsync(c->hsend, send, bytes, cudaMemcpyDeviceToHost, s));
    SG2V_CK(cudaStreamSynchronize(s));
    if (c->cb(c->hsend, c->hrecv, (uint64_t)bytes, c->user) != 0) {
        set_error("all-gather callback failed");
        return SG2V_ENCCL;
    }
    SG2V_CK(cudaMemcpyAsync(recv, c->hrecv, need, cudaMemcpyHostToDevice, s));
    return SG2V_OK;
}

// 1D vertex partition: rank r owns rows [r·nl, r·nl + n_local) of
// every table (nl = ceil(n_global / world)).  Per gather step the passive table is
// exchanged either as whole rows (plan vp_full: one all-gather of every rank's table
// — its table holds nl rows, so it is the send buffer — then the fused single-GPU
// kernels run on the local rows with the staging buffer as the gather source; nothing
// is exchanged at world = 1), or, for passive tables too large to stage, in column
// tiles: pack + all-gather of tile t+1 run on a communication stream while the push
// of tile t's colour-bucket sums into B rows in global memory runs on the compute
// stream (double-buffered staging, events order both ways); the eMA / top then run on
// the local rows.  The per-rank Σ_i are all-gathered and summed in rank order.
struct VpStreams {
    cudaStream_t comm = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr}, src = nullptr;
    ~VpStreams() {
        for (int q = 0; q < 2; ++q) {
            if (ready[q]) cudaEventDestroy(ready[q]);
            if (done[q]) cudaEventDestroy(done[q]);
        }
        if (src) cudaEventDestroy(src);
        if (comm) cudaStreamDestroy(comm);
    }
};

static sg2v_status count_vp(const sg2v_graph *g, const sg2v_template *t, int32_t k, int64_t n_iter, uint64_t seed,
                            sg2v_options o, double *estimate, double *colorful_out, uint64_t *colorful_u64_out) {
    sg2v_comm *c = (sg2v_comm *)o.nccl_comm;
    if (!c) { set_error("mode 1 needs options.nccl_comm (sg2v_comm_init_*)"); return SG2V_EINVAL; }
    if (o.layout == 1) { set_error("the vertex-partitioned mode uses the anchored layout"); return SG2V_EINVAL; }
    const int64_t n_global = g->partitioned ? g->n_global : g->n;
    const int64_t nl = (n_global + c->world - 1) / c->world;
    const int64_t begin = g->partitioned ? g->row_begin : 0;
    if (begin != (int64_t)c->rank * nl || g->n != std::max<int64_t>(0, std::min(nl, n_global - begin))) {
        set_error("partition must be rows [rank*nl, rank*nl + n_local) with nl = ceil(n_global/world)");
        return SG2V_EINVAL;
    }
    const int dev = g->device;
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    sg2v_status st = ensure_device(dev);
    if (st != SG2V_OK) return st;
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev_dev};
    const bool u64mode = o.precision == SG2V_U64;
    cudaStream_t s = (cudaStream_t)o.stream;
    std::vector<double> resf(n_iter, 0.0);
    std::vector<uint64_t> resu(n_iter, 0);
    int ovf = 0;
    if (k == 1) {
        for (int64_t q = 0; q < n_iter; ++q) { resf[q] = (double)n_global; resu[q] = (uint64_t)n_global; }
    } else {
        // plan on nl rows (every rank's tables hold nl rows: the whole-row exchange sends
        // them as they are); staging sized for world·nl global rows
        auto key = std::make_tuple((int)o.precision, nl, g->nnz, -(g->device + 1) - 1000 * c->world, 0,
                                   (uint64_t)o.col_tile, (int64_t)c->world * nl);
        Template &tm = const_cast<Template &>(*(const Template *)t);
        std::unique_lock<std::mutex> plan_lock(tm.mu);
        auto &slot = tm.plans[key];
        if (!slot) {
            std::unique_ptr<Plan> pl;
            st = make_plan(*t, std::max<int64_t>(nl, 1), std::max<int64_t>(g->nnz, 1), o.precision, LAYOUT_ANCHORED,
                           0, pl, (int64_t)c->world * nl, o.col_tile, 0);
            if (st != SG2V_OK) return st;
            slot = std::move(pl);
        }
        Plan *pl = slot.get();
        if (!pl->d_index) {
            SG2V_CK(cudaMalloc(&pl->d_index, pl->index.size() * sizeof(int32_t)));
            SG2V_CK(cudaMemcpy(pl->d_index, pl->index.data(), pl->index.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        }
        plan_lock.unlock();
        char *ws = (char *)o.workspace;
        bool own = false;
        if (ws) {
            if (o.workspace_bytes < (uint64_t)pl->ws_bytes) {
                set_error("workspace too small: need " + std::to_string(pl->ws_bytes) + " bytes");
                return SG2V_ENOMEM;
            }
        } else {
            keep_pool(dev);
            SG2V_CK(cudaMallocAsync((void **)&ws, pl->ws_bytes, s));
            own = true;
        }
        struct Free { char *p; bool own; cudaStream_t s; ~Free() { if (own) cudaFreeAsync(p, s); } } freer{ws, own, s};
        VpStreams vs;
        if (!pl->vp_full) {
            SG2V_CK(cudaStreamCreateWithFlags(&vs.comm, cudaStreamNonBlocking));
            for (int q = 0; q < 2; ++q) {
                SG2V_CK(cudaEventCreateWithFlags(&vs.ready[q], cudaEventDisableTiming));
                SG2V_CK(cudaEventCreateWithFlags(&vs.done[q], cudaEventDisableTiming));
            }
            SG2V_CK(cudaEventCreateWithFlags(&vs.src, cudaEventDisableTiming));
        }
        uint8_t *colors_g = (uint8_t *)(ws + pl->off_colors_g);
        uint8_t *colors_l = colors_g + begin;
        int32_t *hcnt = (int32_t *)(ws + pl->off_hcnt);
        int32_t *bcol = (int32_t *)(ws + pl->off_bcol);
        void *rowval = ws + pl->off_rowval;
        void *partial = ws + pl->off_partial;
        char *part = ws + pl->off_part;  // [0]: this rank's Σ_i, [8..]: all ranks'
        int *dflag = (int *)(ws + pl->off_flag);
        if (!u64mode) SG2V_CK((cudaError_t)ovf_reset(dflag, s));
        const int64_t E = pl->elem, W = pl->tile_w;
        const int vn = 16 / pl->elem;
        std::vector<uint64_t> hpart(c->world);
        int fill = 0;  // tile ordinal (staging parity) across steps
        for (int64_t q = 0; q < n_iter; ++q) {
            const int64_t j = o.iter_offset + q * o.iter_stride;
            // every rank colours every vertex (a pure function of its input id)
            int rc = launch_colorize(seed, j, n_global, k, colors_g, s, g->d_orig);
            if (rc) return cuda_fail("colorize", rc);
            if (g->n > 0 && (rc = launch_bucket(*g, *pl, colors_g, hcnt, bcol, s))) return cuda_fail("bucket", rc);
            for (const Step &stp : pl->steps) {
                if (stp.src == SRC_HIST) {  // local (the histogram is local)
                    rc = launch_astep_vp(*g, *pl, stp, colors_l, hcnt, bcol, ws, rowval, dflag, s, nullptr);
                    if (rc) return cuda_fail("step", rc == -1 ? 0 : rc);
                    continue;
                }
                const char *mp = ws + pl->bufs[stp.buf_p].offset;
                if (pl->vp_full) {
                    // whole rows: one all-gather of the passive table (nl rows per rank)
                    const char *stage = mp;
                    if (c->world > 1) {
                        st = comm_allgather(c, mp, ws + pl->off_stage, (size_t)nl * stp.ldp * E, s);
                        if (st != SG2V_OK) return st;
                        stage = ws + pl->off_stage;
                    }
                    VpArgs va;
                    va.mode = 3;
                    va.stage = stage;
                    va.row_begin = begin;
                    rc = launch_astep_vp(*g, *pl, stp, colors_l, hcnt, bcol, ws, rowval, dflag, s, &va);
                    if (rc) return cuda_fail("step", rc == -1 ? 0 : rc);
                    continue;
                }
                const bool bg_is_out = !stp.top && stp.comb == COMB_ACTIVE_LEAF;
                char *bg = bg_is_out ? ws + pl->bufs[stp.buf_out].offset : ws + pl->off_bg;
                SG2V_CK(cudaMemsetAsync(bg, 0, (size_t)std::max<int64_t>(g->n, 1) * stp.ldb * E, s));
                // the comm stream packs the passive table written by the previous step
                SG2V_CK(cudaEventRecord(vs.src, s));
                SG2V_CK(cudaStreamWaitEvent(vs.comm, vs.src, 0));
                auto exchange = [&](int64_t u0, int par) -> sg2v_status {
                    const int64_t cnt = std::min<int64_t>(W, stp.cp - u0);
                    const int64_t wb = ((cnt + vn - 1) / vn) * vn * E;
                    char *send = ws + pl->off_send + (size_t)par * nl * W * E;
                    char *stage = ws + pl->off_stage + (size_t)par * c->world * nl * W * E;
                    int r2 = g->n > 0 ? launch_pack_tile(g->n, mp, stp.ldp * E, u0 * E, wb, send, W * E, vs.comm) : 0;
                    if (r2) return cuda_fail("pack", r2);
                    sg2v_status s2 = comm_allgather(c, send, stage, (size_t)nl * W * E, vs.comm);
                    if (s2 != SG2V_OK) return s2;
                    SG2V_CK(cudaEventRecord(vs.ready[par], vs.comm));
                    return SG2V_OK;
                };
                const int64_t ntiles = (stp.cp + W - 1) / W;
                // prologue: tile 0 in flight
                if ((st = exchange(0, fill & 1)) != SG2V_OK) return st;
                for (int64_t tt = 0; tt < ntiles; ++tt) {
                    const int par = (fill + (int)tt) & 1;
                    // next tile's exchange overlaps this tile's push (its staging half
                    // was last read by tile tt-1: wait for that push first)
                    if (tt + 1 < ntiles) {
                        if (tt >= 1) SG2V_CK(cudaStreamWaitEvent(vs.comm, vs.done[par ^ 1], 0));
                        if ((st = exchange((tt + 1) * W, par ^ 1)) != SG2V_OK) return st;
                    }
                    SG2V_CK(cudaStreamWaitEvent(s, vs.ready[par], 0));
                    VpArgs va;
                    va.mode = 1;
                    va.stage = ws + pl->off_stage + (size_t)par * c->world * nl * W * E;
                    va.stage_ld = W;
                    va.u0 = tt * W;
                    va.cnt = std::min<int64_t>(W, stp.cp - tt * W);
                    va.bg = bg;
                    rc = launch_astep_vp(*g, *pl, stp, colors_l, hcnt, bcol, ws, rowval, dflag, s, &va);
                    if (rc) return cuda_fail("tile", rc == -1 ? 0 : rc);
                    SG2V_CK(cudaEventRecord(vs.done[par], s));
                }
                fill += (int)ntiles;
                // the comm stream must not run ahead into buffers of the next step
                SG2V_CK(cudaEventRecord(vs.src, s));
                SG2V_CK(cudaStreamWaitEvent(vs.comm, vs.src, 0));
                if (bg_is_out) continue;
                if (stp.top && stp.comb == COMB_ACTIVE_LEAF) {
                    rc = launch_bg_rowval(*pl, g->n, bg, stp.ldb, rowval, s);
                } else {
                    VpArgs va;
                    va.mode = 2;
                    va.bg = bg;
                    rc = launch_astep_vp(*g, *pl, stp, colors_l, hcnt, bcol, ws, rowval, dflag, s, &va);
                }
                if (rc) return cuda_fail("combine", rc == -1 ? 0 : rc);
            }
            if (g->n > 0) {
                rc = launch_reduce(*pl, g->n, rowval, partial, part, s);
                if (rc) return cuda_fail("reduce", rc);
            } else {
                SG2V_CK(cudaMemsetAsync(part, 0, 8, s));
            }
            st = comm_allgather(c, part, part + 8, 8, s);
            if (st != SG2V_OK) return st;
            SG2V_CK(cudaMemcpyAsync(hpart.data(), part + 8, 8 * c->world, cudaMemcpyDeviceToHost, s));
            SG2V_CK(cudaStreamSynchronize(s));
            uint64_t su = 0;
            double sf = 0.0;
            for (int r = 0; r < c->world; ++r) {  // rank order: deterministic
                double f;
                std::memcpy(&f, &hpart[r], 8);
                su += hpart[r];
                sf += f;
            }
            resu[q] = su;
            resf[q] = sf;
        }
        if (vs.comm) SG2V_CK(cudaStreamSynchronize(vs.comm));
        if (!u64mode) SG2V_CK((cudaError_t)ovf_read(dflag, &ovf, s));
    }
    bool finite = ovf == 0;  // a stored F32 table entry overflowed on this rank
    double sum = 0.0;
    for (int64_t q = 0; q < n_iter; ++q) {
        if (colorful_out) colorful_out[q] = u64mode ? (double)resu[q] : resf[q];
        if (colorful_u64_out) colorful_u64_out[q] = u64mode ? resu[q] : (uint64_t)resf[q];
        if (!u64mode) {
            if (!std::isfinite(resf[q])) finite = false;
            sum += resf[q];
        }
    }
    if (estimate) *estimate = u64mode ? std::nan("") : sum / (double)n_iter / (t->P * t->alpha);
    if (!finite) {
        set_error("EOVERFLOW: a colourful count is not finite in F32 (use F64 or U64)");
        return SG2V_EOVERFLOW;
    }
    return SG2V_OK;
}

// Alg. 1 / Alg. 5 outer loop for m templates sharing every colouring (a1 and the
// colour buckets / histogram once per colouring).
// colorful[m * n_iter] / colorful_u64[m * n_iter] template-major.
static sg2v_status count_core(const sg2v_graph *g, const sg2v_template *const *ts, int32_t m, int32_t k,
                              int64_t n_iter, uint64_t seed, const sg2v_options *op, double *estimates,
                              double *colorful_out, uint64_t *colorful_u64_out) {
    if (!g || !ts || m < 1) { set_error("graph or templates NULL / m < 1"); return SG2V_EINVAL; }
    for (int32_t q = 0; q < m; ++q) {
        if (!ts[q]) { set_error("template is NULL"); return SG2V_EINVAL; }
        if (ts[q]->k != k) { set_error("k must equal the number of template vertices of every template (P:161)"); return SG2V_EINVAL; }
    }
    if (n_iter <= 0) { set_error("n_iter must be >= 1"); return SG2V_EINVAL; }
    sg2v_options o;
    if (op) o = *op; else if (g_opts_init) o = g_opts; else sg2v_options_default(&o);
    if (o.precision < SG2V_F32 || o.precision > SG2V_U64) { set_error("bad precision"); return SG2V_EINVAL; }
    if (o.mode < 0 || o.mode > 1) { set_error("mode must be 0 (replicas) or 1 (vertex partition)"); return SG2V_EINVAL; }
    if (o.iter_stride == 0) o.iter_stride = 1;
    if (o.mode == 1) {
        if (m != 1) { set_error("the vertex-partitioned mode counts one template per call"); return SG2V_EINVAL; }
        return count_vp(g, ts[0], k, n_iter, seed, o, estimates, colorful_out, colorful_u64_out);
    }
    const int dev = g->device;
    int prev_dev = 0;
    cudaGetDevice(&prev_dev);
    sg2v_status st = ensure_device(dev);
    if (st != SG2V_OK) return st;
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev_dev};
    const bool u64mode = o.precision == SG2V_U64;
    std::vector<double> resf((size_t)m * n_iter, 0.0);
    std::vector<uint64_t> resu((size_t)m * n_iter, 0);
    int ovf = 0;
    cudaStream_t s = (cudaStream_t)o.stream;

    if (k == 1 || g->n == 0) {
        // single-vertex template: every vertex is a colourful embedding; empty graph: 0
        for (auto &x : resf) x = (double)g->n;
        for (auto &x : resu) x = (uint64_t)g->n;
        if (o.row_values && g->n > 0) {
            std::vector<uint64_t> ones_u(g->n, 1);
            std::vector<double> ones_f(g->n, 1.0);
            const void *srcp = u64mode ? (const void *)ones_u.data() : (const void *)ones_f.data();
            SG2V_CK(cudaMemcpy(o.row_values, srcp, g->n * 8, cudaMemcpyHostToDevice));
        }
    } else {
        std::vector<Plan *> pls;
        st = batch_plans(g, ts, m, o.precision, o.layout, true, o.mem_budget_bytes, pls);
        if (st != SG2V_OK) return st;
        JointPlan J;
        if (pls.size() > 1) joint_schedule(pls, J);
        const BatchLayout L = batch_layout(pls, g->n, g->nnz, pls.size() > 1 ? J.tables_bytes : -1);
        char *ws = (char *)o.workspace;
        bool own = false;
        if (ws) {
            if (o.workspace_bytes < (uint64_t)L.bytes) {
                set_error("workspace too small: need " + std::to_string(L.bytes) + " bytes");
                return SG2V_ENOMEM;
            }
        } else {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            uint64_t budget = o.mem_budget_bytes ? o.mem_budget_bytes : (uint64_t)fr;
            if ((uint64_t)L.bytes > budget) {
                set_error("ENOMEM: plan needs " + std::to_string(L.bytes) + " bytes of device memory, budget " +
                          std::to_string(budget));
                return SG2V_ENOMEM;
            }
            keep_pool(dev);
            SG2V_CK(cudaMallocAsync((void **)&ws, L.bytes, s));
            own = true;
        }
        struct Free { char *p; bool own; cudaStream_t s; ~Free() { if (own) cudaFreeAsync(p, s); } } freer{ws, own, s};
        if (o.mem_budget_bytes && (uint64_t)L.bytes > o.mem_budget_bytes) {
            set_error("ENOMEM: plan needs " + std::to_string(L.bytes) + " bytes, budget " +
                      std::to_string(o.mem_budget_bytes));
            return SG2V_ENOMEM;
        }
        uint8_t *colors = (uint8_t *)(ws + L.off_colors);
        void *H = ws + L.off_hist;
        void *rowval = ws + L.off_rowval;
        void *partial = ws + L.off_partial;
        char *results = ws + L.off_results;
        int32_t *hcnt = (int32_t *)(ws + L.off_hcnt);
        int32_t *bcol = (int32_t *)(ws + L.off_bcol);
        int *dflag = (int *)(ws + L.off_flag);
        // split eMA pipeline: an aux stream + events when some step uses it (SG2V_SPLIT=0 off)
        static int split_on = -1;
        if (split_on < 0) { const char *e = getenv("SG2V_SPLIT"); split_on = e ? atoi(e) : 1; }
        SplitCtx sp;
        struct SplitFree {
            SplitCtx &c;
            ~SplitFree() {
                for (int q = 0; q < 2; ++q) {
                    if (c.ready[q]) cudaEventDestroy(c.ready[q]);
                    if (c.done[q]) cudaEventDestroy(c.done[q]);
                }
                if (c.aux) cudaStreamDestroy((cudaStream_t)c.aux);
            }
        } split_free{sp};
        bool any_split = false;
        for (Plan *p : pls)
            for (const Step &stp : p->steps) any_split = any_split || (stp.split_ema && split_on);
        if (any_split) {
            cudaStream_t aux;
            SG2V_CK(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
            sp.aux = aux;
            for (int q = 0; q < 2; ++q) {
                SG2V_CK(cudaEventCreateWithFlags(&sp.ready[q], cudaEventDisableTiming));
                SG2V_CK(cudaEventCreateWithFlags(&sp.done[q], cudaEventDisableTiming));
            }
            sp.bg = ws + L.off_split;
        }
        const bool anch = pls[0]->layout == LAYOUT_ANCHORED;
        // colour-grouped row order for the steps gathering exclusion-projected segments of
        // >= 1 KB: the light rows sorted by c(i) each colouring (launch_colour_order), so the
        // rows in flight read the same segment of the hub rows; scratch on the call's stream
        // (SG2V_CORDER=0 disables; measured u15-1 0.565 -> 0.539 s: the top, steps 5-7 read the
        //  hub rows' segment c(i) while it is hot in L2, ncu-visible as alg frac > 1 on the top)
        static int corder = -1;
        if (corder < 0) { const char *e = getenv("SG2V_CORDER"); corder = e ? atoi(e) : 1; }
        bool any_proj = false;
        for (Plan *p : pls)
            for (const Step &stp : p->steps) any_proj = any_proj || (stp.proj_p && stp.ldseg_p * p->elem >= 1024);
        int32_t *order_c = nullptr;
        uint8_t *ckeys = nullptr;
        void *ctmp = nullptr;
        size_t ctmp_bytes = 0;
        struct CFree {
            int32_t *&a; uint8_t *&b; void *&c; cudaStream_t s;
            ~CFree() { if (a) cudaFreeAsync(a, s); if (b) cudaFreeAsync(b, s); if (c) cudaFreeAsync(c, s); }
        } cfree{order_c, ckeys, ctmp, s};
        if (corder && anch && any_proj && g->n > 0) {
            ctmp_bytes = colour_order_tmp_bytes(g->n);
            SG2V_CK(cudaMallocAsync((void **)&order_c, g->n * sizeof(int32_t), s));
            SG2V_CK(cudaMallocAsync((void **)&ckeys, 2 * g->n, s));
            SG2V_CK(cudaMallocAsync(&ctmp, std::max<size_t>(ctmp_bytes, 16), s));
        }
        Graph gco = static_cast<const Graph &>(*g);
        if (order_c) gco.d_order = order_c;
        bool need_hist = false;
        for (Plan *p : pls) need_hist = need_hist || p->need_hist;
        std::vector<uint64_t> host_ring((size_t)kResultsRing * m);
        int64_t base = 0;
        if (!u64mode) SG2V_CK((cudaError_t)ovf_reset(dflag, s));
        for (int64_t q = 0; q < n_iter; ++q) {
            const int64_t j = o.iter_offset + q * o.iter_stride;
            int rc = launch_colorize(seed, j, g->n, k, colors, s, g->d_orig);
            if (rc) return cuda_fail("colorize", rc);
            if (need_hist && (rc = launch_hist(*g, *pls[0], colors, H, s))) return cuda_fail("hist", rc);
            if (anch && (rc = launch_bucket(*g, *pls[0], colors, hcnt, bcol, s))) return cuda_fail("bucket", rc);
            if (order_c && (rc = launch_colour_order(*g, colors, order_c, ckeys, ctmp, ctmp_bytes, s)))
                return cuda_fail("colour order", rc);
            for (int32_t tq = 0; tq < m; ++tq) {
                const Plan *pl = pls.size() > 1 ? &J.views[tq] : pls[tq];
                for (const Step &stp : pl->steps) {
                    // (segments >= 1 KB: narrower segments of many rows read at the same offset
                    //  measured slower — u15-1 step 4, 320 B: 20.6 -> 23.5 ms)
                    const bool cgroup = order_c && stp.proj_p && stp.ldseg_p * pl->elem >= 1024;
                    const Graph &gs = cgroup ? gco : static_cast<const Graph &>(*g);
                    if (anch && stp.split_ema && sp.aux) {
                        sp.rows = pl->split_rows;
                        rc = launch_astep_split(gs, *pl, stp, colors, hcnt, bcol, ws, rowval, dflag, s, sp);
                    } else {
                        rc = anch ? launch_astep(gs, *pl, stp, colors, hcnt, bcol, ws, rowval, dflag, s)
                                  : launch_step(*g, *pl, stp, colors, H, ws, rowval, dflag, s);
                    }
                    if (rc == -1) {
                        set_error("row too wide for on-chip B (shared memory > 227 KB)");
                        return SG2V_ENOMEM;
                    }
                    if (rc) return cuda_fail("step", rc);
                }
                rc = launch_reduce(*pl, g->n, rowval, partial, results + ((q - base) * m + tq) * 8, s);
                if (rc) return cuda_fail("reduce", rc);
            }
            if (q - base + 1 == kResultsRing || q == n_iter - 1) {
                int64_t cnt = q - base + 1;
                SG2V_CK(cudaMemcpyAsync(host_ring.data(), results, cnt * m * 8, cudaMemcpyDeviceToHost, s));
                SG2V_CK(cudaStreamSynchronize(s));
                for (int64_t r = 0; r < cnt; ++r)
                    for (int32_t tq = 0; tq < m; ++tq) {
                        const uint64_t bits = host_ring[(size_t)(r * m + tq)];
                        const size_t dst = (size_t)tq * n_iter + (size_t)(base + r);
                        if (u64mode) resu[dst] = bits;
                        else std::memcpy(&resf[dst], &bits, 8);
                    }
                base = q + 1;
            }
        }
        if (o.row_values) {
            SG2V_CK(cudaMemcpyAsync(o.row_values, rowval, g->n * 8, cudaMemcpyDeviceToDevice, s));
            SG2V_CK(cudaStreamSynchronize(s));
        }
        if (!u64mode) SG2V_CK((cudaError_t)ovf_read(dflag, &ovf, s));
    }
    bool finite = ovf == 0;  // a stored F32 table entry overflowed (set by the step kernels)
    for (int32_t tq = 0; tq < m; ++tq) {
        double sum = 0.0;
        for (int64_t q = 0; q < n_iter; ++q) {
            const size_t at = (size_t)tq * n_iter + (size_t)q;
            if (colorful_out) colorful_out[at] = u64mode ? (double)resu[at] : resf[at];
            if (colorful_u64_out) colorful_u64_out[at] = u64mode ? resu[at] : (uint64_t)resf[at];
            if (!u64mode) {
                if (!std::isfinite(resf[at])) finite = false;
                sum += resf[at];
            }
        }
        if (estimates)
            estimates[tq] = u64mode ? std::nan("") : sum / (double)n_iter / (ts[tq]->P * ts[tq]->alpha);
    }
    if (!finite) {
        set_error("EOVERFLOW: a colourful count is not finite in F32 (use F64 or U64)");
        return SG2V_EOVERFLOW;
    }
    return SG2V_OK;
}

}  // namespace sg2v

extern "C" {

sg2v_status sg2v_count_ex(const sg2v_graph *g, const sg2v_template *t, int32_t k, int64_t n_iter, uint64_t seed,
                          const sg2v_options *op, double *estimate_out, double *colorful_out,
                          uint64_t *colorful_u64_out) {
    if (!t) { set_error("graph or template is NULL"); return SG2V_EINVAL; }
    const sg2v_template *ts[1] = {t};
    return count_core(g, ts, 1, k, n_iter, seed, op, estimate_out, colorful_out, colorful_u64_out);
}

sg2v_status sg2v_count_batch(const sg2v_graph *g, const sg2v_template *const *templates, int32_t m, int32_t k,
                             int64_t n_iter, uint64_t seed, const sg2v_options *o, double *estimates_out,
                             double *colorful_out, uint64_t *colorful_u64_out) {
    return count_core(g, templates, m, k, n_iter, seed, o, estimates_out, colorful_out, colorful_u64_out);
}

sg2v_status sg2v_workspace_bytes_batch(const sg2v_graph *g, const sg2v_template *const *templates, int32_t m,
                                       sg2v_precision prec, uint64_t *bytes) {
    if (!g || !templates || m < 1 || !bytes) { set_error("NULL argument"); return SG2V_EINVAL; }
    if (prec < SG2V_F32 || prec > SG2V_U64) { set_error("bad precision"); return SG2V_EINVAL; }
    for (int32_t q = 0; q < m; ++q)
        if (!templates[q]) { set_error("template is NULL"); return SG2V_EINVAL; }
    std::vector<Plan *> pls;
    sg2v_status st = batch_plans(g, templates, m, prec, tls_layout(), false, tls_budget(), pls);
    if (st != SG2V_OK) return st;
    JointPlan J;
    if (pls.size() > 1) joint_schedule(pls, J);
    *bytes = pls.empty() ? 0 : (uint64_t)batch_layout(pls, g->n, g->nnz, pls.size() > 1 ? J.tables_bytes : -1).bytes;
    return SG2V_OK;
}

sg2v_status sg2v_estimate(const sg2v_template *t, int64_t n_iter, const double *colorful, double *estimate_out) {
    if (!t || !colorful || !estimate_out || n_iter < 1) { set_error("bad argument"); return SG2V_EINVAL; }
    double sum = 0.0;
    bool finite = true;
    for (int64_t q = 0; q < n_iter; ++q) {
        finite = finite && std::isfinite(colorful[q]);
        sum += colorful[q];
    }
    *estimate_out = sum / (double)n_iter / (t->P * t->alpha);
    if (!finite) { set_error("EOVERFLOW: a colourful count is not finite"); return SG2V_EOVERFLOW; }
    return SG2V_OK;
}

sg2v_status sg2v_count(const sg2v_graph *g, const sg2v_template *t, int32_t k, int64_t n_iter, uint64_t seed,
                       double *estimate_out, double *colorful_out, uint64_t *colorful_u64_out) {
    return sg2v_count_ex(g, t, k, n_iter, seed, nullptr, estimate_out, colorful_out, colorful_u64_out);
}

sg2v_status sg2v_comm_unique_id(uint8_t id_out[128]) {
    if (!id_out) { set_error("NULL argument"); return SG2V_EINVAL; }
    if (!nccl_api().ok) { set_error("libnccl.so.2 not available"); return SG2V_ENCCL; }
    ncclUniqueId id;
    ncclResult_t r = nccl_api().getUniqueId(&id);
    if (r != ncclSuccess) { set_error(std::string("ncclGetUniqueId: ") + nccl_api().getErrorString(r)); return SG2V_ENCCL; }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id_out, &id, 128);
    return SG2V_OK;
}

sg2v_status sg2v_comm_init_nccl(const uint8_t id[128], int32_t rank, int32_t world, sg2v_comm **out) {
    if (!id || !out || world < 1 || rank < 0 || rank >= world) { set_error("bad argument"); return SG2V_EINVAL; }
    if (!nccl_api().ok) { set_error("libnccl.so.2 not available"); return SG2V_ENCCL; }
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    auto *c = new sg2v_comm();
    c->rank = rank;
    c->world = world;
    ncclResult_t r = nccl_api().commInitRank(&c->nccl, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        set_error(std::string("ncclCommInitRank: ") + nccl_api().getErrorString(r));
        return SG2V_ENCCL;
    }
    *out = c;
    return SG2V_OK;
}

sg2v_status sg2v_comm_init_callback(int32_t rank, int32_t world, sg2v_allgather_fn fn, void *user, sg2v_comm **out) {
    if (!fn || !out || world < 1 || rank < 0 || rank >= world) { set_error("bad argument"); return SG2V_EINVAL; }
    auto *c = new sg2v_comm();
    c->rank = rank;
    c->world = world;
    c->cb = fn;
    c->user = user;
    *out = c;
    return SG2V_OK;
}

void sg2v_comm_free(sg2v_comm *c) {
    if (!c) return;
    if (c->nccl) nccl_api().commDestroy(c->nccl);
    if (c->hsend) cudaFreeHost(c->hsend);
    if (c->hrecv) cudaFreeHost(c->hrecv);
    delete c;
}

sg2v_status sg2v_graph_load_partition(int64_t n_global, int64_t row_begin, int64_t n_local,
                                      const int64_t *row_offsets, const int32_t *col_indices, int64_t nnz,
                                      uint32_t flags, sg2v_graph **out) {
    if (n_global < 0 || row_begin < 0 || n_local < 0 || row_begin + n_local > n_global) {
        set_error("partition out of range");
        return SG2V_EINVAL;
    }
    if (flags & SG2V_GRAPH_VALIDATE) { set_error("VALIDATE needs the whole graph (use sg2v_graph_load_csr)"); return SG2V_EINVAL; }
    sg2v_status st = sg2v_graph_load_csr(n_local, row_offsets, col_indices, nnz, flags, out);
    if (st != SG2V_OK) return st;
    (*out)->partitioned = true;
    (*out)->n_global = n_global;
    (*out)->row_begin = row_begin;
    return SG2V_OK;
}

sg2v_status sg2v_graph_set_vertex_ids(sg2v_graph *g, const int32_t *orig_ids, int64_t count) {
    if (!g || (count > 0 && !orig_ids)) { set_error("NULL argument"); return SG2V_EINVAL; }
    const int64_t want = g->partitioned ? g->n_global : g->n;
    if (count != want) { set_error("count must be n (n_global for a partition)"); return SG2V_EINVAL; }
    for (int64_t v = 0; v < count; ++v)
        if (orig_ids[v] < 0) { set_error("vertex ids must be non-negative"); return SG2V_EINVAL; }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(g->device);
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{cur};
    if (g->d_orig) { cudaFree(g->d_orig); g->d_orig = nullptr; }
    if (count == 0) return SG2V_OK;
    SG2V_CK(cudaMalloc((void **)&g->d_orig, count * sizeof(int32_t)));
    SG2V_CK(cudaMemcpy(g->d_orig, orig_ids, count * sizeof(int32_t), cudaMemcpyHostToDevice));
    return SG2V_OK;
}

sg2v_status sg2v_partition_relabel(int64_t n, const int64_t *row_offsets, const int32_t *col_indices, int32_t world,
                                   int32_t *old_of_new, int64_t *ro_out, int32_t *ci_out) {
    if (n < 0 || world < 1 || !row_offsets || !old_of_new || !ro_out || (row_offsets[n] > 0 && (!col_indices || !ci_out))) {
        set_error("bad argument");
        return SG2V_EINVAL;
    }
    // blocks of nl consecutive new ids (the last one shorter); vertices dealt by degree,
    // heaviest first, in snake order over the blocks that still have room, so every block
    // gets a near-equal share of the edges (nnz) as well as of the rows
    const int64_t nl = (n + world - 1) / world;
    std::vector<int64_t> cap(world), fill(world, 0);
    for (int r = 0; r < world; ++r) cap[r] = std::max<int64_t>(0, std::min(nl, n - (int64_t)r * nl));
    std::vector<int32_t> by_deg(n);
    for (int64_t v = 0; v < n; ++v) by_deg[v] = (int32_t)v;
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int32_t a, int32_t b) {
        return row_offsets[a + 1] - row_offsets[a] > row_offsets[b + 1] - row_offsets[b];
    });
    std::vector<int32_t> new_of_old(n);
    int r = 0, dir = 1;
    for (int64_t q = 0; q < n; ++q) {
        int guard = 0;
        while (fill[r] >= cap[r] && guard++ < 2 * world) {  // skip full blocks
            r += dir;
            if (r == world) { r = world - 1; dir = -1; }
            if (r < 0) { r = 0; dir = 1; }
        }
        const int32_t v = by_deg[q];
        const int64_t id = (int64_t)r * nl + fill[r]++;
        new_of_old[v] = (int32_t)id;
        old_of_new[id] = v;
        r += dir;
        if (r == world) { r = world - 1; dir = -1; }
        if (r < 0) { r = 0; dir = 1; }
    }
    // relabelled CSR: row u = old row old_of_new[u], columns mapped and sorted
    ro_out[0] = 0;
    for (int64_t u = 0; u < n; ++u) {
        const int32_t v = old_of_new[u];
        const int64_t d = row_offsets[v + 1] - row_offsets[v];
        ro_out[u + 1] = ro_out[u] + d;
        int32_t *dst = ci_out + ro_out[u];
        for (int64_t e = 0; e < d; ++e) dst[e] = new_of_old[col_indices[row_offsets[v] + e]];
        std::sort(dst, dst + d);
    }
    return SG2V_OK;
}

sg2v_status sg2v_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof) { g_ev_pool.push_back(r.a); g_ev_pool.push_back(r.b); }
    g_prof.clear();
    g_kernels.store(0);
    g_prof_on = on != 0;
    return SG2V_OK;
}

sg2v_status sg2v_profile_kernel_count(uint64_t *n_out) {
    if (!n_out) {
        set_error("NULL argument");
        return SG2V_EINVAL;
    }
    *n_out = g_kernels.load();
    return SG2V_OK;
}

sg2v_status sg2v_profile_read_launches(int64_t cap, int32_t *cls, double *ms, double *alg_bytes,
                                       double *impl_bytes, double *ema_terms, int64_t *n_out) {
    if (!n_out || (cap > 0 && (!cls || !ms || !alg_bytes || !impl_bytes || !ema_terms))) {
        set_error("NULL argument");
        return SG2V_EINVAL;
    }
    std::lock_guard<std::mutex> lk(g_prof_mu);
    *n_out = (int64_t)g_prof.size();
    for (int64_t q = 0; q < cap && q < (int64_t)g_prof.size(); ++q) {
        const ProfRec &r = g_prof[(size_t)q];
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail("profile event", e);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        cls[q] = r.cls;
        ms[q] = t;
        alg_bytes[q] = r.bytes;
        impl_bytes[q] = r.impl;
        ema_terms[q] = r.terms;
    }
    return SG2V_OK;
}

sg2v_status sg2v_profile_read(int64_t launches[5], double ms[5], double bytes[5]) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int c = 0; c < 5; ++c) { launches[c] = 0; ms[c] = 0.0; bytes[c] = 0.0; }
    for (auto &r : g_prof) {
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail("profile event", e);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        launches[r.cls] += 1;
        ms[r.cls] += t;
        bytes[r.cls] += r.bytes;
    }
    return SG2V_OK;
}

}  // extern "C"
