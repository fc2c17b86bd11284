// planner.cpp — host planner of the colour-coding DP (layer P of SURVEY §1).
//
//  * template validation + α = |Aut(T)| (unrooted, AHU canonical forms)
//  * partition search: root ρ and cut order chosen by a cost
//    model of the B200 kernels (the count is invariant, SURVEY finding 1)
//  * children-first schedule ordered to minimise the peak live set,
//    with each table freed right after its parent's eMA
//  * workspace layout (first-fit arena) and the colour-set index tables:
//    column I_s of a colour set S is its COLEX rank among |S|-subsets of [k]
//    (the paper leaves the map open; the oracle uses lexicographic on
//    purpose so the two share nothing).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <set>
#include <sstream>

#include "sg2v_internal.h"

namespace sg2v {

int64_t binom(int n, int r) {
    if (r < 0 || n < 0 || r > n) return 0;
    static int64_t tab[33][33];
    static bool init = false;
    if (!init) {
        for (int a = 0; a <= 32; ++a) {
            tab[a][0] = 1;
            for (int b = 1; b <= 32; ++b) tab[a][b] = (a == 0) ? 0 : tab[a - 1][b - 1] + tab[a - 1][b];
        }
        init = true;
    }
    return tab[n][r];
}

// colex rank of a subset mask among subsets of equal size: Σ_t C(e_t, t+1)
static int64_t colex_rank(uint32_t mask) {
    int64_t r = 0;
    int t = 0;
    while (mask) {
        int e = __builtin_ctz(mask);
        mask &= mask - 1;
        r += binom(e, t + 1);
        ++t;
    }
    return r;
}

// every s-subset of [k] in increasing mask order (= colex order), Gosper's hack
static void for_each_subset(int k, int s, const std::function<void(uint32_t)> &f) {
    if (s == 0) { f(0u); return; }
    uint64_t m = (1ull << s) - 1, lim = 1ull << k;
    while (m < lim) {
        f((uint32_t)m);
        uint64_t c = m & (~m + 1), r = m + c;
        m = (((r ^ m) >> 2) / c) | r;
    }
}

// ---------------------------------------------------------------------------
sg2v_status validate_template(int k, const int32_t *edges, Template &t) {
    if (k < 1 || k > 31) { set_error("k must be in [1, 31]"); return SG2V_EINVAL; }
    if (k > 1 && !edges) { set_error("edges is NULL"); return SG2V_EINVAL; }
    t.k = k;
    t.adj.assign(k, {});
    t.edges.clear();
    for (int e = 0; e < k - 1; ++e) {
        int u = edges[2 * e], v = edges[2 * e + 1];
        if (u < 0 || v < 0 || u >= k || v >= k) { set_error("template vertex id out of [0,k)"); return SG2V_ENOTTREE; }
        if (u == v) { set_error("template has a self-loop"); return SG2V_ENOTTREE; }
        if (std::find(t.adj[u].begin(), t.adj[u].end(), v) != t.adj[u].end()) {
            set_error("template has a duplicate edge");
            return SG2V_ENOTTREE;
        }
        t.adj[u].push_back(v);
        t.adj[v].push_back(u);
        t.edges.push_back({u, v});
    }
    std::vector<int> seen(k, 0), stack{0};
    seen[0] = 1;
    int cnt = 1;
    while (!stack.empty()) {
        int v = stack.back();
        stack.pop_back();
        for (int w : t.adj[v])
            if (!seen[w]) { seen[w] = 1; ++cnt; stack.push_back(w); }
    }
    if (cnt != k) { set_error("template is not connected (not a tree)"); return SG2V_ENOTTREE; }
    for (auto &a : t.adj) std::sort(a.begin(), a.end());
    return SG2V_OK;
}

// AHU: canonical string + automorphism count of the subtree at v (parent excluded)
static std::pair<std::string, double> ahu(const Template &t, int v, int parent) {
    std::vector<std::pair<std::string, double>> kids;
    for (int c : t.adj[v])
        if (c != parent) kids.push_back(ahu(t, c, v));
    std::sort(kids.begin(), kids.end());
    double aut = 1.0;
    std::string canon = "(";
    for (size_t i = 0; i < kids.size();) {
        size_t j = i;
        while (j < kids.size() && kids[j].first == kids[i].first) ++j;
        for (size_t q = i; q < j; ++q) { aut *= kids[q].second; canon += kids[q].first; }
        for (size_t m = 2; m <= j - i; ++m) aut *= (double)m;   // permute identical subtrees
        i = j;
    }
    canon += ")";
    return {canon, aut};
}

double automorphisms(const Template &t) {
    int k = t.k;
    if (k <= 2) return k == 1 ? 1.0 : 2.0;
    std::vector<int> deg(k);
    std::vector<int> layer;
    for (int v = 0; v < k; ++v) {
        deg[v] = (int)t.adj[v].size();
        if (deg[v] == 1) layer.push_back(v);
    }
    int left = k;
    while (left > 2) {                       // strip leaves to the centre
        left -= (int)layer.size();
        std::vector<int> nxt;
        for (int v : layer)
            for (int u : t.adj[v])
                if (--deg[u] == 1) nxt.push_back(u);
        layer = nxt;
    }
    if (layer.size() == 1) return ahu(t, layer[0], -1).second;
    auto a = ahu(t, layer[0], layer[1]);
    auto b = ahu(t, layer[1], layer[0]);
    return a.second * b.second * (a.first == b.first ? 2.0 : 1.0);
}

// ---------------------------------------------------------------------------
// Partition for a given root and child order.
// ---------------------------------------------------------------------------
struct Chain {
    std::vector<Node> nodes;
    int top = -1;
};

static Chain build_chain(const Template &t, int root, int policy) {
    int k = t.k;
    std::vector<std::vector<int>> children(k);
    std::vector<int> sub(k, 1), parent(k, -1), order;
    std::vector<int> st{root};
    parent[root] = root;
    while (!st.empty()) {
        int v = st.back();
        st.pop_back();
        order.push_back(v);
        for (int w : t.adj[v])
            if (parent[w] < 0) { parent[w] = v; children[v].push_back(w); st.push_back(w); }
    }
    for (int i = (int)order.size() - 1; i >= 0; --i) {
        int v = order[i];
        for (int c : children[v]) sub[v] += sub[c];
    }
    for (int v = 0; v < k; ++v) {
        auto &ch = children[v];
        if (policy == 0)       // smallest subtree cut first (ties: lowest id)
            std::sort(ch.begin(), ch.end(), [&](int a, int b) { return sub[a] != sub[b] ? sub[a] < sub[b] : a < b; });
        else if (policy == 1)  // largest subtree cut first
            std::sort(ch.begin(), ch.end(), [&](int a, int b) { return sub[a] != sub[b] ? sub[a] > sub[b] : a < b; });
        else
            std::sort(ch.begin(), ch.end());
    }
    Chain c;
    std::function<int(int, int)> build = [&](int r, int j) -> int {
        Node nd;
        nd.r = r;
        nd.j = j;
        nd.size = 1;
        for (size_t q = j; q < children[r].size(); ++q) nd.size += sub[children[r][q]];
        if (j < (int)children[r].size()) {
            nd.active = build(r, j + 1);                 // keeps ρ
            nd.passive = build(children[r][j], 0);       // rooted at τ
        }
        c.nodes.push_back(nd);
        return (int)c.nodes.size() - 1;
    };
    c.top = build(root, 0);
    return c;
}

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static int pick_gt(int64_t cols, int vn) {
    // threads per row group: enough lanes that R=4 vectors per lane cover the row
    int64_t nvec = (cols + vn - 1) / vn;
    int64_t want = (nvec + 3) / 4;
    int gt = 4;
    while (gt < want && gt < 256) gt *= 2;
    return gt;
}


static constexpr double kHbm = 6.5e12;     // B/s, MEASURED_PEAKS hbm_gbs (planning only)
static constexpr double kTermRate = 5.0e11; // eMA terms/s (measured order of the index-driven eMA)

// Relabelling of colour sets for the root-colour-anchored layout:
// a set over [k] \ {e} is stored as a set over [k-1] by closing the gap at e.
static uint32_t drop_bit(uint32_t m, int e) { return ((m >> (e + 1)) << e) | (m & ((1u << e) - 1)); }
static uint32_t insert_gap(uint32_t m, int e) { return ((m >> e) << (e + 1)) | (m & ((1u << e) - 1)); }

// Row width of a count table for a node of `size` vertices.
static int64_t table_width(Layout L, int k, int size) {
    return L == LAYOUT_DENSE ? binom(k, size) : binom(k - 1, size - 1);
}

// Arena placement of buffers with the given alloc/free sequence (buffer id, alloc?).
// Returns the arena size and writes each buffer's offset (256-B aligned).
template <typename EvT>
static std::vector<std::pair<int, bool>> events_to_pairs(const std::vector<EvT> &e) {
    std::vector<std::pair<int, bool>> out;
    for (const auto &x : e) out.push_back({x.buf, x.alloc});
    return out;
}

static int64_t place_one(std::vector<Buffer> &bufs, const std::vector<std::pair<int, bool>> &ev,
                         const std::vector<int> &side_hint, bool two_sided) {
    std::vector<int> side(bufs.size(), 0);
    std::vector<int64_t> soff(bufs.size(), 0);                // offset from the side's origin
    std::vector<std::pair<int64_t, int64_t>> live[2];          // (offset, bytes) per side
    int64_t ext[2] = {0, 0}, H = 0;
    for (const auto &e : ev) {
        const int b = e.first;
        const int64_t bytes = round_up(std::max<int64_t>(bufs[b].bytes, 1), 256);
        if (e.second) {
            int sd = 0;
            if (two_sided && side_hint[b] >= 0) sd = 1 - side[side_hint[b]];
            side[b] = sd;
            auto &L = live[sd];
            std::sort(L.begin(), L.end());
            int64_t pos = 0;
            for (auto &iv : L) {
                if (iv.first - pos >= bytes) break;
                pos = std::max(pos, iv.first + iv.second);
            }
            L.push_back({pos, bytes});
            soff[b] = pos;
            ext[sd] = 0;
            for (auto &iv : L) ext[sd] = std::max(ext[sd], iv.first + iv.second);
            H = std::max(H, ext[0] + ext[1]);
        } else {
            auto &L = live[side[b]];
            for (size_t q = 0; q < L.size(); ++q)
                if (L[q].first == soff[b]) { L.erase(L.begin() + q); break; }
            int64_t x = 0;
            for (auto &iv : L) x = std::max(x, iv.first + iv.second);
            ext[side[b]] = x;
        }
    }
    H = round_up(H, 256);
    for (size_t b = 0; b < bufs.size(); ++b)
        bufs[b].offset = side[b] == 0 ? soff[b] : H - soff[b] - round_up(std::max<int64_t>(bufs[b].bytes, 1), 256);
    return H;
}

static int64_t place_arena(std::vector<Buffer> &bufs, const std::vector<std::pair<int, bool>> &ev,
                           const std::vector<int> &side_hint) {
    std::vector<Buffer> one = bufs, two = bufs;
    const int64_t h1 = place_one(one, ev, side_hint, false);
    const int64_t h2 = place_one(two, ev, side_hint, true);
    bufs = h2 < h1 ? two : one;
    return std::min(h1, h2);
}

// Build steps, schedule, buffers and the model for one chain.
static bool plan_chain(const Template &t, const Chain &c, int root, int64_t n, int64_t nnz,
                       sg2v_precision prec, Layout L, Plan &pl, const std::set<std::string> &proj = {}) {
    const int k = t.k;
    pl = Plan();
    pl.proj = proj;
    pl.k = k;
    pl.root = root;
    pl.prec = prec;
    pl.layout = L;
    pl.elem = (prec == SG2V_F32) ? 4 : 8;
    const int vn = 16 / pl.elem;
    pl.nodes = c.nodes;
    const double E = pl.elem;
    const bool anch = (L == LAYOUT_ANCHORED);
    const double live_frac = anch ? (double)(k - 1) / k : 1.0;  // non-monochromatic edges (expected)

    // --- children-first order minimising the peak (Sethi–Ullman style) ---
    std::vector<int64_t> out_bytes(pl.nodes.size(), 0);
    for (size_t i = 0; i < pl.nodes.size(); ++i) {
        const Node &nd = pl.nodes[i];
        if (nd.active >= 0 && (int)i != c.top)
            out_bytes[i] = n * round_up(table_width(L, k, nd.size), vn) * pl.elem;
    }
    // canonical strings first (projected classes change the table sizes)
    std::vector<std::string> canon(pl.nodes.size());
    {
        std::vector<std::vector<std::string>> kids(pl.nodes.size());
        for (size_t v = 0; v < pl.nodes.size(); ++v) {  // children precede parents
            const Node &nd = pl.nodes[v];
            if (nd.active >= 0) {
                kids[v] = kids[nd.active];
                kids[v].push_back(canon[nd.passive]);
                std::sort(kids[v].begin(), kids[v].end());
            }
            std::string cs = "(";
            for (auto &x : kids[v]) cs += x;
            canon[v] = cs + ")";
        }
    }
    for (size_t i = 0; i < pl.nodes.size(); ++i) {
        const Node &nd = pl.nodes[i];
        if (nd.active >= 0 && (int)i != c.top && proj.count(canon[i]))
            out_bytes[i] += n * (int64_t)(k - 1) * round_up(binom(k - 2, nd.size - 1), vn) * pl.elem;
    }
    std::vector<int> sched;
    std::function<int64_t(int, std::vector<int> &)> order = [&](int v, std::vector<int> &seq) -> int64_t {
        const Node &nd = pl.nodes[v];
        if (nd.active < 0) return 0;
        std::vector<int> sa, sp;
        int64_t pa = order(nd.active, sa), pp = order(nd.passive, sp);
        int64_t oa = out_bytes[nd.active], op = out_bytes[nd.passive], os = out_bytes[v];
        int64_t first_a = std::max({pa, oa + pp, oa + op + os});
        int64_t first_p = std::max({pp, op + pa, oa + op + os});
        if (first_a <= first_p) {
            seq.insert(seq.end(), sa.begin(), sa.end());
            seq.insert(seq.end(), sp.begin(), sp.end());
        } else {
            seq.insert(seq.end(), sp.begin(), sp.end());
            seq.insert(seq.end(), sa.begin(), sa.end());
        }
        seq.push_back(v);
        return std::min(first_a, first_p);
    };
    {
        std::vector<int> full;
        order(c.top, full);
        (void)full;
    }
    // --- isomorphic rooted sub-templates share one table ---------------------
    // M_s(i, S) counts colourful embeddings of the ROOTED sub-template T_s with
    // its root at i, so it depends only on T_s's rooted isomorphism
    // class: compute each class once (e.g. the two arms of a path rooted at its
    // middle) and let every parent read it.  canon(node) = AHU string of the
    // rooted sub-template (children multiset, sorted; computed above).
    //
    // Self steps (anchored): T_s = root ρ + two isomorphic child subtrees X, split as
    // active = ρ + X (itself leaf-active over X) and passive = X.  The active row is
    // M_a(i,·) = B_X(i,·) with the same [k-1]-subset indexing as the step's own
    // B_X(i,·) (anchored leaf-active identity), so one gather of X's table gives both:
    // M_s(i,S) = Σ_{A⊂S} B_X(i,A)·B_X(i,S∖A).  The ρ + X table is never built.
    auto self_step = [&](int v) -> bool {
        if (!anch) return false;
        const Node &nd = pl.nodes[v];
        if (nd.active < 0) return false;
        const Node &na = pl.nodes[nd.active];
        return na.active >= 0 && pl.nodes[na.active].active < 0 && canon[na.passive] == canon[nd.passive];
    };
    {
        std::set<std::string> done;
        std::function<void(int)> visit = [&](int v) {
            const Node &nd = pl.nodes[v];
            if (nd.active < 0 || done.count(canon[v])) return;
            if (self_step(v)) {  // the active child is never materialised
                visit(nd.passive);
                done.insert(canon[v]);
                sched.push_back(v);
                return;
            }
            // Sethi–Ullman child order of the tree without sharing
            std::vector<int> sa, sp;
            int64_t pa = order(nd.active, sa), pp = order(nd.passive, sp);
            int64_t oa = out_bytes[nd.active], op = out_bytes[nd.passive];
            if (std::max(pa, oa + pp) <= std::max(pp, op + pa)) { visit(nd.active); visit(nd.passive); }
            else { visit(nd.passive); visit(nd.active); }
            done.insert(canon[v]);
            sched.push_back(v);
        };
        visit(c.top);
    }
    // Exclusion-projected tables: a class read as the PASSIVE side of row-streaming
    // gathers may (also) be stored as k-1 segments per row, one per consumer colour
    // y ≠ c(i), holding the sets that avoid y (C(k-2,s-1) entries): a consumer of
    // colour c(i) streams exactly the sets it can use instead of the whole C(k-1,s-1)
    // row (where a fraction (s-1)/(k-1) contain c(i) and are discarded), for k-s times
    // the table memory.  A class that is also read as an active child M_a (or by a
    // top step with a leaf active child, one column per edge) keeps its plain table
    // too ("dual").  The planner picks the classes (make_plan).
    // gather_reader(v): step v streams its passive child's rows
    auto gather_reader = [&](int v) {
        const Node &nd = pl.nodes[v];
        return anch && pl.nodes[nd.passive].size > 1 && !(v == c.top && pl.nodes[nd.active].size == 1);
    };
    {
        std::set<std::string> seen;
        for (int v : sched)
            if (gather_reader(v) && !seen.count(canon[pl.nodes[v].passive])) {
                seen.insert(canon[pl.nodes[v].passive]);
                pl.proj_cands.push_back(canon[pl.nodes[v].passive]);
            }
    }
    // table key read by step v for its passive child: the projected copy when the class
    // is projected and v streams it, else the plain table
    auto pkey = [&](int v) {
        const std::string &cp = canon[pl.nodes[v].passive];
        return proj.count(cp) && gather_reader(v) ? cp + "|x" : cp;
    };
    // uses of each table by the scheduled steps (a table is freed after its last use)
    std::map<std::string, int> uses;
    for (int v : sched) {
        if (!self_step(v)) uses[canon[pl.nodes[v].active]]++;
        uses[pkey(v)]++;
    }

    // --- table arena over the schedule ---
    // Buffers are recorded as alloc / free events in schedule order and placed after
    // the loop (place_arena): one-sided first fit, or two-sided (a step's output goes
    // to the side opposite its passive input, so a chain of steps ping-pongs between
    // the two ends instead of leaving holes too small for the next, wider table);
    // the smaller arena wins.
    std::map<std::string, int> class_buf;   // canon -> buffer
    std::vector<int> node_buf(pl.nodes.size(), -1);
    struct Ev { int buf; bool alloc; };
    std::vector<Ev> events;
    std::vector<int> side_hint;             // per buffer: the buffer whose side it should avoid (-1: none)
    auto alloc = [&](int64_t bytes, int avoid) -> int64_t {
        Buffer b;
        b.bytes = bytes;
        b.offset = 0;
        pl.bufs.push_back(b);
        side_hint.push_back(avoid);
        events.push_back({(int)pl.bufs.size() - 1, true});
        return 0;
    };
    auto release = [&](int b) {
        if (b >= 0) events.push_back({b, false});
    };

    double model = 0.0, alg_total = 0.0;
    for (int v : sched) {
        const Node &nd = pl.nodes[v];
        Step st;
        st.node = v;
        st.s = nd.size;
        st.a = pl.nodes[nd.active].size;
        st.p = pl.nodes[nd.passive].size;
        st.top = (v == c.top);
        st.src = (st.p == 1) ? SRC_HIST : SRC_GATHER;
        st.comb = (st.a == 1) ? COMB_ACTIVE_LEAF : COMB_GENERAL;
        st.cs = st.top ? 1 : table_width(L, k, st.s);
        st.ca = table_width(L, k, st.a);
        st.cp = table_width(L, k, st.p);
        st.cb = anch ? binom(k - 1, st.p) : st.cp;
        st.proj_out = !st.top && proj.count(canon[v]);
        st.plain_out = !st.top && uses.count(canon[v]) && uses[canon[v]] > 0;  // someone reads the plain table
        st.proj_p = st.src == SRC_GATHER && proj.count(canon[nd.passive]) && gather_reader(v);
        st.lds = st.top ? 1 : round_up(st.cs, vn);
        if (st.proj_out) {
            st.ldseg_out = round_up(binom(k - 2, st.s - 1), vn);
            st.ldsx = (int64_t)(k - 1) * st.ldseg_out;
        }
        st.lda = round_up(st.ca, vn);
        st.ldp = (st.src == SRC_HIST) ? round_up(k, vn) : round_up(st.cp, vn);
        if (st.proj_p) {  // gather width: one segment
            st.cp = binom(k - 2, st.p - 1);
            st.ldseg_p = round_up(st.cp, vn);
            st.ldp = (int64_t)(k - 1) * st.ldseg_p;
        }
        st.ldb = anch ? round_up(st.cb, vn) : st.ldp;
        st.self_a = self_step(v);
        st.canon_out = canon[v];
        st.canon_a = canon[nd.active];
        st.canon_p = pkey(v);
        st.buf_a = (!st.self_a && class_buf.count(st.canon_a)) ? class_buf[st.canon_a] : -1;
        st.buf_p = class_buf.count(st.canon_p) ? class_buf[st.canon_p] : -1;
        if (st.src == SRC_HIST && !anch) pl.need_hist = true;
        if (st.plain_out) {
            alloc(n * st.lds * pl.elem, st.buf_p);
            st.buf_out = (int)pl.bufs.size() - 1;
            node_buf[v] = st.buf_out;
            class_buf[st.canon_out] = st.buf_out;
        }
        if (st.proj_out) {
            alloc(n * st.ldsx * pl.elem, st.buf_p);
            st.buf_outx = (int)pl.bufs.size() - 1;
            class_buf[st.canon_out + "|x"] = st.buf_outx;
        }
        if (!st.self_a && --uses[st.canon_a] == 0) release(st.buf_a);
        if (--uses[st.canon_p] == 0) release(st.buf_p);

        // impl bytes (the implemented layout's compulsory traffic), the model
        // (sector-rounded) and below the method's algorithmic bytes
        double bytes = 0.0, mbytes = 0.0;
        const bool top_leaf = st.top && st.comb == COMB_ACTIVE_LEAF;
        const double hsrc = anch ? n * (double)round_up(k, 4) * 4.0 : n * (double)k * E;
        if (top_leaf) {
            if (st.src == SRC_GATHER) {
                bytes = nnz * 4.0 + nnz * live_frac * E + n * 9.0;
                mbytes = nnz * 4.0 + nnz * live_frac * 32.0 + n * 16.0;
            } else {
                bytes = mbytes = hsrc + n * 9.0;
            }
        } else {
            double gather = (st.src == SRC_GATHER)
                                ? nnz * 4.0 + nnz * live_frac * (double)st.cp * E + n * (12.0 + (anch ? 4.0 * k : 0.0))
                                : hsrc;
            double mg = (st.src == SRC_GATHER)
                            ? nnz * 4.0 + nnz * live_frac * (double)round_up(st.cp * pl.elem, 32) + n * 12.0
                            : hsrc;
            double ma = (st.comb == COMB_GENERAL && !st.self_a) ? n * (double)st.ca * E : n * 1.0;
            double w = st.top ? n * 8.0
                              : (st.plain_out ? n * (double)st.cs * E : 0.0) + (st.proj_out ? n * (double)st.ldsx * E : 0.0);
            bytes = gather + ma + w;
            mbytes = mg + ma + w;
            // GENERAL projected outputs are scattered 4/8-B stores (one per output and
            // segment): model a 32-B sector each (measured: u13-2's 8 = 7 + 1 projected ran
            // slower than the plain plan the model had ranked below it)
            if (st.proj_out && st.comb == COMB_GENERAL)
                mbytes += n * (double)st.cs * (double)(k - st.s) * (32.0 - E);
            if (anch && st.src == SRC_GATHER)  // per-row push of k-1 colour partial sums through smem
                mbytes += n * (double)(k - 1) * (double)st.cp * 4.0 * 0.1;
        }
        if (st.comb == COMB_GENERAL)
            st.nterms = anch ? (st.top ? binom(k - 1, st.a - 1) : binom(st.s - 1, st.a - 1))
                             : (st.top ? binom(k, st.a) : binom(st.s, st.a));
        else
            st.nterms = 1;
        st.ema_terms = (st.comb == COMB_GENERAL) ? (double)n * (double)st.cs * (double)st.nterms : 0.0;
        st.impl_bytes = bytes;
        {
            // SURVEY §8(d) per-step bytes of the method, independent of plain vs projected
            // tables: useful gather (anchored: each live edge carries the C(k-2,p-1) sets
            // avoiding c(i); dense: C(k,p)), CSR + per-row metadata, M_a, and the output
            // written once at plain width (top: one 8-B value per vertex)
            double u = 0.0;
            if (top_leaf) {
                u = st.src == SRC_GATHER ? nnz * 4.0 + nnz * live_frac * E + n * 9.0 : hsrc + n * 9.0;
            } else {
                const double useful_cols = anch ? (double)binom(k - 2, st.p - 1) : (double)binom(k, st.p);
                u = st.src == SRC_GATHER ? nnz * 4.0 + nnz * live_frac * useful_cols * E + n * (12.0 + (anch ? 4.0 * k : 0.0))
                                         : hsrc;
                u += (st.comb == COMB_GENERAL && !st.self_a) ? n * (double)table_width(L, k, st.a) * E : n * 1.0;
                u += st.top ? n * 8.0 : n * (double)table_width(L, k, st.s) * E;
            }
            st.alg_bytes = u;
        }
        {
            // eMA-heavy GENERAL steps run as the split two-stream pipeline
            // (launch_astep_split): same terms-per-byte test as the V-row eMA; gather rows of
            // >= 16 vectors (narrower ones gain nothing from a separate gather launch)
            const int64_t nvec_p = (st.proj_p ? st.ldseg_p : st.ldp) / vn;
            st.split_ema = anch && st.comb == COMB_GENERAL && !st.top && st.src == SRC_GATHER && st.nterms >= 8 &&
                           st.ema_terms >= 0.05 * bytes && nvec_p >= 16;
        }
        st.gt = pick_gt(std::max({st.ldp, st.ldb, st.lds, st.comb == COMB_GENERAL ? st.lda : 0}), vn);
        model += mbytes / kHbm + st.ema_terms / kTermRate;
        alg_total += st.alg_bytes;
        pl.impl_bytes_total += bytes;
        pl.steps.push_back(st);
    }
    pl.tables_bytes = place_arena(pl.bufs, events_to_pairs(events), side_hint);
    pl.ldh = round_up(k, vn);
    pl.kp = round_up(k, 4);
    pl.hist_bytes = pl.need_hist ? n * pl.ldh * pl.elem : 0;
    if (pl.need_hist) {
        double hb = nnz * 4.0 + nnz * 1.0 + n * 12.0 + n * (double)k * E;
        model += (nnz * 4.0 + nnz * 32.0 + pl.hist_bytes) / kHbm;
        alg_total += hb;
        pl.impl_bytes_total += hb;
    }
    if (anch) {  // colour counts + colour-bucketed CSR, once per colouring
        double bb = 2.0 * nnz * 4.0 + nnz * 4.0 + n * 16.0 + n * (double)pl.kp * 4.0;
        model += (bb + nnz * 32.0) / kHbm;
        alg_total += bb;
        pl.impl_bytes_total += bb;
    }
    pl.model_time = model;
    pl.alg_bytes_total = alg_total;

    // split eMA pipeline buffers: two chunks of B rows
    pl.n_rows = n;
    {
        int64_t ldb = 0;
        for (const Step &st : pl.steps)
            if (st.split_ema) ldb = std::max(ldb, st.ldb);
        // 32 chunks: the first chunk's gather (the hub rows) is the part the pipeline
        // cannot hide, so it is kept short
        pl.split_rows = ldb ? std::min<int64_t>(n, std::max<int64_t>(1024, (n + 31) / 32)) : 0;
        pl.split_bytes = 2 * pl.split_rows * ldb * pl.elem;
    }
    // workspace layout
    int64_t off = pl.tables_bytes;
    pl.off_colors = off;  off = round_up(off + std::max<int64_t>(n, 1) + 16, 256);
    pl.off_hist = off;    off = round_up(off + pl.hist_bytes, 256);
    pl.off_hcnt = off;    off = round_up(off + (anch ? n * pl.kp * 4 : 0), 256);
    pl.off_bcol = off;    off = round_up(off + (anch ? nnz * 4 : 0), 256);
    pl.off_rowval = off;  off = round_up(off + std::max<int64_t>(n, 1) * 8, 256);
    pl.off_partial = off; off = round_up(off + kReduceBlocks * 8, 256);
    pl.off_results = off; off = round_up(off + kResultsRing * 8, 256);
    pl.off_flag = off;    off = round_up(off + 16, 256);
    pl.off_split = off;   off = round_up(off + pl.split_bytes, 256);
    pl.ws_bytes = off;
    return true;
}

// Shared-memory bank schedule of the split terms of a GENERAL step (eMA).
// In the V-row eMA each lane owns one output o and reads, per term, the 16-B entries
// M_a(·, ia) and B(·, ib) of its V interleaved rows; a 128-bit shared load is served a
// quarter-warp (8 lanes = 8 consecutive outputs) at a time and is conflict-free only if
// the 8 entries fall in distinct 16-B bank groups (entry mod 8).  The sum over a
// row's terms is order-free (exact in U64; a fixed order in F32/F64), so the terms of
// each output are permuted, quarter by quarter and step by step, to spread both
// operands over the 8 groups (greedy over 8 x 8 (group_a, group_b) buckets).
// SG2V_EMA_SCHED=0 keeps the natural subset order (experiments).
static void schedule_terms(std::vector<std::pair<int32_t, int32_t>> &pairs, int64_t cs, int64_t nt, int64_t aoff) {
    static int on = -1;  // off by default: measured slower (u17 10 = 5 + 5: 780 -> 911 ms), the natural
                         // subset order lets adjacent outputs share entries (broadcast reads)
    if (on < 0) { const char *e = getenv("SG2V_EMA_SCHED"); on = e ? atoi(e) : 0; }
    if (!on) return;
    std::vector<std::pair<int32_t, int32_t>> out(pairs.size());
    for (int64_t o0 = 0; o0 < cs; o0 += 8) {
        const int L = (int)std::min<int64_t>(8, cs - o0);
        // per lane: terms bucketed by (group of M_a entry, group of B entry)
        std::vector<std::vector<int64_t>> bucket((size_t)L * 64);
        for (int l = 0; l < L; ++l)
            for (int64_t w = 0; w < nt; ++w) {
                const auto &pq = pairs[(size_t)((o0 + l) * nt + w)];
                const int ga = (int)((aoff + pq.first) & 7), gb = (int)(pq.second & 7);
                bucket[(size_t)l * 64 + ga * 8 + gb].push_back(w);
            }
        for (int64_t w = 0; w < nt; ++w) {
            unsigned usedA = 0, usedB = 0;
            for (int l = 0; l < L; ++l) {
                int best = -1, bestc = 99;
                for (int b = 0; b < 64 && bestc > 0; ++b) {
                    if (bucket[(size_t)l * 64 + b].empty()) continue;
                    const int c = ((usedA >> (b >> 3)) & 1) + ((usedB >> (b & 7)) & 1);
                    if (c < bestc) { bestc = c; best = b; }
                }
                auto &bk = bucket[(size_t)l * 64 + best];
                const int64_t src = bk.back();
                bk.pop_back();
                out[(size_t)((o0 + l) * nt + w)] = pairs[(size_t)((o0 + l) * nt + src)];
                usedA |= 1u << (best >> 3);
                usedB |= 1u << (best & 7);
            }
        }
    }
    pairs.swap(out);
}

static bool build_index(Plan &pl) {
    const int k = pl.k;
    const uint32_t full = (k == 32) ? 0xffffffffu : ((1u << k) - 1);
    const bool anch = pl.layout == LAYOUT_ANCHORED;
    const int K = anch ? k - 1 : k;                 // universe of the stored colour sets
    const uint32_t fullK = (K >= 32) ? 0xffffffffu : ((1u << K) - 1);
    pl.index.clear();
    auto align = [&]() { while (pl.index.size() % 4) pl.index.push_back(0); };
    std::map<int, int64_t> push_maps;               // anchored push map per passive size p
    std::map<int, int64_t> push_maps_x;             // ... for exclusion-projected sources
    // push-map rows [x][ci] are padded to a multiple of 4 entries (-1), so a lane reads the
    // targets of its 16-B vector with one aligned 16-B (F32) / 8-B (F64, U64) load
    auto pad_row = [&](size_t len) {
        for (size_t q = len; q % 4; ++q) pl.index.push_back(-1);
    };
    for (Step &st : pl.steps) {
        // ---- projected output: write map ----
        if (st.proj_out) {
            const int m = st.s - 1;  // stored sets: (s-1)-subsets of [k-1] (i's universe)
            align();
            st.omap_off = (int64_t)pl.index.size();
            if (st.comb == COMB_ACTIVE_LEAF) {
                // inverse: segment y', position u -> column of B(i,·) (= M_s(i,·)), -1 = pad
                std::vector<uint32_t> us;
                for_each_subset(k - 2, m, [&](uint32_t x) { us.push_back(x); });
                for (int y = 0; y < k - 1; ++y)
                    for (int64_t u = 0; u < st.ldseg_out; ++u)
                        pl.index.push_back(u < (int64_t)us.size() ? (int32_t)colex_rank(insert_gap(us[(size_t)u], y)) : -1);
            } else {
                // forward: output o, segment y' -> position in the segment, -1 if o ∋ y'
                for_each_subset(k - 1, m, [&](uint32_t S) {
                    for (int y = 0; y < k - 1; ++y)
                        pl.index.push_back((S >> y & 1u) ? -1 : (int32_t)colex_rank(drop_bit(S, y)));
                });
            }
        }
        // ---- anchored gather from a projected table: push map [x][ci][u] -> B column ----
        if (st.proj_p) {
            auto it = push_maps_x.find(st.p);
            if (it != push_maps_x.end()) {
                st.map_off = it->second;
            } else {
                align();
                st.map_off = (int64_t)pl.index.size();
                std::vector<uint32_t> us;  // (p-1)-subsets of [k] \ {x, ci}, relabelled into [k-2]
                for_each_subset(k - 2, st.p - 1, [&](uint32_t m) { us.push_back(m); });
                for (int x = 0; x < k; ++x)
                    for (int ci = 0; ci < k; ++ci) {
                        for (uint32_t u : us) {
                            int32_t tcol = -1;
                            if (x != ci) {
                                const int lo = std::min(x, ci), hi = std::max(x, ci);
                                const uint32_t U = insert_gap(insert_gap(u, lo), hi);  // subset of [k] \ {x, ci}
                                tcol = (int32_t)colex_rank(drop_bit(U | (1u << x), ci));
                            }
                            pl.index.push_back(tcol);
                        }
                        pad_row(us.size());
                    }
                push_maps_x[st.p] = st.map_off;
            }
        } else if (anch && st.src == SRC_GATHER && ((pl.vp && !pl.vp_full) || !(st.top && st.comb == COMB_ACTIVE_LEAF))) {
            auto it = push_maps.find(st.p);
            if (it != push_maps.end()) {
                st.map_off = it->second;
            } else {
                double need = (double)k * k * (double)st.cp;
                if (need > 1.5e9) { set_error("push map too large"); return false; }
                align();
                st.map_off = (int64_t)pl.index.size();
                std::vector<uint32_t> us;
                for_each_subset(k - 1, st.p - 1, [&](uint32_t m) { us.push_back(m); });
                for (int x = 0; x < k; ++x)
                    for (int ci = 0; ci < k; ++ci) {
                        for (uint32_t u : us) {
                            int32_t tcol = -1;
                            if (x != ci) {
                                uint32_t U = insert_gap(u, x);            // subset of [k] \ {x}
                                if (!(U >> ci & 1u))
                                    tcol = (int32_t)colex_rank(drop_bit(U | (1u << x), ci));
                            }
                            pl.index.push_back(tcol);
                        }
                        pad_row(us.size());
                    }
                push_maps[st.p] = st.map_off;
            }
        }
        align();
        st.idx_off = (int64_t)pl.index.size();
        if (st.top && st.comb == COMB_ACTIVE_LEAF && pl.vp && !pl.vp_full) {
            pl.index.push_back(0);  // vertex-partitioned: colorful_i = B(i, [k-1]) from bg (push map above)
        } else if (st.top && st.comb == COMB_ACTIVE_LEAF) {
            if (!anch) {
                // colorful_i = B(i, [k] \ {c(i)}): column per colour x
                for (int x = 0; x < k; ++x) pl.index.push_back((int32_t)colex_rank(full ^ (1u << x)));
            } else {
                // colorful_i = Σ_{x≠c(i)} Σ_{j: c(j)=x} M_p(j, [k]\{x,c(i)} relabelled wrt x): [x][ci]
                for (int x = 0; x < k; ++x)
                    for (int ci = 0; ci < k; ++ci)
                        pl.index.push_back(x == ci ? -1
                                                   : (int32_t)colex_rank(drop_bit(full & ~(1u << x) & ~(1u << ci), x)));
            }
            pl.top_leaf_col_off = (int)st.idx_off;
        } else if (st.comb == COMB_ACTIVE_LEAF) {
            if (!anch) {
                // M_s(i,S) = [c(i) ∈ S]·B(i, S \ {c(i)}): map[x][o]
                double need = (double)k * (double)st.cs;
                if (need > 1.5e9) { set_error("index table too large"); return false; }
                std::vector<uint32_t> outs;
                outs.reserve(st.cs);
                for_each_subset(k, st.s, [&](uint32_t m) { outs.push_back(m); });
                for (int x = 0; x < k; ++x)
                    for (uint32_t S : outs)
                        pl.index.push_back((S >> x & 1u) ? (int32_t)colex_rank(S ^ (1u << x)) : -1);
            }
            // anchored leaf-active: M_s(i,·) = B(i,·), no table
        } else {
            // GENERAL: (I_a, I_p) for every split of every output colour set;
            // anchored: universe [k-1], sizes (s-1, a-1, p) — one table for every vertex,
            // stored term-major (entry (w, o) at w*cs + o) and packed ia | ip << 16
            // when both ranks fit 16 bits; dense: output-major int2 pairs
            double need = 2.0 * (double)st.cs * (double)st.nterms;
            if (need > 1.5e9) { set_error("split table too large"); return false; }
            const int asz = anch ? st.a - 1 : st.a;
            std::vector<std::pair<int32_t, int32_t>> pairs;
            pairs.reserve((size_t)(st.cs * st.nterms));
            auto emit = [&](uint32_t S) {
                for (uint32_t sub = S;; sub = (sub - 1) & S) {
                    if (__builtin_popcount(sub) == asz)
                        pairs.push_back({(int32_t)colex_rank(sub), (int32_t)colex_rank(S ^ sub)});
                    if (sub == 0) break;
                }
            };
            if (st.top) emit(fullK);
            else for_each_subset(K, anch ? st.s - 1 : st.s, emit);
            if (!anch) {
                for (auto &pq : pairs) { pl.index.push_back(pq.first); pl.index.push_back(pq.second); }
            } else {
                st.packed = (st.ca < 65536 && st.cb < 65536) ? 1 : 0;
                const int64_t cs = st.cs, nt = st.nterms;
                if (!st.top && nt >= 8) schedule_terms(pairs, cs, nt, st.self_a ? 0 : st.ldb);
                if (st.packed) {
                    size_t base = pl.index.size();
                    pl.index.resize(base + (size_t)(cs * nt));
                    for (int64_t o = 0; o < cs; ++o)
                        for (int64_t w = 0; w < nt; ++w) {
                            const auto &pq = pairs[(size_t)(o * nt + w)];
                            pl.index[base + (size_t)(w * cs + o)] = (int32_t)((uint32_t)pq.first | ((uint32_t)pq.second << 16));
                        }
                } else {
                    size_t base = pl.index.size();
                    pl.index.resize(base + (size_t)(2 * cs * nt));
                    for (int64_t o = 0; o < cs; ++o)
                        for (int64_t w = 0; w < nt; ++w) {
                            const auto &pq = pairs[(size_t)(o * nt + w)];
                            pl.index[base + 2 * (size_t)(w * cs + o)] = pq.first;
                            pl.index[base + 2 * (size_t)(w * cs + o) + 1] = pq.second;
                        }
                }
            }
        }
    }
    if (pl.index.empty()) pl.index.push_back(0);
    return true;
}

// Fastest modelled plan whose workspace fits `budget` (0 = unlimited); when no
// plan fits, the smallest one (sg2v_count then reports ENOMEM with its size).
// Vertex-partitioned extension: per-rank tables hold the local
// rows; every gather step all-gathers the passive table in column tiles of
// tile_w elements into a [n_global][tile_w] staging buffer (double buffered), and
// pushes into B rows in global memory (bg; the output table itself for
// leaf-active steps).
// Full-row exchange (vp_full): when the widest passive table of all ranks fits the
// staging cap, each gather step all-gathers whole rows (every rank's table holds nl
// rows, so its table IS the send buffer) and runs the fused single-GPU kernels on the
// local rows with the staging buffer as the gather source (B stays on chip); at
// world = 1 nothing is exchanged at all.  Otherwise column tiles as above.
static void plan_vp_extend(Plan &pl, int64_t n_local, int64_t n_global, int64_t tile_req) {
    const int vn = 16 / pl.elem;
    int64_t max_cp = 0, max_bg = 0, max_ldp = 0;
    for (Step &st : pl.steps) {
        if (st.src != SRC_GATHER) continue;
        max_cp = std::max(max_cp, round_up(st.cp, vn));
        max_ldp = std::max(max_ldp, st.ldp);
        const bool bg_is_out = !st.top && st.comb == COMB_ACTIVE_LEAF;
        if (!bg_is_out) max_bg = std::max(max_bg, st.ldb);
    }
    static const int64_t kFullCap = 24ll << 30;  // staging bytes allowed for full rows
    pl.n_global = n_global;
    // (at world 1 the local table is the gather source: no staging, so no cap — the cap
    //  once sent the Graph500-like scale-22 graph's u15-1 (50 GB of plain rows) to column
    //  tiles at world 1: 1.92 s instead of ~0.6 s per colouring)
    pl.vp_full = tile_req <= 0 && (n_global <= n_local || n_global * max_ldp * pl.elem <= kFullCap);
    int64_t off = pl.ws_bytes;
    pl.off_colors_g = off; off = round_up(off + std::max<int64_t>(n_global, 1) + 16, 256);
    if (pl.vp_full) {
        pl.tile_w = max_ldp;
        pl.off_stage = off;  off = round_up(off + (n_global > n_local ? n_global * max_ldp * pl.elem : 0), 256);
        pl.off_send = pl.off_bg = off;
    } else {
        int64_t w = tile_req > 0 ? round_up(tile_req, vn)
                                 : std::max<int64_t>(vn, ((2048ll << 20) / std::max<int64_t>(n_global * pl.elem, 1)) / vn * vn);
        w = std::max<int64_t>(vn, std::min(w, std::max<int64_t>(max_cp, vn)));
        pl.tile_w = w;
        pl.off_stage = off;  off = round_up(off + 2 * n_global * w * pl.elem, 256);
        pl.off_send = off;   off = round_up(off + 2 * std::max<int64_t>(n_local, 1) * w * pl.elem, 256);
        pl.off_bg = off;     off = round_up(off + std::max<int64_t>(n_local, 1) * max_bg * pl.elem, 256);
    }
    pl.off_part = off;     off = round_up(off + 4096 * 8, 256);
    pl.ws_bytes = off;
}

sg2v_status make_plan(const Template &t, int64_t n, int64_t nnz, sg2v_precision prec, Layout layout,
                      uint64_t budget, std::unique_ptr<Plan> &out, int64_t vp_n_global, int64_t vp_tile,
                      int proj_mode) {
    std::unique_ptr<Plan> best, smallest;
    int r0 = 0, r1 = t.k - 1;
    if (t.root_hint >= 0) r0 = r1 = t.root_hint;
    const bool try_proj = proj_mode > 0 && layout == LAYOUT_ANCHORED && vp_n_global == 0;
    for (int root = r0; root <= r1; ++root) {
        for (int policy = 0; policy < 3; ++policy) {
            Chain c = build_chain(t, root, policy);
            auto pl = std::make_unique<Plan>();
            plan_chain(t, c, root, n, nnz, prec, layout, *pl);
            if (try_proj && !pl->proj_cands.empty()) {
                // greedy: project the largest classes first while the plan fits the
                // budget and the model says it is faster (proj_mode 2: every class that fits)
                std::vector<std::string> cands = pl->proj_cands;
                std::stable_sort(cands.begin(), cands.end(),
                                 [](const std::string &a, const std::string &b) { return a.size() > b.size(); });
                std::set<std::string> chosen;
                for (const std::string &cl : cands) {
                    std::set<std::string> trial = chosen;
                    trial.insert(cl);
                    Plan q;
                    plan_chain(t, c, root, n, nnz, prec, layout, q, trial);
                    const bool qfits = budget == 0 || (uint64_t)q.ws_bytes <= budget;
                    if (qfits && (proj_mode == 2 || q.model_time < pl->model_time * (1 - 1e-6))) {
                        chosen = trial;
                        *pl = std::move(q);
                    }
                }
            }
            const bool fits = budget == 0 || (uint64_t)pl->ws_bytes <= budget;
            if (!smallest || pl->ws_bytes < smallest->ws_bytes) {
                smallest = std::make_unique<Plan>(*pl);
            }
            if (!fits) continue;
            bool better = !best || pl->model_time < best->model_time * (1 - 1e-9) ||
                          (pl->model_time <= best->model_time * (1 + 1e-9) && pl->ws_bytes < best->ws_bytes);
            if (better) best = std::move(pl);
        }
    }
    if (!best) best = std::move(smallest);
    if (vp_n_global > 0) {
        best->vp = true;
        plan_vp_extend(*best, n, vp_n_global, vp_tile);
    }
    if (!build_index(*best)) return SG2V_ENOMEM;
    out = std::move(best);
    return SG2V_OK;
}

std::string Plan::describe() const {
    std::ostringstream o;
    o << "{\"k\":" << k << ",\"root\":" << root << ",\"elem\":" << elem
      << ",\"layout\":\"" << (layout == LAYOUT_ANCHORED ? "anchored" : "dense") << "\""
      << ",\"precision\":\"" << (prec == SG2V_F32 ? "f32" : prec == SG2V_F64 ? "f64" : "u64") << "\""
      << ",\"need_hist\":" << (need_hist ? "true" : "false") << ",\"hist_bytes\":" << hist_bytes
      << ",\"tables_bytes\":" << tables_bytes << ",\"workspace_bytes\":" << ws_bytes
      << ",\"model_seconds\":" << model_time << ",\"alg_bytes\":" << alg_bytes_total
      << ",\"impl_bytes\":" << impl_bytes_total << ",\"n_rows\":" << n_rows << ",\"split_rows\":" << split_rows
      << ",\"steps\":[";
    for (size_t i = 0; i < steps.size(); ++i) {
        const Step &s = steps[i];
        o << (i ? "," : "") << "{\"s\":" << s.s << ",\"a\":" << s.a << ",\"p\":" << s.p
          << ",\"top\":" << (s.top ? "true" : "false")
          << ",\"src\":\"" << (s.src == SRC_GATHER ? "gather" : "hist") << "\""
          << ",\"comb\":\"" << (s.comb == COMB_ACTIVE_LEAF ? "active_leaf" : "general") << "\""
          << ",\"cs\":" << s.cs << ",\"ca\":" << s.ca << ",\"cp\":" << s.cp
          << ",\"cb\":" << s.cb << ",\"lds\":" << s.lds << ",\"ldp\":" << s.ldp << ",\"nterms\":" << s.nterms
          << ",\"self\":" << (s.self_a ? "true" : "false") << ",\"split_ema\":" << (s.split_ema ? "true" : "false")
          << ",\"proj_out\":" << (s.proj_out ? "true" : "false") << ",\"proj_p\":" << (s.proj_p ? "true" : "false")
          << ",\"plain_out\":" << (s.plain_out ? "true" : "false") << ",\"ldsx\":" << s.ldsx
 << ",\"gt\":" << s.gt << ",\"alg_bytes\":" << s.alg_bytes << ",\"impl_bytes\":" << s.impl_bytes
      << ",\"ema_terms\":" << s.ema_terms << "}";
    }
    o << "]}";
    return o.str();
}

}  // namespace sg2v
