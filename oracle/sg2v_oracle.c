/*
 * sg2v_oracle.c — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2009_11665_b200/) never links, imports or executes it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * What it computes (PAPER.md = P, SPEC.md = S, SURVEY.md §8(c) = readings):
 *   per colouring j, colorful_j = Σ_i M_0(i, I_[k])
 * by the colour-coding dynamic program for a tree template T:
 *   - leaves:     M_s(i, {c(i)}) = 1
 *   - two-stage:  B(i,I_p) = Σ_{j∈N(i)} M_p(j,I_p)                (Alg. 3 l.1-4)
 *                 M_s(i,I_s) += M_a(i,I_a)·B(i,I_p) over splits   (Alg. 3 l.5-8)
 *   - literal Alg. 2: M_s(i,I_s) = Σ_splits Σ_{j∈N(i)} M_a(i,I_a)M_p(j,I_p)
 *                 (with "+=" accumulation: reading "Accumulation")
 * Template partition: SPEC rule S:160 — given root ρ, cut the edge to the
 * lowest-numbered neighbour τ of ρ inside T_s; active child keeps ρ, passive
 * child is rooted at τ.  Children are evaluated before parents
 * ("reverse order of their partitioning").
 * Column index I_s: lexicographic rank of the colour set among all subsets of
 * the same size via a 2^k bitmask -> rank table.  (The CUDA path
 * uses a different bijection on purpose; SURVEY §8(c) "Column index".)
 * Arithmetic: ARITH_U64 = exact residue mod 2^64; ARITH_F64 = IEEE double,
 * plus the running max over every table entry and every B entry, which bounds
 * every intermediate (all values are non-negative sums of products; SURVEY
 * §8(c) pin 6 "Exactness condition").
 * Colouring (P:150, P:158-161 — RNG unspecified): the counter hash of SURVEY
 * §8(c) step 1, colours in [0,k) (reading "Colour range").
 *
 * Loops are plain; OpenMP only splits the independent destination rows
 * (deterministic: each row is summed in CSR order by one thread).
 *
 * Parity pins: tests/test_oracle_pins.py (brute force, closed forms,
 * exhaustive unbiasedness, worked examples from SPEC/SURVEY).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MAXK 24

enum { ORACLE_OK = 0, ORACLE_EINVAL = -1, ORACLE_ENOTTREE = -2, ORACLE_ENOMEM = -3 };
enum { FORM_TWO_STAGE = 0, FORM_ALG2 = 1 };
enum { ARITH_U64 = 0, ARITH_F64 = 1 };

/* ------------------------------------------------------------------------- */
/* 1. Random colouring: SURVEY §8(c) step 1 (counter hash; P:150 is silent).  */
/* ------------------------------------------------------------------------- */
static uint64_t oracle_mix(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

int32_t oracle_color(uint64_t seed, int64_t j, int64_t v, int32_t k)
{
    uint64_t key = oracle_mix(seed + 0x9E3779B97F4A7C15ULL * (uint64_t)(j + 1));
    uint64_t h = oracle_mix(key ^ ((uint64_t)v * 0xD6E8FEB86659FD93ULL));
    return (int32_t)(((h >> 32) * (uint64_t)k) >> 32);
}

void oracle_colors(uint64_t seed, int64_t j, int64_t n, int32_t k, uint8_t *out)
{
    for (int64_t v = 0; v < n; ++v)
        out[v] = (uint8_t)oracle_color(seed, j, v, k);
}

/* ------------------------------------------------------------------------- */
/* 2. Binomials and the lexicographic colour-set rank.            */
/* ------------------------------------------------------------------------- */
int64_t oracle_binom(int32_t n, int32_t r)
{
    if (r < 0 || r > n) return 0;
    int64_t c = 1;
    for (int32_t i = 1; i <= r; ++i) c = c * (n - r + i) / i;
    return c;
}

/* rank[mask] = lexicographic index of the set `mask` among sets of its size. */
static int32_t *oracle_rank_table(int32_t k)
{
    int32_t *rank = (int32_t *)malloc(sizeof(int32_t) << k);
    if (!rank) return NULL;
    for (int32_t s = 0; s <= k; ++s) {
        int32_t c[ORACLE_MAXK + 1];
        for (int32_t i = 0; i < s; ++i) c[i] = i;      /* first combination */
        int32_t r = 0;
        for (;;) {
            uint32_t mask = 0;
            for (int32_t i = 0; i < s; ++i) mask |= 1u << c[i];
            rank[mask] = r++;
            int32_t i = s - 1;                           /* next, lexicographic */
            while (i >= 0 && c[i] == k - s + i) --i;
            if (i < 0) break;
            c[i]++;
            for (int32_t t = i + 1; t < s; ++t) c[t] = c[t - 1] + 1;
        }
    }
    return rank;
}

int32_t oracle_rank(int32_t k, const int32_t *set, int32_t s)
{
    int32_t *rank = oracle_rank_table(k);
    if (!rank) return ORACLE_ENOMEM;
    uint32_t mask = 0;
    for (int32_t i = 0; i < s; ++i) mask |= 1u << set[i];
    int32_t r = rank[mask];
    free(rank);
    return r;
}

/* ------------------------------------------------------------------------- */
/* 3. Template partition (SPEC rule S:160).                        */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t size, root, active, passive; /* active/passive = -1 for a leaf */
    uint32_t mask;
} oracle_node;

typedef struct {
    int32_t k;
    uint32_t adj[ORACLE_MAXK];
    oracle_node nodes[2 * ORACLE_MAXK];
    int32_t n_nodes;
} oracle_tpl;

static int32_t popc(uint32_t x) { return __builtin_popcount(x); }

static int32_t oracle_partition_rec(oracle_tpl *t, uint32_t mask, int32_t root)
{
    oracle_node nd;
    nd.size = popc(mask);
    nd.root = root;
    nd.mask = mask;
    nd.active = nd.passive = -1;
    if (nd.size > 1) {
        uint32_t nb = t->adj[root] & mask;
        int32_t tau = __builtin_ctz(nb);                /* lowest-numbered neighbour */
        uint32_t comp = 1u << tau, prev = 0;            /* subtree of tau without root */
        while (comp != prev) {
            prev = comp;
            for (int32_t v = 0; v < t->k; ++v)
                if (comp & (1u << v)) comp |= t->adj[v] & mask & ~(1u << root);
        }
        nd.active = oracle_partition_rec(t, mask & ~comp, root);
        nd.passive = oracle_partition_rec(t, comp, tau);
    }
    t->nodes[t->n_nodes] = nd;
    return t->n_nodes++;
}

/* Validates a tree on vertices 0..k-1 and partitions it. */
static int32_t oracle_template(int32_t k, const int32_t *edges, int32_t root, oracle_tpl *t)
{
    if (k < 1 || k > ORACLE_MAXK || root < 0 || root >= k) return ORACLE_EINVAL;
    memset(t, 0, sizeof(*t));
    t->k = k;
    for (int32_t e = 0; e < k - 1; ++e) {
        int32_t u = edges[2 * e], v = edges[2 * e + 1];
        if (u < 0 || v < 0 || u >= k || v >= k || u == v) return ORACLE_ENOTTREE;
        if (t->adj[u] & (1u << v)) return ORACLE_ENOTTREE;
        t->adj[u] |= 1u << v;
        t->adj[v] |= 1u << u;
    }
    uint32_t seen = 1u, prev = 0, all = (k == 32) ? 0xffffffffu : ((1u << k) - 1);
    while (seen != prev) {
        prev = seen;
        for (int32_t v = 0; v < k; ++v)
            if (seen & (1u << v)) seen |= t->adj[v];
    }
    if (seen != all) return ORACLE_ENOTTREE; /* k-1 edges + connected = tree */
    oracle_partition_rec(t, all, root);
    return ORACLE_OK;
}

/* Partition as flat arrays (for tests): per node {size, root, active, passive}. */
int32_t oracle_partition(int32_t k, const int32_t *edges, int32_t root, int32_t *out_nodes)
{
    oracle_tpl t;
    int32_t rc = oracle_template(k, edges, root, &t);
    if (rc) return rc;
    for (int32_t i = 0; i < t.n_nodes; ++i) {
        out_nodes[4 * i + 0] = t.nodes[i].size;
        out_nodes[4 * i + 1] = t.nodes[i].root;
        out_nodes[4 * i + 2] = t.nodes[i].active;
        out_nodes[4 * i + 3] = t.nodes[i].passive;
    }
    return t.n_nodes;
}

/* (I_s, I_a, I_p) for every colour set C_s of size s and every split of it
 * into C_a (size a) and C_p = C_s \ C_a. */
static int32_t *oracle_splits(int32_t k, int32_t s, int32_t a, const int32_t *rank, int64_t *count)
{
    int64_t cnt = oracle_binom(k, s) * oracle_binom(s, a);
    int32_t *tr = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)(cnt > 0 ? cnt : 1));
    if (!tr) return NULL;
    int64_t w = 0;
    for (uint32_t S = 0; S < (1u << k); ++S) {
        if (popc(S) != s) continue;
        uint32_t sub = S;
        for (;;) {                                   /* every subset of S */
            if (popc(sub) == a) {
                tr[3 * w + 0] = rank[S];
                tr[3 * w + 1] = rank[sub];
                tr[3 * w + 2] = rank[S ^ sub];
                ++w;
            }
            if (sub == 0) break;
            sub = (sub - 1) & S;
        }
    }
    *count = w;
    return tr;
}

/* ------------------------------------------------------------------------- */
/* 4. Kernels of Alg. 5 as plain loops (exported in fp64 for the SPEC pins).  */
/* ------------------------------------------------------------------------- */
/* Alg. 4 / SpMM: B(i,q) = Σ_{e∈[rowptr[i],rowptr[i+1])} X(col[e], q) */
#define ORACLE_SPMM(T, NAME)                                                            \
    void NAME(int64_t n, const int64_t *rowptr, const int32_t *col, const T *X,       \
              int64_t w, T *B)                                                          \
    {                                                                                   \
        _Pragma("omp parallel for schedule(dynamic, 64)")                               \
        for (int64_t i = 0; i < n; ++i) {                                               \
            T *b = B + (size_t)i * w;                                                   \
            for (int64_t q = 0; q < w; ++q) b[q] = 0;                                   \
            for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {                       \
                const T *x = X + (size_t)col[e] * w;                                    \
                for (int64_t q = 0; q < w; ++q) b[q] += x[q];                           \
            }                                                                           \
        }                                                                               \
    }
ORACLE_SPMM(double, oracle_spmm_f64)
ORACLE_SPMM(uint64_t, oracle_spmm_u64)

/* eMA: dst[i] += a[i]*b[i] */
void oracle_ema_f64(int64_t len, double *dst, const double *a, const double *b)
{
    for (int64_t i = 0; i < len; ++i) dst[i] += a[i] * b[i];
}

/* ------------------------------------------------------------------------- */
/* 5. The DP for one colouring, generic over the arithmetic type.             */
/* ------------------------------------------------------------------------- */
#define ORACLE_DP(T, SUFFIX, TRACK_MAX)                                                  \
static int32_t oracle_dp_##SUFFIX(int64_t n, const int64_t *rowptr, const int32_t *col,  \
                                  const oracle_tpl *t, const int32_t *rank,             \
                                  const uint8_t *colors, int32_t form,                  \
                                  T *out_total, T *out_rows, double *out_max,           \
                                  double *out_max_live)                                 \
{                                                                                       \
    int32_t k = t->k;                                                                   \
    T *M[2 * ORACLE_MAXK];                                                              \
    double vmax = 0.0, vlive = 0.0;                                                     \
    const int32_t top = t->n_nodes - 1;                                                 \
    memset(M, 0, sizeof(M));                                                            \
    int32_t rc = ORACLE_OK;                                                             \
    for (int32_t s = 0; s < t->n_nodes; ++s) {                                          \
        const oracle_node *nd = &t->nodes[s];                                           \
        int64_t cs = oracle_binom(k, nd->size);                                         \
        if (nd->active < 0) {                 /* leaf: P:183-188 */                     \
            M[s] = (T *)calloc((size_t)n * (size_t)cs + 1, sizeof(T));                  \
            if (!M[s]) { rc = ORACLE_ENOMEM; break; }                                   \
            for (int64_t i = 0; i < n; ++i)                                             \
                M[s][(size_t)i * cs + rank[1u << colors[i]]] = 1;                       \
            if (TRACK_MAX && n > 0 && vmax < 1.0) vmax = 1.0;                           \
            if (TRACK_MAX && n > 0 && s != top && vlive < 1.0) vlive = 1.0;             \
            continue;                                                                   \
        }                                                                               \
        const oracle_node *na = &t->nodes[nd->active], *np = &t->nodes[nd->passive];    \
        int64_t ca = oracle_binom(k, na->size), cp = oracle_binom(k, np->size);         \
        int64_t ntr = 0;                                                                \
        int32_t *tr = oracle_splits(k, nd->size, na->size, rank, &ntr);                 \
        if (!tr) { rc = ORACLE_ENOMEM; break; }                                         \
        const T *Ma = M[nd->active];                                                    \
        if (form == FORM_TWO_STAGE) {                                                   \
            /* stage 1 (Alg. 3 l.1-4): B = A_G · M_p.  M_p has no other reader, so it  \
             * is freed before M_s is allocated (memory only: the host-RAM peak is     \
             * max(|M_p|+|B|, |M_a|+|B|+|M_s|) instead of their sum; no arithmetic     \
             * changes) */                                                              \
            T *B = (T *)malloc(sizeof(T) * ((size_t)n * (size_t)cp + 1));               \
            if (!B) { free(tr); rc = ORACLE_ENOMEM; break; }                            \
            oracle_spmm_##SUFFIX(n, rowptr, col, M[nd->passive], cp, B);                \
            if (TRACK_MAX)                                                              \
                for (size_t q = 0; q < (size_t)n * (size_t)cp; ++q)                     \
                    if ((double)B[q] > vmax) vmax = (double)B[q];                       \
            /* live B entries: I_p avoids c(i) (else every product with M_a(i,.) is     \
             * 0, M_a being 0 off c(i) ∈ I_a); the top's B is kept only when  \
             * its active child is not a leaf (with a leaf, B(i,[k]\{c(i)}) is the       \
             * per-vertex total itself) */                                              \
            if (TRACK_MAX && out_max_live && (s != top || na->active >= 0)) {           \
                uint32_t *mask_of = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)cp);  \
                if (!mask_of) { free(B); free(tr); rc = ORACLE_ENOMEM; break; }         \
                for (uint32_t m = 0; m < (1u << k); ++m)                                \
                    if (popc(m) == np->size) mask_of[rank[m]] = m;                      \
                for (int64_t i = 0; i < n; ++i)                                         \
                    for (int64_t q = 0; q < cp; ++q)                                    \
                        if (!((mask_of[q] >> colors[i]) & 1u) &&                        \
                            (double)B[(size_t)i * cp + q] > vlive)                      \
                            vlive = (double)B[(size_t)i * cp + q];                      \
                free(mask_of);                                                          \
            }                                                                           \
            free(M[nd->passive]); M[nd->passive] = NULL;                                \
            M[s] = (T *)calloc((size_t)n * (size_t)cs + 1, sizeof(T));                  \
            if (!M[s]) { free(B); free(tr); rc = ORACLE_ENOMEM; break; }                \
            T *Ms = M[s];                                                               \
            /* stage 2 (Alg. 3 l.5-8): M_s(i,I_s) += M_a(i,I_a)·B(i,I_p) */           \
            _Pragma("omp parallel for schedule(dynamic, 64)")                           \
            for (int64_t i = 0; i < n; ++i)                                             \
                for (int64_t w = 0; w < ntr; ++w)                                       \
                    Ms[(size_t)i * cs + tr[3 * w]] +=                                   \
                        Ma[(size_t)i * ca + tr[3 * w + 1]] *                            \
                        B[(size_t)i * cp + tr[3 * w + 2]];                              \
            free(B);                                                                    \
        } else {                                                                        \
            const T *Mp = M[nd->passive];                                               \
            M[s] = (T *)calloc((size_t)n * (size_t)cs + 1, sizeof(T));                  \
            if (!M[s]) { free(tr); rc = ORACLE_ENOMEM; break; }                         \
            T *Ms = M[s];                                                               \
            /* literal Alg. 2 l.5-9: neighbour loop inside the split loop */           \
            _Pragma("omp parallel for schedule(dynamic, 64)")                           \
            for (int64_t i = 0; i < n; ++i)                                             \
                for (int64_t w = 0; w < ntr; ++w)                                       \
                    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)                 \
                        Ms[(size_t)i * cs + tr[3 * w]] +=                               \
                            Ma[(size_t)i * ca + tr[3 * w + 1]] *                        \
                            Mp[(size_t)col[e] * cp + tr[3 * w + 2]];                    \
        }                                                                               \
        free(tr);                                                                       \
        if (TRACK_MAX)                                                                  \
            for (size_t q = 0; q < (size_t)n * (size_t)cs; ++q)                         \
                if ((double)M[s][q] > vmax) vmax = (double)M[s][q];                     \
        if (TRACK_MAX && s != top)                                                      \
            for (size_t q = 0; q < (size_t)n * (size_t)cs; ++q)                         \
                if ((double)M[s][q] > vlive) vlive = (double)M[s][q];                   \
        free(M[nd->active]);  M[nd->active] = NULL;  /* each child has one parent */  \
        free(M[nd->passive]); M[nd->passive] = NULL;                                    \
    }                                                                                   \
    if (rc == ORACLE_OK) {                                                              \
        /* finalCount numerator: Σ_i Σ_C M_0(i,I_C); C(k,k) = 1 column */      \
        T total = 0;                                                                    \
        for (int64_t i = 0; i < n; ++i) {                                               \
            T v = M[top][i];                                                            \
            if (out_rows) out_rows[i] = v;                                              \
            total += v;                                                                 \
        }                                                                               \
        if (TRACK_MAX && (double)total > vmax) vmax = (double)total;                    \
        *out_total = total;                                                             \
        if (out_max) *out_max = vmax;                                                   \
        if (out_max_live) *out_max_live = vlive;                                        \
    }                                                                                   \
    for (int32_t s = 0; s < t->n_nodes; ++s) free(M[s]);                                \
    return rc;                                                                          \
}
ORACLE_DP(uint64_t, u64, 0)
ORACLE_DP(double, f64, 1)

/*
 * One colouring.  colors[n] in [0,k) (from oracle_colors or any test colouring).
 * arith = ARITH_U64 writes *out_u64 (and out_rows_u64[n] if non-NULL);
 * arith = ARITH_F64 writes *out_f64, *out_max (and out_rows_f64[n]).
 * oracle_count_ex also writes *out_max_live (F64, two-stage form): the max over the
 * entries an F32 pipeline must hold in F32 whatever its layout — every non-top table
 * entry and every live B entry (I_p ∌ c(i)) except the top's B when the top's active
 * child is a leaf.  max_live > FLT_MAX means some stored F32 entry overflows.
 * Returns 0, or ORACLE_EINVAL / ORACLE_ENOTTREE / ORACLE_ENOMEM.
 */
int32_t oracle_count_ex(int64_t n, const int64_t *rowptr, const int32_t *col,
                        int32_t k, const int32_t *edges, int32_t root,
                        const uint8_t *colors, int32_t form, int32_t arith,
                        uint64_t *out_u64, uint64_t *out_rows_u64,
                        double *out_f64, double *out_rows_f64, double *out_max,
                        double *out_max_live)
{
    oracle_tpl t;
    int32_t rc = oracle_template(k, edges, root, &t);
    if (rc) return rc;
    for (int64_t i = 0; i < n; ++i)
        if (colors[i] >= k) return ORACLE_EINVAL;
    int32_t *rank = oracle_rank_table(k);
    if (!rank) return ORACLE_ENOMEM;
    if (arith == ARITH_U64)
        rc = oracle_dp_u64(n, rowptr, col, &t, rank, colors, form, out_u64, out_rows_u64, NULL, NULL);
    else
        rc = oracle_dp_f64(n, rowptr, col, &t, rank, colors, form, out_f64, out_rows_f64, out_max,
                           out_max_live);
    free(rank);
    return rc;
}

int32_t oracle_count(int64_t n, const int64_t *rowptr, const int32_t *col,
                     int32_t k, const int32_t *edges, int32_t root,
                     const uint8_t *colors, int32_t form, int32_t arith,
                     uint64_t *out_u64, uint64_t *out_rows_u64,
                     double *out_f64, double *out_rows_f64, double *out_max)
{
    return oracle_count_ex(n, rowptr, col, k, edges, root, colors, form, arith, out_u64, out_rows_u64,
                           out_f64, out_rows_f64, out_max, NULL);
}

void oracle_set_threads(int32_t nt)
{
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
#else
    (void)nt;
#endif
}

int32_t oracle_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
