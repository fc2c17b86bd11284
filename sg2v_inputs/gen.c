/*
 * gen.c — fast deterministic RMAT graph construction for sg2v_inputs.
 * INPUT GENERATION ONLY: no arithmetic of the colour-coding method lives here.
 *
 * RMAT(a,b,c,d) edge draw (Chakrabarti et al.): each of the m
 * directed draws picks one quadrant per level; the uniform for (edge e, level l)
 * is a counter hash of (seed, e, l), so the result does not depend on the
 * thread count.  Vertex ids are relabelled by a Fisher–Yates permutation keyed
 * by perm_seed.  The CSR is then symmetrised, self-loops dropped, rows sorted
 * and deduplicated (SURVEY §8(d) D4 recipe).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t gmix(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double gunif(uint64_t seed, uint64_t a, uint64_t b)
{
    uint64_t h = gmix(gmix(seed ^ gmix(a)) + b);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

static int cmp_i32(const void *x, const void *y)
{
    int32_t a = *(const int32_t *)x, b = *(const int32_t *)y;
    return (a > b) - (a < b);
}

/* Pass 1: returns nnz after symmetrise/dedupe; fills row_offsets (n+1) and
 * col (capacity 2*m).  Caller allocates col with 2*m entries. */
int64_t gen_rmat(int32_t scale, int64_t m, double a, double b, double c, uint64_t seed,
                 int64_t perm_seed, int64_t *row_offsets, int32_t *col)
{
    const int64_t n = (int64_t)1 << scale;
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * n);
    int32_t *src = (int32_t *)malloc(sizeof(int32_t) * m);
    int32_t *dst = (int32_t *)malloc(sizeof(int32_t) * m);
    int64_t *cur = (int64_t *)calloc(n + 1, sizeof(int64_t));
    if (!perm || !src || !dst || !cur) return -1;
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    if (perm_seed >= 0)
        for (int64_t i = n - 1; i > 0; --i) {
            int64_t j = (int64_t)(gunif((uint64_t)perm_seed, 0xFEEDULL, (uint64_t)i) * (double)(i + 1));
            if (j > i) j = i;
            int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
        }
    const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        int64_t u = 0, v = 0;
        for (int32_t l = 0; l < scale; ++l) {
            double r = gunif(seed, (uint64_t)e, (uint64_t)l);
            int64_t bit = (int64_t)1 << (scale - 1 - l);
            if (r >= ab) u |= bit;
            if ((r >= a && r < ab) || r >= abc) v |= bit;
        }
        src[e] = perm[u];
        dst[e] = perm[v];
    }
    /* counts, both directions, no self loops */
    for (int64_t e = 0; e < m; ++e)
        if (src[e] != dst[e]) { cur[src[e] + 1]++; cur[dst[e] + 1]++; }
    for (int64_t i = 0; i < n; ++i) cur[i + 1] += cur[i];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    memcpy(fill, cur, sizeof(int64_t) * (n + 1));
    for (int64_t e = 0; e < m; ++e)
        if (src[e] != dst[e]) { col[fill[src[e]]++] = dst[e]; col[fill[dst[e]]++] = src[e]; }
    free(fill);
    free(src);
    free(dst);
    free(perm);
    /* sort + dedupe each row in place, record new lengths */
    int64_t *len = (int64_t *)malloc(sizeof(int64_t) * n);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        int32_t *r = col + cur[i];
        int64_t d = cur[i + 1] - cur[i], w = 0;
        qsort(r, (size_t)d, sizeof(int32_t), cmp_i32);
        for (int64_t q = 0; q < d; ++q)
            if (q == 0 || r[q] != r[q - 1]) r[w++] = r[q];
        len[i] = w;
    }
    /* compact */
    int64_t out = 0;
    row_offsets[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        memmove(col + out, col + cur[i], sizeof(int32_t) * len[i]);
        out += len[i];
        row_offsets[i + 1] = out;
    }
    free(len);
    free(cur);
    return out;
}
