// akernels.cu — root-colour-anchored kernels.
//
// A table row of vertex i for a sub-template of size s stores only the colour
// sets S ∋ c(i): M_s(i,S) = 0 whenever c(i) ∉ S (the root is mapped to i), so the
// row is indexed by S∖{c(i)} relabelled into [k-1] (colex rank), C(k-1,s-1)
// columns instead of C(k,s).  The DP of Alg. 3 is unchanged:
//   B(i,T)   = Σ_{j∈N(i)} M_p(j,T)             only T ∌ c(i) are ever used, and
//              only neighbours with c(j) ∈ T contribute: grouping N(i) by colour x,
//            = Σ_{x∈T} R_x(T∖{x}),  R_x = Σ_{j∈N(i), c(j)=x} M_p(j,·)      (a4)
//   M_s(i,S) = Σ_{S_a} M_a(i,S_a)·B(i,S∖S_a)  over the universe [k-1] with one
//              split table for every vertex; = B(i,·) itself when |T_a| = 1   (a5)
// Monochromatic edges (c(j) = c(i)) contribute nothing and are skipped.
//
//  bucket_kernel  per colouring: colour counts H(i,x) and a colour-bucketed copy
//                 of every CSR row (stable), one warp per row
//  astep_kernel   fused gather (per-colour register sums R_x, pushed into B in
//                 shared memory through the [x][c(i)] map) + eMA + store
//  atop_leaf_kernel  top step with a leaf active child: one column per edge
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "kcommon.cuh"
#include "sg2v_internal.h"

namespace sg2v {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// colour counts + colour-bucketed CSR (stable within each colour)
// ---------------------------------------------------------------------------
// bcol entries carry the neighbour's degree-rank class in bits 26..30 when
// n < 2^26 (the L2 residency hint of the gather; kClassShift), else bare ids.
static constexpr int kClassShift = 26;
// rows with >= 2^kHeavyLog2 neighbours (a prefix of the degree-descending order) are
// walked by a whole CTA in the bucket, heavy-row and ring kernels
static constexpr int kHeavyLog2 = 11;

__global__ void __launch_bounds__(256) bucket_kernel(int64_t n, int k, int kp, const int64_t *__restrict__ rowptr,
                                                     const int32_t *__restrict__ col,
                                                     const uint8_t *__restrict__ colors,
                                                     const uint8_t *__restrict__ vclass,
                                                     int32_t *__restrict__ hcnt, int32_t *__restrict__ bcol,
                                                     int64_t heavy_min) {
    // rows are local (row_begin + i is the global id); neighbour ids are global.
    // Per warp-row: pass 1 counts colours (lanes of equal colour found by match_any, the
    // lowest lane adds the group size to the warp's shared counter: integer, exact);
    // pass 2 writes each neighbour at its colour bucket's running position + its rank
    // among equal-colour lanes of the chunk (stable within a colour).
    __shared__ int cnt_s[8][32];
    const bool tag = vclass != nullptr && n < (int64_t(1) << kClassShift);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int *cnt = cnt_s[w];
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + w; i < n; i += warps) {
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        if (e1 - e0 >= heavy_min) continue;  // bucket_heavy_kernel's row
        cnt[lane] = 0;
        __syncwarp();
        // 128 neighbours (4 chunks of 32) in flight per pass; a row of <= 128 neighbours
        // (~3/4 of RMAT-1M-like rows) is loaded once and placed from registers
        int32_t jj[4];
        int cc[4];
        auto load4 = [&](int64_t base) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t e = base + q * 32 + lane;
                jj[q] = e < e1 ? __ldg(col + e) : -1;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) cc[q] = jj[q] >= 0 ? (int)colors[jj[q]] : 255;
        };
        auto count4 = [&]() {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const unsigned m = __match_any_sync(0xffffffffu, cc[q]);
                if (cc[q] != 255 && (__ffs(m) - 1) == lane) atomicAdd(&cnt[cc[q]], __popc(m));
            }
        };
        auto place4 = [&]() {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int c = cc[q];
                const unsigned m = __match_any_sync(0xffffffffu, c);
                if (c != 255) {
                    const int pos = cnt[c] + __popc(m & lanemask_lt());
                    const int32_t j = jj[q];
                    SG2V_DASSERT(pos >= 0 && pos < e1 - e0);
                    bcol[e0 + pos] = tag ? (j | ((int32_t)min((int)vclass[j], 31) << kClassShift)) : j;
                }
                __syncwarp();
                if (c != 255 && (__ffs(m) - 1) == lane) cnt[c] += __popc(m);
                __syncwarp();
            }
        };
        // pass 1: colour counts (integer adds, exact)
        load4(e0);
        count4();
        for (int64_t base = e0 + 128; base < e1; base += 128) {
            load4(base);
            count4();
        }
        __syncwarp();
        const int mine = lane < k ? cnt[lane] : 0;
        if (lane < kp) hcnt[i * kp + lane] = mine;
        // exclusive scan over colours -> start of each colour's bucket
        int incl = mine;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        __syncwarp();
        cnt[lane] = incl - mine;  // running write position per colour
        __syncwarp();
        // pass 2: stable placement (position = running start of the colour + rank among
        // equal-colour lanes of the chunk)
        if (e1 - e0 <= 128) {
            place4();
        } else {
            for (int64_t base = e0; base < e1; base += 128) {
                load4(base);
                place4();
            }
        }
    }
}

// Heavy rows (degree >= 2^kHeavyLog2, rows [0, n_heavy) of the degree order): one CTA
// per row, so a 56K-neighbour hub is not walked by one warp (it was the whole kernel's
// critical path).  Same result as bucket_kernel: colour counts (integer adds, exact) and
// the stable colour-bucketed copy — chunks of 256 neighbours in CSR order, each
// neighbour's position = its bucket's running start + the counts of its colour in the
// chunk's earlier warps + its rank among equal-colour lanes of its warp.  Loads of four
// chunks are in flight together.
__global__ void __launch_bounds__(256) bucket_heavy_kernel(int64_t n_heavy, int k, int kp, const int64_t *__restrict__ rowptr,
                                                           const int32_t *__restrict__ col, const uint8_t *__restrict__ colors,
                                                           const uint8_t *__restrict__ vclass, const int32_t *__restrict__ order,
                                                           int32_t *__restrict__ hcnt, int32_t *__restrict__ bcol, int64_t nfull) {
    constexpr int CH = 4;  // chunks of 256 in flight
    __shared__ int cnt[32];
    __shared__ int wcnt[8][32];
    __shared__ int wbase[8][32];
    __shared__ int run[32];
    const bool tag = vclass != nullptr && nfull < (int64_t(1) << kClassShift);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int64_t r = blockIdx.x; r < n_heavy; r += gridDim.x) {
        const int64_t i = order[r];
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        if (tid < 32) cnt[tid] = 0;
        __syncthreads();
        // pass 1: colour counts
        for (int64_t base = e0; base < e1; base += 256 * CH) {
            int c[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int64_t e = base + q * 256 + tid;
                const int32_t j = e < e1 ? __ldg(col + e) : -1;
                c[q] = j >= 0 ? (int)colors[j] : 255;
            }
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const unsigned m = __match_any_sync(0xffffffffu, c[q]);
                if (c[q] != 255 && (__ffs(m) - 1) == lane) atomicAdd(&cnt[c[q]], __popc(m));
            }
        }
        __syncthreads();
        if (tid < 32) {
            const int mine = tid < k ? cnt[tid] : 0;
            if (tid < kp) hcnt[i * kp + tid] = mine;
            int incl = mine;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (tid >= off) incl += y;
            }
            run[tid] = incl - mine;
        }
        __syncthreads();
        // pass 2: stable placement, CH chunks of loads in flight
        for (int64_t base = e0; base < e1; base += 256 * CH) {
            int32_t jj[CH];
            int c[CH];
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int64_t e = base + q * 256 + tid;
                jj[q] = e < e1 ? __ldg(col + e) : -1;
                c[q] = jj[q] >= 0 ? (int)colors[jj[q]] : 255;
            }
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                wcnt[w][lane] = 0;
                __syncwarp();
                const unsigned m = __match_any_sync(0xffffffffu, c[q]);
                const int rank = __popc(m & lanemask_lt());
                if (c[q] != 255 && (__ffs(m) - 1) == lane) wcnt[w][c[q]] = __popc(m);
                __syncthreads();
                if (tid < 32) {  // per colour: exclusive prefix over the 8 warps of the chunk
                    int s = run[tid];
#pragma unroll
                    for (int w2 = 0; w2 < 8; ++w2) {
                        wbase[w2][tid] = s;
                        s += wcnt[w2][tid];
                    }
                    run[tid] = s;
                }
                __syncthreads();
                if (c[q] != 255) {
                    const int32_t j = jj[q];
                    SG2V_DASSERT(wbase[w][c[q]] + rank >= 0 && wbase[w][c[q]] + rank < e1 - e0);
                    bcol[e0 + wbase[w][c[q]] + rank] = tag ? (j | ((int32_t)min((int)vclass[j], 31) << kClassShift)) : j;
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// fused anchored step
// ---------------------------------------------------------------------------
struct AStepArgs {
    int64_t n;
    int k, kp;
    const int64_t *rowptr;
    const int32_t *bcol;
    const int32_t *hcnt;
    const int32_t *order;
    const uint8_t *colors;
    const char *mp;     // passive anchored table (gather source)
    int64_t ldp, cp;    // its row stride / width C(k-1,p-1)
    int src_hist;       // p = 1: B(i,{y}) = H(i,y)
    const int32_t *pmap;  // push map [x][c(i)][cp] -> B column or -1
    int64_t ldseg_p;    // > 0: the passive table is exclusion-projected: k-1 segments of
                        //   ldseg_p elements per row, segment y' = sets avoiding colour y
    int64_t ldseg_out;  // > 0: write the exclusion-projected output table msx (stride ldsx)
    char *msx;
    int64_t ldsx;
    const int32_t *omap;  // its write map (leaf-active: inverse [y'][ldseg_out]; general:
                          //   forward [o][k-1] -> position in segment y', or -1)
    int64_t ocols;      // eMA outputs per row, padded to 16 B
    const char *ma;     // active anchored table (GENERAL)
    int64_t lda;
    char *ms;           // output table (non-top)
    int64_t lds, cs;
    int64_t ldb, cb;    // B row: C(k-1,p) columns
    int comb, top;
    const int32_t *idx; // GENERAL split pairs over [k-1]
    int64_t nterms;
    void *rowval;
    int64_t smem_group;
    int tagged;         // bcol carries rank classes
    int hot_log2;       // neighbours with class < hot_log2 are kept in L2 (evict_last)
    int hint;           // use the L2 policies at all
    int packed;         // split pairs packed as ia | ip << 16 (both < 2^16)
    int stage_a;        // M_a row staged in shared memory (else read through L1)
    int tpo;            // lanes per output in the eMA (power of 2, <= 32)
    double terms_per_byte;  // eMA split terms per algorithmic byte of the step (launch config)
    int64_t aoff;       // offset of the M_a row in a group's shared memory: ldb, or 0 when
                        // M_a(i,·) IS B(i,·) (self step: T_s = root + two copies of X)
    // vertex-partitioned mode: B rows live in global memory
    int64_t cp_map;     // row stride of the push map: cp rounded up to 4 entries
    int64_t u0;         // first passive column of this tile (push-map offset)
    int tile_mode;      // stage 1 only: gather a staged column tile, push into bg rows
    int bsrc_global;    // stage 1 = copy the completed B row from bg
    char *bg;           // [n_local][ldb] B rows (tile_mode / bsrc_global)
    int *ovf;           // F32 overflow flag of this sg2v_count call (in its workspace)
    int64_t n_heavy;    // rows [0, n_heavy) of `order` have >= 2^kHeavyLog2 neighbours
    // split eMA pipeline (GENERAL eMA-heavy steps): the gather launch stores each finished
    // B row at b_out + r·ldb (r = position in `order`) instead of running the eMA; the
    // combine launch (MODE 2) reads bg by that position (bg_pos)
    char *b_out;
    int bg_pos;
};

// F32 overflow flag (AStepArgs::ovf, one int in the calling sg2v_count's workspace, so
// concurrent calls on other streams cannot clear or raise it): set by any step that
// stores a non-finite table entry (EOVERFLOW contract of sg2v.h).  Checked at the
// stores, so the report does not depend on how inf / NaN propagate later.

template <typename T>
__device__ __forceinline__ bool nonfinite(T x) {
    if constexpr (std::is_same<T, float>::value) return !isfinite(x);
    else return false;
}
template <typename T>
__device__ __forceinline__ bool nonfinite4(const uint4 &w) {
    if constexpr (std::is_same<T, float>::value)
        return !isfinite(__uint_as_float(w.x)) || !isfinite(__uint_as_float(w.y)) ||
               !isfinite(__uint_as_float(w.z)) || !isfinite(__uint_as_float(w.w));
    else return false;
}

// push targets of the VN elements of 16-B vector v (one aligned vector load of the
// padded push-map row; -1 = the set contains c(i), nothing to add)
template <typename T>
__device__ __forceinline__ void load_targets(const int32_t *mp, int64_t v, int32_t (&tt)[Vec<T>::N]) {
    if constexpr (Vec<T>::N == 4) {
        const int4 q = __ldg(reinterpret_cast<const int4 *>(mp) + v);
        tt[0] = q.x; tt[1] = q.y; tt[2] = q.z; tt[3] = q.w;
    } else {
        const int2 q = __ldg(reinterpret_cast<const int2 *>(mp) + v);
        tt[0] = q.x; tt[1] = q.y;
    }
}

// ---- stage 1 for one row: B(i,·) over T ⊂ [k]∖{c(i)} into sB (group-uniform) ----
// STRIDE: element stride of B in sB (V when V rows are interleaved in shared memory)
template <typename T, int GT, int R, int U, int STRIDE = 1>
__device__ __forceinline__ void gather_row(const AStepArgs &A, int64_t i, int ci, T *sB, int t, int g,
                                           uint64_t pol_last, uint64_t pol_first) {
    constexpr int VN = Vec<T>::N;
    constexpr int32_t kIdMask = (1 << kClassShift) - 1;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const size_t row_bytes = (size_t)A.ldp * sizeof(T);
    const int k = A.k;
    const int32_t *h = A.hcnt + (size_t)i * A.kp;
    if (A.src_hist) {
        for (int64_t y = t; y < A.cb; y += GT) sB[y * STRIDE] = (T)__ldg(h + y + (y >= ci ? 1 : 0));
        return;
    }
    int64_t e = A.rowptr[i];
    for (int x = 0; x < k; ++x) {
        const int cnt = __ldg(h + x);
        if (x != ci && cnt > 0) {
            const int r = ci - (ci > x ? 1 : 0);  // c(i)'s element in x's universe [k-1]
            const int32_t *mp = A.pmap + ((size_t)x * k + ci) * A.cp_map + A.u0;
            // byte offset of this lane's vector in a neighbour row; a projected source
            // is read in segment r (the sets avoiding c(i))
            const int64_t sbase = (A.ldseg_p > 0 ? (int64_t)r * A.ldseg_p * (int64_t)sizeof(T) : 0) + (int64_t)t * 16;
            for (int64_t v0 = 0; v0 < nvec_p; v0 += GT * R) {
                uint4 acc[R];
                bool need[R];
                int32_t tt[R][VN];  // push targets, loaded before the neighbour loads
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    acc[q] = make_uint4(0, 0, 0, 0);
                    need[q] = v0 + q * GT + t < nvec_p;
                    if (need[q]) load_targets<T>(mp, v0 + q * GT + t, tt[q]);
                }
                int64_t e2 = e;
                const int64_t e3 = e + cnt;
                for (; e2 + U <= e3; e2 += U) {
                    int32_t jj[U];
                    uint64_t pol[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int32_t b = __ldg(A.bcol + e2 + u);
                        jj[u] = A.tagged ? (b & kIdMask) : b;
                        pol[u] = (A.tagged && (b >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                    }
                    uint4 xv[U][R];
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int q = 0; q < R; ++q) {
                            const int64_t v = v0 + q * GT + t;
                            const char *src = A.mp + (size_t)jj[u] * row_bytes + sbase + (v - t) * 16;
                            xv[u][q] = ldg16_pred(src, need[q], pol[u]);
                        }
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int q = 0; q < R; ++q) Vec<T>::add(acc[q], xv[u][q]);
                }
                if (e2 < e3) {  // tail: one predicated batch, all loads in flight together
                    constexpr int UT = U < 8 ? U : 8;
                    for (; e2 < e3; e2 += UT) {
                        int32_t jj[UT];
                        uint64_t pol[UT];
#pragma unroll
                        for (int u = 0; u < UT; ++u) {
                            const int32_t b1 = (e2 + u < e3) ? __ldg(A.bcol + e2 + u) : -1;
                            jj[u] = (b1 >= 0 && A.tagged) ? (b1 & kIdMask) : b1;
                            pol[u] = (A.tagged && b1 >= 0 && (b1 >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                        }
                        uint4 xv[UT][R];
#pragma unroll
                        for (int u = 0; u < UT; ++u)
#pragma unroll
                            for (int q = 0; q < R; ++q) {
                                const int64_t v = v0 + q * GT + t;
                                xv[u][q] = ldg16_pred(A.mp + (size_t)(jj[u] >= 0 ? jj[u] : 0) * row_bytes + sbase + (v - t) * 16,
                                                      jj[u] >= 0 && need[q], pol[u]);
                            }
#pragma unroll
                        for (int u = 0; u < UT; ++u)
#pragma unroll
                            for (int q = 0; q < R; ++q) Vec<T>::add(acc[q], xv[u][q]);
                    }
                }
                // push R_x into B: distinct targets within one colour
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    if (need[q]) {
#pragma unroll
                        for (int el = 0; el < VN; ++el)  // (u < cp: a column tile's last vector
                                                          //  may run into the next tile)
                            if (tt[q][el] >= 0 && (v0 + q * GT + t) * VN + el < A.cp) {
                                SG2V_DASSERT(A.tile_mode || tt[q][el] < A.ldb);
                                sB[(size_t)tt[q][el] * STRIDE] += vget<T>(acc[q], el);
                            }
                    }
                }
            }
            group_sync<GT>(g);  // colours x and x' may push to the same T
        }
        e += cnt;
    }
}

// ---- stage 2 for one slot (V rows of a group): eMA over the universe [k-1] and the
// stores, or the top dot product + per-vertex value (shared by the register-gather and
// the bulk-staged kernels) ----
template <typename T, typename RT, int GT, int V>
__device__ __forceinline__ void ema_stage(const AStepArgs &A, T *sBase, const int64_t *iv, const bool *actv, int t,
                                          int g, RT *red, bool &bad) {
    constexpr int VN = Vec<T>::N;
    RT racc = 0;
    if (!A.top && A.comb == COMB_ACTIVE_LEAF) {
        // M_s(i,·) = B(i,·): |T_s| - 1 = |T_p| and the colour sets coincide
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (actv[v]) {
                const T *sB = sBase + (size_t)v * A.smem_group;
                if (A.ms) {  // plain table
                    T *out = reinterpret_cast<T *>(A.ms) + (size_t)iv[v] * A.lds;
                    for (int64_t q = t; q < A.lds / VN; q += GT) {
                        const uint4 w = reinterpret_cast<const uint4 *>(sB)[q];
                        bad |= nonfinite4<T>(w);
                        __stcs(reinterpret_cast<uint4 *>(out) + q, w);
                    }
                }
                if (A.msx) {
                    // projected: segment y' position u <- B(i, omap[y'][u]) (16-B stores)
                    T *out = reinterpret_cast<T *>(A.msx) + (size_t)iv[v] * A.ldsx;
                    for (int64_t q = t; q < A.ldsx / VN; q += GT) {
                        uint4 w;
                        int32_t c[VN];  // one aligned vector load of the map (segments padded to 16 B)
                        load_targets<T>(A.omap, q, c);
#pragma unroll
                        for (int el = 0; el < VN; ++el) vset<T>(w, el, c[el] >= 0 ? sB[c[el]] : (T)0);
                        bad |= nonfinite4<T>(w);
                        __stcs(reinterpret_cast<uint4 *>(out) + q, w);
                    }
                }
            }
    } else if (!A.top) {
        // split table term-major: entry (w, o) at w*cs + o, so the lanes (consecutive
        // outputs o) read consecutive words; each entry serves the group's V rows.
        // With few outputs (cs < GT) tpo consecutive lanes share an output.
        const int tpo = A.tpo, cs = (int)A.cs, nt = (int)A.nterms, lds = (int)A.ocols;
        const int l = t % tpo;
        for (int ob = 0; ob < lds; ob += GT / tpo) {
            const int o = ob + t / tpo;
            T acc[V];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = 0;
            if (o < cs) {
                if (V > 1 && A.packed && A.stage_a) {
                    // interleaved rows: entry e of the V rows is sBase[e*V .. e*V+V)
                    // (measured: batching the 16 table loads with a predicated remainder, or a
                    //  running pointer, ran the u17 10 = 5 + 5 eMA 20 % slower than this form)
                    const uint32_t *p = reinterpret_cast<const uint32_t *>(A.idx) + o;
                    constexpr int NV = (V * (int)sizeof(T)) / 16;  // 16-B vectors per entry
#pragma unroll 16
                    for (int w = l; w < nt; w += tpo) {
                        const uint32_t q = __ldg(p + w * cs);
                        const uint32_t ia = (q & 0xffffu) + (uint32_t)A.aoff, ib = q >> 16;
                        SG2V_DASSERT(ia < (uint32_t)A.smem_group && ib < (uint32_t)A.ldb);
                        const uint4 *pa = reinterpret_cast<const uint4 *>(sBase + (size_t)ia * V);
                        const uint4 *pb = reinterpret_cast<const uint4 *>(sBase + (size_t)ib * V);
#pragma unroll
                        for (int z = 0; z < NV; ++z) {
                            const uint4 va = pa[z], vb = pb[z];
#pragma unroll
                            for (int e = 0; e < 16 / (int)sizeof(T); ++e)
                                acc[z * (16 / (int)sizeof(T)) + e] += vget<T>(va, e) * vget<T>(vb, e);
                        }
                    }
                } else if (A.packed && A.stage_a) {
                    const uint32_t *p = reinterpret_cast<const uint32_t *>(A.idx) + o;
#pragma unroll 4
                    for (int w = l; w < nt; w += tpo) {
                        const uint32_t q = __ldg(p + w * cs);
                        const uint32_t ia = q & 0xffffu, ib = q >> 16;
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            const T *sB = sBase + (size_t)v * A.smem_group;
                            acc[v] += sB[A.aoff + ia] * sB[ib];
                        }
                    }
                } else {
                    for (int w = l; w < nt; w += tpo) {
                        int32_t ia, ib;
                        if (A.packed) {
                            const uint32_t q = __ldg(reinterpret_cast<const uint32_t *>(A.idx) + o + (size_t)w * cs);
                            ia = (int32_t)(q & 0xffffu);
                            ib = (int32_t)(q >> 16);
                        } else {
                            const int2 q = __ldg(reinterpret_cast<const int2 *>(A.idx) + o + (size_t)w * cs);
                            ia = q.x;
                            ib = q.y;
                        }
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            const T *sB = V > 1 ? sBase + v : sBase + (size_t)v * A.smem_group;
                            const int64_t sv = V > 1 ? V : 1;
                            const T av = A.stage_a ? sB[(A.aoff + ia) * sv]
                                                   : __ldg(reinterpret_cast<const T *>(A.ma) + (size_t)iv[v] * A.lda + ia);
                            acc[v] += av * sB[ib * sv];
                        }
                    }
                }
            }
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if (tpo > 1) {  // tpo <= 32 and GT >= 32: whole warps, uniform trip count
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1)
                        if (off < tpo) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
                }
                if (actv[v] && l == 0 && o < lds) {
                    bad |= nonfinite<T>(acc[v]);
                    if (A.ms) __stcs(reinterpret_cast<T *>(A.ms) + (size_t)iv[v] * A.lds + o, acc[v]);
                    if (A.msx && o < cs) {  // projected: every segment y' ∌ o
                        T *orow = reinterpret_cast<T *>(A.msx) + (size_t)iv[v] * A.ldsx;
#pragma unroll 1
                        for (int y = 0; y < A.k - 1; ++y) {
                            const int32_t pos = __ldg(A.omap + (size_t)o * (A.k - 1) + y);
                            if (pos >= 0) __stcs(orow + (size_t)y * A.ldseg_out + pos, acc[v]);
                        }
                    }
                }
            }
        }
    } else if (actv[0]) {
        // top (V == 1): colorful_i = Σ_{I_a} M_a(i,I_a)·B(i,[k-1]∖I_a)
        const T *sB = sBase;
        const T *ga = reinterpret_cast<const T *>(A.ma) + (size_t)iv[0] * A.lda;
        for (int64_t w = t; w < A.nterms; w += GT) {
            int32_t ia, ib;
            if (A.packed) {
                const uint32_t q = __ldg(reinterpret_cast<const uint32_t *>(A.idx) + w);
                ia = (int32_t)(q & 0xffffu);
                ib = (int32_t)(q >> 16);
            } else {
                const int2 q = __ldg(reinterpret_cast<const int2 *>(A.idx) + w);
                ia = q.x;
                ib = q.y;
            }
            const T av = A.stage_a ? sB[A.aoff + ia] : __ldg(ga + ia);
            racc += (RT)av * (RT)sB[ib];
        }
    }
    if (A.top) {
        RT s = group_reduce<RT, GT>(racc, g, red);
        if (actv[0] && t == 0) reinterpret_cast<RT *>(A.rowval)[iv[0]] = s;
    }
}

// GT threads per row group; R 16-B vectors per thread per pass; U neighbours in
// flight; V rows per group per slot (V > 1 only for GENERAL non-top steps: each
// split-table entry is loaded once and applied to V rows).
// MODE: 0 = fused single-GPU step, 1 = vertex-partitioned column-tile gather into
// bg rows, 2 = vertex-partitioned combine from bg (compile-time so the fused
// kernel keeps its register allocation).
// Register budget: the single-row gather variants keep 3 (U = 16) or 4 (U = 8) CTAs of
// 256 threads per SM (<= 80 / 64 registers), the V-row eMA variants 2 (<= 128) —
// ptxas otherwise spends registers on the epilogue paths / eMA unrolling and loses
// CTAs of memory parallelism per SM.
#ifndef XP_MINB16
#define XP_MINB16 3  // ... of the U = 16 variants
#endif
#ifndef XP_MINB8
#define XP_MINB8 4  // CTAs per SM of the U = 8 single-row variants (experiments: -DXP_MINB8=5)
#endif
template <int U, int V, int MODE, int GT = 256>
struct AStepMinBlocks {
    static constexpr int value = GT > 256 ? 1 : V == 1 ? (U >= 16 ? XP_MINB16 : XP_MINB8) : 2;
};

// CTA size: 256 threads, or one 512-thread group (GT = 512: V-row eMA steps whose V rows
// take more shared memory than two 256-thread CTAs can share, so the SM's one CTA
// brings 16 warps instead of 8 to hide the split-table and shared-memory latencies)
template <int GT>
struct AStepThreads {
    static constexpr int value = GT > 256 ? GT : 256;
};

template <typename T, typename RT, int GT, int R, int U, int V, int MODE>
__global__ void __launch_bounds__(AStepThreads<GT>::value, AStepMinBlocks<U, V, MODE, GT>::value) astep_kernel(AStepArgs A) {
    constexpr int G = AStepThreads<GT>::value / GT;
    constexpr int VN = Vec<T>::N;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ RT red[AStepThreads<GT>::value / 32];
    const int g = threadIdx.x / GT, t = threadIdx.x % GT;
    T *sBase = reinterpret_cast<T *>(smem) + (size_t)g * V * A.smem_group;
    const int64_t per_slot = (int64_t)G * V;
    const int64_t nslots = (A.n + per_slot - 1) / per_slot;
    // Count-table rows are written with streaming stores (__stcs: read by a later
    // launch only, so they should not displace the hub rows kept in L2).
    // L2 policies of the gathers: hub rows evict_last, the rest evict_first (no hints:
    // evict_normal for everything, e.g. the re-read staging tiles of the vertex mode)
    const uint64_t pol_last = policy_evict_last(), pol_first = A.hint ? policy_evict_first() : policy_evict_normal();

    bool bad = false;  // a stored F32 entry is not finite
    for (int64_t slot = blockIdx.x; slot < nslots; slot += gridDim.x) {
        int64_t iv[V];
        bool actv[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int64_t r = (slot * G + g) * V + v;
            actv[v] = r < A.n;
            iv[v] = actv[v] ? A.order[r] : 0;
        }
        // ---- stage 1: B rows (and staged M_a rows) into shared memory -----------
        // V = 1: [B | M_a] per group.  V > 1: the V rows are interleaved element by
        // element ([ldb][V] then [lda][V]) so one 16-byte shared load fetches an entry
        // of all V rows in the eMA.
        if constexpr (V == 1) {
            T *sB = sBase;
            T *sA = sB + A.ldb;
            const int64_t i = iv[0];
            if constexpr (MODE == 1) {
                // vertex-partitioned: push this column tile's R_x sums into the row's
                // B in global memory (zeroed before the first tile)
                T *gB = reinterpret_cast<T *>(A.bg) + (size_t)i * A.ldb;
                if (actv[0]) gather_row<T, GT, R, U>(A, i, (int)A.colors[i], gB, t, g, pol_last, pol_first);
                group_sync<GT>(g);
                continue;
            }
            if (actv[0]) {
                if (MODE == 2) {
                    const int64_t br = A.bg_pos ? (slot * G + g) : i;
                    const char *b = A.bg + (size_t)br * A.ldb * sizeof(T);
                    for (int64_t q = t; q < A.ldb / VN; q += GT) reinterpret_cast<uint4 *>(sB)[q] = ldg16(b + q * 16);
                } else {
                    for (int64_t q = t; q < A.ldb / VN; q += GT) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
                }
                if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
                    const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
                    for (int64_t q = t; q < A.lda / VN; q += GT) reinterpret_cast<uint4 *>(sA)[q] = ldg16(a + q * 16);
                }
            }
            group_sync<GT>(g);
            if (MODE == 0 && actv[0]) gather_row<T, GT, R, U>(A, i, (int)A.colors[i], sB, t, g, pol_last, pol_first);
            if (MODE == 0 && A.b_out) {  // split pipeline: hand the B row to the eMA launch
                group_sync<GT>(g);
                if (actv[0]) {
                    uint4 *o = reinterpret_cast<uint4 *>(A.b_out + (size_t)(slot * G + g) * A.ldb * sizeof(T));
                    for (int64_t q = t; q < A.ldb / VN; q += GT) __stcg(o + q, reinterpret_cast<const uint4 *>(sB)[q]);
                }
                group_sync<GT>(g);
                continue;
            }
        } else {
            static_assert(MODE != 1, "tile mode runs one row per group");
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int64_t i = iv[v];
                if (actv[v]) {
                    if (MODE == 2) {
                        const int64_t br = A.bg_pos ? (slot * G + g) * V + v : i;
                        const T *b = reinterpret_cast<const T *>(A.bg) + (size_t)br * A.ldb;
                        for (int64_t q = t; q < A.ldb; q += GT) sBase[q * V + v] = b[q];
                    } else {
                        for (int64_t q = t; q < A.ldb; q += GT) sBase[q * V + v] = 0;
                    }
                    if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
                        const T *a = reinterpret_cast<const T *>(A.ma) + (size_t)i * A.lda;
                        for (int64_t q = t; q < A.lda; q += GT) sBase[(A.ldb + q) * V + v] = __ldg(a + q);
                    }
                } else {  // (only this slot's own entries: smem_group per row)
                    for (int64_t q = t; q < A.smem_group; q += GT) sBase[q * V + v] = 0;
                }
            }
            group_sync<GT>(g);
            if (MODE == 0) {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (actv[v]) gather_row<T, GT, R, U, V>(A, iv[v], (int)A.colors[iv[v]], sBase + v, t, g, pol_last, pol_first);
            }
        }
        group_sync<GT>(g);
        ema_stage<T, RT, GT, V>(A, sBase, iv, actv, t, g, red, bad);
        group_sync<GT>(g);
    }
    if (bad) atomicOr(A.ovf, 1);
}

// ---------------------------------------------------------------------------
// heavy rows of narrow steps (north_star "CTA-per-heavy-row"): a row
// with thousands of neighbours walked by the small row group of a narrow step (4-32
// lanes) would run for milliseconds after every other row is done.  The rows with
// degree >= 2^kHeavyLog2 — a prefix of the degree-descending order — are taken first
// by this kernel, one CTA per row: the 256 threads form NG = 256/SG sub-groups of SG
// lanes (lane l owns 16-B vectors l, l+SG, ...), sub-group g takes the neighbours
// c ≡ g (mod NG) of each colour bucket, and the NG partial sums are added in a fixed
// order (g = 0..NG-1) before the push — deterministic, no atomics.  Same stage 2.
// ---------------------------------------------------------------------------
template <typename T, typename RT, int SG, int R, int U>
__global__ void __launch_bounds__(256) astep_heavy_kernel(AStepArgs A) {
    constexpr int NG = 256 / SG;
    constexpr int VN = Vec<T>::N;
    constexpr int32_t kIdMask = (1 << kClassShift) - 1;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ RT red[8];
    T *sB = reinterpret_cast<T *>(smem);
    uint4 *scratch = reinterpret_cast<uint4 *>(smem + ((A.smem_group * sizeof(T) + 15) / 16) * 16);
    const int t = threadIdx.x, sg = t / SG, l = t % SG;
    const int k = A.k;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const size_t row_bytes = (size_t)A.ldp * sizeof(T);
    const uint64_t pol_last = policy_evict_last(), pol_first = A.hint ? policy_evict_first() : policy_evict_normal();
    bool bad = false;
    for (int64_t r = blockIdx.x; r < A.n; r += gridDim.x) {
        int64_t iv[1];
        bool actv[1] = {true};
        const int64_t i = A.order[r];
        iv[0] = i;
        const int ci = A.colors[i];
        for (int64_t q = t; q < A.ldb / VN; q += 256) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
        if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
            const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
            for (int64_t q = t; q < A.lda / VN; q += 256) reinterpret_cast<uint4 *>(sB + A.ldb)[q] = ldg16(a + q * 16);
        }
        group_sync<256>(0);
        const int32_t *h = A.hcnt + (size_t)i * A.kp;
        int64_t e = A.rowptr[i];
        for (int x = 0; x < k; ++x) {
            const int cnt = __ldg(h + x);
            if (x != ci && cnt > 0) {
                const int rr = ci - (ci > x ? 1 : 0);
                const int64_t sbase = A.ldseg_p > 0 ? (int64_t)rr * A.ldseg_p * (int64_t)sizeof(T) : 0;
                uint4 acc[R];
#pragma unroll
                for (int q = 0; q < R; ++q) acc[q] = make_uint4(0, 0, 0, 0);
                for (int c0 = sg; c0 < cnt; c0 += NG * U) {
                    int32_t jj[U];
                    uint64_t pol[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int c = c0 + u * NG;
                        const int32_t b = c < cnt ? __ldg(A.bcol + e + c) : -1;
                        jj[u] = (b >= 0 && A.tagged) ? (b & kIdMask) : b;
                        pol[u] = (A.tagged && b >= 0 && (b >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                    }
                    uint4 xv[U][R];
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int q = 0; q < R; ++q) {
                            const int64_t v = l + q * SG;
                            xv[u][q] = ldg16_pred(A.mp + (size_t)(jj[u] >= 0 ? jj[u] : 0) * row_bytes + sbase + v * 16,
                                                  jj[u] >= 0 && v < nvec_p, pol[u]);
                        }
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int q = 0; q < R; ++q) Vec<T>::add(acc[q], xv[u][q]);
                }
#pragma unroll
                for (int q = 0; q < R; ++q) scratch[(size_t)sg * SG * R + q * SG + l] = acc[q];
                group_sync<256>(0);
                // fixed-order sum of the NG partials, then push R_x into B (distinct targets)
                const int32_t *mp = A.pmap + ((size_t)x * k + ci) * A.cp_map + A.u0;
                for (int64_t v = t; v < nvec_p; v += 256) {
                    const int q = (int)(v / SG), ll = (int)(v % SG);
                    int32_t tt[VN];
                    load_targets<T>(mp, v, tt);
                    uint4 sum = scratch[q * SG + ll];
                    for (int g2 = 1; g2 < NG; ++g2) Vec<T>::add(sum, scratch[(size_t)g2 * SG * R + q * SG + ll]);
#pragma unroll
                    for (int el = 0; el < VN; ++el)
                        if (tt[el] >= 0 && v * VN + el < A.cp) {
                            SG2V_DASSERT(tt[el] < A.ldb);
                            sB[tt[el]] += vget<T>(sum, el);
                        }
                }
                group_sync<256>(0);
            }
            e += cnt;
        }
        ema_stage<T, RT, 256, 1>(A, sB, iv, actv, t, 0, red, bad);
        group_sync<256>(0);
    }
    if (bad) atomicOr(A.ovf, 1);
}

template <typename T, typename RT, int SG, int R, int U>
static int launch_astep_heavy_t(const AStepArgs &A, void *stream) {
    constexpr int NG = 256 / SG;
    const size_t smem = ((A.smem_group * sizeof(T) + 15) / 16) * 16 + (size_t)NG * SG * R * 16;
    if (smem > 227 * 1024) return -1;
    auto kern = astep_heavy_kernel<T, RT, SG, R, U>;
    if (cudaError_t e = ensure_dyn_smem((const void *)kern, smem)) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    if (occ < 1) occ = 1;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(A.n, (int64_t)occ * num_sms()));
    kern<<<(unsigned)blocks, 256, smem, (cudaStream_t)stream>>>(A);
    note_launch();
    return (int)cudaGetLastError();
}

// rows [0, A.n) of A.order are the heavy prefix; nvec = the gather row's 16-B vectors
template <typename T, typename RT>
static int launch_astep_heavy(const AStepArgs &A, int64_t nvec, void *stream) {
    if (nvec <= 4) return launch_astep_heavy_t<T, RT, 4, 1, 4>(A, stream);
    if (nvec <= 8) return launch_astep_heavy_t<T, RT, 8, 1, 4>(A, stream);
    if (nvec <= 16) return launch_astep_heavy_t<T, RT, 16, 1, 4>(A, stream);
    if (nvec <= 32) return launch_astep_heavy_t<T, RT, 16, 2, 4>(A, stream);
    if (nvec <= 64) return launch_astep_heavy_t<T, RT, 16, 4, 2>(A, stream);
    return launch_astep_heavy_t<T, RT, 16, 8, 1>(A, stream);
}

// ---------------------------------------------------------------------------
// bulk-staged fused step (wide rows): the gather of stage 1 is fed by the TMA engine.
// One producer warp walks the neighbour list of the CTA's rows in colour-bucket order
// (the row's own colour skipped) and issues one cp.async.bulk per neighbour — its whole
// anchored row, or for an exclusion-projected source its segment c(i) — into a ring of
// S shared-memory stages (full/empty mbarriers); the 256 consumer threads add each
// staged row into per-colour register sums R_x (lane t owns 16-B vectors t, t+256, ...),
// push R_x into B(i,·) through the [x][c(i)] map at every colour boundary (one named
// barrier per colour, as in gather_row), then run the same eMA / top epilogue
// (ema_stage).  Loads need no registers and run up to S rows ahead across colour and
// row boundaries, so memory-level parallelism no longer depends on the consumers'
// register budget, and a consumer spends ~6 instructions per 16-B vector instead of
// the register-gather's index/policy/address work per neighbour.
// ---------------------------------------------------------------------------
// NC consumer threads (64, 128 or 256: sized to the row) + one producer warp.
template <int NC>
struct BulkMinBlocks {
    static constexpr int value = NC == 256 ? 3 : NC == 128 ? 5 : 8;
};

template <typename T, typename RT, int R, int NC>
__global__ void __launch_bounds__(NC + 32, BulkMinBlocks<NC>::value) astep_bulk_kernel(AStepArgs A, int S, uint32_t stage_bytes) {
    constexpr int kBulkConsumers = NC;
    constexpr int VN = Vec<T>::N;
    constexpr int32_t kIdMask = (1 << kClassShift) - 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ RT red[8];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + S;
    T *sB = reinterpret_cast<T *>(smem + ((2 * S * 8 + 127) / 128) * 128);
    unsigned char *stages = reinterpret_cast<unsigned char *>(sB) + ((A.smem_group * sizeof(T) + 127) / 128) * 128;
    const int tid = threadIdx.x;
    const int k = A.k;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const uint32_t seg_bytes = (uint32_t)(nvec_p * 16);
    const size_t row_bytes = (size_t)A.ldp * sizeof(T);
    if (tid == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, kBulkConsumers / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t n = A.n;
    if (tid >= kBulkConsumers) {
        // ---------------- producer warp ----------------
        const int lane = tid & 31;
        const uint64_t pol_last = policy_evict_last(), pol_first = A.hint ? policy_evict_first() : policy_evict_normal();
        int slot = 0;
        uint32_t ph = 0;
        for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
            const int64_t i = A.order[r];
            const int ci = A.colors[i];
            const int64_t e0 = A.rowptr[i];
            // lane x holds this row's count of colour x
            const int hx = lane < k ? __ldg(A.hcnt + (size_t)i * A.kp + lane) : 0;
            int x = -1, left = 0;     // current colour bucket and its remaining neighbours
            int64_t e = e0;
            for (;;) {
                // advance to the next non-empty bucket of a colour != ci (warp-uniform)
                while (left == 0) {
                    ++x;
                    if (x >= k) break;
                    const int c = __shfl_sync(0xffffffffu, hx, x);
                    if (x == ci) { e += c; continue; }
                    left = c;
                }
                if (x >= k) break;
                const int take = left < 32 ? left : 32;
                const int32_t b = lane < take ? __ldg(A.bcol + e + lane) : 0;
                const int rr = ci - (ci > x ? 1 : 0);
                const int64_t sbase = A.ldseg_p > 0 ? (int64_t)rr * A.ldseg_p * (int64_t)sizeof(T) : 0;
                for (int q = 0; q < take; ++q) {
                    const int32_t bj = __shfl_sync(0xffffffffu, b, q);
                    if (lane == 0) {
                        const int32_t j = A.tagged ? (bj & kIdMask) : bj;
                        const uint64_t pol = (A.tagged && (bj >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                        mbar_wait(empty + slot, ph ^ 1);
                        mbar_arrive_expect_tx(full + slot, seg_bytes);
                        bulk_g2s(stages + (size_t)slot * stage_bytes, A.mp + (size_t)j * row_bytes + sbase, seg_bytes,
                                 full + slot, pol);
                    }
                    if (++slot == S) { slot = 0; ph ^= 1; }
                }
                e += take;
                left -= take;
            }
        }
        return;
    }
    // ---------------- consumers (256 threads = one row group) ----------------
    const int t = tid;
    const int lane = tid & 31;
    bool bad = false;
    int slot = 0;
    uint32_t ph = 0;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        int64_t iv[1];
        bool actv[1] = {true};
        const int64_t i = A.order[r];
        iv[0] = i;
        const int ci = A.colors[i];
        for (int64_t q = t; q < A.ldb / VN; q += kBulkConsumers) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
        if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
            const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
            for (int64_t q = t; q < A.lda / VN; q += kBulkConsumers)
                reinterpret_cast<uint4 *>(sB + A.ldb)[q] = ldg16(a + q * 16);
        }
        group_sync<kBulkConsumers>(0);
        const int32_t *h = A.hcnt + (size_t)i * A.kp;
        for (int x = 0; x < k; ++x) {
            const int cnt = __ldg(h + x);
            if (x == ci || cnt == 0) continue;
            uint4 acc[R];
            // push targets of this colour, loaded before the stages are consumed
            const int32_t *mp = A.pmap + ((size_t)x * k + ci) * A.cp_map + A.u0;
            int32_t tt[R][VN];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                acc[q] = make_uint4(0, 0, 0, 0);
                const int v = t + q * kBulkConsumers;
                if (v < nvec_p) load_targets<T>(mp, v, tt[q]);
            }
            for (int c = 0; c < cnt; ++c) {
                mbar_wait(full + slot, ph);
                const unsigned char *st = stages + (size_t)slot * stage_bytes;
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int v = t + q * kBulkConsumers;
                    if (v < nvec_p) Vec<T>::add(acc[q], lds16(st + (size_t)v * 16));
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + slot);
                if (++slot == S) { slot = 0; ph ^= 1; }
            }
            // push R_x into B: distinct targets within one colour
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t v = t + q * kBulkConsumers;
                if (v < nvec_p) {
#pragma unroll
                    for (int el = 0; el < VN; ++el)
                        if (tt[q][el] >= 0 && v * VN + el < A.cp) {
                            SG2V_DASSERT(tt[q][el] < A.ldb);
                            sB[tt[q][el]] += vget<T>(acc[q], el);
                        }
                }
            }
            group_sync<kBulkConsumers>(0);  // colours x and x' may push to the same T
        }
        if (A.b_out) {  // split pipeline: hand the B row to the eMA launch
            uint4 *o = reinterpret_cast<uint4 *>(A.b_out + (size_t)r * A.ldb * sizeof(T));
            for (int64_t q = t; q < A.ldb / VN; q += kBulkConsumers) __stcg(o + q, reinterpret_cast<const uint4 *>(sB)[q]);
        } else {
            ema_stage<T, RT, kBulkConsumers, 1>(A, sB, iv, actv, t, 0, red, bad);
        }
        group_sync<kBulkConsumers>(0);
    }
    if (bad) atomicOr(A.ovf, 1);
}

// ---------------------------------------------------------------------------
// self-fed warp rings (narrow and medium gather rows: u15-1 steps 3-5).  The CTA-wide
// kernels above spend every neighbour on a block-wide hand-off (mbarrier wait/arrive by
// every consumer warp, or a group barrier per colour bucket) whose cost does not shrink
// with the row: at 0.3-1.2 KB per neighbour that overhead, not HBM, set the pace
// (~100-140 warp instructions per neighbour).  Here a warp owns a row: it is its own
// producer — up to 32 lanes issue one cp.async.bulk each (the neighbour's plain row or
// projected segment c(i)) into the warp's ring of S stages — and its own consumer: lane l
// adds 16-B vectors l, l+32, ... of each staged row into per-colour sums R_x and pushes
// them into B(i,·) in the warp's shared memory at each colour boundary (a __syncwarp,
// no block barrier), then runs the shared eMA / top epilogue with a 32-lane group.
// The issue cursor runs ahead of the consumer across colour buckets AND rows (a queue of
// the rows it entered), so the ring stays full through row boundaries and epilogues.
// Rows with >= 2^kHeavyLog2 neighbours (the degree-ordered prefix) are taken first, one
// row per CTA: warp w takes the neighbours c ≡ w (mod W) of every colour bucket into its
// own copy of B, and the W copies are added in the fixed order w = 0..W-1 (deterministic,
// no atomics); light rows are then handed out to warps in chunks (an atomic counter).
// ---------------------------------------------------------------------------
static constexpr int kRingQ = 32;      // rows the issue cursor may run ahead of the consumer
static constexpr int kRingChunk = 4;   // light rows per counter grab

template <int W>
__device__ __forceinline__ void team_sync() {
    if constexpr (W == 8) asm volatile("bar.sync 1, 256;" ::: "memory");
    else asm volatile("bar.sync 1, %0;" ::"n"(W * 32) : "memory");
}

template <typename T, typename RT, int R, int W>
__global__ void __launch_bounds__(W * 32) astep_ring_kernel(AStepArgs A, int S, uint32_t stage_bytes, uint32_t warp_bytes,
                                                            int64_t n_heavy, int *ctr) {
    constexpr int VN = Vec<T>::N;
    constexpr int32_t kIdMask = (1 << kClassShift) - 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ RT red[8];
    __shared__ int s_row;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *wb = smem + (size_t)w * warp_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(wb);
    int32_t *rq = reinterpret_cast<int32_t *>(wb + (size_t)S * 8);
    T *sB = reinterpret_cast<T *>(wb + (((size_t)S * 8 + kRingQ * 4 + 127) / 128) * 128);
    unsigned char *stages = reinterpret_cast<unsigned char *>(sB) + ((A.smem_group * sizeof(T) + 127) / 128) * 128;
    const int k = A.k;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const uint32_t seg_bytes = (uint32_t)(nvec_p * 16);
    const size_t row_bytes = (size_t)A.ldp * sizeof(T);
    const int ls = 31 - __clz(S);  // S is a power of two
    const uint64_t pol_last = policy_evict_last(), pol_first = A.hint ? policy_evict_first() : policy_evict_normal();
    if (lane == 0) {
        for (int q = 0; q < S; ++q) mbar_init(full + q, 1);
        fence_mbar_init();
    }
    __syncthreads();

    // ring counters (warp-uniform): stages issued / consumed, rows entered / consumed
    uint32_t issued = 0, consumed = 0, q_in = 0, q_out = 0;
    // issue cursor (warp-uniform; hx: lane x holds the row's count of colour x)
    int64_t cr = -1, ce = 0, cbase = 0;
    int cci = 0, cx = k, cleft = 0, chx = 0;
    int cm = 1, cw = 0;         // member w of m: neighbours c ≡ w (mod m) of each bucket
    bool cdone = false;         // no more rows for this cursor
    bool team = false;          // heavy phase: one row, no row queue
    int64_t chunk = 0;          // light phase: current chunk of rows, position in it
    int cpos = kRingChunk;
    int nxt = 0;                // lane 0: the next chunk (counter prefetch)

    // move the cursor to its next row; false when there is none (or the queue is full)
    auto next_row = [&]() -> bool {
        if (team || cdone) { cdone = true; return false; }
        if (q_in - q_out >= (uint32_t)kRingQ) return false;
        if (cpos == kRingChunk) {
            chunk = (int64_t)__shfl_sync(0xffffffffu, nxt, 0) * kRingChunk;
            if (lane == 0) nxt = atomicAdd(ctr + 1, 1);
            cpos = 0;
        }
        const int64_t r = n_heavy + chunk + cpos;
        if (r >= A.n) { cdone = true; return false; }
        ++cpos;
        cr = r;
        const int64_t i = A.order[r];
        cci = A.colors[i];
        cbase = A.rowptr[i];
        chx = lane < k ? __ldg(A.hcnt + (size_t)i * A.kp + lane) : 0;
        cx = -1;
        cleft = 0;
        if (lane == 0) rq[q_in & (kRingQ - 1)] = (int32_t)r;
        ++q_in;
        return true;
    };
    // issue up to `budget` stages (warp-uniform)
    auto issue = [&](int budget) {
        while (budget > 0) {
            if (cleft == 0) {
                // next bucket of a colour != c(i) with neighbours for this member
                if (cx >= k || cr < 0) {
                    if (!next_row()) return;
                }
                for (;;) {
                    ++cx;
                    if (cx >= k) break;
                    const int c = __shfl_sync(0xffffffffu, chx, cx);
                    const int64_t b0 = cbase;
                    cbase += c;
                    if (cx == cci || c <= cw) continue;
                    cleft = (c - cw + cm - 1) / cm;
                    ce = b0 + cw;
                    break;
                }
                if (cx >= k) continue;  // row finished: next row on the next pass
            }
            const int take = min(min(cleft, budget), 32);
            if (lane < take) {
                const int32_t b = __ldg(A.bcol + ce + (int64_t)lane * cm);
                const int32_t j = A.tagged ? (b & kIdMask) : b;
                const uint64_t pol = (A.tagged && (b >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                const int rr = cci - (cci > cx ? 1 : 0);
                const int64_t sbase = A.ldseg_p > 0 ? (int64_t)rr * A.ldseg_p * (int64_t)sizeof(T) : 0;
                const int slot = (int)((issued + lane) & (uint32_t)(S - 1));
                mbar_arrive_expect_tx(full + slot, seg_bytes);
                bulk_g2s(stages + (size_t)slot * stage_bytes, A.mp + (size_t)j * row_bytes + sbase, seg_bytes, full + slot, pol);
            }
            issued += take;
            ce += (int64_t)take * cm;
            cleft -= take;
            budget -= take;
        }
    };
    const int refill = S >= 8 ? S / 4 : 1;
    // gather of one row into sB (this member's neighbours), consuming the ring in order
    auto gather = [&](int64_t i, int ci, int hx) {
        for (int x = 0; x < k; ++x) {
            const int c = __shfl_sync(0xffffffffu, hx, x);
            if (x == ci || c <= cw) continue;
            const int cnt = (c - cw + cm - 1) / cm;
            const int32_t *mp = A.pmap + ((size_t)x * k + ci) * A.cp_map + A.u0;
            uint4 acc[R];
            int32_t tt[R][VN];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                acc[q] = make_uint4(0, 0, 0, 0);
                const int v = lane + q * 32;
                if (v < nvec_p) load_targets<T>(mp, v, tt[q]);
            }
            for (int e = 0; e < cnt; ++e) {
                const int fr = S - (int)(issued - consumed);
                if (fr >= refill || issued == consumed) issue(fr);
                const int slot = (int)(consumed & (uint32_t)(S - 1));
                SG2V_DASSERT(issued != consumed && issued - consumed <= (uint32_t)S);
                mbar_wait(full + slot, (consumed >> ls) & 1u);
                const unsigned char *st = stages + (size_t)slot * stage_bytes;
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int v = lane + q * 32;
                    if (v < nvec_p) Vec<T>::add(acc[q], lds16(st + (size_t)v * 16));
                }
                ++consumed;
            }
            // (the lanes' reads of a stage are done before any lane re-issues into it:
            //  the refill follows this warp's __syncwarp in program order)
            __syncwarp();
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t v = lane + q * 32;
                if (v < nvec_p) {
#pragma unroll
                    for (int el = 0; el < VN; ++el)
                        if (tt[q][el] >= 0 && v * VN + el < A.cp) {
                            SG2V_DASSERT(tt[q][el] < A.ldb);
                            sB[tt[q][el]] += vget<T>(acc[q], el);
                        }
                }
            }
            __syncwarp();  // colours x and x' may push to the same T
        }
    };

    bool bad = false;
    // ---------------- heavy rows: one row per CTA, W members ----------------
    if (n_heavy > 0) {
        team = true;
        cm = W;
        cw = w;
        for (;;) {
            if (threadIdx.x == 0) s_row = atomicAdd(ctr, 1);
            __syncthreads();
            const int64_t r = s_row;
            __syncthreads();
            if (r >= n_heavy) break;
            const int64_t i = A.order[r];
            const int ci = A.colors[i];
            const int hx = lane < k ? __ldg(A.hcnt + (size_t)i * A.kp + lane) : 0;
            // cursor on this row only
            cr = r; cci = ci; cbase = A.rowptr[i]; chx = hx; cx = -1; cleft = 0; cdone = false;
            for (int64_t q = lane; q < A.ldb / VN; q += 32) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
            __syncwarp();
            gather(i, ci, hx);
            team_sync<W>();
            // fixed-order sum of the W copies into warp 0's B; M_a staged next to it
            T *sB0 = reinterpret_cast<T *>(smem + (((size_t)S * 8 + kRingQ * 4 + 127) / 128) * 128);
            for (int64_t q = threadIdx.x; q < A.ldb / VN; q += W * 32) {
                uint4 s = reinterpret_cast<const uint4 *>(sB0)[q];
                for (int w2 = 1; w2 < W; ++w2)
                    Vec<T>::add(s, reinterpret_cast<const uint4 *>(
                                       reinterpret_cast<const unsigned char *>(sB0) + (size_t)w2 * warp_bytes)[q]);
                reinterpret_cast<uint4 *>(sB0)[q] = s;
            }
            if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
                const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
                for (int64_t q = threadIdx.x; q < A.lda / VN; q += W * 32)
                    reinterpret_cast<uint4 *>(sB0 + A.ldb)[q] = ldg16(a + q * 16);
            }
            team_sync<W>();
            int64_t iv[1] = {i};
            bool actv[1] = {true};
            ema_stage<T, RT, W * 32, 1>(A, sB0, iv, actv, threadIdx.x, 0, red, bad);
            team_sync<W>();
        }
        team = false;
        cdone = false;
        cm = 1;
        cw = 0;
        cr = -1;
        cx = k;
        cleft = 0;
    }
    // ---------------- light rows: a warp per row ----------------
    if (lane == 0) nxt = atomicAdd(ctr + 1, 1);
    for (;;) {
        if (q_in == q_out) {
            issue(S - (int)(issued - consumed));
            if (q_in == q_out) break;
        }
        __syncwarp();
        const int64_t r = rq[q_out & (kRingQ - 1)];
        ++q_out;
        const int64_t i = A.order[r];
        const int ci = A.colors[i];
        const int hx = lane < k ? __ldg(A.hcnt + (size_t)i * A.kp + lane) : 0;
        for (int64_t q = lane; q < A.ldb / VN; q += 32) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
        if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
            const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
            for (int64_t q = lane; q < A.lda / VN; q += 32) reinterpret_cast<uint4 *>(sB + A.ldb)[q] = ldg16(a + q * 16);
        }
        __syncwarp();
        gather(i, ci, hx);
        int64_t iv[1] = {i};
        bool actv[1] = {true};
        ema_stage<T, RT, 32, 1>(A, sB, iv, actv, lane, w, red, bad);
        __syncwarp();
    }
    if (bad) atomicOr(A.ovf, 1);
}

// ---------------------------------------------------------------------------
// warp-per-row register gather across colour buckets (narrow and medium rows).
// tools/gather_roof.cu measured the TMA engine at ~4.5e9 bulk copies/s per chip, so a
// bulk copy per neighbour only pays from ~1.5 KB segments; below that, 128-bit loads into
// registers reach 4.4-6.5 TB/s on random segments.  The register kernels above gather one
// colour bucket at a time (a group barrier per bucket, ~13 neighbours per bucket on
// RMAT-1M-like rows, so most loads come from a partly filled tail batch).  Here a warp
// owns a row and walks the row's live neighbours (its own colour's bucket skipped) as ONE
// stream in batches of U: the U indices of the next batch are loaded while the current
// batch's R·U 128-bit loads are in flight, each neighbour's colour comes from a ballot
// over the bucket ends (lane x holds the end of bucket x), and the per-colour sums R_x
// are pushed into B(i,·) (warp shared memory, __syncwarp) whenever the colour changes.
// Rows with >= 2^kHeavyLog2 neighbours are split over the W warps of a CTA (stream
// elements s ≡ w mod W, private B copies added in the fixed order w = 0..W-1), as in
// astep_ring_kernel.  Same epilogue (ema_stage).
// ---------------------------------------------------------------------------
template <int R, int U>
struct WrowMinBlocks {
    static constexpr int value = R <= 2 ? 6 : R == 3 ? 5 : 4;  // 128-thread CTAs (80 / 96 / 128 registers)
};

// NVP > 0: narrow rows (<= NVP <= 16 vectors): lane = (slot, vector), P = 32/NVP slots each
// take one neighbour per load, so a warp load covers P neighbours; the row is gathered a
// colour bucket at a time (rounds of P·U neighbours, indices loaded coalesced once per
// round), the slots' sums added by shuffles at the bucket's end and pushed by slot 0 —
// the eMA / stores then use all 32 lanes (the register row groups size one group for both,
// leaving gather lanes idle on narrow-gather GENERAL steps: u14-2's 5 = 3 + 2 ran 4 of 64).
template <typename T, typename RT, int R, int U, int W, int NVP = 0>
__global__ void __launch_bounds__(W * 32, WrowMinBlocks<R, U>::value) astep_wrow_kernel(AStepArgs A, uint32_t warp_bytes,
                                                                                       int64_t n_heavy, int *ctr) {
    constexpr int VN = Vec<T>::N;
    constexpr int32_t kIdMask = (1 << kClassShift) - 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ RT red[8];
    __shared__ int s_row;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T *sB = reinterpret_cast<T *>(smem + (size_t)w * warp_bytes);
    const int k = A.k;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const size_t row_bytes = (size_t)A.ldp * sizeof(T);
    const int64_t segb = A.ldseg_p * (int64_t)sizeof(T);
    const uint64_t pol_last = policy_evict_last(), pol_first = A.hint ? policy_evict_first() : policy_evict_normal();
    bool bad = false;

    // gather of row i (member mw of mm) into sB
    auto gather = [&](int64_t i, int ci, int mw, int mm) {
        const int64_t e0 = A.rowptr[i];
        const int hx = lane < k ? __ldg(A.hcnt + (size_t)i * A.kp + lane) : 0;
        int incl = hx;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const int endx = lane < k ? incl : 0x7fffffff;  // end of bucket `lane` (row-relative)
        const int cnt_ci = __shfl_sync(0xffffffffu, hx, ci);
        const int sci = __shfl_sync(0xffffffffu, incl, ci) - cnt_ci;
        const int live = __shfl_sync(0xffffffffu, incl, 31) - cnt_ci;
        const int len = live > mw ? (live - mw + mm - 1) / mm : 0;  // this member's stream
        auto pos = [&](int s) { return s < sci ? s : s + cnt_ci; };
        // indices of batch 0 (lane u < U holds neighbour u of the batch)
        int32_t bnext = -1;
        if (lane < U && lane < len) bnext = __ldg(A.bcol + e0 + pos(mw + lane * mm));
        int curx = -1;
        uint4 acc[R];
        int32_t tt[R][VN];
#pragma unroll
        for (int q = 0; q < R; ++q) acc[q] = make_uint4(0, 0, 0, 0);
        auto push = [&]() {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t v = lane + q * 32;
                if (v < nvec_p) {
#pragma unroll
                    for (int el = 0; el < VN; ++el)
                        if (tt[q][el] >= 0 && v * VN + el < A.cp) {
                            SG2V_DASSERT(tt[q][el] < A.ldb);
                            sB[tt[q][el]] += vget<T>(acc[q], el);
                        }
                }
                acc[q] = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();  // colours x and x' may push to the same T
        };
        for (int b0 = 0; b0 < len; b0 += U) {
            const int32_t bcur = bnext;
            if (b0 + U < len && lane < U && b0 + U + lane < len) bnext = __ldg(A.bcol + e0 + pos(mw + (b0 + U + lane) * mm));
            uint4 xv[U][R];
            int xu[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = b0 + u < len;
                const int32_t b = __shfl_sync(0xffffffffu, bcur, u);
                const int p = pos(mw + (b0 + u) * mm);
                xu[u] = ok ? __popc(__ballot_sync(0xffffffffu, endx <= p)) : -1;
                const int32_t j = A.tagged ? (b & kIdMask) : b;
                const uint64_t pol = (A.tagged && (b >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                const int rr = ci - (ci > xu[u] ? 1 : 0);
                const char *src = A.mp + (size_t)(ok ? j : 0) * row_bytes + (A.ldseg_p > 0 ? (int64_t)rr * segb : 0) + lane * 16;
#pragma unroll
                for (int q = 0; q < R; ++q) xv[u][q] = ldg16_pred(src + q * 512, ok && lane + q * 32 < nvec_p, pol);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (xu[u] < 0) break;
                if (xu[u] != curx) {
                    if (curx >= 0) push();
                    curx = xu[u];
                    const int32_t *mp = A.pmap + ((size_t)curx * k + ci) * A.cp_map + A.u0;
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int v = lane + q * 32;
                        if (v < nvec_p) load_targets<T>(mp, v, tt[q]);
                    }
                }
#pragma unroll
                for (int q = 0; q < R; ++q) Vec<T>::add(acc[q], xv[u][q]);
            }
        }
        if (curx >= 0) push();
    };
    // narrow rows: P slots of NVP lanes, a colour bucket at a time (NVP > 0)
    auto gather_narrow = [&](int64_t i, int ci, int mw, int mm) {
        constexpr int NV = NVP > 0 ? NVP : 1;
        constexpr int P = 32 / NV;
        constexpr int PU = P * U <= 32 ? P * U : 32;
        const int slot = lane / NV, v = lane % NV;
        const int64_t e0 = A.rowptr[i];
        const int hx = lane < k ? __ldg(A.hcnt + (size_t)i * A.kp + lane) : 0;
        int64_t eb = e0;
        for (int x = 0; x < k; ++x) {
            const int c = __shfl_sync(0xffffffffu, hx, x);
            const int64_t ex = eb;
            eb += c;
            if (x == ci || c <= mw) continue;
            const int cnt = (c - mw + mm - 1) / mm;  // this member's neighbours: mw, mw+mm, ...
            const int32_t *mp = A.pmap + ((size_t)x * k + ci) * A.cp_map + A.u0;
            int32_t tt[VN];
            if (v < nvec_p) load_targets<T>(mp, v, tt);
            const int rr = ci - (ci > x ? 1 : 0);
            const char *base = A.mp + (A.ldseg_p > 0 ? (int64_t)rr * segb : 0) + v * 16;
            uint4 acc = make_uint4(0, 0, 0, 0);
            for (int c0 = 0; c0 < cnt; c0 += PU) {
                const int take = min(cnt - c0, PU);
                const int32_t b = lane < take ? __ldg(A.bcol + ex + mw + (int64_t)(c0 + lane) * mm) : -1;
                uint4 xv[PU / P];
#pragma unroll
                for (int u = 0; u < PU / P; ++u) {
                    const int32_t bj = __shfl_sync(0xffffffffu, b, u * P + slot);
                    const int32_t j = A.tagged ? (bj & kIdMask) : bj;
                    const uint64_t pol = (A.tagged && (bj >> kClassShift) < A.hot_log2) ? pol_last : pol_first;
                    xv[u] = ldg16_pred(base + (size_t)(bj >= 0 ? j : 0) * row_bytes, bj >= 0 && v < nvec_p, pol);
                }
#pragma unroll
                for (int u = 0; u < PU / P; ++u) Vec<T>::add(acc, xv[u]);
            }
            // slots' partial sums (fixed butterfly order: deterministic)
#pragma unroll
            for (int off = NV; off < 32; off <<= 1) {
                uint4 o;
                o.x = __shfl_xor_sync(0xffffffffu, acc.x, off);
                o.y = __shfl_xor_sync(0xffffffffu, acc.y, off);
                o.z = __shfl_xor_sync(0xffffffffu, acc.z, off);
                o.w = __shfl_xor_sync(0xffffffffu, acc.w, off);
                Vec<T>::add(acc, o);
            }
            if (slot == 0 && v < nvec_p) {
#pragma unroll
                for (int el = 0; el < VN; ++el)
                    if (tt[el] >= 0 && (int64_t)v * VN + el < A.cp) {
                            SG2V_DASSERT(tt[el] < A.ldb);
                            sB[tt[el]] += vget<T>(acc, el);
                        }
            }
            __syncwarp();  // colours x and x' may push to the same T
        }
    };

    // ---------------- heavy rows: one row per CTA, W members ----------------
    if (n_heavy > 0) {
        for (;;) {
            if (threadIdx.x == 0) s_row = atomicAdd(ctr, 1);
            __syncthreads();
            const int64_t r = s_row;
            __syncthreads();
            if (r >= n_heavy) break;
            const int64_t i = A.order[r];
            const int ci = A.colors[i];
            for (int64_t q = lane; q < A.ldb / VN; q += 32) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
            __syncwarp();
            if constexpr (NVP > 0) gather_narrow(i, ci, w, W);
            else gather(i, ci, w, W);
            team_sync<W>();
            T *sB0 = reinterpret_cast<T *>(smem);
            for (int64_t q = threadIdx.x; q < A.ldb / VN; q += W * 32) {
                uint4 s = reinterpret_cast<const uint4 *>(sB0)[q];
                for (int w2 = 1; w2 < W; ++w2)
                    Vec<T>::add(s, reinterpret_cast<const uint4 *>(smem + (size_t)w2 * warp_bytes)[q]);
                reinterpret_cast<uint4 *>(sB0)[q] = s;
            }
            if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
                const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
                for (int64_t q = threadIdx.x; q < A.lda / VN; q += W * 32)
                    reinterpret_cast<uint4 *>(sB0 + A.ldb)[q] = ldg16(a + q * 16);
            }
            team_sync<W>();
            int64_t iv[1] = {i};
            bool actv[1] = {true};
            ema_stage<T, RT, W * 32, 1>(A, sB0, iv, actv, threadIdx.x, 0, red, bad);
            team_sync<W>();
        }
    }
    // ---------------- light rows: a warp per row, chunks of rows from a counter ----------------
    int nxt = lane == 0 ? atomicAdd(ctr + 1, 1) : 0;
    for (;;) {
        const int64_t chunk = (int64_t)__shfl_sync(0xffffffffu, nxt, 0) * kRingChunk;
        if (n_heavy + chunk >= A.n) break;
        if (lane == 0) nxt = atomicAdd(ctr + 1, 1);  // prefetch the next chunk
        for (int c = 0; c < kRingChunk; ++c) {
            const int64_t r = n_heavy + chunk + c;
            if (r >= A.n) break;
            const int64_t i = A.order[r];
            const int ci = A.colors[i];
            for (int64_t q = lane; q < A.ldb / VN; q += 32) reinterpret_cast<uint4 *>(sB)[q] = make_uint4(0, 0, 0, 0);
            if (A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0) {
                const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
                for (int64_t q = lane; q < A.lda / VN; q += 32) reinterpret_cast<uint4 *>(sB + A.ldb)[q] = ldg16(a + q * 16);
            }
            __syncwarp();
            if constexpr (NVP > 0) gather_narrow(i, ci, 0, 1);
            else gather(i, ci, 0, 1);
            int64_t iv[1] = {i};
            bool actv[1] = {true};
            ema_stage<T, RT, 32, 1>(A, sB, iv, actv, lane, w, red, bad);
            __syncwarp();
        }
    }
    if (bad) atomicOr(A.ovf, 1);
}

// ---------------------------------------------------------------------------
// top step, leaf active child: colorful_i = Σ_{j∈N(i), c(j)≠c(i)} M_p(j, topcol[c(j)][c(i)])
// ---------------------------------------------------------------------------
// colors: indexed by global vertex id (neighbours); row i's own colour is colors[row_begin + i]
template <typename T, typename RT>
__global__ void __launch_bounds__(256) atop_leaf_kernel(int64_t n, int k, int kp, const int64_t *__restrict__ rowptr,
                                                        const int32_t *__restrict__ col,
                                                        const uint8_t *__restrict__ colors,
                                                        const int32_t *__restrict__ hcnt, const T *__restrict__ src,
                                                        int64_t ldp, int src_hist, const int32_t *__restrict__ topcol,
                                                        RT *__restrict__ rowval, int64_t row_begin) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        const int ci = colors[row_begin + i];
        RT acc = 0;
        if (src_hist) {  // k = 2: the one other colour
            if (lane == 0) acc = (RT)hcnt[(size_t)i * kp + (ci == 0 ? 1 : 0)];
        } else {
            const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
            for (int64_t e = e0 + lane; e < e1; e += 32) {
                const int32_t j = __ldg(col + e);
                const int cj = colors[j];
                if (cj != ci) acc += (RT)__ldg(src + (size_t)j * ldp + __ldg(topcol + cj * k + ci));
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
        }
        if (lane == 0) rowval[i] = acc;
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int ovf_reset(int *dflag, void *stream) {
    return (int)cudaMemsetAsync(dflag, 0, sizeof(int), (cudaStream_t)stream);
}

int ovf_read(const int *dflag, int *flag, void *stream) {
    cudaError_t e = cudaMemcpyAsync(flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaStreamSynchronize((cudaStream_t)stream);
}

int launch_bucket(const Graph &g, const Plan &pl, const uint8_t *colors, int32_t *hcnt, int32_t *bcol,
                  void *stream) {
    if (g.n <= 0) return 0;
    int64_t blocks = std::min<int64_t>((g.n + 7) / 8, (int64_t)num_sms() * 8);
    double bytes = g.nnz * 9.0 + g.nnz * 4.0 + g.n * 16.0 + (double)g.n * pl.kp * 4.0;
    // heavy rows (a prefix of the degree order) by a CTA each, the rest by a warp each
    static int heavy = -1;
    if (heavy < 0) { const char *e = getenv("SG2V_HEAVY"); heavy = e ? atoi(e) : 1; }
    const int64_t n_heavy = (heavy && g.d_order) ? g.n_deg_ge[kHeavyLog2] : 0;
    const uint8_t *vcl = g.partitioned ? nullptr : g.d_vclass;
    prof_begin(1, stream);
    if (n_heavy > 0) {
        note_launch();
        bucket_heavy_kernel<<<(unsigned)std::min<int64_t>(n_heavy, (int64_t)num_sms() * 4), 256, 0, (cudaStream_t)stream>>>(
            n_heavy, pl.k, (int)pl.kp, g.d_rowptr, g.d_col, colors, vcl, g.d_order, hcnt, bcol, g.n);
    }
    bucket_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        g.n, pl.k, (int)pl.kp, g.d_rowptr, g.d_col, colors, vcl, hcnt, bcol,
        n_heavy > 0 ? (int64_t(1) << kHeavyLog2) : (int64_t(1) << 62));
    note_launch();
    prof_end(1, bytes, stream);
    return (int)cudaGetLastError();
}

template <typename T, typename RT, int GT, int R, int U, int V = 1, int MODE = 0>
static int launch_astep_t(const AStepArgs &A, void *stream) {
    auto kern = astep_kernel<T, RT, GT, R, U, V, MODE>;
    constexpr int NT = AStepThreads<GT>::value;
    constexpr int G = NT / GT;
    size_t smem = (size_t)G * V * A.smem_group * sizeof(T);
    if (smem > 227 * 1024) return -1;
    if (cudaError_t e = ensure_dyn_smem((const void *)kern, smem)) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (occ < 1) occ = 1;
    int64_t nslots = (A.n + (int64_t)G * V - 1) / ((int64_t)G * V);
    int64_t blocks = std::min<int64_t>(nslots, (int64_t)occ * num_sms());
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, NT, smem, (cudaStream_t)stream>>>(A);
    note_launch();
    return (int)cudaGetLastError();
}

// Bulk-staged launch (astep_bulk_kernel): R 16-B vectors per consumer lane, S stages
// sized for ~48 KB of bulk copies in flight per CTA (3 CTAs per SM).
template <typename T, typename RT, int R, int NC>
static int launch_astep_bulk_t(const AStepArgs &A, void *stream) {
    constexpr int kBulkThreads = NC + 32;
    constexpr int VN = Vec<T>::N;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const uint32_t stage_bytes = (uint32_t)(((nvec_p * 16) + 127) / 128 * 128);
    static int want_kb = -1;  // SG2V_BULK_KB (experiments): bulk bytes in flight per 256 consumers
    if (want_kb < 0) { const char *e = getenv("SG2V_BULK_KB"); want_kb = e ? atoi(e) : 48; }
    const int64_t kb = std::max<int64_t>(8, (int64_t)want_kb * NC / 256);
    int S = (int)std::max<int64_t>(3, std::min<int64_t>(16, (kb * 1024) / stage_bytes));
    auto smem_of = [&](int s) {
        return (size_t)((2 * s * 8 + 127) / 128 * 128) + (size_t)((A.smem_group * sizeof(T) + 127) / 128 * 128) +
               (size_t)s * stage_bytes;
    };
    while (S > 3 && smem_of(S) > 220 * 1024) --S;
    // one CTA per SM (B + M_a rows too wide for two): the register gather keeps more
    // loads in flight there (u17 16 = 10 + 6: 0.88 s vs 1.10 s bulk, 1.30 s bulk with
    // every stage that fits) -> caller falls back
    static int bulk1 = -1;  // SG2V_BULK1=1 (experiments): allow the one-CTA-per-SM configuration
    if (bulk1 < 0) { const char *e = getenv("SG2V_BULK1"); bulk1 = e ? atoi(e) : 0; }
    if (smem_of(3) > 110 * 1024 && !bulk1) return -2;
    const size_t smem = smem_of(S);
    if (smem > 227 * 1024) return -1;
    auto kern = astep_bulk_kernel<T, RT, R, NC>;
    if (cudaError_t e = ensure_dyn_smem((const void *)kern, smem)) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBulkThreads, smem);
    if (occ < 1) occ = 1;
    int64_t blocks = std::min<int64_t>(A.n, (int64_t)occ * num_sms());
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, kBulkThreads, smem, (cudaStream_t)stream>>>(A, S, stage_bytes);
    note_launch();
    return (int)cudaGetLastError();
}

// Self-fed warp rings (astep_ring_kernel): W = 4 warps per CTA, each with a ring of S
// (a power of two) stages of ~SG2V_RING_KB (16) KB.
template <typename T, typename RT, int R>
static int launch_astep_ring_t(const AStepArgs &A0, void *stream) {
    constexpr int W = 4;
    AStepArgs A = A0;
    // eMA lanes per output for a 32-lane group (GENERAL steps with few outputs)
    A.tpo = 1;
    if (A.comb == COMB_GENERAL && !A.top)
        while (A.tpo < 32 && A.cs * A.tpo * 2 <= 32) A.tpo *= 2;
    constexpr int VN = Vec<T>::N;
    const int64_t nvec_p = (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    const uint32_t stage_bytes = (uint32_t)(nvec_p * 16);
    static int ring_kb = -1;
    if (ring_kb < 0) { const char *e = getenv("SG2V_RING_KB"); ring_kb = e ? atoi(e) : 16; }
    int S = 64;
    while (S > 2 && (int64_t)S * stage_bytes > (int64_t)ring_kb * 1024) S >>= 1;
    auto warp_bytes_of = [&](int s) {
        return (uint32_t)((((size_t)s * 8 + kRingQ * 4 + 127) / 128) * 128 + ((A.smem_group * sizeof(T) + 127) / 128) * 128 +
                          (((size_t)s * stage_bytes + 127) / 128) * 128);
    };
    while (S > 2 && (size_t)W * warp_bytes_of(S) > 220 * 1024) S >>= 1;
    const uint32_t warp_bytes = warp_bytes_of(S);
    const size_t smem = (size_t)W * warp_bytes;
    if (smem > 227 * 1024) return -2;
    auto kern = astep_ring_kernel<T, RT, R, W>;
    if (cudaError_t e = ensure_dyn_smem((const void *)kern, smem)) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W * 32, smem);
    if (occ < 1) occ = 1;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((A.n + W - 1) / W, (int64_t)occ * num_sms()));
    int *ctr = A.ovf + 1;  // two scheduling counters next to the overflow flag (workspace)
    if (cudaError_t e = cudaMemsetAsync(ctr, 0, 2 * sizeof(int), (cudaStream_t)stream)) return (int)e;
    const int64_t n_heavy = std::min<int64_t>(A.n_heavy, A.n);
    kern<<<(unsigned)blocks, W * 32, smem, (cudaStream_t)stream>>>(A, S, stage_bytes, warp_bytes, n_heavy, ctr);
    note_launch();
    return (int)cudaGetLastError();
}

// Warp-per-row register gather (astep_wrow_kernel): W = 4 warps per CTA
template <typename T, typename RT, int R, int U, int NVP = 0>
static int launch_astep_wrow_t(const AStepArgs &A0, void *stream) {
    constexpr int W = 4;
    AStepArgs A = A0;
    A.tpo = 1;  // eMA lanes per output for a 32-lane group (GENERAL steps with few outputs)
    if (A.comb == COMB_GENERAL && !A.top)
        while (A.tpo < 32 && A.cs * A.tpo * 2 <= 32) A.tpo *= 2;
    const uint32_t warp_bytes = (uint32_t)(((A.smem_group * sizeof(T) + 127) / 128) * 128);
    const size_t smem = (size_t)W * warp_bytes;
    if (smem > 227 * 1024) return -2;
    auto kern = astep_wrow_kernel<T, RT, R, U, W, NVP>;
    if (cudaError_t e = ensure_dyn_smem((const void *)kern, smem)) return (int)e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W * 32, smem);
    if (occ < 1) occ = 1;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((A.n + W - 1) / W, (int64_t)occ * num_sms()));
    int *ctr = A.ovf + 1;  // two scheduling counters next to the overflow flag (workspace)
    if (cudaError_t e = cudaMemsetAsync(ctr, 0, 2 * sizeof(int), (cudaStream_t)stream)) return (int)e;
    const int64_t n_heavy = std::min<int64_t>(A.n_heavy, A.n);
    kern<<<(unsigned)blocks, W * 32, smem, (cudaStream_t)stream>>>(A, warp_bytes, n_heavy, ctr);
    note_launch();
    return (int)cudaGetLastError();
}

template <typename T, typename RT>
static int launch_astep_wrow(const AStepArgs &A, int64_t nvec, int ucfg, void *stream) {
    // narrow rows: lane-packed slots (U = 32 / P neighbours per round: one index load each)
    if (nvec <= 2) return launch_astep_wrow_t<T, RT, 1, 2, 2>(A, stream);
    if (nvec <= 4) return launch_astep_wrow_t<T, RT, 1, 4, 4>(A, stream);
    if (nvec <= 8) return launch_astep_wrow_t<T, RT, 1, 8, 8>(A, stream);
    if (nvec <= 16) return launch_astep_wrow_t<T, RT, 1, 8, 16>(A, stream);
    if (nvec <= 32) {
        if (ucfg == 4) return launch_astep_wrow_t<T, RT, 1, 4>(A, stream);
        return launch_astep_wrow_t<T, RT, 1, 8>(A, stream);
    }
    if (nvec <= 64) {
        if (ucfg == 2) return launch_astep_wrow_t<T, RT, 2, 2>(A, stream);
        return launch_astep_wrow_t<T, RT, 2, 4>(A, stream);
    }
    if (nvec <= 96) {
        if (ucfg == 2) return launch_astep_wrow_t<T, RT, 3, 2>(A, stream);
        return launch_astep_wrow_t<T, RT, 3, 4>(A, stream);
    }
    if (nvec <= 128) return launch_astep_wrow_t<T, RT, 4, 2>(A, stream);
    if (nvec <= 192) {
        if (ucfg == 3) return launch_astep_wrow_t<T, RT, 6, 3>(A, stream);
        return launch_astep_wrow_t<T, RT, 6, 2>(A, stream);
    }
    return -2;
}

// Row-group configuration: narrow rows give every vector of the passive row its own
// lane (R = 1) and keep U = 8 neighbours in flight; rows wider than 256 vectors use
// the whole CTA, one vector per lane per pass, also U = 8 (64 registers, 4 CTAs per
// SM; on RMAT-1M-like graphs a colour bucket holds ~200/k neighbours, so most loads
// are issued by the 8-wide tail batch anyway; U = 16 at 3 CTAs/SM measured 5 % slower).
template <typename T, typename RT, int R, int U, int MODE = 0>
static int launch_astep_gt(const AStepArgs &A, int gt, void *stream) {
    switch (gt) {
        case 4: return launch_astep_t<T, RT, 4, R, U, 1, MODE>(A, stream);
        case 8: return launch_astep_t<T, RT, 8, R, U, 1, MODE>(A, stream);
        case 16: return launch_astep_t<T, RT, 16, R, U, 1, MODE>(A, stream);
        case 32: return launch_astep_t<T, RT, 32, R, U, 1, MODE>(A, stream);
        case 64: return launch_astep_t<T, RT, 64, R, U, 1, MODE>(A, stream);
        case 128: return launch_astep_t<T, RT, 128, R, U, 1, MODE>(A, stream);
        default: return launch_astep_t<T, RT, 256, R, U, 1, MODE>(A, stream);
    }
}

template <typename T, typename RT, int MODE = 0>
static int launch_astep_cfg(const AStepArgs &A0, void *stream) {
    AStepArgs A = A0;
    constexpr int VN = Vec<T>::N;
    static int tune = -1;  // SG2V_TUNE (experiments only): 1 narrow U=16; 2 wide R=2/U=8; 4 wide R=4/U=4; 5 no V-rows;
                           // 16 wide U=16 (default U=8 under the 4-CTA register cap: measured faster, r1s18)
    if (tune < 0) {
        const char *e = getenv("SG2V_TUNE");
        tune = e ? atoi(e) : 0;
    }
    const int64_t nvec = A.src_hist ? 1 : (A.ldseg_p > 0 ? A.ldseg_p : A.ldp) / VN;
    // (a projected output row is written by the same lanes in more passes: the group
    // is sized by the gather and the eMA, not by the k-1 output segments)
    const int64_t nout = std::max(A.ldb, A.ocols) / VN;
    // Row-group width: the gather's vectors, widened for the epilogue only on eMA-heavy
    // GENERAL steps (>= SG2V_VTPB split terms per byte: the V-row eMA wants >= 32 lanes).
    // Sizing narrow groups by the gather alone leaves no idle lanes in the gather, which
    // dominates those steps (measured: u17 4 = 2 + 2 32.3 -> 7.6 ms, u15-1 step 3 7.6 ->
    // 5.1 ms).  SG2V_GTDIV (experiments): want = max(gather vectors, output vectors /
    // GTDIV) on the other steps too (4 = the previous sizing).
    static int gtdiv = -1;
    if (gtdiv < 0) { const char *e = getenv("SG2V_GTDIV"); gtdiv = e ? std::max(1, atoi(e)) : 1 << 20; }
    static double vtpb0 = -1;
    if (vtpb0 < 0) { const char *e = getenv("SG2V_VTPB"); vtpb0 = e ? atof(e) : 0.05; }
    const bool ema_heavy = A.comb == COMB_GENERAL && !A.top && A.terms_per_byte >= vtpb0 && A.nterms >= 8;
    // (a leaf-passive step gathers nothing per neighbour: B = H, its epilogue is the work)
    const int64_t div = (ema_heavy || A.src_hist) ? 4 : gtdiv;
    int64_t want = std::max<int64_t>(nvec, (nout + div - 1) / div);
    int gt = 4;
    while (gt < want && gt < 256) gt *= 2;
    // the 256/gt row groups of a CTA must hold their B (+ M_a) rows in shared memory
    while (gt < 256 && (size_t)(256 / gt) * A.smem_group * sizeof(T) > 160 * 1024) gt *= 2;
    if (nvec > 256) gt = 256;
    // eMA with few outputs: tpo lanes per output (whole warps only)
    A.tpo = 1;
    if (A.comb == COMB_GENERAL && !A.top && gt >= 32)
        while (A.tpo < 32 && A.cs * A.tpo * 2 <= gt) A.tpo *= 2;
    // eMA-heavy GENERAL steps: V = 4 rows share every split-table load
    static int ema512 = -1;  // SG2V_EMA512=0: V-row eMA CTAs of 256 threads only
    if (ema512 < 0) { const char *e = getenv("SG2V_EMA512"); ema512 = e ? atoi(e) : 1; }
    static double vtpb = -1;  // SG2V_VTPB (experiments): the terms-per-byte threshold
    if (vtpb < 0) { const char *e = getenv("SG2V_VTPB"); vtpb = e ? atof(e) : 0.05; }
    // (only where the eMA is a real share of the step: >= 0.05 split terms per gathered
    // byte; gather-dominated GENERAL steps such as u14-2's 13 = 5 + 8 (0.011) run one row
    // per group so the gathers of different rows overlap)
    const bool multi = A.comb == COMB_GENERAL && !A.top && A.nterms >= 8 && gt >= 32 && tune != 5 && !A.b_out &&
                       (A.terms_per_byte >= vtpb || tune == 9) &&
                       (size_t)(256 / gt) * 4 * A.smem_group * sizeof(T) <= 200 * 1024;
    // wide gather rows without V-row batching: bulk-staged loads (SG2V_BULK=0 disables,
    // SG2V_BULK_MIN sets the minimum row width in 16-B vectors)
    static int bulk = -1, bulk_min = -1;
    if (bulk < 0) {
        const char *e = getenv("SG2V_BULK");
        bulk = e ? atoi(e) : 1;
        const char *m = getenv("SG2V_BULK_MIN");
        bulk_min = m ? atoi(m) : 64;
    }
    // narrow and medium gather rows: warp-per-row register gather across colour buckets
    // (SG2V_WROW=0 disables; SG2V_WROW_MIN / _MAX: row widths in 16-B vectors; SG2V_WROW_U:
    // neighbours in flight per batch, among the compiled variants)
    static int wrow = -1, wrow_min = -1, wrow_max = -1, wrow_u = -1;
    if (wrow < 0) {
        const char *e = getenv("SG2V_WROW");
        wrow = e ? atoi(e) : 1;
        const char *a = getenv("SG2V_WROW_MIN");
        wrow_min = a ? atoi(a) : 24;
        const char *b = getenv("SG2V_WROW_MAX");
        wrow_max = b ? atoi(b) : 192;
        const char *u = getenv("SG2V_WROW_U");
        wrow_u = u ? atoi(u) : 0;
    }
    // SG2V_NARROW=1 (experiments): lane-packed warp rows for rows of <= 16 vectors.  Measured
    // slower than gather-sized register row groups on the 64-B steps (u15-1 step 3 6.2 vs
    // 4.9 ms, u12-1 5.5 vs 3.7, Orkut u12-1 12.9 vs 7.2: a bucket at a time, its latency is
    // exposed per bucket), faster on u13-2's step 4 (11.8 vs 13.0 ms): off by default.
    static int narrow = -1;
    if (narrow < 0) { const char *e = getenv("SG2V_NARROW"); narrow = e ? atoi(e) : 0; }
    if (MODE == 0 && wrow && !multi && !A.b_out && !A.src_hist && A.pmap != nullptr &&
        ((narrow && nvec <= 16) || (nvec >= wrow_min && nvec <= wrow_max && nvec <= 192))) {
        const int rc = launch_astep_wrow<T, RT>(A, nvec, wrow_u, stream);
        if (rc != -2) return rc;
    }
    // self-fed warp rings of bulk copies (experiments: SG2V_RING=1; SG2V_RING_MAX sets
    // the widest row in 16-B vectors)
    static int ring = -1, ring_max = -1;
    if (ring < 0) {
        const char *e = getenv("SG2V_RING");
        ring = e ? atoi(e) : 0;
        const char *m = getenv("SG2V_RING_MAX");
        ring_max = m ? atoi(m) : 96;
    }
    if (MODE == 0 && ring && !multi && !A.b_out && !A.src_hist && A.pmap != nullptr && nvec <= ring_max && nvec <= 256) {
        int rc;
        if (nvec <= 32) rc = launch_astep_ring_t<T, RT, 1>(A, stream);
        else if (nvec <= 64) rc = launch_astep_ring_t<T, RT, 2>(A, stream);
        else if (nvec <= 96) rc = launch_astep_ring_t<T, RT, 3>(A, stream);
        else if (nvec <= 128) rc = launch_astep_ring_t<T, RT, 4>(A, stream);
        else if (nvec <= 192) rc = launch_astep_ring_t<T, RT, 6>(A, stream);
        else rc = launch_astep_ring_t<T, RT, 8>(A, stream);
        if (rc != -2) return rc;
    }
    if (MODE == 0 && bulk && !multi && !A.src_hist && A.pmap != nullptr && nvec >= bulk_min && nvec <= 2048) {
        auto bulk_launch = [&](const AStepArgs &X) {
            if (nvec <= 64) return launch_astep_bulk_t<T, RT, 1, 64>(X, stream);
            if (nvec <= 128) return launch_astep_bulk_t<T, RT, 1, 128>(X, stream);
            if (nvec <= 256) return launch_astep_bulk_t<T, RT, 1, 256>(X, stream);
            if (nvec <= 512) return launch_astep_bulk_t<T, RT, 2, 256>(X, stream);
            if (nvec <= 1024) return launch_astep_bulk_t<T, RT, 4, 256>(X, stream);
            return launch_astep_bulk_t<T, RT, 8, 256>(X, stream);
        };
        int rc = bulk_launch(A);
        if (rc != -2) return rc;  // -2: not a bulk configuration, register gather below
        // gather-dominated GENERAL steps (few split terms per byte, e.g. u17's 16 = 10 + 6:
        // 0.025) whose staged M_a row keeps two CTAs from an SM: read M_a through L1 in the
        // eMA instead and gather with bulk copies (SG2V_UNSTAGE=1; measured slower on u17:
        // 16 = 10 + 6 922 vs 808 ms, so off by default)
        static int unstage = -1;
        if (unstage < 0) { const char *e = getenv("SG2V_UNSTAGE"); unstage = e ? atoi(e) : 0; }
        if (unstage && A.comb == COMB_GENERAL && A.stage_a && A.aoff != 0 && A.terms_per_byte < vtpb) {
            AStepArgs B2 = A;
            B2.stage_a = 0;
            B2.smem_group = A.ldb;
            rc = bulk_launch(B2);
            if (rc != -2) return rc;
        }
    }
    // heavy rows of narrow register-gather steps: CTA per row first, the rest after
    // (SG2V_HEAVY=0 disables)
    static int heavy = -1;
    if (heavy < 0) { const char *e = getenv("SG2V_HEAVY"); heavy = e ? atoi(e) : 1; }
    if (MODE == 0 && heavy && !multi && !A.b_out && !A.src_hist && A.pmap != nullptr && gt < 256 && nvec <= 32 &&
        A.n_heavy > 0 && A.n_heavy < A.n) {
        AStepArgs H = A;
        H.n = A.n_heavy;
        int rc = launch_astep_heavy<T, RT>(H, nvec, stream);
        if (rc) return rc;
        A.order += A.n_heavy;
        A.n -= A.n_heavy;
    }
    if constexpr (MODE != 0) {
        if constexpr (MODE == 2) {
            if (multi) {
                // V = 4 rows alone on the SM (> ~113 KB): one 512-thread CTA (SG2V_EMA512=0: 256)
                if (ema512 && (size_t)4 * A.smem_group * sizeof(T) > 113 * 1024) {
                    if (ema512 == 2) return launch_astep_t<T, RT, 1024, 1, 8, 4, MODE>(A, stream);  // (experiment)
                    return launch_astep_t<T, RT, 512, 1, 8, 4, MODE>(A, stream);
                }
                // (experiment, SG2V_EMA512=3): 8 interleaved rows per 512-thread group, each
                // split-table load serving 8 rows
                if (ema512 == 3 && (size_t)8 * A.smem_group * sizeof(T) <= 200 * 1024)
                    return launch_astep_t<T, RT, 512, 1, 8, 8, MODE>(A, stream);
                if (nvec > 256) return launch_astep_t<T, RT, 256, 1, 16, 4, MODE>(A, stream);
                return launch_astep_t<T, RT, 256, 1, 8, 4, MODE>(A, stream);
            }
        }
        if (nvec > 256) return launch_astep_t<T, RT, 256, 1, 16, 1, MODE>(A, stream);
        return launch_astep_gt<T, RT, 1, 8, MODE>(A, gt, stream);
    }
    if (multi) {
        // V = 4 rows per group while they fit in ~100 KB (two CTAs per SM), else V = 2
        const size_t per4 = (size_t)(256 / gt) * 4 * A.smem_group * sizeof(T);
        // V = 4 rows that only fit one CTA per SM: a 512-thread group (16 warps)
        if (ema512 && gt == 256 && per4 > 113 * 1024 && per4 <= 200 * 1024 && tune != 6)
            return launch_astep_t<T, RT, 512, 1, 8, 4>(A, stream);
        if (nvec > 256) {
            if (per4 > 100 * 1024 && tune != 6) return launch_astep_t<T, RT, 256, 1, 16, 2>(A, stream);
            return launch_astep_t<T, RT, 256, 1, 16, 4>(A, stream);
        }
        if (per4 > 100 * 1024 && gt == 256 && tune != 6) return launch_astep_t<T, RT, 256, 1, 8, 2>(A, stream);
        switch (gt) {
            case 32: return launch_astep_t<T, RT, 32, 1, 8, 4>(A, stream);
            case 64: return launch_astep_t<T, RT, 64, 1, 8, 4>(A, stream);
            case 128: return launch_astep_t<T, RT, 128, 1, 8, 4>(A, stream);
            default: return launch_astep_t<T, RT, 256, 1, 8, 4>(A, stream);
        }
    }
    if (nvec > 256) {
        if (tune == 2) return launch_astep_t<T, RT, 256, 2, 8>(A, stream);
        if (tune == 4) return launch_astep_t<T, RT, 256, 4, 4>(A, stream);
        // very wide top steps (>= 4 passes, e.g. u16/u17 paths: 6435 / 11440 columns) keep
        // 16 neighbours in flight (r1s20: u16-1 top 1201 -> 987 ms, u17-1 2069 -> 1718 ms);
        // everything else U = 8 (u15-1: 0.799 -> 0.762 s)
        if (tune == 16 || (A.top && nvec > 1024 && tune != 8)) return launch_astep_t<T, RT, 256, 1, 16>(A, stream);
        return launch_astep_t<T, RT, 256, 1, 8>(A, stream);
    }
    if (tune == 1) return launch_astep_gt<T, RT, 1, 16>(A, gt, stream);
    return launch_astep_gt<T, RT, 1, 8>(A, gt, stream);
}

int launch_astep(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const int32_t *hcnt,
                 const int32_t *bcol, char *tables, void *rowval, int *ovf, void *stream) {
    return launch_astep_vp(g, pl, st, colors, hcnt, bcol, tables, rowval, ovf, stream, nullptr);
}

int launch_astep_vp(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const int32_t *hcnt,
                    const int32_t *bcol, char *tables, void *rowval, int *ovf, void *stream, const VpArgs *vp) {
    if (g.n <= 0) return 0;
    const int32_t *idx = pl.d_index + st.idx_off;
    const char *src = (st.src == SRC_HIST || (vp && vp->mode == 2)) ? nullptr
                      : (vp && vp->mode == 3) ? vp->stage : tables + pl.bufs[st.buf_p].offset;
    // vertex mode, whole rows: neighbour ids are global, this rank's rows start at row_begin
    const int64_t colour_off = (vp && vp->mode == 3) ? vp->row_begin : 0;
    if (st.top && st.comb == COMB_ACTIVE_LEAF && (!vp || vp->mode == 3)) {
        int64_t blocks = std::min<int64_t>((g.n + 7) / 8, (int64_t)num_sms() * 8);
        int srch = st.src == SRC_HIST;
        prof_begin(3, stream);
        if (pl.prec == SG2V_F32)
            atop_leaf_kernel<float, double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
                g.n, pl.k, (int)pl.kp, g.d_rowptr, g.d_col, colors - colour_off, hcnt, (const float *)src, st.ldp, srch, idx,
                (double *)rowval, colour_off);
        else if (pl.prec == SG2V_F64)
            atop_leaf_kernel<double, double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
                g.n, pl.k, (int)pl.kp, g.d_rowptr, g.d_col, colors - colour_off, hcnt, (const double *)src, st.ldp, srch, idx,
                (double *)rowval, colour_off);
        else
            atop_leaf_kernel<u64, u64><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
                g.n, pl.k, (int)pl.kp, g.d_rowptr, g.d_col, colors - colour_off, hcnt, (const u64 *)src, st.ldp, srch, idx,
                (u64 *)rowval, colour_off);
        note_launch();
        prof_end(3, st.alg_bytes, stream, st.impl_bytes, 0.0);
        return (int)cudaGetLastError();
    }
    AStepArgs A;
    A.n = g.n;
    A.k = pl.k;
    A.kp = (int)pl.kp;
    A.rowptr = g.d_rowptr;
    A.bcol = bcol;
    A.hcnt = hcnt;
    A.order = g.d_order;
    A.colors = colors;
    A.mp = src;
    A.ldp = st.ldp;
    A.cp = st.cp;
    A.src_hist = st.src == SRC_HIST;
    A.pmap = st.map_off >= 0 ? pl.d_index + st.map_off : nullptr;
    A.ma = (st.comb == COMB_GENERAL && st.buf_a >= 0) ? tables + pl.bufs[st.buf_a].offset : nullptr;
    A.lda = st.lda;
    A.ms = (st.top || st.buf_out < 0) ? nullptr : tables + pl.bufs[st.buf_out].offset;
    A.lds = st.lds;
    A.cs = st.cs;
    A.ldseg_p = st.proj_p ? st.ldseg_p : 0;
    A.ldseg_out = st.proj_out ? st.ldseg_out : 0;
    A.msx = (!st.top && st.proj_out && st.buf_outx >= 0) ? tables + pl.bufs[st.buf_outx].offset : nullptr;
    A.ldsx = st.ldsx;
    A.terms_per_byte = st.impl_bytes > 0 ? st.ema_terms / st.impl_bytes : 1.0;
    A.omap = st.omap_off >= 0 ? pl.d_index + st.omap_off : nullptr;
    A.ocols = st.top ? 1 : (st.cs + (16 / pl.elem) - 1) / (16 / pl.elem) * (16 / pl.elem);
    A.ldb = st.ldb;
    A.cb = st.cb;
    A.comb = st.comb;
    A.top = st.top;
    A.idx = idx;
    A.nterms = st.nterms;
    A.rowval = rowval;
    A.packed = st.packed;
    A.cp_map = (st.cp + 3) / 4 * 4;  // push-map rows are padded to 4 entries
    A.u0 = 0;
    A.tile_mode = 0;
    A.bsrc_global = 0;
    A.bg = nullptr;
    A.ovf = ovf;
    A.n_heavy = g.n_deg_ge[kHeavyLog2];
    A.b_out = nullptr;
    A.bg_pos = 0;
    // stage M_a next to B only while both fit comfortably (occupancy); else L1
    A.aoff = st.self_a ? 0 : st.ldb;
    static int stage_kb = -1;  // SG2V_STAGE_KB (experiments): M_a staging threshold
    if (stage_kb < 0) { const char *e = getenv("SG2V_STAGE_KB"); stage_kb = e ? atoi(e) : 100; }
    A.stage_a = (st.comb == COMB_GENERAL) && (st.self_a || (st.ldb + st.lda) * pl.elem <= (int64_t)stage_kb * 1024);
    A.tpo = 1;  // set per launch configuration (launch_astep_cfg)
    A.smem_group = st.ldb + (A.stage_a && !st.self_a ? st.lda : 0);
    A.tagged = std::max(g.n, pl.n_rows) < (int64_t(1) << kClassShift);  // as bucket_kernel tagged (full n)
    {
        // rows of the hottest H neighbours fit in ~75 MB of the 126 MB L2
        static int64_t l2 = 0;
        if (!l2) {
            int dev = 0, v = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
            l2 = v > 0 ? v : (126ll << 20);
        }
        static double hotfrac = -1;  // SG2V_HOTFRAC (experiments): share of L2 for hub rows
        if (hotfrac < 0) { const char *e = getenv("SG2V_HOTFRAC"); hotfrac = e ? atof(e) : 0.6; }
        const double H = hotfrac * (double)l2 / (double)(st.ldp * pl.elem);
        int hl = 0;
        while (hl < 31 && (double)(1ll << (hl + 1)) <= H) ++hl;
        A.hot_log2 = hl;
        static int hint = -1;  // SG2V_HINT=0 disables the L2 policy (experiments)
        if (hint < 0) { const char *e = getenv("SG2V_HINT"); hint = e ? atoi(e) : 1; }
        A.hint = hint;
    }
    A.tagged = A.tagged && g.d_vclass != nullptr && !g.partitioned;
    if (vp && vp->mode == 1) {  // column tile of the all-gathered passive table -> bg
        A.mp = vp->stage;
        A.ldp = vp->stage_ld;
        A.cp = vp->cnt;
        A.u0 = vp->u0;
        A.tile_mode = 1;
        A.bg = vp->bg;
        A.smem_group = 0;
        A.stage_a = 0;
        A.hint = 0;
    } else if (vp && vp->mode == 2) {  // combine: B rows complete in bg
        A.bsrc_global = 1;
        A.bg = vp->bg;
        A.src_hist = 0;
    } else if (vp && vp->mode == 3) {  // fused step, whole rows from the staging buffer
        A.hint = 0;
    } else if (vp && vp->mode == 4) {  // split pipeline, gather half: B rows -> bg by position
        A.b_out = vp->bg;
        A.stage_a = 0;
        A.smem_group = st.ldb;
    } else if (vp && vp->mode == 5) {  // split pipeline, eMA half: B rows from bg by position
        A.bsrc_global = 1;
        A.bg = vp->bg;
        A.bg_pos = 1;
        A.src_hist = 0;
    }
    int cls = st.top ? 3 : 2;
    prof_begin(cls, stream);
    int rc;
    const int md = !vp ? 0 : vp->mode == 3 || vp->mode == 4 ? 0 : vp->mode == 5 ? 2 : vp->mode;
    if (pl.prec == SG2V_F32)
        rc = md == 1 ? launch_astep_cfg<float, double, 1>(A, stream)
                     : md == 2 ? launch_astep_cfg<float, double, 2>(A, stream) : launch_astep_cfg<float, double, 0>(A, stream);
    else if (pl.prec == SG2V_F64)
        rc = md == 1 ? launch_astep_cfg<double, double, 1>(A, stream)
                     : md == 2 ? launch_astep_cfg<double, double, 2>(A, stream) : launch_astep_cfg<double, double, 0>(A, stream);
    else
        rc = md == 1 ? launch_astep_cfg<u64, u64, 1>(A, stream)
                     : md == 2 ? launch_astep_cfg<u64, u64, 2>(A, stream) : launch_astep_cfg<u64, u64, 0>(A, stream);
    // algorithmic bytes of a column tile: its share of the step's gather
    // profile records: a column tile carries its share of the gather; a split-pipeline
    // chunk carries its share of the step (gather bytes on the gather launch, eMA terms
    // on the eMA launch)
    const double rows_frac = (double)g.n / (double)std::max<int64_t>(pl.n_rows, 1);
    double fb = 1.0, ft = 1.0;
    if (vp && vp->mode == 1) { fb = (double)vp->cnt / (double)std::max<int64_t>(st.cp, 1); ft = 0.0; }
    else if (vp && vp->mode == 2) { fb = 0.0; }
    else if (vp && vp->mode == 4) { fb = rows_frac; ft = 0.0; }
    else if (vp && vp->mode == 5) { fb = 0.0; ft = rows_frac; }
    prof_end(cls, st.alg_bytes * fb, stream, st.impl_bytes * fb, st.ema_terms * ft);
    return rc;
}

// ---------------------------------------------------------------------------
// split eMA pipeline (GENERAL eMA-heavy steps, Step::split_ema): the rows (degree
// order) are cut into chunks of sp.rows; chunk c's gather (bulk / register kernel, B
// rows to bg[c % 2]) runs on the main stream while chunk c-1's eMA (MODE 2 combine,
// V interleaved rows) runs on the aux stream, so the HBM-bound gather and the
// shared-memory-bound eMA of different rows overlap on the SMs (one kernel of each
// kind co-resident per SM) instead of alternating inside one CTA.
// ---------------------------------------------------------------------------
int launch_astep_split(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const int32_t *hcnt,
                       const int32_t *bcol, char *tables, void *rowval, int *ovf, void *stream, const SplitCtx &sp) {
    cudaStream_t s0 = (cudaStream_t)stream, s1 = (cudaStream_t)sp.aux;
    const int64_t nchunks = (g.n + sp.rows - 1) / sp.rows;
    const size_t half = (size_t)sp.rows * st.ldb * pl.elem;
    cudaError_t e;
    if ((e = cudaEventRecord(sp.ready[0], s0))) return (int)e;  // aux must see the previous steps
    if ((e = cudaStreamWaitEvent(s1, sp.ready[0], 0))) return (int)e;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int par = (int)(c & 1);
        const int64_t r0 = c * sp.rows, r1 = std::min<int64_t>(g.n, r0 + sp.rows);
        if (c >= 2 && (e = cudaStreamWaitEvent(s0, sp.done[par], 0))) return (int)e;  // bg[par] consumed
        Graph gc = g;  // rows r0..r1 of the degree order
        gc.d_order = g.d_order + r0;
        gc.n = r1 - r0;
        gc.n_deg_ge[kHeavyLog2] = std::max<int64_t>(0, std::min<int64_t>(g.n_deg_ge[kHeavyLog2], r1) - r0);
        VpArgs va;
        va.mode = 4;  // gather only -> bg
        va.bg = sp.bg + par * half;
        int rc = launch_astep_vp(gc, pl, st, colors, hcnt, bcol, tables, rowval, ovf, s0, &va);
        if (rc) return rc;
        if ((e = cudaEventRecord(sp.ready[par], s0))) return (int)e;
        if ((e = cudaStreamWaitEvent(s1, sp.ready[par], 0))) return (int)e;
        va.mode = 5;  // eMA from bg (by position)
        rc = launch_astep_vp(gc, pl, st, colors, hcnt, bcol, tables, rowval, ovf, s1, &va);
        if (rc) return rc;
        if ((e = cudaEventRecord(sp.done[par], s1))) return (int)e;
    }
    // join: the main stream continues after every eMA chunk
    for (int par = 0; par < 2 && par < nchunks; ++par)
        if ((e = cudaStreamWaitEvent(s0, sp.done[par], 0))) return (int)e;
    return 0;
}

// ---------------------------------------------------------------------------
// vertex-partitioned mode helpers
// ---------------------------------------------------------------------------
// dst[i][0..w) = src[i][u0..u0+w) (16-B vectors; row strides ldv / dstv vectors)
__global__ void pack_tile_kernel(int64_t n, const uint4 *__restrict__ src, int64_t ldv, int64_t u0v, int64_t wv,
                                 uint4 *__restrict__ dst, int64_t dstv) {
    const int64_t total = n * wv;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / wv, v = q - i * wv;
        dst[i * dstv + v] = src[i * ldv + u0v + v];
    }
}

int launch_pack_tile(int64_t n, const char *src, int64_t ld_bytes, int64_t u0_bytes, int64_t w_bytes, char *dst,
                     int64_t dst_ld_bytes, void *stream) {
    if (n <= 0 || w_bytes <= 0) return 0;
    const int64_t total = n * (w_bytes / 16);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
    pack_tile_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        n, (const uint4 *)src, ld_bytes / 16, u0_bytes / 16, w_bytes / 16, (uint4 *)dst, dst_ld_bytes / 16);
    note_launch();
    return (int)cudaGetLastError();
}

template <typename T, typename RT>
__global__ void bg_rowval_kernel(int64_t n, const T *__restrict__ bg, int64_t ldb, RT *__restrict__ rowval) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        rowval[i] = (RT)bg[i * ldb];
}

int launch_bg_rowval(const Plan &pl, int64_t n, const char *bg, int64_t ldb, void *rowval, void *stream) {
    if (n <= 0) return 0;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    cudaStream_t s = (cudaStream_t)stream;
    if (pl.prec == SG2V_F32) bg_rowval_kernel<float, double><<<(unsigned)blocks, 256, 0, s>>>(n, (const float *)bg, ldb, (double *)rowval);
    else if (pl.prec == SG2V_F64) bg_rowval_kernel<double, double><<<(unsigned)blocks, 256, 0, s>>>(n, (const double *)bg, ldb, (double *)rowval);
    else bg_rowval_kernel<u64, u64><<<(unsigned)blocks, 256, 0, s>>>(n, (const u64 *)bg, ldb, (u64 *)rowval);
    note_launch();
    return (int)cudaGetLastError();
}

}  // namespace sg2v
