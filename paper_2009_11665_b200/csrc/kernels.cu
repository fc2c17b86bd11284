// kernels.cu — sm_100a kernels of the colour-coding hot path.
//
//  a1  colorize_kernel   c(v) = COLOR(seed, j, v, k)
//  a4′ hist_kernel       H(i,x) = #{j∈N(i): c(j)=x}  (leaf-passive SpMM, P:446 with M_p one-hot)
//  a4+a5 step_kernel     fused SpMM + eMA, one row group per vertex:
//                          B(i,·) = Σ_{j∈N(i)} M_p(j,·)  on chip (smem)
//                          M_s(i,I_s) = Σ_splits M_a(i,I_a)·B(i,I_p)
//                        leaf-active form M_s(i,S) = [c(i)∈S]·B(i,S∖c(i))   (a = 1)
//  a6  top_leaf_kernel   colorful_i = Σ_{j∈N(i)} M_p(j, [k]∖c(i))  (top step, a = 1)
//      step_kernel(top)  colorful_i = Σ_{I_a} M_a(i,I_a)·B(i,[k]∖I_a)
//      reduce kernels    colorful_j = Σ_i colorful_i, fixed-order tree (deterministic)
//
// Layout (SURVEY §8(a) "Types"; north_star "vertex-major"): every count table
// is n × ld row-major (vertex-major), the colour-set columns of a vertex
// contiguous and padded to 16 B, so each neighbour contributes one coalesced
// 128-bit-vectorised row read.  No tensor cores: this is a sparse,
// bandwidth-bound contraction (north_star).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdio>
#include <type_traits>

#include "kcommon.cuh"
#include "sg2v_internal.h"

namespace sg2v {

// ---------------------------------------------------------------------------
// a1: colouring (SURVEY §8(c) step 1 counter hash; bias <= k/2^32)
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 mix64(u64 z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

// ids (optional): vertex v is input vertex ids[v] (relabelled graphs colour by input id)
__global__ void colorize_kernel(u64 seed, int64_t j, int64_t n, int k, uint8_t *__restrict__ out,
                                const int32_t *__restrict__ ids) {
    const u64 key = mix64(seed + 0x9E3779B97F4A7C15ULL * (u64)(j + 1));
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const u64 id = ids ? (u64)(uint32_t)ids[v] : (u64)v;
        u64 h = mix64(key ^ (id * 0xD6E8FEB86659FD93ULL));
        out[v] = (uint8_t)(((h >> 32) * (u64)k) >> 32);
    }
}

// ---------------------------------------------------------------------------
// a4′: neighbour colour histogram, warp per row, ballot per colour
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) hist_kernel(int64_t n, int k, const int64_t *__restrict__ rowptr,
                                                   const int32_t *__restrict__ col,
                                                   const uint8_t *__restrict__ colors, T *__restrict__ H,
                                                   int64_t ldh) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        unsigned cnt = 0;
        for (int64_t base = e0; base < e1; base += 32) {
            const int64_t e = base + lane;
            int c = (e < e1) ? (int)colors[__ldg(col + e)] : 255;
            for (int x = 0; x < k; ++x) {
                unsigned b = __ballot_sync(0xffffffffu, c == x);
                if (lane == x) cnt += __popc(b);
            }
        }
        for (int64_t x = lane; x < ldh; x += 32) H[i * ldh + x] = (T)(x < k ? cnt : 0u);
    }
}

// ---------------------------------------------------------------------------
// a4 + a5: fused SpMM + eMA, row-group per vertex, B kept in shared memory
// ---------------------------------------------------------------------------
struct StepArgs {
    int64_t n;
    int k;
    const int64_t *rowptr;
    const int32_t *col;
    const int32_t *order;
    const uint8_t *colors;
    const char *src;   // M_p (gather) or H (src_hist)
    int64_t ldp;       // elements per source row (multiple of 16 B)
    int src_hist;
    const char *ma;    // M_a (GENERAL)
    int64_t lda;
    char *ms;          // M_s (non-top)
    int64_t lds, cs;
    int comb, top;
    const int32_t *idx;
    int64_t nterms;
    void *rowval;      // top: per-vertex values (RT)
    int64_t smem_group;  // elements of shared memory per row group
    int *ovf;          // F32 overflow flag of the call (workspace)
};

template <typename T, typename RT, int GT>
__global__ void __launch_bounds__(256) step_kernel(StepArgs A) {
    constexpr int G = 256 / GT;
    constexpr int VN = Vec<T>::N;
    constexpr int R = 4;  // 16-B vectors per lane per pass
    constexpr int U = 4;  // neighbours in flight per lane
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ RT red[8];
    const int g = threadIdx.x / GT, t = threadIdx.x % GT;
    T *sB = reinterpret_cast<T *>(smem) + (size_t)g * A.smem_group;
    T *sA = sB + A.ldp;
    const int64_t nslots = (A.n + G - 1) / G;
    const int64_t nvec = A.ldp / VN;
    const size_t row_bytes = (size_t)A.ldp * sizeof(T);
    bool bad = false;  // a stored F32 table entry is not finite (EOVERFLOW)

    for (int64_t slot = blockIdx.x; slot < nslots; slot += gridDim.x) {
        const int64_t r = slot * G + g;
        const bool act = r < A.n;
        const int64_t i = act ? A.order[r] : 0;
        // ---- stage 1: B(i,·) into shared memory -------------------------------
        if (act) {
            if (A.src_hist) {
                const char *h = A.src + (size_t)i * row_bytes;
                for (int64_t v = t; v < nvec; v += GT) reinterpret_cast<uint4 *>(sB)[v] = ldg16(h + v * 16);
            } else {
                const int64_t e0 = A.rowptr[i], e1 = A.rowptr[i + 1];
                for (int64_t v0 = 0; v0 < nvec; v0 += GT * R) {
                    uint4 acc[R];
#pragma unroll
                    for (int q = 0; q < R; ++q) acc[q] = make_uint4(0, 0, 0, 0);
                    int64_t e = e0;
                    for (; e + U <= e1; e += U) {
                        int32_t jj[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) jj[u] = __ldg(A.col + e + u);
                        uint4 x[U][R];
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int q = 0; q < R; ++q) {
                                const int64_t v = v0 + q * GT + t;
                                x[u][q] = (v < nvec) ? ldg16(A.src + (size_t)jj[u] * row_bytes + v * 16)
                                                     : make_uint4(0, 0, 0, 0);
                            }
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int q = 0; q < R; ++q) Vec<T>::add(acc[q], x[u][q]);
                    }
                    for (; e < e1; ++e) {
                        const int32_t j1 = __ldg(A.col + e);
#pragma unroll
                        for (int q = 0; q < R; ++q) {
                            const int64_t v = v0 + q * GT + t;
                            if (v < nvec) Vec<T>::add(acc[q], ldg16(A.src + (size_t)j1 * row_bytes + v * 16));
                        }
                    }
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int64_t v = v0 + q * GT + t;
                        if (v < nvec) reinterpret_cast<uint4 *>(sB)[v] = acc[q];
                    }
                }
            }
            if (A.comb == COMB_GENERAL) {
                const char *a = A.ma + (size_t)i * A.lda * sizeof(T);
                for (int64_t v = t; v < A.lda / VN; v += GT) reinterpret_cast<uint4 *>(sA)[v] = ldg16(a + v * 16);
            }
        }
        group_sync<GT>(g);
        // ---- stage 2: eMA into M_s (or the top per-vertex value) ---------------
        RT racc = 0;
        if (act) {
            if (!A.top) {
                T *out = reinterpret_cast<T *>(A.ms) + (size_t)i * A.lds;
                if (A.comb == COMB_ACTIVE_LEAF) {
                    const int32_t *m = A.idx + (size_t)A.colors[i] * A.cs;
                    for (int64_t o = t; o < A.lds; o += GT) {
                        T val = 0;
                        if (o < A.cs) {
                            const int32_t q = __ldg(m + o);
                            if (q >= 0) val = sB[q];
                        }
                        if constexpr (std::is_same<T, float>::value) bad |= !isfinite(val);
                        out[o] = val;
                    }
                } else {
                    const int2 *sp = reinterpret_cast<const int2 *>(A.idx);
                    for (int64_t o = t; o < A.lds; o += GT) {
                        T acc = 0;
                        if (o < A.cs) {
                            const int2 *p = sp + (size_t)o * A.nterms;
                            for (int64_t w = 0; w < A.nterms; ++w) {
                                const int2 q = __ldg(p + w);
                                acc += sA[q.x] * sB[q.y];
                            }
                        }
                        if constexpr (std::is_same<T, float>::value) bad |= !isfinite(acc);
                        out[o] = acc;
                    }
                }
            } else {
                const int2 *sp = reinterpret_cast<const int2 *>(A.idx);
                for (int64_t w = t; w < A.nterms; w += GT) {
                    const int2 q = __ldg(sp + w);
                    racc += (RT)sA[q.x] * (RT)sB[q.y];
                }
            }
        }
        if (A.top) {
            RT s = group_reduce<RT, GT>(racc, g, red);
            if (act && t == 0) reinterpret_cast<RT *>(A.rowval)[i] = s;
        }
        group_sync<GT>(g);
    }
    if (bad) atomicOr(A.ovf, 1);
}

// ---------------------------------------------------------------------------
// a6 (leaf-active top): colorful_i = Σ_{j∈N(i)} M_p(j, topcol[c(i)])
// ---------------------------------------------------------------------------
template <typename T, typename RT>
__global__ void __launch_bounds__(256) top_leaf_kernel(int64_t n, const int64_t *__restrict__ rowptr,
                                                       const int32_t *__restrict__ col,
                                                       const uint8_t *__restrict__ colors,
                                                       const T *__restrict__ src, int64_t ldp, int src_hist,
                                                       const int32_t *__restrict__ topcol, RT *__restrict__ rowval) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        const int q = __ldg(topcol + colors[i]);
        RT acc = 0;
        if (src_hist) {
            if (lane == 0) acc = (RT)src[(size_t)i * ldp + q];
        } else {
            const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
            for (int64_t e = e0 + lane; e < e1; e += 32) acc += (RT)__ldg(src + (size_t)__ldg(col + e) * ldp + q);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
        }
        if (lane == 0) rowval[i] = acc;
    }
}

// ---------------------------------------------------------------------------
// deterministic Σ_i (fixed grid, fixed tree) — P:154 finalCount numerator
// ---------------------------------------------------------------------------
template <typename RT>
__global__ void __launch_bounds__(256) reduce_partial_kernel(const RT *__restrict__ v, int64_t n, RT *__restrict__ partial) {
    __shared__ RT sh[256];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    RT s = 0;
    for (int64_t q = b0 + threadIdx.x; q < b1; q += blockDim.x) s += v[q];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

template <typename RT>
__global__ void __launch_bounds__(256) reduce_final_kernel(const RT *__restrict__ partial, int nb, RT *__restrict__ out) {
    __shared__ RT sh[256];
    RT s = 0;
    for (int q = threadIdx.x; q < nb; q += blockDim.x) s += partial[q];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// ---------------------------------------------------------------------------
// graph preprocessing: degree-descending order; CSR validation
// ---------------------------------------------------------------------------
__global__ void degree_kernel(int64_t n, const int64_t *__restrict__ rowptr, int32_t *__restrict__ deg,
                              int32_t *__restrict__ ids) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        deg[i] = (int32_t)(rowptr[i + 1] - rowptr[i]);
        ids[i] = (int32_t)i;
    }
}

// cnt[q] = number of rows with degree >= 2^q in the descending degree array
__global__ void deg_count_kernel(const int32_t *__restrict__ deg_sorted, int64_t n, int64_t *__restrict__ cnt) {
    const int q = threadIdx.x;
    if (q >= 32) return;
    const int64_t thr = int64_t(1) << q;
    int64_t lo = 0, hi = n;  // first position with degree < thr
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if ((int64_t)deg_sorted[mid] >= thr) lo = mid + 1; else hi = mid;
    }
    cnt[q] = lo;
}

__global__ void vclass_kernel(int64_t n, const int32_t *__restrict__ order, uint8_t *__restrict__ vclass) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        vclass[order[r]] = (uint8_t)(63 - __clzll((unsigned long long)(r + 1)));
}

__global__ void validate_kernel(int64_t n, int64_t nnz, const int64_t *__restrict__ rowptr,
                                const int32_t *__restrict__ col, int *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        if (e0 > e1 || e1 > nnz || e0 < 0) { atomicOr(bad, 1); continue; }
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t j = col[e];
            if (j < 0 || j >= n) { atomicOr(bad, 2); break; }
            if (j == i) atomicOr(bad, 4);
            if (e > e0 && col[e - 1] >= j) atomicOr(bad, 8);
            // symmetry: binary search i in N(j)
            int64_t lo = rowptr[j], hi = rowptr[j + 1];
            bool found = false;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                int32_t x = col[mid];
                if (x == i) { found = true; break; }
                if (x < i) lo = mid + 1; else hi = mid;
            }
            if (!found) atomicOr(bad, 16);
        }
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

int launch_colorize(uint64_t seed, int64_t j, int64_t n, int k, uint8_t *out, void *stream, const int32_t *ids) {
    if (n <= 0) return 0;
    int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    prof_begin(0, stream);
    colorize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(seed, j, n, k, out, ids);
    note_launch();
    prof_end(0, (double)n, stream);
    return (int)cudaGetLastError();
}

int launch_hist(const Graph &g, const Plan &pl, const uint8_t *colors, void *H, void *stream) {
    if (g.n <= 0) return 0;
    int64_t blocks = std::min<int64_t>((g.n + 7) / 8, (int64_t)num_sms() * 8);
    double bytes = g.nnz * 5.0 + g.n * 12.0 + (double)g.n * pl.k * pl.elem;
    prof_begin(1, stream);
    if (pl.prec == SG2V_F32)
        hist_kernel<float><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(g.n, pl.k, g.d_rowptr, g.d_col, colors, (float *)H, pl.ldh);
    else if (pl.prec == SG2V_F64)
        hist_kernel<double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(g.n, pl.k, g.d_rowptr, g.d_col, colors, (double *)H, pl.ldh);
    else
        hist_kernel<u64><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(g.n, pl.k, g.d_rowptr, g.d_col, colors, (u64 *)H, pl.ldh);
    note_launch();
    prof_end(1, bytes, stream);
    return (int)cudaGetLastError();
}

template <typename T, typename RT, int GT>
static int launch_step_t(const StepArgs &A, void *stream) {
    auto kern = step_kernel<T, RT, GT>;
    constexpr int G = 256 / GT;
    size_t smem = (size_t)G * A.smem_group * sizeof(T);
    if (smem > 227 * 1024) return -1;
    if (cudaError_t e = ensure_dyn_smem((const void *)kern, smem)) return (int)e;    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    if (occ < 1) occ = 1;
    int64_t nslots = (A.n + G - 1) / G;
    int64_t blocks = std::min<int64_t>(nslots, (int64_t)occ * num_sms());
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, smem, (cudaStream_t)stream>>>(A);
    note_launch();
    return (int)cudaGetLastError();
}

template <typename T, typename RT>
static int launch_step_gt(const StepArgs &A, int gt, void *stream) {
    switch (gt) {
        case 4: return launch_step_t<T, RT, 4>(A, stream);
        case 8: return launch_step_t<T, RT, 8>(A, stream);
        case 16: return launch_step_t<T, RT, 16>(A, stream);
        case 32: return launch_step_t<T, RT, 32>(A, stream);
        case 64: return launch_step_t<T, RT, 64>(A, stream);
        case 128: return launch_step_t<T, RT, 128>(A, stream);
        default: return launch_step_t<T, RT, 256>(A, stream);
    }
}

int launch_step(const Graph &g, const Plan &pl, const Step &st, const uint8_t *colors, const void *H,
                char *tables, void *rowval, int *ovf, void *stream) {
    if (g.n <= 0) return 0;
    const int32_t *idx = pl.d_index + st.idx_off;
    const char *src = (st.src == SRC_HIST) ? (const char *)H : tables + pl.bufs[st.buf_p].offset;
    if (st.top && st.comb == COMB_ACTIVE_LEAF) {
        int64_t blocks = std::min<int64_t>((g.n + 7) / 8, (int64_t)num_sms() * 8);
        int srch = st.src == SRC_HIST;
        prof_begin(3, stream);
        if (pl.prec == SG2V_F32)
            top_leaf_kernel<float, double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
                g.n, g.d_rowptr, g.d_col, colors, (const float *)src, st.ldp, srch, idx, (double *)rowval);
        else if (pl.prec == SG2V_F64)
            top_leaf_kernel<double, double><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
                g.n, g.d_rowptr, g.d_col, colors, (const double *)src, st.ldp, srch, idx, (double *)rowval);
        else
            top_leaf_kernel<u64, u64><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
                g.n, g.d_rowptr, g.d_col, colors, (const u64 *)src, st.ldp, srch, idx, (u64 *)rowval);
        note_launch();
        prof_end(3, st.alg_bytes, stream, st.impl_bytes, 0.0);
        return (int)cudaGetLastError();
    }
    StepArgs A;
    A.n = g.n;
    A.k = pl.k;
    A.rowptr = g.d_rowptr;
    A.col = g.d_col;
    A.order = g.d_order;
    A.colors = colors;
    A.src = src;
    A.ldp = st.ldp;
    A.src_hist = st.src == SRC_HIST;
    A.ma = (st.comb == COMB_GENERAL && st.buf_a >= 0) ? tables + pl.bufs[st.buf_a].offset : nullptr;
    A.lda = st.lda;
    A.ms = st.top ? nullptr : tables + pl.bufs[st.buf_out].offset;
    A.lds = st.lds;
    A.cs = st.cs;
    A.comb = st.comb;
    A.top = st.top;
    A.idx = idx;
    A.nterms = st.nterms;
    A.rowval = rowval;
    A.smem_group = st.ldp + (st.comb == COMB_GENERAL ? st.lda : 0);
    A.ovf = ovf;
    int cls = st.top ? 3 : 2;
    prof_begin(cls, stream);
    int rc;
    if (pl.prec == SG2V_F32) rc = launch_step_gt<float, double>(A, st.gt, stream);
    else if (pl.prec == SG2V_F64) rc = launch_step_gt<double, double>(A, st.gt, stream);
    else rc = launch_step_gt<u64, u64>(A, st.gt, stream);
    prof_end(cls, st.alg_bytes, stream, st.impl_bytes, st.ema_terms);
    return rc;
}

int launch_reduce(const Plan &pl, int64_t n, const void *rowval, void *partial, void *result, void *stream) {
    prof_begin(4, stream);
    if (pl.prec == SG2V_U64) {
        reduce_partial_kernel<u64><<<kReduceBlocks, 256, 0, (cudaStream_t)stream>>>((const u64 *)rowval, n, (u64 *)partial);
        note_launch();
        reduce_final_kernel<u64><<<1, 256, 0, (cudaStream_t)stream>>>((const u64 *)partial, kReduceBlocks, (u64 *)result);
        note_launch();
    } else {
        reduce_partial_kernel<double><<<kReduceBlocks, 256, 0, (cudaStream_t)stream>>>((const double *)rowval, n, (double *)partial);
        note_launch();
        reduce_final_kernel<double><<<1, 256, 0, (cudaStream_t)stream>>>((const double *)partial, kReduceBlocks, (double *)result);
        note_launch();
    }
    prof_end(4, (double)n * 8.0, stream);
    return (int)cudaGetLastError();
}

// Colour-grouped processing order (SG2V_CORDER, on): the heavy prefix of the
// degree order unchanged, the light rows stably sorted by their colour c(i) (degree order
// kept within a colour), so the CTAs of a wide step gather the SAME segment c(i) of the
// hub rows at the same time — segment-sized (not row-sized) hot rows for the L2.
__global__ void colour_keys_kernel(int64_t n, const int32_t *__restrict__ order, const uint8_t *__restrict__ colors,
                                   uint8_t *__restrict__ keys) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        keys[r] = colors[order[r]];
}

size_t colour_order_tmp_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint8_t *)nullptr, (uint8_t *)nullptr, (const int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)std::max<int64_t>(n, 1), 0, 8);
    return t;
}

int launch_colour_order(const Graph &g, const uint8_t *colors, int32_t *order_out, uint8_t *keys, void *tmp,
                        size_t tmp_bytes, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nh = std::min<int64_t>(g.n_deg_ge[11], g.n), nl = g.n - nh;
    if (nh > 0) {
        cudaError_t e = cudaMemcpyAsync(order_out, g.d_order, nh * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return (int)e;
    }
    if (nl <= 0) return 0;
    colour_keys_kernel<<<(unsigned)std::min<int64_t>((nl + 255) / 256, 4096), 256, 0, s>>>(nl, g.d_order + nh, colors, keys);
    note_launch();
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys + nl, g.d_order + nh, order_out + nh,
                                                    (int)nl, 0, 8, s);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

int graph_build_order(Graph &g, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n = g.n;
    if (n <= 0) return 0;
    int32_t *deg = nullptr, *deg_sorted = nullptr, *ids = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaMallocAsync((void **)&deg, n * sizeof(int32_t) * 3, s);
    if (e != cudaSuccess) return (int)e;
    deg_sorted = deg + n;
    ids = deg + 2 * n;
    degree_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(n, g.d_rowptr, deg, ids);
    note_launch();
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, deg, deg_sorted, ids, g.d_order, (int)n, 0, 32, s);
    e = cudaMallocAsync(&tmp, tmp_bytes, s);
    if (e == cudaSuccess) {
        cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, deg, deg_sorted, ids, g.d_order, (int)n, 0, 32, s);
        vclass_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(n, g.d_order, g.d_vclass);
        note_launch();
        int32_t mx = 0;
        cudaMemcpyAsync(&mx, deg_sorted, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(tmp, s);
        e = cudaStreamSynchronize(s);
        g.max_deg = mx;
        // rows with degree >= 2^q (a prefix of the descending order), one thread per q
        int64_t *d_cnt = nullptr;
        if (e == cudaSuccess && (e = cudaMallocAsync((void **)&d_cnt, 32 * sizeof(int64_t), s)) == cudaSuccess) {
            deg_count_kernel<<<1, 32, 0, s>>>(deg_sorted, n, d_cnt);
            note_launch();
            cudaMemcpyAsync(g.n_deg_ge, d_cnt, 32 * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
            cudaFreeAsync(d_cnt, s);
            e = cudaStreamSynchronize(s);
        }
    }
    cudaFreeAsync(deg, s);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

int graph_validate(const Graph &g, int *bad, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    int *d_bad = nullptr;
    cudaError_t e = cudaMalloc(&d_bad, sizeof(int));
    if (e != cudaSuccess) return (int)e;
    cudaMemsetAsync(d_bad, 0, sizeof(int), s);
    if (g.n > 0) {
        validate_kernel<<<(unsigned)std::min<int64_t>((g.n + 255) / 256, 8192), 256, 0, s>>>(g.n, g.nnz, g.d_rowptr, g.d_col, d_bad);
        note_launch();
    }
    cudaMemcpyAsync(bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    cudaFree(d_bad);
    return (int)e;
}

}  // namespace sg2v
