// kcommon.cuh — device helpers shared by the dense (kernels.cu) and the
// root-colour-anchored (akernels.cu) kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <utility>

namespace sg2v {

// Device bounds checks of the check build (libsg2v_check.so, build(check=True)): shared-
// memory push targets, ring slots, bucket positions.  compute-sanitizer is not available
// on the GPU pool, so the GPU parity suite is run once against this build as well
// (tools/check_run.sh); the product build compiles them out.
#ifdef SG2V_CHECK
#define SG2V_DASSERT(c)                                                                          \
    do {                                                                                        \
        if (!(c)) {                                                                             \
            printf("SG2V_CHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define SG2V_DASSERT(c) \
    do {                \
    } while (0)
#endif

typedef unsigned long long u64;

// 16-byte vector arithmetic on raw uint4 bits, per element type
template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int N = 4;
    __device__ __forceinline__ static void add(uint4 &a, const uint4 &b) {
        a.x = __float_as_uint(__uint_as_float(a.x) + __uint_as_float(b.x));
        a.y = __float_as_uint(__uint_as_float(a.y) + __uint_as_float(b.y));
        a.z = __float_as_uint(__uint_as_float(a.z) + __uint_as_float(b.z));
        a.w = __float_as_uint(__uint_as_float(a.w) + __uint_as_float(b.w));
    }
};
template <> struct Vec<double> {
    static constexpr int N = 2;
    __device__ __forceinline__ static void add(uint4 &a, const uint4 &b) {
        double2 x = *reinterpret_cast<double2 *>(&a);
        const double2 y = *reinterpret_cast<const double2 *>(&b);
        x.x += y.x;
        x.y += y.y;
        a = *reinterpret_cast<uint4 *>(&x);
    }
};
template <> struct Vec<u64> {
    static constexpr int N = 2;
    __device__ __forceinline__ static void add(uint4 &a, const uint4 &b) {
        ulonglong2 x = *reinterpret_cast<ulonglong2 *>(&a);
        const ulonglong2 y = *reinterpret_cast<const ulonglong2 *>(&b);
        x.x += y.x;  // wraps mod 2^64 (exact residue arithmetic)
        x.y += y.y;
        a = *reinterpret_cast<uint4 *>(&x);
    }
};

// read-only 128-bit load through the non-coherent path
__device__ __forceinline__ uint4 ldg16(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 128-bit load with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ uint4 ldg16_pol(const void *p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
// predicated 128-bit load with an L2 policy: zero when !pred.  The predicate is
// applied to the load instruction itself (no branch), so a batch of these stays
// in flight together whatever control flow the compiler would otherwise choose.
__device__ __forceinline__ uint4 ldg16_pred(const void *p, bool pred, uint64_t pol) {
    uint4 r = make_uint4(0, 0, 0, 0);
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
        "@q ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%5], %6;\n\t}"
        : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
        : "r"((int)pred), "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Synchronise the GT threads of row group g (GT | 256).  Groups narrower than a
// warp sync only their own lanes, so the call is legal inside group-uniform
// (but warp-divergent) control flow.
template <int GT>
__device__ __forceinline__ void group_sync(int g) {
    if constexpr (GT < 32) {
        const unsigned lane = threadIdx.x & 31u;
        const unsigned mask = ((1u << GT) - 1u) << (lane & ~(unsigned)(GT - 1));
        __syncwarp(mask);
    } else if constexpr (GT == 32) {
        __syncwarp();
    } else if constexpr (GT == 256) {
        // named barrier 1 of 256 threads (not bar 0): the bulk-staged kernel runs a
        // producer warp beside the 256 consumer threads, which must not join
        asm volatile("bar.sync 1, 256;" ::: "memory");
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(GT) : "memory");
    }
}

// Sum over the GT threads of group g (must be called by every thread of the
// block, in uniform control flow).  Result valid in the group's thread 0.
template <typename RT, int GT>
__device__ __forceinline__ RT group_reduce(RT v, int g, RT *red) {
    const int lane = threadIdx.x & 31;
    constexpr int W = GT < 32 ? GT : 32;
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off, W);
    if constexpr (GT > 32) {
        const int warp = threadIdx.x >> 5;
        if (lane == 0) red[warp] = v;
        group_sync<GT>(g);
        RT s = 0;
        if ((threadIdx.x % GT) == 0)
            for (int w = 0; w < GT / 32; ++w) s += red[g * (GT / 32) + w];
        return s;
    } else {
        return v;
    }
}

// element e (0..VN-1) of a 16-B vector as T
template <typename T>
__device__ __forceinline__ T vget(const uint4 &v, int e) {
    return reinterpret_cast<const T *>(&v)[e];
}

// set element e (0..VN-1) of a 16-B vector
template <typename T>
__device__ __forceinline__ void vset(uint4 &v, int e, T x) {
    reinterpret_cast<T *>(&v)[e] = x;
}

// ---- mbarrier + bulk-copy (TMA engine, non-tensor) helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both ends 16-B aligned), completion
// counted on `bar` (complete_tx), L2 eviction policy `pol` (createpolicy)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint4 lds16(const void *p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(smem_u32(p)));
    return r;
}

int num_sms();

// Opt a kernel into `smem` bytes of dynamic shared memory on the CURRENT device.
// The attribute is per (function, device), so it is tracked per (kernel, device)
// under a lock (launches may come from several threads / devices).
inline cudaError_t ensure_dyn_smem(const void *kern, size_t smem) {
    if (smem <= 48 * 1024) return cudaSuccess;
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t &have = done[{kern, dev}];
    if (have >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = smem;
    return e;
}

}  // namespace sg2v
