// smcsd_device.cuh -- device helpers for libsmcsd (sm_100a).  No host code, no torch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace smcsd {

constexpr int kThreads = 256;            // CTA size of every kernel in the library
constexpr int kWarps = kThreads / 32;
constexpr int kSeg = 8192;               // SMCSD_SEGMENT: fixed in-row segment (G17)
constexpr int kTailMaxN = 1024;          // fused tail / resample keep per-prompt state in smem

// ---- scalars -------------------------------------------------------------------------
// Packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2 / FMUL2): two lanes of IEEE fp32 per issue
// slot, each lane rounded exactly as its scalar counterpart (fma fused, add/mul rn).
__device__ __forceinline__ unsigned long long pk2(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return upk2(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}

// 2^x on the FMA pipe (packed fp32x2), x <= 0: x = n + f with n = round(x) by the 1.5 * 2^23
// trick (f in [-1/2, 1/2], exact), 2^f by a degree-4 minimax polynomial (max relative error
// 2.7e-6 in fp32 Horner), times 2^n built from exponent bits (exact).  x is clamped at -127
// first, so -inf (masked columns) gives exactly 0; NaN is NOT propagated (callers must detect
// NaN elsewhere).  Used for the PowerSMC second sum only, where the MUFU pipe is the limit
// (two ex2 per element); the plain exp-sum measured slower with it (profiles/r01f_ab_poly_exp2.txt).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -127.0f);
    x.y = fmaxf(x.y, -127.0f);
    const float2 y = fadd2(x, make_float2(12582912.0f, 12582912.0f));     // 1.5 * 2^23 + round(x)
    const float2 r = fadd2(y, make_float2(-12582912.0f, -12582912.0f));   // round(x)
    const float2 f = fadd2(x, make_float2(-r.x, -r.y));                   // x - round(x)
    float2 p = ffma2(make_float2(0.009570609778165817f, 0.009570609778165817f), f,
                     make_float2(0.055917903780937195f, 0.055917903780937195f));
    p = ffma2(p, f, make_float2(0.24024732410907745f, 0.24024732410907745f));
    p = ffma2(p, f, make_float2(0.6931217908859253f, 0.6931217908859253f));
    p = ffma2(p, f, make_float2(0.9999992847442627f, 0.9999992847442627f));
    const float sx = __uint_as_float((__float_as_uint(y.x) - 0x4B3FFF81u) << 23);   // 2^n
    const float sy = __uint_as_float((__float_as_uint(y.y) - 0x4B3FFF81u) << 23);
    return fmul2(p, make_float2(sx, sy));
}

__device__ __forceinline__ float ex2_approx(float x) {
#ifdef SMCSD_EXPERIMENT_NO_EX2          // timing experiment only: wrong numerics
    return x * 0.5f;
#else
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#endif
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Streaming 16-byte load: read-only path, no L1 allocation (each logit byte is read once).
__device__ __forceinline__ uint4 ld_stream(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream(void *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Butterfly sum: every lane ends with the same bits (x+y == y+x at each level).
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---- optional timeline trace (debug builds only: -DSMCSD_TRACE) ---------------------------
#ifdef SMCSD_TRACE
__device__ unsigned long long g_trace[4096];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SMCSD_TRACE_AT(slot) do { g_trace[(slot)] = gtimer(); } while (0)
#define SMCSD_CLK_AT(slot) do { g_trace[(slot)] = clock64(); } while (0)
#else
#define SMCSD_TRACE_AT(slot) do { } while (0)
#define SMCSD_CLK_AT(slot) do { } while (0)
#endif

// ---- mbarrier + bulk async copy (TMA 1-D) --------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}"
        :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
// 1-D bulk copy global -> shared, completion counted in bytes on `bar` (16-B aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---- Philox4x32-10 (Salmon et al. SC'11), own implementation (reading G5) ---------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            key.x += 0x9E3779B9u;
            key.y += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * ctr.x, hi0 = __umulhi(0xD2511F53u, ctr.x);
        const uint32_t lo1 = 0xCD9E8D57u * ctr.z, hi1 = __umulhi(0xCD9E8D57u, ctr.z);
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    }
    return ctr;
}

// ---- block-wide exclusive scan of int over n <= kTailMaxN entries held in smem -------------
// Returns the total.  All threads of the CTA must call it.  `wtot` is kWarps+1 ints of smem.
__device__ __forceinline__ int block_exclusive_scan(int *data, int n, int *wtot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int carry = 0;
    for (int base = 0; base < n; base += kThreads) {
        const int i = base + tid;
        const int v = i < n ? data[i] : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtot[warp] = x;
        __syncthreads();
        if (tid == 0) {
            int acc = 0;
            for (int w = 0; w < kWarps; ++w) {
                const int t = wtot[w];
                wtot[w] = acc;
                acc += t;
            }
            wtot[kWarps] = acc;
        }
        __syncthreads();
        if (i < n) data[i] = carry + wtot[warp] + x - v;
        carry += wtot[kWarps];
        __syncthreads();
    }
    return carry;
}

}  // namespace smcsd
