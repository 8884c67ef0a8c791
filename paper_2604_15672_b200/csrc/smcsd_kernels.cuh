// smcsd_kernels.cuh -- the sm_100a kernels of libsmcsd.
//
//  K1  k_rowstats<DT, PW>    S1: per (logit row, fixed 8192-element segment) work item, one
//                            streaming pass: m = max t, s = sum 2^(t - m) (PowerSMC: and
//                            s2 = sum 2^(alpha (t - m))), t = inv_temp * z * log2(e)
//                            (Eq. 1a).  Persistent warp-specialised
//                            CTAs: a producer warp streams items into a 2-stage shared-memory
//                            ring with cp.async.bulk (TMA), 8 consumer warps reduce them.
//  K2  k_tail                PDL-launched behind K1, one CTA per 32 (particle, position) pairs
//                            of a prompt: S2 merge segments in fixed order -> ell and the S3
//                            terms; the prompt's last CTA (completion counter) runs S3, S4 fp64
//                            normalise + ESS, S5-S7 resampling from Philox, reset.  Bonus-token
//                            CTAs (NEXT #2) in the same grid.
//  K3  k_kv_reindex          S8/S9 source-major bitwise gather of per-particle blocks of up to
//                            256 state tensors.
//  and k_merge_rows / k_tail_large / k_resample / k_power_tail / k_select / k_paged_* (see each).
//
// Determinism (reading G17): every row uses the same segment boundaries and the same
// element->thread->warp->segment reduction order, so bitwise-equal p and q rows give
// bitwise-equal ell (p == q => Delta == 0 exactly) and every run is bit-reproducible.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>
#include "smcsd_device.cuh"

namespace smcsd {


constexpr uint32_t ST_DEGENERATE = 1u, ST_NOT_ABSCONT = 2u, ST_BAD_TOKEN = 4u, ST_NONFINITE = 8u;
constexpr uint32_t ST_BAD_PAGE = 16u;
constexpr uint32_t ST_EXCHANGE = 32u;                         // S10 peer flag wait timed out
constexpr uint32_t ST_BAD_INDEX = 64u;                        // reindex: src_index out of range / hazard
constexpr uint64_t kXTimeoutNs = 20000000000ull;              // 20 s
#ifndef SMCSD_PHASE
#ifdef SMCSD_TRACE
// S4-S7 phase clocks of prompt 0 (trace build): g_trace[2300 + i]
#define SMCSD_PHASE(i) do { if (lane == 0 && p == 0) g_trace[2300 + (i)] = clock64(); } while (0)
#else
#define SMCSD_PHASE(i) do { } while (0)
#endif
#endif
}  // namespace smcsd
#include "smcsd_warp_tail.cuh"
namespace smcsd {
constexpr double kLn2 = 0.693147180559945309417232121458176568;
constexpr int kRowStatSmem = 2048;                           // rows whose S2 stats fit in smem

struct Params {
    // ---- inputs (S1)
    const char *lp;  int64_t ld_p; int rpp_p;   // target logits (bytes base), ld in elements
    const char *lq;  int64_t ld_q; int rpp_q;   // draft logits
    const int32_t *tokens;                      // [P][N][K]
    const int32_t *n_drafted;                   // [P][N] or null
    const float *logw_prev;                     // [P][N] or null (-ln N)
    int P, N, K;
    int64_t V;                                  // full vocabulary (token range check)
    int64_t v_begin, v_len;                     // columns held by these rows (shard)
    int nseg;                                   // ceil(v_len / kSeg)
    float c_p, c_q;                             // inv_temp * log2(e)
    double alpha;
    // ---- resampling
    double eta;
    uint64_t seed, step;
    int64_t prompt_base;
    const uint32_t *uniforms;
    // ---- outputs
    float *logw_out, *logw_pre, *logp_tok, *logq_tok, *wnorm;
    double *lse, *ess;
    uint32_t *status;
    int32_t *ancestors, *offspring, *slot_src, *n_ties;
    int32_t *bonus_tok;                         // [P][N] bonus token (NEXT #2) or null
    long long main_items;                       // K1 items of the weight rows
    long long bonus_items;                      // K1 items of the bonus rows (P*N*nseg or 0)
    uint8_t *resampled;
    float4 *partials_out;                       // MODE_PARTIAL: [P*2*N*K] {m, s, x, 0}
    // ---- S2 sources: row r's parts at parts[r*part_row_stride + i*part_seg_stride], i < nparts
    const float4 *parts;
    int64_t part_row_stride, part_seg_stride;
    int nparts;
    // ---- workspace
    float4 *part_ws;                            // [P*2*N*K*nseg]
    unsigned long long *lt_words;               // polling tails: [nseg][P*2*N*K] {m, s} words
                                                // K1 publishes, zero between steps; or null
    double *ell_ws;                             // [P*2*N*K]
    float *lam_ws;                              // [P*N]   (N > kTailMaxN path)
    double *e_ws, *c_ws;                        // [P*N]
    float4 *rowstat_ws;                         // [P*2*N*K] (rows > kRowStatSmem)
    unsigned long long mg_nseg, mg_K, mg_N;     // magic multipliers: x / d == (x * mg) >> (32 + sh)
    int sh_nseg, sh_K, sh_N;
    int dtype;                                  // 0 fp32, 1 bf16 (logits)
    int scheme;                                 // 0 systematic, 1 multinomial
    int n_models;                               // 2: target + draft rows; 1: PowerSMC (target only)
    float alpha_f;                              // PowerSMC exponent (K1 second sum)
    int32_t *selected;                          // smcsd_select output [P]
    int x_from_logits;                          // 1: tail loads t_d from the logits; 0: from parts
    int late_claim;                             // K1: claim items only when a ring slot is free
    unsigned gate_ctr;                          // k_tail_small: work_ctr once every K1 item is claimed
    unsigned *work_ctr;                         // K1 dynamic work counter (re-armed by K2)
    unsigned *prompt_ctr;                       // [P] K2 chunk completion counters
    uint32_t *st_ws;                            // [P] K2 status accumulation
    // ---- S10 fused peer-memory exchange (TP): K1 pushes each segment partial to every rank
    char *const *xpeer;                         // [G] device array: every rank's exchange buffer
    char *xlocal;                               // this rank's exchange buffer (tail reads it)
    int xrank, xG, xnseg;                       // rank, ranks, segment slots per rank
    uint32_t xepoch;                            // this step's epoch (>= 1), or 0: device epoch
    unsigned *xctr;                             // K1 CTA completion counter (workspace)
    int64_t xhalf;                              // tail, device epoch: float4 elements per half
};

// Exchange buffer layout (one per rank, peer-mapped): uint32 flags[64] (flags[g] = last epoch
// rank g finished pushing here; word kXEpochWord = this rank's last completed epoch and word
// kXTailCtrWord = the tail's CTA completion count, both local, device-epoch mode only), then two
// parity halves of [rows][G * xnseg] float4 partials {m, s, x, 0}; row r's slot g * xnseg + s
// holds segment s of rank g's shard, so the rank-order merge of a row's G * xnseg parts is the
// global column order.
constexpr int kXFlagBytes = 256;
constexpr int kXEpochWord = 48, kXTailCtrWord = 49;         // flags[g] use words 0 .. 31
// This launch's epoch: the host's, or (xepoch == 0) one past the last epoch this rank completed
// -- device-resident, so a captured CUDA graph advances it on every replay.
__device__ __forceinline__ uint32_t x_epoch(const Params &prm) {
    return prm.xepoch ? prm.xepoch
                      : __ldcg(reinterpret_cast<const uint32_t *>(prm.xlocal) + kXEpochWord) + 1u;
}
__host__ __device__ inline size_t x_half_elems(int rows, int G, int xnseg) {
    return (size_t)rows * G * xnseg;
}
__device__ __forceinline__ float4 *x_parts(char *base, int rows, int G, int xnseg, uint32_t epoch) {
    return reinterpret_cast<float4 *>(base + kXFlagBytes) + (epoch & 1u) * x_half_elems(rows, G, xnseg);
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Store into cluster rank `rank`'s copy of a shared-memory object (distributed shared memory).
__device__ __forceinline__ void st_cluster_f32(float *local, unsigned rank, float v) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(r), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_f64(double *local, unsigned rank, double v) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(r), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t *local, unsigned rank, uint32_t v) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(local), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(r), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(void *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu_b64(void *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_b64(const void *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const void *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------------------------------
// Programmatic dependent launch (PDL): the tail / gather kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, start while their predecessor drains,
// and block in griddepcontrol.wait until its memory is visible.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------------------------------
// K1: S1 over (row, 8192-column segment) work items.  Persistent CTAs own contiguous item
// ranges; every thread keeps the NEXT item's 16-byte loads in flight (register double
// buffer) while it reduces the current one, so the per-item block merge never drains the
// memory pipe.  One CTA-wide barrier per item; warp 0 merges the 8 warp partials with a
// fixed-order shuffle tree and stores {m, s, x, 0}.
// ------------------------------------------------------------------------------------------
template <int DT>
struct ItemTraits {
    static constexpr int kEsz = DT == 1 ? 2 : 4;
    static constexpr int kVec = 16 / kEsz;                   // elements per 16-byte vector
    static constexpr int kLoads = kSeg / (kThreads * kVec);  // vectors per thread: 4 / 8
    static constexpr uint32_t kNegInf = DT == 1 ? 0xFF80FF80u : 0xFF800000u;
};

__device__ __forceinline__ int drafted_len(const Params &prm, int64_t pn) {
    return prm.n_drafted ? prm.n_drafted[pn] : prm.K;
}

// t_d = inv_temp * z_d * log2(e) for global token d of row (model, pn, j), or -inf when d is not
// among this row's columns [v_begin, v_begin + v_len).
__device__ __forceinline__ float load_x(const Params &prm, int model, int64_t pn, int j, int64_t d) {
    const int64_t dl = d - prm.v_begin;
    if (dl < 0 || dl >= prm.v_len) return -INFINITY;
    const int esz = prm.dtype == 1 ? 2 : 4;
    const char *row = model == 0 ? prm.lp + ((pn * prm.rpp_p + j) * prm.ld_p) * esz
                                 : prm.lq + ((pn * prm.rpp_q + j) * prm.ld_q) * esz;
    const float z = prm.dtype == 1 ? bf16lo(__ldg((const unsigned short *)row + dl))
                                   : __ldg((const float *)row + dl);
    return z * (model == 0 ? prm.c_p : prm.c_q);
}

// Reduce one item held in registers: lane 0 of each warp writes red[warp] = {m_w, s_w, s2_w}
// with s2 = sum 2^(alpha (t - m)) for PowerSMC (PW != 0), 0 otherwise.  PW = -1: general alpha,
// a second ex2 per element; PW = k in 1..4: alpha == k, 2^(k t') = (2^t')^k by k-1 multiplies of
// the ex2 already taken for s (no second MUFU op; keeps the power sum at the HBM roofline).
#ifndef SMCSD_K1_POLY_K
#define SMCSD_K1_POLY_K 4             // plain exp-sum: all on MUFU (see reduce_item)
#endif
#ifndef SMCSD_POW_POLY_K
#define SMCSD_POW_POLY_K 2            // pairs k >= this (of 4 per 16-byte vector) on the FMA pipe
#endif
template <int PW>
__device__ __forceinline__ float2 pow_acc(float2 acc, float2 e, float2 t, float alpha, bool fma_pipe = false) {
    if (PW == -1) {
        // general alpha: a second exp per element (MUFU-bound); fma_pipe moves it to the FMA
        // pipe (polynomial) for the caller's share of the elements
        const float2 ta = fmul2(t, make_float2(alpha, alpha));
        return fadd2(acc, fma_pipe ? ex2_poly2(ta) : make_float2(ex2_approx(ta.x), ex2_approx(ta.y)));
    }
    if (PW == 1) return fadd2(acc, e);
    if (PW == 2) return ffma2(e, e, acc);
    if (PW == 3) return ffma2(fmul2(e, e), e, acc);
    const float2 e2 = fmul2(e, e);
    return ffma2(e2, e2, acc);
}

// Half-integer alpha = k + 1/2 (PW = 10 + k, k = 0..3): one ex2 per element, y = 2^(t'/2) with
// t'/2 = fma(z, c/2, -m/2) (bit-exactly t'/2: scaling by 2^-1), then 2^t' = y^2 for s and
// 2^(alpha t') = y (y^2)^k for s2 -- multiplies instead of a second MUFU op.
template <int PW>
__device__ __forceinline__ float2 half_pow(float2 y, float2 e) {
    if (PW == 10) return y;
    if (PW == 11) return fmul2(y, e);
    if (PW == 12) return fmul2(fmul2(y, e), e);
    return fmul2(fmul2(y, e), fmul2(e, e));
}

template <int DT, int PW = 0>
__device__ __forceinline__ void reduce_item(uint4 (&v)[ItemTraits<DT>::kLoads], int nv, float c,
                                            float4 *red, float alpha = 1.0f) {
    using T = ItemTraits<DT>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (nv < kSeg) {                                          // ragged last segment: mask >= V
#pragma unroll
        for (int i = 0; i < T::kLoads; ++i) {
            const int e = (i * kThreads + tid) * T::kVec;
            uint32_t *w = reinterpret_cast<uint32_t *>(&v[i]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (DT == 1) {
                    if (e + 2 * k >= nv)     w[k] = (w[k] & 0xffff0000u) | 0x0000FF80u;
                    if (e + 2 * k + 1 >= nv) w[k] = (w[k] & 0x0000ffffu) | 0xFF800000u;
                } else {
                    if (e + k >= nv) w[k] = T::kNegInf;
                }
            }
        }
    }
    // max over the warp's elements (raw logits; c > 0 so max(z)*c = max(z*c))
    float mt;
    if (DT == 1) {
        uint32_t acc = v[0].x;
#pragma unroll
        for (int i = 0; i < T::kLoads; ++i) {
            const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (SMCSD_K1_POLY_K < 4 && PW == 0)             // the polynomial does not carry NaN
                    asm("max.NaN.bf16x2 %0, %0, %1;" : "+r"(acc) : "r"(w4[k]));
                else
                    asm("max.bf16x2 %0, %0, %1;" : "+r"(acc) : "r"(w4[k]));
            }
        }
        mt = fmaxf(bf16lo(acc), bf16hi(acc));
    } else {
        mt = -INFINITY;
#pragma unroll
        for (int i = 0; i < T::kLoads; ++i)
            mt = fmaxf(mt, fmaxf(fmaxf(__uint_as_float(v[i].x), __uint_as_float(v[i].y)),
                                 fmaxf(__uint_as_float(v[i].z), __uint_as_float(v[i].w))));
    }
    const float mw = warp_max(mt) * c;                       // warp max of t = z*c
    const float off = mw == -INFINITY ? 0.0f : mw;           // all -inf: sum(2^-inf) = 0, NaN kept
    // sum of 2^(t - m): exactly one ex2 per element; t and the sums in packed fp32x2 (element
    // pairs), halving the FMA-pipe issue slots of this issue-bound loop
    const float2 cc = make_float2(c, c), mo = make_float2(-off, -off);
    const float2 cch = make_float2(0.5f * c, 0.5f * c), moh = make_float2(-0.5f * off, -0.5f * off);
    float2 acc[T::kLoads], acc2[T::kLoads];
#pragma unroll
    for (int i = 0; i < T::kLoads; ++i) {
        const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        float2 a = make_float2(0.0f, 0.0f), a2 = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int k = 0; k < (DT == 1 ? 4 : 2); ++k) {
            const float2 z = DT == 1 ? make_float2(bf16lo(w4[k]), bf16hi(w4[k]))
                                     : make_float2(__uint_as_float(w4[2 * k]), __uint_as_float(w4[2 * k + 1]));
            if (PW >= 10) {
                const float2 th = ffma2(z, cch, moh);
                const float2 y = make_float2(ex2_approx(th.x), ex2_approx(th.y));
                const float2 e = fmul2(y, y);
                a = fadd2(a, e);
                a2 = fadd2(a2, half_pow<PW>(y, e));
                continue;
            }
            const float2 t = ffma2(z, cc, mo);
            // (A/B option SMCSD_K1_POLY_K < 4: pairs k >= it of each bf16 vector on the FMA-pipe
            // polynomial instead of MUFU -- slower burst and sustained, profiles/r02c_ab_k1_poly_sustained.txt)
            const float2 e = PW == 0 && DT == 1 && k >= SMCSD_K1_POLY_K ? ex2_poly2(t)
                                                                        : make_float2(ex2_approx(t.x), ex2_approx(t.y));
            a = fadd2(a, e);
            if (PW) a2 = pow_acc<PW>(a2, e, t, alpha, PW == -1 && DT == 1 && k >= SMCSD_POW_POLY_K);
        }
        acc[i] = a;
        acc2[i] = a2;
    }
    float s = acc[0].x + acc[0].y, s2 = acc2[0].x + acc2[0].y;
#pragma unroll
    for (int i = 1; i < T::kLoads; ++i) {
        s += acc[i].x + acc[i].y;
        s2 += acc2[i].x + acc2[i].y;
    }
    s = warp_sum(s);
    if (PW) s2 = warp_sum(s2);
    if (lane == 0) red[warp] = make_float4(mw, s, s2, 0.0f);
}

// Unsigned division by a runtime constant d via a precomputed magic number (host computes
// mg = ceil(2^(32+sh) / d) with sh = ceil(log2 d), < 2^33); exact for x, d < 2^31.
__device__ __forceinline__ unsigned fastdiv(unsigned x, unsigned long long mg, int sh) {
    return (unsigned)(((unsigned long long)x * mg) >> (32 + sh));
}

// Per-item data derived from the item index (every thread, no broadcast).
struct ItemInfo {
    const char *seg;        // first byte of the segment
    int nv;                 // valid elements in the segment
    float c;                // inv_temp * log2(e) of the row's model
    int valid;              // row is read (j < k_n)
    int64_t tok;            // index of the row's drafted token in tokens[] (weight rows), else -1
    int64_t v0;             // first column of the segment (shard-local)
};

template <int DT>
__device__ __forceinline__ ItemInfo item_info(const Params &prm, long long item) {
    ItemInfo f;
    constexpr int kEsz0 = ItemTraits<DT>::kEsz;
    if (item >= prm.main_items) {                           // bonus row k_n of target particle pn
        const unsigned b = (unsigned)(item - prm.main_items);
        const unsigned pn = fastdiv(b, prm.mg_nseg, prm.sh_nseg);
        const int seg = (int)(b - pn * (unsigned)prm.nseg);
        const int kn = prm.n_drafted ? prm.n_drafted[pn] : prm.K;
        f.valid = kn >= 0 && kn <= prm.K;
        const int64_t v0 = (int64_t)seg * kSeg;
        f.seg = prm.lp + (((int64_t)pn * prm.rpp_p + (f.valid ? kn : 0)) * prm.ld_p + v0) * kEsz0;
        f.nv = (int)min((int64_t)kSeg, prm.v_len - v0);
        f.c = prm.c_p;
        f.tok = -1;
        f.v0 = v0;
        return f;
    }
    const unsigned u = (unsigned)item;                      // total < 2^31 (validated)
    unsigned row = fastdiv(u, prm.mg_nseg, prm.sh_nseg);
    const int seg = (int)(u - row * (unsigned)prm.nseg);
    const unsigned r1 = fastdiv(row, prm.mg_K, prm.sh_K);
    const int j = (int)(row - r1 * (unsigned)prm.K);
    const unsigned r2 = fastdiv(r1, prm.mg_N, prm.sh_N);
    const int n = (int)(r1 - r2 * (unsigned)prm.N);
    const int model = prm.n_models == 2 ? (int)(r2 & 1u) : 0;
    const int64_t pn = (int64_t)(prm.n_models == 2 ? (r2 >> 1) : r2) * prm.N + n;
    const int kn = prm.n_drafted ? prm.n_drafted[pn] : prm.K;
    f.valid = kn >= 0 && kn <= prm.K && j < kn;
    constexpr int kEsz = ItemTraits<DT>::kEsz;
    const int64_t v0 = (int64_t)seg * kSeg;
    const char *row_ptr = model == 0 ? prm.lp + ((pn * prm.rpp_p + j) * prm.ld_p) * kEsz
                                     : prm.lq + ((pn * prm.rpp_q + j) * prm.ld_q) * kEsz;
    f.seg = row_ptr + v0 * kEsz;
    f.nv = (int)min((int64_t)kSeg, prm.v_len - v0);
    f.c = model == 0 ? prm.c_p : prm.c_q;
    f.tok = pn * prm.K + j;
    f.v0 = v0;
    return f;
}

// Issue this thread's loads of one decoded item.
template <int DT>
__device__ __forceinline__ void load_seg(uint4 (&v)[ItemTraits<DT>::kLoads], const ItemInfo &f) {
    using T = ItemTraits<DT>;
    const int tid = threadIdx.x;
    if (f.nv == kSeg) {
#pragma unroll
        for (int i = 0; i < T::kLoads; ++i) v[i] = ld_stream(f.seg + (size_t)(i * kThreads + tid) * 16);
    } else {
#pragma unroll
        for (int i = 0; i < T::kLoads; ++i) {
            const int e = (i * kThreads + tid) * T::kVec;
            v[i] = e < f.nv ? ld_stream(f.seg + (size_t)(i * kThreads + tid) * 16)
                            : make_uint4(T::kNegInf, T::kNegInf, T::kNegInf, T::kNegInf);
        }
    }
}

// K1 kernel: warp-specialised bulk-copy (TMA) pipeline, no CTA-wide barriers.
//   warp 8 (producer, lane 0): takes items in global order from an atomic counter (first item
//     per CTA static), decodes them, and streams each item's bytes into a kStages-deep
//     shared-memory ring with cp.async.bulk (completion counted on full[s] in bytes);
//   warps 0..7 (consumers): wait full[s], reduce the item from shared memory, write their
//     warp partial; the last consumer warp to finish an item (shared-memory counter) merges
//     the 8 partials in fixed tree order, stores {m, s, -inf, 0}, and every warp releases the
//     slot on empty[s].
// The drafted-token logit is not taken here (the tail loads it).  grid = min(items, SMs x
// resident CTAs), block = kK1Threads, dynamic smem = kStages x stage + bookkeeping.
constexpr int kK1Threads = kThreads + 32;
#ifndef SMCSD_K1_STAGES
#define SMCSD_K1_STAGES 2
#endif
#ifndef SMCSD_K1_MINB
#define SMCSD_K1_MINB 6
#endif
constexpr int kStages = SMCSD_K1_STAGES;

struct StageMeta {
    long long item;         // global item index, or -1: no more work
    int nv;                 // valid elements in the segment
    float c;                // inv_temp * log2(e) of the row's model
    int valid;              // row is read (j < k_n)
    int dloc;               // S10 exchange: drafted token's column in this segment, else -1
};

constexpr int kXMaxG = 32;                                  // S10: ranks of one exchange
static_assert(kXMaxG <= kXEpochWord, "flag words of the ranks must not reach the epoch words");

template <int DT, bool XP = false>
constexpr size_t rowstats_smem_bytes() {
    return (size_t)kStages * kSeg * ItemTraits<DT>::kEsz            // data ring
         + kStages * (2 * sizeof(uint64_t) + sizeof(StageMeta) + kWarps * sizeof(float4) + 16)
         + (XP ? kXMaxG * sizeof(float4 *) + 16 : 0);                // S10: per-rank destinations, epoch
}

// bf16 path: SMCSD_K1_MINB CTAs/SM (32 registers); the general-alpha and cube power sums need
// a few more live registers, one CTA/SM fewer.
template <int DT, int PW>
constexpr int k1_min_blocks() { return DT != 1 ? 1 : (PW == -1 || PW == 3) ? SMCSD_K1_MINB - 1 : SMCSD_K1_MINB; }

// XP: the S10 fused-exchange variant (smcsd_tp_step), a separate instance so that the plain
// kernel carries none of its code.
// S10: the drafted token of a K1 item's row (-1 when the row has none), loaded by the producer
// one item ahead of its use.
template <int DT>
__device__ __forceinline__ int xp_token(const Params &prm, long long item) {
    const ItemInfo f = item_info<DT>(prm, item);
    return f.valid && f.tok >= 0 ? __ldg(prm.tokens + f.tok) : -1;
}

template <int DT, int PW, bool XP = false>
__global__ void __launch_bounds__(kK1Threads, k1_min_blocks<DT, PW>()) k_rowstats(const __grid_constant__ Params prm) {
    using T = ItemTraits<DT>;
    constexpr uint32_t kStageBytes = (uint32_t)kSeg * T::kEsz;
    extern __shared__ __align__(128) char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
    uint64_t *empty = full + kStages;
    StageMeta *meta = reinterpret_cast<StageMeta *>(empty + kStages);
    float4 *red = reinterpret_cast<float4 *>(meta + kStages);       // [kStages][kWarps]
    int *done = reinterpret_cast<int *>(red + kStages * kWarps);    // [kStages]
    float4 **xdst = reinterpret_cast<float4 **>(done + kStages);     // [kXMaxG] (XP only)
    static_assert(kStages % 2 == 0, "xdst must stay 8-byte aligned");
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long total = prm.main_items + prm.bonus_items;

    if (tid == 0) {
        SMCSD_TRACE_AT(blockIdx.x & 1023);                      // K1 CTA start
#ifdef SMCSD_TRACE
        { unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid)); g_trace[3072 + (blockIdx.x & 1023)] = smid; }
#endif
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
            done[s] = 0;
        }
        fence_mbar_init();
    }
    uint32_t *xep = reinterpret_cast<uint32_t *>(xdst + kXMaxG);     // S10: this launch's epoch
    __syncthreads();
    if (!XP && PW == 0 && prm.lt_words) {
        // Polling tail: the tail polls lt_words (k_tail_small even runs beside this grid), so let
        // it launch now -- after the wait, so that it too sees the predecessor's outputs.  Every
        // thread (the consumers would wait for the producer's first copy anyway).
        pdl_wait();
        pdl_trigger();
    }
    if (XP && warp < kWarps) {
        // consumers only (named barrier 1), so the producer's first TMA is not held back: the
        // epoch word is advanced by the previous step's tail, so read it after that completes,
        // then this epoch's half of each rank's buffer (used at the first item's merge)
        if (tid == 0) {
            pdl_wait();
            *xep = x_epoch(prm);
        }
        named_bar_sync(1, kWarps * 32);
        if (tid < prm.xG)
            xdst[tid] = x_parts(prm.xpeer[tid], 2 * prm.P * prm.N * prm.K, prm.xG, prm.xnseg, *xep);
        named_bar_sync(1, kWarps * 32);
    }

    if (warp == kWarps) {
        // ------------------------------------------------------------------ producer
        if (prm.bonus_tok) {
            // status[] is OR-ed by the bonus CTAs of the tail: zero it here, after the
            // predecessor (the previous call's tail) has completed.
            pdl_wait();
            for (int q = (int)blockIdx.x * 32 + lane; q < prm.P; q += (int)gridDim.x * 32) prm.status[q] = 0u;
        }
        if (lane == 0) {
            // The predecessor may have produced the logits (or re-armed work_ctr): wait for it
            // before the first global access.  Setup above overlapped its tail.
            pdl_wait();
            long long item = blockIdx.x;
            int xtok = -1;                                  // S10: drafted token of `item`
            if (XP && item < total) xtok = xp_token<DT>(prm, item);
            for (long long it = 0;; ++it) {
                const int s = (int)(it % kStages);
                mbar_wait(&empty[s], (uint32_t)(((it / kStages) & 1) ^ 1));   // slot released
                // short streams (a few items per CTA: the latency-bound single-prompt steps)
                // claim the next item only once a slot is free, so no CTA holds an item while
                // its ring is full and the last items go to CTAs that can start them at once;
                // long streams claim one item ahead (hides the atomic behind the copies)
                if (!XP && prm.late_claim && it > 0) item = (long long)gridDim.x + atomicAdd(prm.work_ctr, 1u);
                StageMeta m;
                m.item = item < total ? item : -1;
                m.valid = 0;
                m.nv = 0;
                m.c = 0.0f;
                m.dloc = -1;
                const char *src = nullptr;
                if (item < total) {
                    const ItemInfo f = item_info<DT>(prm, item);
                    m.valid = f.valid;
                    m.nv = f.nv;
                    m.c = f.c;
                    src = f.seg;
                    if (XP && f.valid && f.tok >= 0) {
                        // S10: x = t_d comes from the staged segment; d was loaded one
                        // iteration ahead (xtok), so no dependent load delays the TMA issue
                        const int64_t dl = (int64_t)xtok - prm.v_begin - f.v0;
                        m.dloc = dl >= 0 && dl < f.nv ? (int)dl : -1;
                    }
                }
                meta[s] = m;
                if (m.valid) {
                    const uint32_t bytes = (uint32_t)(((m.nv + T::kVec - 1) / T::kVec) * 16);
                    mbar_arrive_expect_tx(&full[s], bytes);
                    bulk_g2s(smem + (size_t)s * kStageBytes, src, bytes, &full[s]);
                } else {
                    mbar_arrive(&full[s]);                    // metadata only (release)
                }
                if (item >= total) break;
                if (XP || !prm.late_claim) item = (long long)gridDim.x + atomicAdd(prm.work_ctr, 1u);
                if (XP && item < total) xtok = xp_token<DT>(prm, item);   // used after the next wait
            }
        }
    } else {
        // ------------------------------------------------------------------ consumers
        uint4 v[T::kLoads];
        for (long long it = 0;; ++it) {
            const int s = (int)(it % kStages);
            mbar_wait(&full[s], (uint32_t)((it / kStages) & 1));
            const StageMeta m = meta[s];
            if (m.item < 0) break;
            float4 *r = red + s * kWarps;
            if (m.valid) {
                const char *sl = smem + (size_t)s * kStageBytes;
#pragma unroll
                for (int i = 0; i < T::kLoads; ++i)
                    v[i] = *reinterpret_cast<const uint4 *>(sl + (size_t)(i * kThreads + tid) * 16);
                reduce_item<DT, PW>(v, m.nv, m.c, r, prm.alpha_f);
            }
            __syncwarp();
            int last = 0;
            if (lane == 0) {
                __threadfence_block();                        // red[warp] before the count
                last = atomicAdd(&done[s], 1) == kWarps - 1;
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence_block();
                // fixed-order (tree) merge of the 8 warp partials on lanes 0..7
                float4 out = make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f);
                if (m.valid) {
                    const float4 rw = lane < kWarps ? r[lane] : make_float4(-INFINITY, 0.0f, 0.0f, 0.0f);
                    float M = rw.x;
                    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 4));
                    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 2));
                    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
                    const float d = rw.x == M ? 0.0f : rw.x - M;
                    float t = lane < kWarps ? rw.y * (rw.x == M ? 1.0f : ex2_approx(d)) : 0.0f;
                    t += __shfl_xor_sync(0xffffffffu, t, 4);
                    t += __shfl_xor_sync(0xffffffffu, t, 2);
                    t += __shfl_xor_sync(0xffffffffu, t, 1);
                    float t2 = 0.0f;
                    if (PW) {
                        t2 = lane < kWarps ? rw.z * (rw.x == M ? 1.0f : ex2_approx(d * prm.alpha_f)) : 0.0f;
                        t2 += __shfl_xor_sync(0xffffffffu, t2, 4);
                        t2 += __shfl_xor_sync(0xffffffffu, t2, 2);
                        t2 += __shfl_xor_sync(0xffffffffu, t2, 1);
                    }
                    out = make_float4(M, t, -INFINITY, t2);
                }
                if (XP) {
                    // S10 fused exchange: x = t_d when the drafted token is in this segment
                    // (taken from the staged segment), then one 16-byte store per rank
                    const unsigned row = fastdiv((unsigned)m.item, prm.mg_nseg, prm.sh_nseg);
                    const int sg = (int)((unsigned)m.item - row * (unsigned)prm.nseg);
                    if (m.valid && m.dloc >= 0) {
                        const char *sl = smem + (size_t)s * kStageBytes;
                        const float z = DT == 1 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(sl)[m.dloc] << 16)
                                                : reinterpret_cast<const float *>(sl)[m.dloc];
                        out.z = z * m.c;
                    }
                    if (lane < prm.xG) {
                        // two single-copy-atomic 8-byte words, both nonzero whenever written
                        // ({m, s}: m finite => s >= 1, an empty segment has m = -inf; {x, 1}),
                        // so the tail polls the data itself -- no fence or flag per step
                        float4 *slot = xdst[lane] + (size_t)row * prm.xG * prm.xnseg + prm.xrank * prm.xnseg + sg;
                        st_relaxed_sys_u64(slot, (unsigned long long)__float_as_uint(out.x) |
                                                 ((unsigned long long)__float_as_uint(out.y) << 32));
                        st_relaxed_sys_u64(reinterpret_cast<unsigned long long *>(slot) + 1,
                                           (unsigned long long)__float_as_uint(out.z) | (1ull << 32));
                        // this rank's shard has fewer segments than the exchange's slots: the
                        // row's last segment also fills the unused slots with neutral parts
                        for (int u = sg + 1; sg == prm.nseg - 1 && u < prm.xnseg; ++u) {
                            st_relaxed_sys_u64(slot + (u - sg), 0xFF800000ull);        // {-inf, 0}
                            st_relaxed_sys_u64(reinterpret_cast<unsigned long long *>(slot + (u - sg)) + 1,
                                               0xFF800000ull | (1ull << 32));          // {-inf, 1}
                        }
                    }
                    if (lane == 0) done[s] = 0;
                } else if (lane == 0) {
                    if (PW == 0 && prm.lt_words) {            // polling tail: data and flag in
                        // one word, segment-major ([seg][row]): the tail's lanes that take part
                        // k of consecutive rows read consecutive words
                        const unsigned row = fastdiv((unsigned)m.item, prm.mg_nseg, prm.sh_nseg);
                        const unsigned sg = (unsigned)m.item - row * (unsigned)prm.nseg;
                        st_relaxed_gpu_b64(prm.lt_words + (size_t)sg * (unsigned)(2 * prm.P * prm.N * prm.K) + row,
                                           (unsigned long long)__float_as_uint(out.x) |
                                           ((unsigned long long)__float_as_uint(out.y) << 32));
                    }
                    else
                        prm.part_ws[m.item] = out;
                    done[s] = 0;
                }
                __syncwarp();
            }
            if (lane == 0) mbar_arrive(&empty[s]);            // this warp is done with slot s
        }
    }
    if (tid == 0) SMCSD_TRACE_AT(1024 + (blockIdx.x & 1023));    // K1 CTA done
    if (XP) pdl_trigger();                 // the tail's only dependency is the pushed words
    if (!XP) pdl_trigger();
}

// S2, phase A: merged {M, S, X} of every row of prompt p into rowstat[0 .. 2NK).  Chunks of
// 256 rows x 16 parts are read with coalesced 16-byte loads (16 per thread in flight), staged in
// shared memory (row pitch 17 float4: conflict-free), then thread t merges row t of the chunk
// in part order (online rescale across part chunks when a row has more than 16 parts).
constexpr int kStagePitch = 17;
constexpr size_t kTailStageBytes = (size_t)kThreads * kStagePitch * sizeof(float4);

__device__ __forceinline__ void tail_rowstats(const Params &prm, int p, float4 *rowstat, float4 *stage) {
    const int tid = threadIdx.x;
    const int rows = 2 * prm.N * prm.K, np_all = prm.nparts;
    const int64_t gbase = (int64_t)p * rows;
    for (int r0 = 0; r0 < rows; r0 += kThreads) {
        const int cr = min(kThreads, rows - r0);
        float M = -INFINITY, S = 0.0f, X = -INFINITY;
        for (int pc = 0; pc < np_all; pc += 16) {
            const int np = min(16, np_all - pc);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                const int e = tid + kThreads * kk, r = e >> 4, i = e & 15;
                if (r < cr && i < np)
                    stage[r * kStagePitch + i] =
                        __ldcg(&prm.parts[(gbase + r0 + r) * prm.part_row_stride + (int64_t)(pc + i) * prm.part_seg_stride]);
            }
            __syncthreads();
            if (tid < cr) {
                const float4 *row = stage + tid * kStagePitch;
                float Mc = -INFINITY;
                for (int i = 0; i < np; ++i) Mc = fmaxf(Mc, row[i].x);
                const float Mn = fmaxf(M, Mc);
                S = S * (M == Mn ? 1.0f : ex2_approx(M - Mn));
                for (int i = 0; i < np; ++i) {
                    const float4 q = row[i];
                    S += q.y * (q.x == Mn ? 1.0f : ex2_approx(q.x - Mn));
                    X = fmaxf(X, q.z);
                }
                M = Mn;
            }
            __syncthreads();
        }
        if (tid < cr) rowstat[r0 + tid] = make_float4(M, S, X, 0.0f);
    }
}

// S2, phase B + per-row part of S3.  Thread pairs (2q, 2q+1) take the target and draft rows of
// (particle n, position j), q = n*K + j: ell from rowstat, then term[q] = alpha*ell^p - ell^q
// (fp64); NaN marks an invalid pair (flag already raised).  term is shared memory when
// term_smem != nullptr, else prm.ell_ws (global, L2).
__device__ __forceinline__ void tail_scores(const Params &prm, int p, const float4 *rowstat, double *term_smem,
                                            uint32_t *sh_st, float x_pre) {
    const int N = prm.N, K = prm.K, tid = threadIdx.x;
    const int NK = N * K, rows = 2 * NK;
    double *term_g = prm.ell_ws + (int64_t)p * NK;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    uint32_t st = 0;
    for (int base = 0; base < rows; base += kThreads) {      // uniform trip count per warp
        const int r2 = base + tid;
        const bool active = r2 < rows;
        const int model = r2 & 1;
        const int q = r2 >> 1;
        const int n = active ? q / K : 0, j = active ? q - (q / K) * K : 0;
        const int64_t pn = (int64_t)p * N + n;
        double ell = 0.0;
        bool valid = false;
        if (active) {
            const int kn = drafted_len(prm, pn);
            const int64_t d = prm.tokens[pn * K + j];
            float4 m = rowstat[model * NK + q];
            valid = kn >= 0 && kn <= K && j < kn;
            if (prm.x_from_logits)                            // prefetched for the first rows
                m.z = base == 0 ? x_pre : (valid && d >= 0 && d < prm.V ? load_x(prm, model, pn, j, d) : -INFINITY);
            if (!valid) {
                ell = 0.0;
            } else if (d < 0 || d >= prm.V) {
                st |= ST_BAD_TOKEN;
                ell = qnan;
            } else if (!isfinite(m.x) || !isfinite(m.y)) {
                st |= ST_NONFINITE;
                ell = qnan;
            } else {
                // ell = (x - m - log2 s) * ln 2  (natural log of the softmax at d); s in [1, V]
                ell = __dmul_rn(__dsub_rn(__dsub_rn((double)m.z, (double)m.x), (double)log2f(m.y)), kLn2);
            }
            float *outp = model == 0 ? prm.logp_tok : prm.logq_tok;
            if (outp) outp[pn * K + j] = (float)ell;
        }
        const double other = __shfl_xor_sync(0xffffffffu, ell, 1);
        if (active && model == 0 && valid) {
            const double lp = ell, lq = other;
            double term;
            if (isnan(lp) || isnan(lq)) {
                term = qnan;
            } else if (lq == -INFINITY) {
                st |= ST_NOT_ABSCONT;
                term = qnan;
            } else {
                term = __dsub_rn(__dmul_rn(prm.alpha, lp), lq);
            }
            if (term_smem) term_smem[q] = term;
            else __stcg(&term_g[q], term);
        }
    }
    if (st) atomicOr(sh_st, st);
}

// Rest of S3 for particle n: lam' = fl32(prev + sum_{j<k_n} term_j) in j order.
__device__ __forceinline__ float tail_reweight(const Params &prm, int p, int n, const double *term_smem,
                                               float prev, uint32_t *st) {
    const int N = prm.N, K = prm.K;
    const int64_t pn = (int64_t)p * N + n;
    const double *tg = prm.ell_ws + (int64_t)p * N * K + (int64_t)n * K;
    const double *ts = term_smem ? term_smem + (int64_t)n * K : nullptr;
    int kn = drafted_len(prm, pn);
    bool bad = false;
    if (kn < 0 || kn > K) {
        *st |= ST_BAD_TOKEN;
        bad = true;
        kn = 0;
    }
    double delta = 0.0;
    for (int j = 0; j < kn; ++j) delta = __dadd_rn(delta, ts ? ts[j] : __ldcg(&tg[j]));
    if (isnan(delta)) bad = true;                           // an invalid pair (flag raised in S2)
    if (isnan(prev) || prev == INFINITY) {
        *st |= ST_NONFINITE;
        bad = true;
    }
    return bad ? -INFINITY : (float)__dadd_rn((double)prev, delta);
}

// ------------------------------------------------------------------------------------------
// S4-S7 for prompt p from sh.lam[0..N), executed by warp 0 alone (warp-synchronous: no block
// barriers on the critical path).  Lane l owns particles [l*B, min(N, (l+1)*B)), B = ceil(N/32).
// All threads may call; warps other than 0 return at once.  The caller synchronises after.
// ------------------------------------------------------------------------------------------
struct TailSmem {
    double e[kTailMaxN];
    double C[kTailMaxN];
    float lam[kTailMaxN];
    int o[kTailMaxN];
    int ex[kTailMaxN];          // E list: source of the i-th extra copy
    uint32_t st;
    double U;                   // systematic uniform (drawn before the predecessor finishes)
    float reset;                // fl32(-ln N)
};

// Weight-independent tail inputs: U = word0(Philox4x32-10(...)) * 2^-32 and fl32(-ln N).
// Called by thread 0 before griddepcontrol.wait so they overlap the predecessor kernel.
__device__ __forceinline__ void tail_prologue(const Params &prm, int p, TailSmem &sh) {
    uint32_t x = 0;
    if (prm.scheme != 0) {
        x = 0;                                                  // multinomial: per-particle draws
    } else if (prm.uniforms) {
        x = prm.uniforms[p];
    } else {
        const uint64_t g = (uint64_t)(prm.prompt_base + p);
        const uint4 r = philox4x32_10(
            make_uint4((uint32_t)prm.step, (uint32_t)(prm.step >> 32), (uint32_t)g, 0u),
            make_uint2((uint32_t)prm.seed, (uint32_t)(prm.seed >> 32)));
        x = r.x;
    }
    sh.U = (double)x * 2.3283064365386962890625e-10;          // 2^-32, exact
    sh.reset = (float)(-log((double)prm.N));
}

// Uniform of particle n (weight-independent): systematic u_n = (n + U) / N with U = word 0 of
// Philox(step, prompt, 0) (or uniforms[p]) times 2^-32; multinomial u_n = word n & 3 of
// Philox(step, prompt, 1 + n / 4) (or uniforms[p][n]) times 2^-32.  Exactly the values
// normalise_resample forms.
__device__ __forceinline__ double tail_uniform(const Params &prm, int p, int n) {
    const uint64_t gp = (uint64_t)(prm.prompt_base + p);
    const uint2 key = make_uint2((uint32_t)prm.seed, (uint32_t)(prm.seed >> 32));
    uint32_t x;
    if (prm.scheme == 0) {
        x = prm.uniforms ? prm.uniforms[p]
                         : philox4x32_10(make_uint4((uint32_t)prm.step, (uint32_t)(prm.step >> 32), (uint32_t)gp, 0u), key).x;
        return __ddiv_rn(__dadd_rn((double)n, (double)x * 2.3283064365386962890625e-10), (double)prm.N);
    }
    if (prm.uniforms) {
        x = n < prm.N ? prm.uniforms[(int64_t)p * prm.N + n] : 0u;
    } else {
        const uint4 r = philox4x32_10(
            make_uint4((uint32_t)prm.step, (uint32_t)(prm.step >> 32), (uint32_t)gp, 1u + (uint32_t)(n >> 2)), key);
        const int w = n & 3;
        x = w == 0 ? r.x : w == 1 ? r.y : w == 2 ? r.z : r.w;
    }
    return (double)x * 2.3283064365386962890625e-10;
}

__device__ __forceinline__ void normalise_resample(const Params &prm, int p, bool resample_mode, TailSmem &sh) {
    if (threadIdx.x >= 32) return;
    const unsigned FULL = 0xffffffffu;
    const int N = prm.N, lane = threadIdx.x;
    const int B = (N + 31) >> 5;
    const int b0 = min(N, lane * B), b1 = min(N, b0 + B);
    const int64_t base = (int64_t)p * N;
    double U = sh.U;
    SMCSD_PHASE(0);
    // ---- S4: M = max lam (order-free), e_n = exp(lam_n - M)
    float mloc = -INFINITY;
    for (int n = b0; n < b1; ++n) mloc = fmaxf(mloc, sh.lam[n]);
    const double M = (double)warp_max(mloc);
    if (M == -INFINITY) {                                     // degenerate prompt
        for (int n = b0; n < b1; ++n) {
            if (prm.wnorm) prm.wnorm[base + n] = 0.0f;
            if (resample_mode) {
                prm.ancestors[base + n] = n;
                if (prm.offspring) prm.offspring[base + n] = 1;
                if (prm.slot_src) prm.slot_src[base + n] = n;
                prm.logw_out[base + n] = sh.lam[n];
            }
        }
        if (lane == 0) {
            sh.st |= ST_DEGENERATE;
            if (prm.lse) prm.lse[p] = -INFINITY;
            if (prm.ess) prm.ess[p] = 0.0;
            if (resample_mode) {
                prm.resampled[p] = 0;
                if (prm.n_ties) prm.n_ties[p] = 0;
            }
        }
        return;
    }
    SMCSD_PHASE(1);
    for (int n = b0; n < b1; ++n) sh.e[n] = exp(__dsub_rn((double)sh.lam[n], M));
    __syncwarp();
    SMCSD_PHASE(2);
    // sequential fp64 prefix and sum of squares in particle order (reading G6): one lane
    double S = 0.0, ess = 0.0;
    int do_res = 0;
    if (lane == 0) {
        double acc = 0.0, sq = 0.0;
        for (int m = 0; m < N; ++m) {
            const double e = sh.e[m];
            acc = __dadd_rn(acc, e);
            sq = __dadd_rn(sq, __dmul_rn(e, e));
            sh.C[m] = acc;
        }
        S = acc;
        ess = __ddiv_rn(__dmul_rn(S, S), sq);
        do_res = resample_mode && ess < prm.eta;
        if (prm.ess) prm.ess[p] = ess;
        if (prm.lse) prm.lse[p] = __dadd_rn(M, log(S));
    }
    SMCSD_PHASE(3);
    S = __shfl_sync(FULL, S, 0);
    do_res = __shfl_sync(FULL, do_res, 0);
    __syncwarp();
    if (prm.wnorm)
        for (int n = b0; n < b1; ++n) prm.wnorm[base + n] = (float)__ddiv_rn(sh.e[n], S);
    if (!resample_mode) return;
    if (!do_res) {
        for (int n = b0; n < b1; ++n) {
            prm.ancestors[base + n] = n;
            if (prm.offspring) prm.offspring[base + n] = 1;
            if (prm.slot_src) prm.slot_src[base + n] = n;
            prm.logw_out[base + n] = sh.lam[n];
        }
        if (lane == 0) {
            prm.resampled[p] = 0;
            if (prm.n_ties) prm.n_ties[p] = 0;
        }
        return;
    }
    SMCSD_PHASE(4);
    // ---- S6: systematic ancestors by inverse CDF: C_m = P_m / S, u_n = (n + U) / N
    for (int m = b0; m < b1; ++m) {
        sh.C[m] = __ddiv_rn(sh.C[m], S);
        sh.o[m] = 0;
    }
    __syncwarp();
    SMCSD_PHASE(5);
    const double tie = 9.094947017729282379150390625e-13;     // 2^-40
    int ties = 0;
    const uint64_t gp = (uint64_t)(prm.prompt_base + p);
    for (int n = b0; n < b1; ++n) {
        double u;
        if (prm.scheme == 0) {                                  // systematic: (n + U) / N
            u = __ddiv_rn(__dadd_rn((double)n, U), (double)N);
        } else {                                                // multinomial
            uint32_t x;
            if (prm.uniforms) {
                x = prm.uniforms[base + n];
            } else {
                const uint4 r = philox4x32_10(
                    make_uint4((uint32_t)prm.step, (uint32_t)(prm.step >> 32), (uint32_t)gp, 1u + (uint32_t)(n >> 2)),
                    make_uint2((uint32_t)prm.seed, (uint32_t)(prm.seed >> 32)));
                const int w = n & 3;
                x = w == 0 ? r.x : w == 1 ? r.y : w == 2 ? r.z : r.w;
            }
            u = (double)x * 2.3283064365386962890625e-10;
        }
        int lo = 0, hi = N;                                     // a = #{m : C_m <= u}
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sh.C[mid] <= u) lo = mid + 1; else hi = mid;
        }
        const int a = lo < N ? lo : N - 1;                      // lo < N always (C_{N-1} = 1 > u)
        prm.ancestors[base + n] = a;
        atomicAdd(&sh.o[a], 1);
        for (int m = a - 1; m >= 0 && fabs(__dsub_rn(u, sh.C[m])) <= tie; --m) ++ties;
        for (int m = a; m < N && fabs(__dsub_rn(u, sh.C[m])) <= tie; ++m) ++ties;
    }
    __syncwarp();
    SMCSD_PHASE(6);
    // ---- in-place slot plan (G14): dead slots (o = 0, ascending) take the extra copies
    // (source m repeated o_m - 1 times, ascending m).  Per-lane block totals + warp scans.
    int dead_l = 0, extra_l = 0;
    for (int m = b0; m < b1; ++m) {
        const int o = sh.o[m];
        dead_l += o == 0;
        extra_l += o > 1 ? o - 1 : 0;
    }
    int dead_x = dead_l, extra_x = extra_l;                     // inclusive scans
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int dv = __shfl_up_sync(FULL, dead_x, s), ev = __shfl_up_sync(FULL, extra_x, s);
        if (lane >= s) { dead_x += dv; extra_x += ev; }
    }
    int d_rank = dead_x - dead_l, x_pos = extra_x - extra_l;   // exclusive
    for (int m = b0; m < b1; ++m) {
        const int o = sh.o[m];
        for (int c = 1; c < o; ++c) sh.ex[x_pos++] = m;
    }
    ties = __reduce_add_sync(FULL, ties);
    __syncwarp();
    SMCSD_PHASE(7);
    const float reset = sh.reset;                              // S7
    for (int m = b0; m < b1; ++m) {
        const int o = sh.o[m];
        if (prm.offspring) prm.offspring[base + m] = o;
        if (prm.slot_src) prm.slot_src[base + m] = o != 0 ? m : sh.ex[d_rank++];
        prm.logw_out[base + m] = reset;
    }
    if (lane == 0) {
        prm.resampled[p] = 1;
        if (prm.n_ties) prm.n_ties[p] = ties;
    }
    SMCSD_PHASE(8);
}

// K2: the tail, distributed.  grid = P x chunks_per_prompt; CTA (p, c) owns the (particle,
// position) pairs q in [32c, 32c + 32) of prompt p, i.e. 64 rows (32 target + 32 draft):
//   S2  16 lanes per row merge the row's parts (coalesced 16-byte loads, fixed 16-lane tree),
//       ell = (x - m - log2 s) ln 2 with x = t_d read from the logits before the wait;
//   S3  term_q = alpha ell^p_q - ell^q_q (fp64) -> workspace, status bits -> workspace;
// then a per-prompt completion counter: the last CTA of the prompt sums the terms in j order
// (S3), and warp 0 runs S4 (weights) or S4-S7 (step).  Launched with PDL behind K1 (or behind
// the NCCL exchange for the combine path): inputs are read before griddepcontrol.wait.
constexpr int kPairsPerCta = 32;

// S10, device epoch: every tail CTA counts itself once it no longer reads the exchange buffer;
// the last one records the epoch as this rank's completed one (the next step's K1 reads it after
// griddepcontrol.wait, i.e. after this whole grid) and re-arms the count.
// S10: re-arm K1's work counter once this rank's K1 grid has completed (CTA 0, at its exit:
// off the critical path; the next step's K1 reads the counter after its own griddepcontrol.wait)
__device__ __forceinline__ void x_tail_rearm(const Params &prm) {
    if ((prm.xlocal || prm.lt_words) && prm.work_ctr && blockIdx.x == 0 && threadIdx.x == 0) {
        pdl_wait();
        *prm.work_ctr = 0u;
    }
}

__device__ __forceinline__ void x_tail_done(const Params &prm, uint32_t xe) {
    if (!prm.xlocal || prm.xepoch) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t *w = reinterpret_cast<uint32_t *>(prm.xlocal);
        if (atomicAdd(w + kXTailCtrWord, 1u) == gridDim.x - 1) {
            w[kXTailCtrWord] = 0u;
            w[kXEpochWord] = xe;
        }
    }
}

// S10 exchange slots (smcsd_tp_step): a slot is two 8-byte words {m, s}, {x, 1}, both nonzero
// once written by the owning rank's K1 (single-copy-atomic relaxed system-scope stores); the
// tail polls them and zeroes them after reading (each slot has one reader per step), so the
// parity half is zero again before any rank can write it next (two steps later).  Bounded: a
// slot still empty after kXTimeoutNs returns a neutral part and `true` (-> SMCSD_ST_EXCHANGE).
__device__ __forceinline__ float4 xp_decode(unsigned long long a, unsigned long long b) {
    return make_float4(__uint_as_float((uint32_t)a), __uint_as_float((uint32_t)(a >> 32)),
                       __uint_as_float((uint32_t)b), 0.0f);
}
// Polling tail (prm.lt_words): of global row g, the KV groups of 4 parts starting at part
// pi0 + pstep * v (v < KV) from K1's segment-major {m, s} words (nonzero once written; zeroed here
// for the next step), all loads in flight at once.  Returns true on timeout (the missing parts
// become neutral {-inf, 0}).
template <int KV>
__device__ __forceinline__ bool lt_take(unsigned long long *words, int64_t total_rows, int64_t g, int pi0, int pstep,
                                        int nparts, float4 (&t)[4 * KV]) {
    unsigned long long a[4 * KV];
    bool nd[4 * KV];
#pragma unroll
    for (int i = 0; i < 4 * KV; ++i) {
        const int pi = pi0 + pstep * (i >> 2) + (i & 3);
        nd[i] = pi < nparts;
        a[i] = nd[i] ? ld_relaxed_gpu_b64(words + pi * total_rows + g) : 0x00000000FF800000ull;
    }
    bool late = false;
    uint64_t t0 = 0;
    for (;;) {
        bool all = true;
#pragma unroll
        for (int i = 0; i < 4 * KV; ++i) all &= a[i] != 0ull;
        if (all) break;
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > kXTimeoutNs) { late = true; break; }
#pragma unroll
        for (int i = 0; i < 4 * KV; ++i)
            if (a[i] == 0ull) a[i] = ld_relaxed_gpu_b64(words + (pi0 + pstep * (i >> 2) + (i & 3)) * total_rows + g);
    }
#pragma unroll
    for (int i = 0; i < 4 * KV; ++i) {
        if (a[i] == 0ull) a[i] = 0x00000000FF800000ull;
        t[i] = make_float4(__uint_as_float((uint32_t)a[i]), __uint_as_float((uint32_t)(a[i] >> 32)), -INFINITY, 0.0f);
        if (nd[i]) __stcg(words + (pi0 + pstep * (i >> 2) + (i & 3)) * total_rows + g, 0ull);
    }
    return late;
}

__device__ __forceinline__ bool xp_take4(const float4 *pr, int64_t stride, int pi0, int nparts, float4 (&t)[4]) {
    const unsigned long long *w[4];
    unsigned long long a[4], b[4];
    bool nd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        nd[k] = pi0 + k < nparts;
        w[k] = reinterpret_cast<const unsigned long long *>(pr + (nd[k] ? (int64_t)(pi0 + k) * stride : 0));
        a[k] = nd[k] ? ld_relaxed_sys_u64(w[k]) : 1ull;
        b[k] = nd[k] ? ld_relaxed_sys_u64(w[k] + 1) : 1ull;
    }
    bool late = false;
    uint64_t t0 = 0;
    for (;;) {
        bool all = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) all &= a[k] != 0ull && b[k] != 0ull;
        if (all) break;
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > kXTimeoutNs) { late = true; break; }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (a[k] == 0ull) a[k] = ld_relaxed_sys_u64(w[k]);
            if (b[k] == 0ull) b[k] = ld_relaxed_sys_u64(w[k] + 1);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        t[k] = nd[k] && a[k] && b[k] ? xp_decode(a[k], b[k]) : make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f);
        if (nd[k]) {
            unsigned long long *ww = const_cast<unsigned long long *>(w[k]);
            ww[0] = 0ull;
            ww[1] = 0ull;
        }
    }
    return late;
}
// one slot, polled (no zeroing): the first pass of a row with more than 16 parts
__device__ __forceinline__ float4 xp_peek(const float4 *slot, bool &late) {
    const unsigned long long *w = reinterpret_cast<const unsigned long long *>(slot);
    unsigned long long a = ld_relaxed_sys_u64(w), b = ld_relaxed_sys_u64(w + 1);
    const uint64_t t0 = globaltimer_ns();
    while (a == 0ull || b == 0ull) {
        if (globaltimer_ns() - t0 > kXTimeoutNs) { late = true; return make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f); }
        if (a == 0ull) a = ld_relaxed_sys_u64(w);
        if (b == 0ull) b = ld_relaxed_sys_u64(w + 1);
    }
    return xp_decode(a, b);
}
// the second pass: read (already seen nonzero) and zero
__device__ __forceinline__ float4 xp_read_zero(const float4 *slot) {
    unsigned long long *w = reinterpret_cast<unsigned long long *>(const_cast<float4 *>(slot));
    const unsigned long long a = ld_relaxed_sys_u64(w), b = ld_relaxed_sys_u64(w + 1);
    w[0] = 0ull;
    w[1] = 0ull;
    return a && b ? xp_decode(a, b) : make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f);
}

__device__ __forceinline__ float3 lane_premerge(const Params &prm, int64_t grow, int li) {
    // parts li, li+16, li+32, ... of one row, merged in index order (nparts > 16 only)
    float M = -INFINITY, S = 0.0f, X = -INFINITY;
    for (int i = li; i < prm.nparts; i += 16)
        M = fmaxf(M, __ldcg(&prm.parts[grow * prm.part_row_stride + (int64_t)i * prm.part_seg_stride]).x);
    for (int i = li; i < prm.nparts; i += 16) {
        const float4 t = __ldcg(&prm.parts[grow * prm.part_row_stride + (int64_t)i * prm.part_seg_stride]);
        S += t.y * (t.x == M ? 1.0f : ex2_approx(t.x - M));
        X = fmaxf(X, t.z);
    }
    return make_float3(M, S, X);
}


// ---- bonus token (NEXT #2; "sample x+ ~ p(. | x, y)"; reading G22) -------------
// One CTA per particle n of prompt p, inside k_tail's grid.  Exact draw from softmax(tau z) of
// target row k_n: (1) segment a by inverse CDF over the K1 segment masses w_i = s_i 2^(m_i - M)
// with U = word0(Philox(ctr = (step, prompt, 2^31 + 2^20 n))); (2) Gumbel-max over segment a:
// key_v = tau z_v log2(e) - log2(E_v), E_v = -ln u_v from Philox word k of
// ctr word3 = 2^31 + 2^20 n + 1 + q (column 4q + k of the segment).  The Gumbel terms do not
// depend on a, so they are drawn before griddepcontrol.wait, overlapping K1's drain.
constexpr int kBonusBlocks = kSeg / 4 / kThreads;           // Philox blocks per thread (8)
constexpr int kBonusMaxSeg = 256;                           // V <= 2^21 for the bonus row

__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// -log2(E), E = -ln u, u = (w + 1/2) 2^-32, branch-free.  Small E (u near 1) decides the
// argmax, so E keeps ~1e-6 relative accuracy everywhere: u < 1/2: -ln u; u >= 1/2 with
// r = 1 - u = (~w + 1/2) 2^-32 (exact to 2^-24 relative): r < 1/16: the log1p series
// r + r^2/2 + ... + r^7/7 (truncation < r^8/8 < 2^-26 r); else -ln(1 - r).
__device__ __forceinline__ float gumbel2(uint32_t w) {
    const float u = fmaf((float)w, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
    const float r = fmaf((float)(~w), 2.3283064365386963e-10f, 1.1641532182693481e-10f);
    const float Ea = -lg2_approx(u) * 0.6931471805599453f;
    const float Eb = -lg2_approx(1.0f - r) * 0.6931471805599453f;
    float Ec = fmaf(r, 1.0f / 7.0f, 1.0f / 6.0f);
    Ec = fmaf(r, Ec, 0.2f);
    Ec = fmaf(r, Ec, 0.25f);
    Ec = fmaf(r, Ec, 1.0f / 3.0f);
    Ec = fmaf(r, Ec, 0.5f);
    Ec = fmaf(r, Ec, 1.0f);
    Ec *= r;
    const float E = w < 0x80000000u ? Ea : (r < 0.0625f ? Ec : Eb);
    return -lg2_approx(E);
}

struct BonusSmem {
    float4 g2[kSeg / 4];        // Gumbel terms -log2(E) of the segment's columns (pre-wait)
    double C[kBonusMaxSeg];
    float m[kBonusMaxSeg], s[kBonusMaxSeg];
    float bk[kWarps];
    int bi[kWarps];
    int a;
    uint32_t st;
};

template <int DT>
__device__ __noinline__ uint32_t bonus_role(const Params &prm, int p, int n, BonusSmem &bs) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t pn = (int64_t)p * prm.N + n;
    const uint2 key = make_uint2((uint32_t)prm.seed, (uint32_t)(prm.seed >> 32));
    const uint32_t prompt = (uint32_t)(uint64_t)(prm.prompt_base + p);
    const uint32_t w3 = 0x80000000u + ((uint32_t)n << 20);
    const uint32_t s0 = (uint32_t)prm.step, s1 = (uint32_t)(prm.step >> 32);
    const int kn = prm.n_drafted ? prm.n_drafted[pn] : prm.K;
    double U = 0.0;
    if (tid == 0) U = (double)philox4x32_10(make_uint4(s0, s1, prompt, w3), key).x * 2.3283064365386962890625e-10;
    // The Gumbel terms do not depend on the segment: draw them before griddepcontrol.wait so
    // they overlap K1's drain (this CTA becomes resident as K1 CTAs retire).
#pragma unroll 2
    for (int r = 0; r < kBonusBlocks; ++r) {
        const int q = tid + kThreads * r;
        const uint4 w = philox4x32_10(make_uint4(s0, s1, prompt, w3 + 1u + (uint32_t)q), key);
        bs.g2[q] = make_float4(gumbel2(w.x), gumbel2(w.y), gumbel2(w.z), gumbel2(w.w));
    }
    pdl_wait();
    const int nseg = prm.nseg;
    if (warp == 0) {
        // (1) segment masses from K1's partials (one L2 round trip), fp64 prefix on lane 0,
        // (2) a = #{i : C_i <= U W} counted across lanes
        const float4 *parts = prm.part_ws + prm.main_items + pn * nseg;
        float mloc = -INFINITY;
        for (int i = lane; i < nseg; i += 32) {
            const float4 q = __ldcg(&parts[i]);
            bs.m[i] = q.x;
            bs.s[i] = q.y;
            mloc = fmaxf(mloc, q.x);
        }
        const float M = warp_max(mloc);
        __syncwarp();
        uint32_t st = 0;
        double W = 0.0;
        if (lane == 0) {
            if (kn < 0 || kn > prm.K) {
                st = ST_BAD_TOKEN;
            } else if (!isfinite(M)) {
                st = ST_NONFINITE;
            } else {
                for (int i = 0; i < nseg; ++i) {
                    const float w = bs.s[i] * (bs.m[i] == M ? 1.0f : ex2_approx(bs.m[i] - M));
                    W = __dadd_rn(W, (double)w);
                    bs.C[i] = W;
                }
                if (isnan(W)) st = ST_NONFINITE;
            }
        }
        st = __shfl_sync(0xffffffffu, st, 0);
        const double T = __shfl_sync(0xffffffffu, U * W, 0);
        __syncwarp();
        int cnt = 0;
        if (!st)
            for (int i = lane; i < nseg; i += 32) cnt += bs.C[i] <= T;
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) {
            bs.a = st ? -1 : min(cnt, nseg - 1);
            bs.st = st;
        }
    }
    __syncthreads();
    const int a = bs.a;
    const uint32_t st = bs.st;
    if (a < 0) {
        if (tid == 0) prm.bonus_tok[pn] = -1;
        return st;
    }
    const int64_t v0 = (int64_t)a * kSeg;
    const int nv = (int)min((int64_t)kSeg, prm.V - v0);
    const float c = prm.c_p;
    const char *row = prm.lp + ((int64_t)pn * prm.rpp_p + kn) * prm.ld_p * (DT == 1 ? 2 : 4);
    // (3) Gumbel-max over segment a: key = z c + g2 (log2 units), smallest column on ties
    using Raw = typename std::conditional<DT == 1, uint2, uint4>::type;
    Raw raw[kBonusBlocks];
#pragma unroll
    for (int r = 0; r < kBonusBlocks; ++r) {
        const int i0 = 4 * (tid + kThreads * r);
        if (i0 < nv) raw[r] = __ldcs(reinterpret_cast<const Raw *>(row + (v0 + i0) * (DT == 1 ? 2 : 4)));
    }
    float best = -INFINITY;
    int bi = 0x7fffffff;
#pragma unroll
    for (int r = 0; r < kBonusBlocks; ++r) {
        const int q = tid + kThreads * r, i0 = 4 * q;
        if (i0 < nv) {
            const float4 g = bs.g2[q];
            const float gk[4] = {g.x, g.y, g.z, g.w};
            float z[4];
            if (DT == 1) {
                const uint2 b = *reinterpret_cast<const uint2 *>(&raw[r]);
                z[0] = bf16lo(b.x); z[1] = bf16hi(b.x); z[2] = bf16lo(b.y); z[3] = bf16hi(b.y);
            } else {
                const uint4 b = *reinterpret_cast<const uint4 *>(&raw[r]);
                z[0] = __uint_as_float(b.x); z[1] = __uint_as_float(b.y);
                z[2] = __uint_as_float(b.z); z[3] = __uint_as_float(b.w);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float kv = fmaf(z[k], c, gk[k]);
                if (i0 + k < nv && kv > best) {
                    best = kv;
                    bi = i0 + k;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0) {
        bs.bk[warp] = best;
        bs.bi[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
        best = bs.bk[0];
        bi = bs.bi[0];
        for (int w = 1; w < kWarps; ++w)
            if (bs.bk[w] > best || (bs.bk[w] == best && bs.bi[w] < bi)) {
                best = bs.bk[w];
                bi = bs.bi[w];
            }
        prm.bonus_tok[pn] = bi == 0x7fffffff ? -1 : (int32_t)(v0 + bi);
    }
    return st;
}

__global__ void __launch_bounds__(kThreads, 4) k_tail(const __grid_constant__ Params prm, int resample_mode,
                                                   int chunks_per_prompt, int bonus_ctas, int cluster) {
    // chunk CTAs and bonus CTAs use disjoint shared state: one buffer, two views
    struct ChunkSmem {
        TailSmem sh;
        float4 rs[2 * kPairsPerCta];
        double ell_s[2 * kPairsPerCta];
    };
    constexpr size_t kSmemBytes = sizeof(ChunkSmem) > sizeof(BonusSmem) ? sizeof(ChunkSmem) : sizeof(BonusSmem);
    __shared__ __align__(16) unsigned char smem_raw[kSmemBytes];
    ChunkSmem &cs = *reinterpret_cast<ChunkSmem *>(smem_raw);
    BonusSmem &bsm = *reinterpret_cast<BonusSmem *>(smem_raw);
    TailSmem &sh = cs.sh;
    float4 *rs = cs.rs;
    double *ell_s = cs.ell_s;
    __shared__ int s_last;
    __shared__ uint32_t s_xe;                                   // S10: this launch's epoch
    // cluster tail with whole particles per chunk (K divides 32): S3 runs in the chunk CTAs and
    // each pushes its particles' lam' and its status bits into cluster rank 0's shared memory
    // (DSMEM stores, ordered by the cluster barrier), so rank 0 goes straight to S4-S7
    __shared__ double term_s[kPairsPerCta];
    __shared__ uint32_t s_cst;                                  // this chunk's status bits
    __shared__ uint32_t s_flags[16];                            // rank 0: every chunk's bits
    __shared__ __align__(16) WtSmem wts;                        // N <= 32: warp-synchronous S4-S7
    const int tid = threadIdx.x;
    const int N = prm.N, K = prm.K, NK = N * K, rows = 2 * NK;
    const int chunk_ctas = prm.P * chunks_per_prompt;
    if ((int)blockIdx.x >= chunk_ctas) {
        // bonus-token CTA (NEXT #2), after every chunk CTA in launch order.  Off the S3-S7
        // critical path: it does not take part in the completion count, and its flags are
        // OR-ed into status[p] (zeroed by K1's producer warp after its griddepcontrol.wait;
        // the last chunk CTA ORs its own bits when bonus CTAs exist).
        const int b = (int)blockIdx.x - chunk_ctas, p = b / N;
        const uint32_t bst = prm.dtype == 1 ? bonus_role<1>(prm, p, b - p * N, bsm)
                                            : bonus_role<0>(prm, p, b - p * N, bsm);
        if (tid == 0 && bst) atomicOr(&prm.status[p], bst);
        pdl_trigger();
        return;
    }
    const int per_prompt = chunks_per_prompt;
    const int p = blockIdx.x / per_prompt, c = blockIdx.x - p * per_prompt;
    const int q0 = c * kPairsPerCta, nq = min(kPairsPerCta, NK - q0);
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    const bool s3_local = cluster && (kPairsPerCta % K) == 0;   // uniform
    // Distributed shared memory may only be written once the target CTA has started: every
    // thread arrives on the cluster barrier now and waits before the first remote store (the
    // other CTAs have long arrived by then, so the wait does not stall)
    if (s3_local) asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
    // N <= 32: this lane's uniform for warp_tail (weight-independent, drawn before the wait)
    const double u_lane = (N <= 64 && resample_mode && tid < 32) ? tail_uniform(prm, p, tid) : 0.0;
    const double u_lane2 = (N > 32 && N <= 64 && resample_mode && tid < 32) ? tail_uniform(prm, p, tid + 32) : 0.0;
    int lr_model = 0, lr_q = 0;
    int64_t lr_pn = 0;
    float prev3 = 0.0f;                                         // S3 in the chunk: lam_prev, then lam'
    const bool row_thread = tid < 2 * kPairsPerCta && (tid & (kPairsPerCta - 1)) < nq;
    {

    // ---- inputs (not produced by the predecessor): before the wait
    int lr_kn = 0;
    int64_t lr_d = -1;
    float x_pre = -INFINITY;
    if (row_thread) {
        lr_model = tid / kPairsPerCta;
        lr_q = q0 + (tid & (kPairsPerCta - 1));
        const int n = lr_q / K, j = lr_q - n * K;
        lr_pn = (int64_t)p * N + n;
        lr_kn = drafted_len(prm, lr_pn);
        lr_d = prm.tokens[lr_pn * K + j];
        if (prm.x_from_logits && lr_kn >= 0 && lr_kn <= K && j < lr_kn && lr_d >= 0 && lr_d < prm.V)
            x_pre = load_x(prm, lr_model, lr_pn, j, lr_d);
    }
    // k_n of this thread's pair (terms) and, with S3 in the chunk, of its particle and lam_prev
    // (logw_prev may be the previous step's output: complete before K1 launched this grid)
    const int kn_t = tid < nq ? drafted_len(prm, (int64_t)p * N + (q0 + tid) / K) : 0;
    int kn3 = 0;
    if (s3_local && tid < nq / K) {
        const int64_t pn = (int64_t)p * N + q0 / K + tid;
        kn3 = drafted_len(prm, pn);
        prev3 = prm.logw_prev ? prm.logw_prev[pn] : (float)(-log((double)N));
    }
    if (tid == 0) {
        sh.st = 0;
        s_cst = 0;
        if (resample_mode) tail_prologue(prm, p, sh);
        wts.a = WtArgs{prm.logw_out, prm.wnorm, prm.lse, prm.ess, prm.ancestors, prm.offspring,
                       prm.slot_src, prm.n_ties, prm.resampled, prm.eta, prm.N, prm.scheme};
        wts.st = 0u;
    }
    if (tid == 0 && blockIdx.x == 0) SMCSD_TRACE_AT(2048);      // tail CTA resident
    // S10 (xlocal): the pushed words themselves are the dependency (the tail polls them), so
    // the tail does not wait for K1's grid to complete and flush.
    // Polling tail (lt_words): likewise K1's {m, s} words are the dependency; K1's counter is
    // re-armed at exit, once K1's grid has completed (x_tail_rearm).
    if (!prm.xlocal && !prm.lt_words) pdl_wait();
    if (tid == 0 && blockIdx.x == 0) {
        SMCSD_TRACE_AT(2049);                                   // predecessor complete
        SMCSD_CLK_AT(2200);
        if (prm.work_ctr && !prm.xlocal && !prm.lt_words) *prm.work_ctr = 0u;    // re-arm K1's counter
    }
    if (prm.xlocal) {
        // this launch's epoch (device epoch: advanced by the previous step's tail, which
        // completed before this step's K1 passed its griddepcontrol.wait) picks the half
        if (tid == 0) s_xe = x_epoch(prm);
        __syncthreads();
    }

    // ---- S2: 4 lanes per row, 64 rows per CTA in one pass.  Lane l4 of a row merges parts
    // 4 l4 .. 4 l4 + 3 (+ 16 c for rows with more than 16 parts) in index order in registers
    // (coalesced: a row's 16 parts are 256 contiguous bytes), then a fixed 2-step shuffle tree
    // (xor 2, xor 1).  x = t_d is taken from the logits (x_from_logits) or as the max of the
    // parts' x (TP combine).
    if (tid == 0 && blockIdx.x == 0) SMCSD_CLK_AT(2201);
    // S10 with the device epoch: this epoch's parity half of the exchange buffer
    const float4 *parts = prm.xlocal && !prm.xepoch ? prm.parts + (int64_t)(s_xe & 1u) * prm.xhalf : prm.parts;
    bool s2_late = false;                                       // polling tail: a word timed out
    {
        const int l4 = tid & 3, lr = tid >> 2;                  // local row: model = lr / 32
        const int qq = lr & (kPairsPerCta - 1);
        const int64_t grow = (int64_t)p * rows + (int64_t)(lr / kPairsPerCta) * NK + q0 + qq;
        const float4 *pr = parts + grow * prm.part_row_stride;
        float Ml = -INFINITY, Sl = 0.0f, Xl = -INFINITY;
        if (qq < nq) {
            if (prm.nparts <= 16) {
                float4 t[4];
                if (prm.xlocal) {
                    if (xp_take4(pr, prm.part_seg_stride, 4 * l4, prm.nparts, t)) atomicOr(&prm.st_ws[p], ST_EXCHANGE);
                } else if (prm.lt_words) {
                    s2_late = lt_take<1>(prm.lt_words, 2ll * prm.P * NK, grow, 4 * l4, 0, prm.nparts, t);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int pi = 4 * l4 + k;
                        t[k] = pi < prm.nparts ? __ldcg(pr + (int64_t)pi * prm.part_seg_stride)
                                               : make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f);
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    Ml = fmaxf(Ml, t[k].x);
                    Xl = fmaxf(Xl, t[k].z);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    Sl = __fmaf_rn(t[k].y, t[k].x == Ml ? 1.0f : ex2_approx(t[k].x - Ml), Sl);
            } else {
                bool late = false;
                for (int c = 0; 4 * l4 + 16 * c < prm.nparts; ++c)
                    for (int k = 0; k < 4; ++k) {
                        const int pi = 4 * l4 + 16 * c + k;
                        if (pi < prm.nparts) {
                            const float4 *sp = pr + (int64_t)pi * prm.part_seg_stride;
                            const float4 t = prm.xlocal ? xp_peek(sp, late) : __ldcg(sp);
                            Ml = fmaxf(Ml, t.x);
                            Xl = fmaxf(Xl, t.z);
                        }
                    }
                for (int c = 0; 4 * l4 + 16 * c < prm.nparts; ++c)
                    for (int k = 0; k < 4; ++k) {
                        const int pi = 4 * l4 + 16 * c + k;
                        if (pi < prm.nparts) {
                            const float4 *sp = pr + (int64_t)pi * prm.part_seg_stride;
                            const float4 t = prm.xlocal ? xp_read_zero(sp) : __ldcg(sp);
                            Sl = __fmaf_rn(t.y, t.x == Ml ? 1.0f : ex2_approx(t.x - Ml), Sl);
                        }
                    }
                if (late) atomicOr(&prm.st_ws[p], ST_EXCHANGE);
            }
        }
        float M = fmaxf(Ml, __shfl_xor_sync(0xffffffffu, Ml, 2));
        M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
        float X = Xl;
        if (!prm.x_from_logits) {                               // uniform branch
            X = fmaxf(X, __shfl_xor_sync(0xffffffffu, X, 2));
            X = fmaxf(X, __shfl_xor_sync(0xffffffffu, X, 1));
        }
        float S = __fmul_rn(Sl, Ml == M ? 1.0f : ex2_approx(Ml - M));
        S = __fadd_rn(S, __shfl_xor_sync(0xffffffffu, S, 2));
        S = __fadd_rn(S, __shfl_xor_sync(0xffffffffu, S, 1));
        if (l4 == 0) rs[lr] = make_float4(M, S, X, 0.0f);
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) SMCSD_CLK_AT(2202);
    // ---- ell per row (thread = local row), then terms per pair
    uint32_t st = s2_late ? ST_EXCHANGE : 0u;
    if (row_thread) {
        const int j = lr_q - (lr_q / K) * K;
        const bool valid = lr_kn >= 0 && lr_kn <= K && j < lr_kn;
        const float4 m = rs[tid];
        const float x = prm.x_from_logits ? x_pre : m.z;
        double ell = 0.0;
        if (!valid) {
            ell = 0.0;
        } else if (lr_d < 0 || lr_d >= prm.V) {
            st |= ST_BAD_TOKEN;
            ell = qnan;
        } else if (!isfinite(m.x) || !isfinite(m.y)) {
            st |= ST_NONFINITE;
            ell = qnan;
        } else {
            ell = __dmul_rn(__dsub_rn(__dsub_rn((double)x, (double)m.x), (double)log2f(m.y)), kLn2);
        }
        ell_s[tid] = ell;
        // with S3 in the chunk these output stores go after the cluster barrier's arrive (a
        // release would wait for them)
        float *outp = lr_model == 0 ? prm.logp_tok : prm.logq_tok;
        if (outp && !s3_local) outp[lr_pn * K + j] = (float)ell;
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) SMCSD_CLK_AT(2203);
    if (tid < nq) {
        const int qq = q0 + tid, j = qq - (qq / K) * K;
        const int kn = kn_t;
        double term = 0.0;
        if (kn >= 0 && kn <= K && j < kn) {
            const double lp = ell_s[tid], lq = ell_s[kPairsPerCta + tid];
            if (isnan(lp) || isnan(lq)) {
                term = qnan;
            } else if (lq == -INFINITY) {
                st |= ST_NOT_ABSCONT;
                term = qnan;
            } else {
                term = __dsub_rn(__dmul_rn(prm.alpha, lp), lq);
            }
        }
        if (s3_local) term_s[tid] = term;
        else __stcg(&prm.ell_ws[(int64_t)p * NK + qq], term);
    }
    if (s3_local) {
        if (st) atomicOr(&s_cst, st);
        asm volatile("barrier.cluster.wait;" ::: "memory");     // every CTA of the cluster started
        __syncthreads();
        // S3 for this chunk's whole particles, exactly as the rank-0 loop below does it
        const int np_chunk = nq / K;
        unsigned crank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
        if (tid < np_chunk) {
            const int n = q0 / K + tid;
            int kn = kn3;
            uint32_t st3 = 0;
            bool bad = false;
            if (kn < 0 || kn > K) {
                st3 |= ST_BAD_TOKEN;
                bad = true;
                kn = 0;
            }
            double delta = 0.0;
            for (int j = 0; j < kn; ++j) delta = __dadd_rn(delta, term_s[tid * K + j]);
            if (isnan(delta)) bad = true;
            const float prev = prev3;
            if (isnan(prev) || prev == INFINITY) {
                st3 |= ST_NONFINITE;
                bad = true;
            }
            const float lam = bad ? -INFINITY : (float)__dadd_rn((double)prev, delta);
            st_cluster_f32(&sh.lam[n], 0u, lam);
            prev3 = lam;                                        // stored after the arrive
            if (st3) atomicOr(&s_cst, st3);
        }
        __syncthreads();
        if (tid == 0) st_cluster_u32(&s_flags[crank], 0u, s_cst);
    } else if (st) {
        atomicOr(&prm.st_ws[p], st);
    }
    if (tid == 0 && blockIdx.x == 0) { SMCSD_TRACE_AT(2053); SMCSD_CLK_AT(2204); }      // chunk 0 S2 done
    }
    // ---- completion: the last CTA of the prompt finishes it.  Release chain: the barrier
    // orders every thread's terms / flags before thread 0's gpu-scope release fence and count;
    // the CTA completing the count acquires (fence) and its barrier passes that on to its
    // threads, whose reads of the other CTAs' terms go to L2 (ld.cg).
    if (cluster) {
        // the prompt's chunk CTAs are one thread-block cluster: a cluster barrier (release /
        // acquire at cluster scope, covering the global terms and flags) replaces the counter,
        // and cluster rank 0 finishes the prompt
        if (tid == 0 && blockIdx.x == 0) SMCSD_CLK_AT(2205);
        asm volatile("barrier.cluster.arrive.release;" ::: "memory");
        if (s3_local) {
            // this chunk's outputs, after the arrive: nothing in the cluster reads them
            if (row_thread) {
                float *outp = lr_model == 0 ? prm.logp_tok : prm.logq_tok;
                if (outp) outp[lr_pn * K + (lr_q - (lr_q / K) * K)] = (float)ell_s[tid];
            }
            if (tid < nq / K) {
                const int64_t pn = (int64_t)p * N + q0 / K + tid;
                if (prm.logw_pre) prm.logw_pre[pn] = prev3;
                if (!resample_mode) prm.logw_out[pn] = prev3;
            }
        }
        asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
        if (tid == 0) {
            unsigned r;
            asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
            s_last = r == 0u;
        }
    } else {
        __syncthreads();
        if (tid == 0 && blockIdx.x == 0) SMCSD_CLK_AT(2205);
        if (tid == 0) {
            fence_acq_rel_gpu();
            s_last = atomicAdd(&prm.prompt_ctr[p], 1u) == (unsigned)(per_prompt - 1);
            if (s_last) fence_acq_rel_gpu();
        }
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x == 0) SMCSD_CLK_AT(2206);
    if (!s_last) {
        x_tail_rearm(prm);
        x_tail_done(prm, s_xe);
        pdl_trigger();
        return;
    }
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2050);
    if (s3_local) {
        // S3 ran in the chunk CTAs: lam' is in sh.lam (visible after the cluster barrier), the
        // chunks' status bits in s_flags.  With N <= 64 warp 2 merges the bits while warps 0-1
        // run S4-S7 (the barrier after S4-S7 orders sh.st before the status write).
        if (tid == 64) {
            uint32_t f = 0;
            for (int r = 0; r < per_prompt; ++r) f |= s_flags[r];
            sh.st |= f;
        }
        if (N > 64) __syncthreads();
    } else {
    // ---- S3: lam' = fl32(prev + sum_{j<k_n} term_j) in j order
    const double *terms = prm.ell_ws + (int64_t)p * NK;
    uint32_t st3 = 0;
    const float neglogN = (float)(-log((double)N));
    for (int n = tid; n < N; n += kThreads) {
        const int64_t pn = (int64_t)p * N + n;
        int kn = drafted_len(prm, pn);
        bool bad = false;
        if (kn < 0 || kn > K) {
            st3 |= ST_BAD_TOKEN;
            bad = true;
            kn = 0;
        }
        double delta = 0.0;
        for (int j0 = 0; j0 < kn; j0 += 8) {                // loads first, then the j-order sum
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = j0 + u < kn ? __ldcg(&terms[n * K + j0 + u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (j0 + u < kn) delta = __dadd_rn(delta, t[u]);
        }
        if (isnan(delta)) bad = true;                       // an invalid pair (flag raised in S2)
        const float prev = prm.logw_prev ? prm.logw_prev[pn] : neglogN;
        if (isnan(prev) || prev == INFINITY) {
            st3 |= ST_NONFINITE;
            bad = true;
        }
        const float lam = bad ? -INFINITY : (float)__dadd_rn((double)prev, delta);
        sh.lam[n] = lam;
        if (prm.logw_pre) prm.logw_pre[pn] = lam;
        if (!resample_mode) prm.logw_out[pn] = lam;
    }
    if (st3) atomicOr(&sh.st, st3);
    __syncthreads();
    if (tid == 0) {
        sh.st |= __ldcg(&prm.st_ws[p]);                         // flags of every chunk
        prm.st_ws[p] = 0u;
        prm.prompt_ctr[p] = 0u;                                  // graph-replay safe
    }
    __syncthreads();
    }
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2051);
    if (N <= 64) {
        if (tid < 64) {
            if (N <= 32) warp_tail<1>(tid >> 5, p, resample_mode, 0, sh.lam, u_lane, 0.0, sh.reset, wts);
            else warp_tail<2>(tid >> 5, p, resample_mode, 0, sh.lam, u_lane, u_lane2, sh.reset, wts);
        }
    } else {
        normalise_resample(prm, p, resample_mode != 0, sh);
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t st_all = sh.st | wts.st;
        if (bonus_ctas) atomicOr(&prm.status[p], st_all);
        else prm.status[p] = st_all;
    }
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2052);
    x_tail_rearm(prm);
    x_tail_done(prm, s_xe);
    pdl_trigger();
}

// K2 (TP partial path): merge each row's segment partials into one {m, s, x, 0}.  grid =
// P x ceil(2NK / 64): one CTA per 64 rows, 16 lanes per row (coalesced 16-byte loads, the fixed
// 16-lane tree of k_tail), 4 passes; x = t_d (when the drafted token is in this shard) read from
// the logits before griddepcontrol.wait by the row's first thread.
constexpr int kMergeRowsPerCta = 64;
__global__ void __launch_bounds__(kThreads) k_merge_rows(const __grid_constant__ Params prm) {
    const int tid = threadIdx.x, N = prm.N, K = prm.K, NK = N * K, rows = 2 * NK;
    const int chunks = (rows + kMergeRowsPerCta - 1) / kMergeRowsPerCta;
    const int p = blockIdx.x / chunks, r0 = (blockIdx.x - p * chunks) * kMergeRowsPerCta;
    __shared__ float xs[kMergeRowsPerCta];
    if (tid < kMergeRowsPerCta) {                              // inputs only: safe before the wait
        const int r = r0 + tid;
        float x = -INFINITY;
        if (r < rows) {
            const int model = r / NK, q = r - model * NK, n = q / K, j = q - n * K;
            const int64_t pn = (int64_t)p * N + n;
            const int kn = drafted_len(prm, pn);
            if (kn >= 0 && kn <= K && j < kn) x = load_x(prm, model, pn, j, prm.tokens[pn * K + j]);
        }
        xs[tid] = x;
    }
    pdl_wait();
    if (tid == 0 && blockIdx.x == 0) *prm.work_ctr = 0u;      // re-arm K1's counter
    __syncthreads();
    const int li = tid & 15, rsub = tid >> 4;
    float3 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int r = r0 + rsub + 16 * u;
        const int64_t grow = (int64_t)p * rows + r;
        q[u] = make_float3(-INFINITY, 0.0f, -INFINITY);
        if (r < rows) {
            if (prm.nparts <= 16) {
                if (li < prm.nparts) {
                    const float4 t = __ldcg(&prm.parts[grow * prm.part_row_stride + (int64_t)li * prm.part_seg_stride]);
                    q[u] = make_float3(t.x, t.y, t.z);
                }
            } else {
                q[u] = lane_premerge(prm, grow, li);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        float M = q[u].x;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        float S = q[u].y * (q[u].x == M ? 1.0f : ex2_approx(q[u].x - M));
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        const int lr = rsub + 16 * u, r = r0 + lr;
        if (li == 0 && r < rows) prm.partials_out[(int64_t)p * rows + r] = make_float4(M, S, xs[lr], 0.0f);
    }
    pdl_trigger();
}

// S4-S7 from fp32 log-weights, grid = P (smcsd_resample).
__global__ void __launch_bounds__(kThreads) k_resample(const __grid_constant__ Params prm) {
    __shared__ TailSmem sh;
    const int p = blockIdx.x, N = prm.N;
    if (threadIdx.x == 0) {
        sh.st = 0;
        tail_prologue(prm, p, sh);
    }
    pdl_wait();
    __syncthreads();
    uint32_t st = 0;
    for (int n = threadIdx.x; n < N; n += kThreads) {
        float v = prm.logw_prev[(int64_t)p * N + n];
        if (isnan(v) || v == INFINITY) {
            st |= ST_NONFINITE;
            v = -INFINITY;
        }
        sh.lam[n] = v;
    }
    if (st) atomicOr(&sh.st, st);
    __syncthreads();
    normalise_resample(prm, p, true, sh);
    __syncthreads();
    if (threadIdx.x == 0) prm.status[p] = sh.st;
    pdl_trigger();
}

// Large-N weights path (N > kTailMaxN): S2+S3 in parallel, S4 serial over global workspace.
__global__ void __launch_bounds__(kThreads) k_tail_large(const __grid_constant__ Params prm) {
    __shared__ uint32_t s_st;
    __shared__ float s_red[kWarps];
    __shared__ double s_M, s_S;
    const int p = blockIdx.x, N = prm.N, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)p * N;
    if (tid == 0) s_st = 0;
    pdl_wait();
    if (tid == 0 && p == 0) *prm.work_ctr = 0u;               // re-arm K1's counter
    __syncthreads();
    extern __shared__ float4 dyn_smem[];
    float4 *rowstat = prm.rowstat_ws + (int64_t)p * 2 * N * prm.K;
    tail_rowstats(prm, p, rowstat, dyn_smem);
    __syncthreads();
    float x_pre = -INFINITY;
    if (prm.x_from_logits && tid < 2 * N * prm.K) {
        const int model = tid & 1, q = tid >> 1, n = q / prm.K, j = q - n * prm.K;
        const int64_t pn = (int64_t)p * N + n;
        const int kn = drafted_len(prm, pn);
        const int64_t d = prm.tokens[pn * prm.K + j];
        if (kn >= 0 && kn <= prm.K && j < kn && d >= 0 && d < prm.V) x_pre = load_x(prm, model, pn, j, d);
    }
    tail_scores(prm, p, rowstat, nullptr, &s_st, x_pre);
    __syncthreads();
    const float neglogN = (float)(-log((double)N));
    uint32_t st = 0;
    float mloc = -INFINITY;
    for (int n = tid; n < N; n += kThreads) {
        const float lam = tail_reweight(prm, p, n, nullptr,
                                        prm.logw_prev ? prm.logw_prev[base + n] : neglogN, &st);
        __stcg(&prm.lam_ws[base + n], lam);
        prm.logw_out[base + n] = lam;
        if (prm.logw_pre) prm.logw_pre[base + n] = lam;
        mloc = fmaxf(mloc, lam);
    }
    if (st) atomicOr(&s_st, st);
    mloc = warp_max(mloc);
    if (lane == 0) s_red[warp] = mloc;
    __syncthreads();
    if (tid == 0) {
        float M = s_red[0];
        for (int w = 1; w < kWarps; ++w) M = fmaxf(M, s_red[w]);
        s_M = (double)M;
    }
    __syncthreads();
    const double M = s_M;
    if (M == -INFINITY) {
        for (int n = tid; n < N; n += kThreads) if (prm.wnorm) prm.wnorm[base + n] = 0.0f;
        if (tid == 0) {
            if (prm.lse) prm.lse[p] = -INFINITY;
            if (prm.ess) prm.ess[p] = 0.0;
            prm.status[p] = s_st | ST_DEGENERATE;
        }
        return;
    }
    for (int n = tid; n < N; n += kThreads)
        __stcg(&prm.e_ws[base + n], exp(__dsub_rn((double)__ldcg(&prm.lam_ws[base + n]), M)));
    __syncthreads();
    if (tid == 0) {
        double acc = 0.0, sq = 0.0;
        for (int m = 0; m < N; ++m) {
            const double e = __ldcg(&prm.e_ws[base + m]);
            acc = __dadd_rn(acc, e);
            sq = __dadd_rn(sq, __dmul_rn(e, e));
        }
        s_S = acc;
        if (prm.lse) prm.lse[p] = __dadd_rn(M, log(acc));
        if (prm.ess) prm.ess[p] = __ddiv_rn(__dmul_rn(acc, acc), sq);
        prm.status[p] = s_st;
    }
    __syncthreads();
    if (prm.wnorm)
        for (int n = tid; n < N; n += kThreads)
            prm.wnorm[base + n] = (float)__ddiv_rn(__ldcg(&prm.e_ws[base + n]), s_S);
}

// PowerSMC tail (NEXT #4; App. F), grid = P: per particle, merge the row's
// segment partials {m, s, -, s2} in index order, log w = ln 2 (log2 S2 - alpha log2 S1) =
// ln sum_v p_v^alpha, lam' = fl32(lam_prev + log w), then S4 (weights mode).
__global__ void __launch_bounds__(kThreads) k_power_tail(const __grid_constant__ Params prm) {
    __shared__ TailSmem sh;
    const int p = blockIdx.x, N = prm.N, tid = threadIdx.x;
    const float neglogN = (float)(-log((double)N));
    if (tid == 0) sh.st = 0;
    pdl_wait();
    if (tid == 0 && p == 0) *prm.work_ctr = 0u;               // re-arm K1's counter
    __syncthreads();
    uint32_t st = 0;
    const double a = (double)prm.alpha_f;
    for (int n = tid; n < N; n += kThreads) {
        const int64_t pn = (int64_t)p * N + n;
        const float4 *parts = prm.part_ws + pn * prm.nseg;     // rows [P][N] (K = 1, one model)
        // the row's parts in chunks of 16 loaded together (one L2 round trip per chunk, not
        // one per part); within a chunk: max, then the sums in part order.  A later chunk
        // with a larger max rescales the running sums (V > 16 segments only).
        float M = -INFINITY, S1 = 0.0f, S2 = 0.0f;
        for (int i0 = 0; i0 < prm.nseg; i0 += 16) {
            float4 q[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
                q[u] = i0 + u < prm.nseg ? __ldcg(&parts[i0 + u]) : make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f);
            float Mc = M;
#pragma unroll
            for (int u = 0; u < 16; ++u) Mc = fmaxf(Mc, q[u].x);
            if (Mc != M && M != -INFINITY) {
                S1 *= ex2_approx(M - Mc);
                S2 *= ex2_approx((M - Mc) * prm.alpha_f);
            }
            M = Mc;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (i0 + u >= prm.nseg) break;
                const float d = q[u].x == M ? 0.0f : q[u].x - M;
                S1 += q[u].y * (q[u].x == M ? 1.0f : ex2_approx(d));
                S2 += q[u].w * (q[u].x == M ? 1.0f : ex2_approx(d * prm.alpha_f));
            }
        }
        const float prev = prm.logw_prev ? prm.logw_prev[pn] : neglogN;
        bool bad = false;
        double inc = __longlong_as_double(0x7ff8000000000000ll);
        if (!isfinite(M) || !isfinite(S1) || !isfinite(S2)) {
            st |= ST_NONFINITE;
            bad = true;
        } else {
            inc = __dmul_rn(__dsub_rn(log2((double)S2), __dmul_rn(a, log2((double)S1))), kLn2);
        }
        if (isnan(prev) || prev == INFINITY) {
            st |= ST_NONFINITE;
            bad = true;
        }
        const float lam = bad ? -INFINITY : (float)__dadd_rn((double)prev, inc);
        sh.lam[n] = lam;
        prm.logw_out[pn] = lam;
        if (prm.logp_tok) prm.logp_tok[pn] = (float)inc;        // per-particle log w
    }
    if (st) atomicOr(&sh.st, st);
    __syncthreads();
    normalise_resample(prm, p, false, sh);
    __syncthreads();
    if (tid == 0) prm.status[p] = sh.st;
    pdl_trigger();
}

// S10, all-reduce form (the north star's literal "NCCL all-reduces the per-row max/sum-exp"):
// between all_reduce(MAX) of {m, s, x, 0} (only m and x are used) and all_reduce(SUM) of the
// rescaled sums, each rank maps its local row sum to the global max:
//   s'_r = s_r 2^(m_r - M_r)   (s_r when m_r == M_r; 0 when s_r == 0; NaN propagates)
// and writes {M_r, s'_r, X_r, 0} so that after the SUM of field 1 across ranks the row holds the
// merged {M, S, X} that smcsd_weights_combine takes with G = 1.
__global__ void __launch_bounds__(kThreads) k_partials_rescale(const float4 *local, const float4 *mx,
                                                              float4 *out, int64_t rows) {
    for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < rows; r += (int64_t)gridDim.x * kThreads) {
        const float4 l = local[r], g = mx[r];
        const float sc = l.y == 0.0f ? 0.0f : __fmul_rn(l.y, l.x == g.x ? 1.0f : ex2_approx(l.x - g.x));
        out[r] = make_float4(g.x, sc, g.z, 0.0f);
    }
}

// Exchange-buffer init: control words and every slot zero (= not yet written).
__global__ void k_xinit(char *base, size_t n_parts) {
    if (blockIdx.x == 0 && threadIdx.x < kXFlagBytes / 4) reinterpret_cast<uint32_t *>(base)[threadIdx.x] = 0u;
    float4 *parts = reinterpret_cast<float4 *>(base + kXFlagBytes);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_parts; i += (size_t)gridDim.x * blockDim.x)
        parts[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
}

// Terminal selection: one index per prompt from the normalised weights by the
// same inverse CDF, u = word0(Philox(key = seed, ctr = (step_lo, step_hi, prompt, 0xFFFFFFFF))).
// grid = P, one warp per prompt; lane 0 runs the sequential fp64 prefix.
__global__ void __launch_bounds__(32) k_select(const __grid_constant__ Params prm) {
    const int p = blockIdx.x, N = prm.N, lane = threadIdx.x;
    const int64_t base = (int64_t)p * N;
    pdl_wait();
    float mloc = -INFINITY;
    uint32_t st = 0;
    for (int n = lane; n < N; n += 32) {
        float v = prm.logw_prev[base + n];
        if (isnan(v) || v == INFINITY) { st |= ST_NONFINITE; v = -INFINITY; }
        mloc = fmaxf(mloc, v);
    }
    const double M = (double)warp_max(mloc);
    st = __reduce_or_sync(0xffffffffu, st);
    if (lane == 0) {
        if (M == -INFINITY) {
            prm.selected[p] = -1;
            prm.status[p] = st | ST_DEGENERATE;
        } else {
            uint32_t x;
            if (prm.uniforms) {
                x = prm.uniforms[p];
            } else {
                const uint64_t g = (uint64_t)(prm.prompt_base + p);
                x = philox4x32_10(make_uint4((uint32_t)prm.step, (uint32_t)(prm.step >> 32), (uint32_t)g, 0xFFFFFFFFu),
                                  make_uint2((uint32_t)prm.seed, (uint32_t)(prm.seed >> 32))).x;
            }
            const double u = (double)x * 2.3283064365386962890625e-10;
            double acc = 0.0;
            for (int m = 0; m < N; ++m) {
                float v = prm.logw_prev[base + m];
                if (isnan(v) || v == INFINITY) v = -INFINITY;
                acc = __dadd_rn(acc, exp(__dsub_rn((double)v, M)));
                prm.e_ws[base + m] = acc;
            }
            int count = 0;
            for (int m = 0; m < N; ++m) count += __ddiv_rn(prm.e_ws[base + m], acc) <= u;
            prm.selected[p] = count;
            prm.status[p] = st;
        }
    }
    pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// K5: paged (pointer) KV reindex -- the paper's own mechanism ("copying page
// metadata and incrementing the reference counts").  No KV content moves.
//   k_paged_gather (grid P): table_dst[p][n][:] = table_src[p][a_n][:], n_pages_dst = the
//     ancestor's length, refcount += 1 per new reference and -= 1 per old reference (integer
//     atomics: order-free, exact);
//   k_paged_freed (grid P, PDL): freed[pg] = (refcount[pg] == 0) for every old-list page.
// ------------------------------------------------------------------------------------------
struct PagedParams {
    const int32_t *table_src, *n_src, *idx;
    int32_t *table_dst, *n_dst, *refcount;
    uint8_t *freed;
    uint32_t *status;
    int P, N, max_pages, num_pages;
};

// grid = (ceil(N * max_pages / kThreads), P): one (particle, slot) entry per thread, so a long
// list's loads are independent.  status[p] was zeroed by the caller's stream (memset) before.
__global__ void __launch_bounds__(kThreads) k_paged_gather(const __grid_constant__ PagedParams q) {
    const int p = blockIdx.y, N = q.N, MP = q.max_pages;
    pdl_wait();
    uint32_t st = 0;
    const int64_t base = (int64_t)p * N;
    const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (e < (int64_t)N * MP) {
        const int n = (int)(e / MP), i = (int)(e - (int64_t)n * MP);
        // new list of n = old list of its ancestor
        const int a = q.idx[base + n];
        int len = 0;
        if (a < 0 || a >= N) {
            st |= ST_BAD_PAGE;
        } else {
            len = q.n_src[base + a];
            if (len < 0 || len > MP) { st |= ST_BAD_PAGE; len = 0; }
        }
        int32_t pg = -1;
        if (i < len) {
            pg = q.table_src[(base + a) * MP + i];
            if (pg < 0 || pg >= q.num_pages) { st |= ST_BAD_PAGE; pg = -1; }
            else atomicAdd(&q.refcount[pg], 1);
        }
        q.table_dst[(base + n) * MP + i] = pg;
        if (i == 0) q.n_dst[base + n] = len;
        // old list of n drops its references
        const int olen = q.n_src[base + n];
        if (olen < 0 || olen > MP) {
            if (i == 0) st |= ST_BAD_PAGE;
        } else if (i < olen) {
            const int32_t og = q.table_src[(base + n) * MP + i];
            if (og < 0 || og >= q.num_pages) st |= ST_BAD_PAGE;
            else atomicSub(&q.refcount[og], 1);
        }
    }
    st = __reduce_or_sync(0xffffffffu, st);
    if (st && (threadIdx.x & 31) == 0 && q.status) atomicOr(&q.status[p], st);
    pdl_trigger();
}

__global__ void __launch_bounds__(kThreads) k_paged_freed(const __grid_constant__ PagedParams q) {
    const int p = blockIdx.y, N = q.N, MP = q.max_pages;
    pdl_wait();
    const int64_t base = (int64_t)p * N;
    const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (e < (int64_t)N * MP) {
        const int n = (int)(e / MP), i = (int)(e - (int64_t)n * MP);
        const int olen = q.n_src[base + n];
        if (olen >= 0 && olen <= MP && i < olen) {
            const int32_t og = q.table_src[(base + n) * MP + i];
            if (og >= 0 && og < q.num_pages) q.freed[og] = (uint8_t)(__ldcg(&q.refcount[og]) == 0);
        }
    }
    pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// K3: S8/S9 source-major block gather.  grid = n_outer * P * nchunks, block = kThreads.
// ------------------------------------------------------------------------------------------
constexpr int kKvUnroll = 4;
constexpr int kKvChunkVec = kThreads * kKvUnroll;             // 16-byte vectors per CTA chunk

// One state tensor of a reindex launch (byte geometry; see smcsd_kv_tensor in smcsd.h).
struct KvTensor {
    char *dst;
    const char *src;
    int64_t outer_stride, prompt_stride, particle_stride, seg_stride;
    uint32_t vps;                 // 16-byte vectors per segment
    int in_place;                 // dst == src: apply the slot plan (skip src_index[n] == n)
    uint64_t vecs;                // vectors per block = seg_count * vps
    int64_t nchunks;              // CTA chunks per block
    int64_t item_end;             // exclusive prefix of items (n_outer * P * nchunks) over tensors
};
constexpr int kMaxKvTensors = 256;        // 256 x 72 B of __grid_constant__ parameters

struct KvParams {
    const int32_t *idx;           // [P][N] src_index (ancestors, or the slot plan in place)
    uint32_t *status;             // [P] or null: ST_BAD_INDEX per prompt (written by chunk 0)
    int P, N, n_tensors;
    int any_in_place;             // some tensor is reindexed in place
    KvTensor t[kMaxKvTensors];
};

// Grid = sum over tensors of n_outer * P * nchunks items; item -> (tensor by binary search over
// item_end, outer plane, prompt, chunk).  Every CTA builds its prompt's copy plan (destinations
// grouped by source, counting sort) and copies its chunk source-major: each source vector is
// loaded once and stored to every destination.
__global__ void __launch_bounds__(kThreads) k_kv_reindex(const __grid_constant__ KvParams prm) {
    __shared__ int cnt[kTailMaxN], start[kTailMaxN], fill[kTailMaxN], dsts[kTailMaxN], srcs[kTailMaxN];
    __shared__ int wtot[kWarps + 1];
    const int tid = threadIdx.x, N = prm.N;
    int lo = 0, hi = prm.n_tensors - 1;                        // first tensor with item_end > item
    const int64_t gitem = blockIdx.x;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (prm.t[mid].item_end > gitem) hi = mid; else lo = mid + 1;
    }
    const KvTensor &T = prm.t[lo];
    const int64_t item = gitem - (lo > 0 ? prm.t[lo - 1].item_end : 0);
    const int64_t chunk = item % T.nchunks;
    const int64_t op = item / T.nchunks;
    const int p = (int)(op % prm.P);
    const int64_t o = op / prm.P;
    const int in_place = T.in_place;
    const int32_t *idx = prm.idx + (int64_t)p * N;
    pdl_wait();                                                // src_index from the tail kernel

    // ---- copy plan for prompt p: destinations grouped by source (counting sort).  Entries
    // outside [0, N) are skipped; an in-place plan in which some index is both a source and a
    // destination (not hazard-free) is skipped whole.  Both raise ST_BAD_INDEX.
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    for (int n = tid; n < N; n += kThreads) {
        cnt[n] = 0;
        srcs[n] = idx[n];                                      // staged copy (srcs is rebuilt below)
    }
    __syncthreads();
    int bad = 0;
    for (int n = tid; n < N; n += kThreads) {
        const int s = srcs[n];
        if ((unsigned)s >= (unsigned)N) bad |= 1;
        else if (s != n && srcs[s] != s) bad |= 2;             // source s is itself overwritten
        if ((unsigned)s < (unsigned)N && (!in_place || s != n)) atomicAdd(&cnt[s], 1);
    }
    if (bad) atomicOr(&s_bad, bad);
    __syncthreads();
    const int pbad = s_bad;
    if (prm.status && lo == 0 && o == 0 && chunk == 0 && tid == 0)
        prm.status[p] = ((pbad & 1) || ((pbad & 2) && prm.any_in_place)) ? ST_BAD_INDEX : 0u;
    if (in_place && (pbad & 2)) return;                        // uniform across the CTA
    for (int n = tid; n < N; n += kThreads) {
        start[n] = cnt[n];
        fill[n] = cnt[n] > 0;
    }
    __syncthreads();
    block_exclusive_scan(start, N, wtot);
    const int nsrc = block_exclusive_scan(fill, N, wtot);
    for (int m = tid; m < N; m += kThreads)
        if (cnt[m] > 0) srcs[fill[m]] = m;
    __syncthreads();
    for (int m = tid; m < N; m += kThreads) fill[m] = 0;
    __syncthreads();
    for (int n = tid; n < N; n += kThreads) {
        const int s = idx[n];
        if ((unsigned)s < (unsigned)N && (!in_place || s != n))
            dsts[start[s] + atomicAdd(&fill[s], 1)] = n;
    }
    __syncthreads();

    // ---- byte offsets of this thread's vectors inside a block
    int64_t voff[kKvUnroll];
    bool valid[kKvUnroll];
#pragma unroll
    for (int i = 0; i < kKvUnroll; ++i) {
        const uint64_t v = (uint64_t)chunk * kKvChunkVec + (uint64_t)i * kThreads + tid;
        valid[i] = v < T.vecs;
        const uint64_t g = v / T.vps, w = v - g * T.vps;
        voff[i] = (int64_t)g * T.seg_stride + (int64_t)w * 16;
    }
    const int64_t pbase = o * T.outer_stride + (int64_t)p * T.prompt_stride;
    for (int k = 0; k < nsrc; ++k) {
        const int s = srcs[k];
        const char *sb = T.src + pbase + (int64_t)s * T.particle_stride;
        uint4 r[kKvUnroll];
#pragma unroll
        for (int i = 0; i < kKvUnroll; ++i)
            if (valid[i]) r[i] = ld_stream(sb + voff[i]);
        const int c = cnt[s], st0 = start[s];
        for (int q = 0; q < c; ++q) {
            char *db = T.dst + pbase + (int64_t)dsts[st0 + q] * T.particle_stride;
#pragma unroll
            for (int i = 0; i < kKvUnroll; ++i)
                if (valid[i]) st_stream(db + voff[i], r[i]);
        }
    }
}

}  // namespace smcsd
