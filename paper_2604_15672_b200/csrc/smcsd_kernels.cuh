// smcsd_kernels.cuh -- the sm_100a kernels of libsmcsd.
//
//  K1  k_rowstats<DT, MODE>  S1: per (logit row, fixed 8192-element segment) work item, one
//                            streaming pass: m = max t, s = sum 2^(t - m), x = t_d, with
//                            t = inv_temp * z * log2(e)  (Eq. 1a).
//                            MODE_WEIGHTS / MODE_STEP: the last CTA of each prompt (completion
//                            counter) runs the tail below in the same launch.
//  K2  tail_prompt           S2 merge segments in fixed order -> ell, S3 reweight, S4 fp64
//                            normalise + ESS, S5-S7 systematic resampling from Philox, reset.
//  K3  k_kv_reindex          S8/S9 source-major bitwise gather of per-particle blocks.
//
// Determinism (reading G17): every row uses the same segment boundaries and the same
// element->thread->warp->segment reduction order, so bitwise-equal p and q rows give
// bitwise-equal ell (p == q => Delta == 0 exactly) and every run is bit-reproducible.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "smcsd_device.cuh"

namespace smcsd {

enum { MODE_WEIGHTS = 0, MODE_STEP = 1, MODE_PARTIAL = 2, MODE_ROWS_ONLY = 3 };

constexpr uint32_t ST_DEGENERATE = 1u, ST_NOT_ABSCONT = 2u, ST_BAD_TOKEN = 4u, ST_NONFINITE = 8u;
constexpr double kLn2 = 0.693147180559945309417232121458176568;

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
    uint8_t *resampled;
    float4 *partials_out;                       // MODE_PARTIAL: [P*2*N*K] {m, s, x, 0}
    // ---- S2 sources: row r's parts at parts[r*part_row_stride + i*part_seg_stride], i < nparts
    const float4 *parts;
    int64_t part_row_stride, part_seg_stride;
    int nparts;
    // ---- workspace
    unsigned *counters;                         // [P]
    float4 *part_ws;                            // [P*2*N*K*nseg]
    double *ell_ws;                             // [P*2*N*K]
    float *lam_ws;                              // [P*N]   (N > kTailMaxN path)
    double *e_ws, *c_ws;                        // [P*N]
};

// ------------------------------------------------------------------------------------------
// S1 for one (row, segment).  Returns {m, s, x, 0} at thread 0 (log2 domain).
// ------------------------------------------------------------------------------------------
template <int DT>  // 0 = fp32, 1 = bf16
__device__ __forceinline__ float4 segment_stats(const char *row, int64_t v_len, int seg, float c,
                                                int64_t d_local, float2 *red) {
    constexpr int kEsz = DT == 1 ? 2 : 4;
    constexpr int kVec = 16 / kEsz;                          // elements per 16-byte load
    constexpr int kLoads = kSeg / (kThreads * kVec);         // 4 (bf16) or 8 (fp32)
    constexpr uint32_t kNegInf = DT == 1 ? 0xFF80FF80u : 0xFF800000u;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t v0 = (int64_t)seg * kSeg;

    // drafted-token logit: issued first so its latency hides under the stream
    float zd = -INFINITY;
    const bool has_d = tid == 0 && d_local >= v0 && d_local < v0 + kSeg && d_local < v_len;
    if (has_d) {
        if (DT == 1) zd = bf16lo((uint32_t)__ldg((const unsigned short *)row + d_local));
        else         zd = __ldg((const float *)row + d_local);
    }

    uint4 v[kLoads];
    if (v0 + kSeg <= v_len) {
#pragma unroll
        for (int i = 0; i < kLoads; ++i)
            v[i] = ld_stream(row + (v0 + (int64_t)(i * kThreads + tid) * kVec) * kEsz);
    } else {
#pragma unroll
        for (int i = 0; i < kLoads; ++i) {
            const int64_t e = v0 + (int64_t)(i * kThreads + tid) * kVec;
            if (e < v_len) {
                v[i] = ld_stream(row + e * kEsz);
                uint32_t *w = reinterpret_cast<uint32_t *>(&v[i]);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (DT == 1) {
                        if (e + 2 * k >= v_len)     w[k] = (w[k] & 0xffff0000u) | 0x0000FF80u;
                        if (e + 2 * k + 1 >= v_len) w[k] = (w[k] & 0x0000ffffu) | 0xFF800000u;
                    } else {
                        if (e + k >= v_len) w[k] = kNegInf;
                    }
                }
            } else {
                v[i] = make_uint4(kNegInf, kNegInf, kNegInf, kNegInf);
            }
        }
    }

    // ---- max over the warp's 1024 elements (raw logits; c > 0 so max(z)*c = max(z*c))
    float mt;
    if (DT == 1) {
        uint32_t acc = v[0].x;
#pragma unroll
        for (int i = 0; i < kLoads; ++i) {
            const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) asm("max.bf16x2 %0, %0, %1;" : "+r"(acc) : "r"(w4[k]));
        }
        mt = fmaxf(bf16lo(acc), bf16hi(acc));
    } else {
        mt = -INFINITY;
#pragma unroll
        for (int i = 0; i < kLoads; ++i) {
            mt = fmaxf(mt, fmaxf(fmaxf(__uint_as_float(v[i].x), __uint_as_float(v[i].y)),
                                 fmaxf(__uint_as_float(v[i].z), __uint_as_float(v[i].w))));
        }
    }
    const float mw = warp_max(mt) * c;                       // warp max of t = z*c
    const float off = mw == -INFINITY ? 0.0f : mw;           // all -inf: sum(2^-inf) = 0, NaN kept

    // ---- sum of 2^(t - m): exactly one ex2 per element
    float s_acc[kLoads];
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
        const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
        float a = 0.0f;
        if (DT == 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                a += ex2_approx(fmaf(bf16lo(w4[k]), c, -off));
                a += ex2_approx(fmaf(bf16hi(w4[k]), c, -off));
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) a += ex2_approx(fmaf(__uint_as_float(w4[k]), c, -off));
        }
        s_acc[i] = a;
    }
    float s = s_acc[0];
#pragma unroll
    for (int i = 1; i < kLoads; ++i) s += s_acc[i];
    s = warp_sum(s);
    if (lane == 0) red[warp] = make_float2(mw, s);
    __syncthreads();
    float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
        float M = red[0].x;
#pragma unroll
        for (int w = 1; w < kWarps; ++w) M = fmaxf(M, red[w].x);
        float S = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float mwv = red[w].x;
            S += red[w].y * (mwv == M ? 1.0f : ex2_approx(mwv - M));
        }
        out = make_float4(M, S, has_d ? zd * c : -INFINITY, 0.0f);
    }
    return out;
}

// Merge row parts in fixed index order: M = max m_i, S = sum s_i 2^(m_i - M), X = max x_i.
__device__ __forceinline__ float4 merge_parts(const float4 *parts, int64_t stride, int count) {
    float M = -INFINITY;
    for (int i = 0; i < count; ++i) M = fmaxf(M, __ldcg(&parts[i * stride]).x);
    float S = 0.0f, X = -INFINITY;
    for (int i = 0; i < count; ++i) {
        const float4 q = __ldcg(&parts[i * stride]);
        S += q.y * (q.x == M ? 1.0f : ex2_approx(q.x - M));
        X = fmaxf(X, q.z);
    }
    return make_float4(M, S, X, 0.0f);
}

__device__ __forceinline__ int drafted_len(const Params &prm, int64_t pn) {
    return prm.n_drafted ? prm.n_drafted[pn] : prm.K;
}

// ------------------------------------------------------------------------------------------
// Tail state in shared memory (N <= kTailMaxN) for the fused path and smcsd_resample.
// ------------------------------------------------------------------------------------------
struct TailSmem {
    double e[kTailMaxN];
    double C[kTailMaxN];
    float lam[kTailMaxN];
    int o[kTailMaxN];
    float2 red[kWarps];
    float fred[kWarps];
    int wtot[kWarps + 1];
    uint32_t st;
    int do_res, degenerate, ties;
    double S, U, M;
};

// S2 for every row of prompt p: ell -> ell_ws (+ optional fp32 outputs); flags into sh_st.
__device__ void tail_rows(const Params &prm, int p, uint32_t *sh_st) {
    const int N = prm.N, K = prm.K;
    const int64_t rows = 2ll * N * K;
    uint32_t st = 0;
    for (int64_t rl = threadIdx.x; rl < rows; rl += kThreads) {
        const int j = (int)(rl % K);
        const int n = (int)((rl / K) % N);
        const int model = (int)(rl / ((int64_t)N * K));
        const int64_t pn = (int64_t)p * N + n;
        const int64_t r = (int64_t)p * rows + rl;           // global row index
        const int kn = drafted_len(prm, pn);
        double ell = 0.0;
        if (kn >= 0 && kn <= K && j < kn) {
            const int64_t d = prm.tokens[pn * K + j];
            if (d < 0 || d >= prm.V) {
                st |= ST_BAD_TOKEN;
                ell = __longlong_as_double(0x7ff8000000000000ll);
            } else {
                const float4 q = merge_parts(prm.parts + r * prm.part_row_stride,
                                             prm.part_seg_stride, prm.nparts);
                if (!isfinite(q.x) || !isfinite(q.y)) {
                    st |= ST_NONFINITE;
                    ell = __longlong_as_double(0x7ff8000000000000ll);
                } else {
                    // ell = (x - m - log2 s) * ln 2   (natural log of the softmax at d)
                    ell = __dmul_rn(__dsub_rn(__dsub_rn((double)q.z, (double)q.x), log2((double)q.y)), kLn2);
                }
            }
        }
        __stcg(&prm.ell_ws[r], ell);
        float *outp = model == 0 ? prm.logp_tok : prm.logq_tok;
        if (outp) outp[pn * K + j] = (float)ell;
    }
    if (st) atomicOr(sh_st, st);
}

// S3 for particle n of prompt p: returns lam' (fp32); flags OR-ed into *st.
__device__ __forceinline__ float reweight_particle(const Params &prm, int p, int n, float neglogN,
                                                   uint32_t *st) {
    const int N = prm.N, K = prm.K;
    const int64_t pn = (int64_t)p * N + n;
    const int64_t rows = 2ll * N * K;
    const double *ellp = prm.ell_ws + (int64_t)p * rows + (int64_t)n * K;
    const double *ellq = ellp + (int64_t)N * K;
    int kn = drafted_len(prm, pn);
    bool bad = false;
    if (kn < 0 || kn > K) {
        *st |= ST_BAD_TOKEN;
        bad = true;
        kn = 0;
    }
    double delta = 0.0;
    for (int j = 0; j < kn; ++j) {
        const double lp = __ldcg(&ellp[j]), lq = __ldcg(&ellq[j]);
        if (isnan(lp) || isnan(lq)) {
            bad = true;                                      // flag already raised in S2
        } else if (lq == -INFINITY) {
            *st |= ST_NOT_ABSCONT;
            bad = true;
        } else {
            delta = __dadd_rn(delta, __dsub_rn(__dmul_rn(prm.alpha, lp), lq));
        }
    }
    const float prev = prm.logw_prev ? prm.logw_prev[pn] : neglogN;
    if (isnan(prev) || prev == INFINITY) {
        *st |= ST_NONFINITE;
        bad = true;
    }
    return bad ? -INFINITY : (float)__dadd_rn((double)prev, delta);
}

// S4-S7 for prompt p from lam[0..N) (smem).  All threads call.  resample_mode = false: S4 only.
__device__ void normalise_resample(const Params &prm, int p, bool resample_mode, TailSmem &sh) {
    const int N = prm.N, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)p * N;
    // ---- S4: M = max lam (order-free), e_n = exp(lam_n - M)
    float mloc = -INFINITY;
    for (int n = tid; n < N; n += kThreads) mloc = fmaxf(mloc, sh.lam[n]);
    mloc = warp_max(mloc);
    if (lane == 0) sh.fred[warp] = mloc;
    __syncthreads();
    if (tid == 0) {
        float M = sh.fred[0];
        for (int w = 1; w < kWarps; ++w) M = fmaxf(M, sh.fred[w]);
        sh.M = (double)M;
        sh.degenerate = M == -INFINITY;
    }
    __syncthreads();
    if (sh.degenerate) {
        for (int n = tid; n < N; n += kThreads) {
            if (prm.wnorm) prm.wnorm[base + n] = 0.0f;
            if (resample_mode) {
                prm.ancestors[base + n] = n;
                if (prm.offspring) prm.offspring[base + n] = 1;
                if (prm.slot_src) prm.slot_src[base + n] = n;
                prm.logw_out[base + n] = sh.lam[n];
            }
        }
        if (tid == 0) {
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
    for (int n = tid; n < N; n += kThreads) sh.e[n] = exp(__dsub_rn((double)sh.lam[n], sh.M));
    __syncthreads();
    if (tid == 0) {
        // sequential fp64 prefix and sum of squares (reading G6): same order as the oracle
        double acc = 0.0, sq = 0.0;
        for (int m = 0; m < N; ++m) {
            acc = __dadd_rn(acc, sh.e[m]);
            sh.C[m] = acc;
        }
        for (int m = 0; m < N; ++m) sq = __dadd_rn(sq, __dmul_rn(sh.e[m], sh.e[m]));
        const double S = acc;
        const double ess = __ddiv_rn(__dmul_rn(S, S), sq);
        sh.S = S;
        if (prm.lse) prm.lse[p] = __dadd_rn(sh.M, log(S));
        if (prm.ess) prm.ess[p] = ess;
        sh.do_res = resample_mode && ess < prm.eta;
        if (sh.do_res) {
            uint32_t x;
            if (prm.uniforms) {
                x = prm.uniforms[p];
            } else {
                const uint64_t g = (uint64_t)(prm.prompt_base + p);
                const uint4 r = philox4x32_10(
                    make_uint4((uint32_t)prm.step, (uint32_t)(prm.step >> 32), (uint32_t)g, 0u),
                    make_uint2((uint32_t)prm.seed, (uint32_t)(prm.seed >> 32)));
                x = r.x;
            }
            sh.U = (double)x * 2.3283064365386962890625e-10;   // 2^-32, exact
        }
        sh.ties = 0;
    }
    __syncthreads();
    const double S = sh.S;
    if (prm.wnorm)
        for (int n = tid; n < N; n += kThreads) prm.wnorm[base + n] = (float)__ddiv_rn(sh.e[n], S);
    if (!resample_mode) return;
    if (!sh.do_res) {
        for (int n = tid; n < N; n += kThreads) {
            prm.ancestors[base + n] = n;
            if (prm.offspring) prm.offspring[base + n] = 1;
            if (prm.slot_src) prm.slot_src[base + n] = n;
            prm.logw_out[base + n] = sh.lam[n];
        }
        if (tid == 0) {
            prm.resampled[p] = 0;
            if (prm.n_ties) prm.n_ties[p] = 0;
        }
        return;
    }
    // ---- S6: systematic ancestors by inverse CDF
    for (int m = tid; m < N; m += kThreads) {
        sh.C[m] = __ddiv_rn(sh.C[m], S);
        sh.o[m] = 0;
    }
    __syncthreads();
    const double U = sh.U;
    const double tie = 9.094947017729282379150390625e-13;     // 2^-40
    int ties = 0;
    for (int n = tid; n < N; n += kThreads) {
        const double u = __ddiv_rn(__dadd_rn((double)n, U), (double)N);
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
    if (ties) atomicAdd(&sh.ties, ties);
    __syncthreads();
    // ---- S7 reset and per-particle outputs
    const float reset = (float)(-log((double)N));
    for (int n = tid; n < N; n += kThreads) {
        if (prm.offspring) prm.offspring[base + n] = sh.o[n];
        prm.logw_out[base + n] = reset;
    }
    if (tid == 0) {
        prm.resampled[p] = 1;
        if (prm.n_ties) prm.n_ties[p] = sh.ties;
        if (prm.slot_src) {
            // in-place plan (G14): dead slots ascending <- extra copies, ascending source
            int32_t *plan = prm.slot_src + base;
            int src = 0, left = 0;
            for (int m = 0; m < N; ++m) {
                if (sh.o[m] != 0) {
                    plan[m] = m;
                    continue;
                }
                while (left == 0) {
                    if (sh.o[src] >= 2) left = sh.o[src] - 1;
                    if (left == 0) ++src;
                }
                plan[m] = src;
                if (--left == 0) ++src;
            }
        }
    }
}

// Whole tail for prompt p: S2, S3, then S4 (MODE_WEIGHTS) or S4-S7 (MODE_STEP).  N <= kTailMaxN.
__device__ void tail_prompt(const Params &prm, int p, bool resample_mode, TailSmem &sh) {
    const int N = prm.N, tid = threadIdx.x;
    if (tid == 0) sh.st = 0;
    __syncthreads();
    tail_rows(prm, p, &sh.st);
    __syncthreads();
    const float neglogN = (float)(-log((double)N));
    uint32_t st = 0;
    for (int n = tid; n < N; n += kThreads) {
        const float lam = reweight_particle(prm, p, n, neglogN, &st);
        sh.lam[n] = lam;
        const int64_t pn = (int64_t)p * N + n;
        if (prm.logw_pre) prm.logw_pre[pn] = lam;
        if (!resample_mode) prm.logw_out[pn] = lam;
    }
    if (st) atomicOr(&sh.st, st);
    __syncthreads();
    normalise_resample(prm, p, resample_mode, sh);
    __syncthreads();
    if (tid == 0) prm.status[p] = sh.st;
}

// ------------------------------------------------------------------------------------------
// K1 (+ fused tail).  grid = P * 2 * N * K * nseg, block = kThreads.
// ------------------------------------------------------------------------------------------
template <int DT, int MODE>
__global__ void __launch_bounds__(kThreads) k_rowstats(const __grid_constant__ Params prm) {
    __shared__ float2 red[kWarps];
    __shared__ int s_last;
    const int64_t item = blockIdx.x;
    const int seg = (int)(item % prm.nseg);
    const int64_t row = item / prm.nseg;                    // ((p*2 + model)*N + n)*K + j
    const int K = prm.K, N = prm.N;
    const int j = (int)(row % K);
    const int n = (int)((row / K) % N);
    const int model = (int)((row / ((int64_t)K * N)) % 2);
    const int p = (int)(row / (2ll * K * N));
    const int64_t pn = (int64_t)p * N + n;
    const int kn = drafted_len(prm, pn);
    if (kn >= 0 && kn <= K && j < kn) {
        const char *base = model == 0
            ? prm.lp + ((pn * prm.rpp_p + j) * prm.ld_p) * (DT == 1 ? 2 : 4)
            : prm.lq + ((pn * prm.rpp_q + j) * prm.ld_q) * (DT == 1 ? 2 : 4);
        const float c = model == 0 ? prm.c_p : prm.c_q;
        const int64_t d = prm.tokens[pn * K + j];
        const float4 r = segment_stats<DT>(base, prm.v_len, seg, c, d - prm.v_begin, red);
        if (threadIdx.x == 0) prm.part_ws[item] = r;
    } else if (threadIdx.x == 0) {
        prm.part_ws[item] = make_float4(-INFINITY, 0.0f, -INFINITY, 0.0f);
    }
    if constexpr (MODE == MODE_ROWS_ONLY) return;

    // ---- completion counting: the last CTA of prompt p runs its tail (threadFenceReduction)
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned total = (unsigned)(2ll * N * K * prm.nseg);
        const unsigned prev = atomicAdd(&prm.counters[p], 1u);
        s_last = prev == total - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    if constexpr (MODE == MODE_PARTIAL) {
        const int64_t rows = 2ll * N * K;
        for (int64_t rl = threadIdx.x; rl < rows; rl += kThreads) {
            const int64_t r = (int64_t)p * rows + rl;
            prm.partials_out[r] = merge_parts(prm.part_ws + r * prm.nseg, 1, prm.nseg);
        }
    } else {
        __shared__ TailSmem sh;
        tail_prompt(prm, p, MODE == MODE_STEP, sh);
    }
    if (threadIdx.x == 0) prm.counters[p] = 0u;             // graph-replay safe
}

// Tail-only kernel, grid = P: S2-S7 from prm.parts (combine path, N <= kTailMaxN).
__global__ void __launch_bounds__(kThreads) k_tail(const __grid_constant__ Params prm, int resample_mode) {
    __shared__ TailSmem sh;
    tail_prompt(prm, blockIdx.x, resample_mode != 0, sh);
}

// S4-S7 from fp32 log-weights, grid = P (smcsd_resample).
__global__ void __launch_bounds__(kThreads) k_resample(const __grid_constant__ Params prm) {
    __shared__ TailSmem sh;
    const int p = blockIdx.x, N = prm.N;
    if (threadIdx.x == 0) sh.st = 0;
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
}

// Large-N weights path (N > kTailMaxN): S2+S3 in parallel, S4 serial over global workspace.
__global__ void __launch_bounds__(kThreads) k_tail_large(const __grid_constant__ Params prm) {
    __shared__ uint32_t s_st;
    __shared__ float s_red[kWarps];
    __shared__ double s_M, s_S;
    const int p = blockIdx.x, N = prm.N, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = (int64_t)p * N;
    if (tid == 0) s_st = 0;
    __syncthreads();
    tail_rows(prm, p, &s_st);
    __syncthreads();
    const float neglogN = (float)(-log((double)N));
    uint32_t st = 0;
    float mloc = -INFINITY;
    for (int n = tid; n < N; n += kThreads) {
        const float lam = reweight_particle(prm, p, n, neglogN, &st);
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
        for (int m = 0; m < N; ++m) acc = __dadd_rn(acc, __ldcg(&prm.e_ws[base + m]));
        for (int m = 0; m < N; ++m) {
            const double e = __ldcg(&prm.e_ws[base + m]);
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

// ------------------------------------------------------------------------------------------
// K3: S8/S9 source-major block gather.  grid = n_outer * P * nchunks, block = kThreads.
// ------------------------------------------------------------------------------------------
constexpr int kKvUnroll = 4;
constexpr int kKvChunkVec = kThreads * kKvUnroll;             // 16-byte vectors per CTA chunk

struct KvParams {
    char *dst;
    const char *src;
    int64_t outer_stride, prompt_stride, particle_stride, seg_stride;
    uint32_t vps;                 // 16-byte vectors per segment
    uint64_t vecs;                // vectors per block = seg_count * vps
    int64_t nchunks;
    const int32_t *idx;
    int P, N, in_place;
};

__global__ void __launch_bounds__(kThreads) k_kv_reindex(const __grid_constant__ KvParams prm) {
    __shared__ int cnt[kTailMaxN], start[kTailMaxN], fill[kTailMaxN], dsts[kTailMaxN], srcs[kTailMaxN];
    __shared__ int wtot[kWarps + 1];
    const int tid = threadIdx.x, N = prm.N;
    const int64_t item = blockIdx.x;
    const int64_t chunk = item % prm.nchunks;
    const int64_t op = item / prm.nchunks;
    const int p = (int)(op % prm.P);
    const int64_t o = op / prm.P;
    const int32_t *idx = prm.idx + (int64_t)p * N;

    // ---- copy plan for prompt p: destinations grouped by source (counting sort)
    for (int n = tid; n < N; n += kThreads) cnt[n] = 0;
    __syncthreads();
    for (int n = tid; n < N; n += kThreads) {
        const int s = idx[n];
        if ((unsigned)s < (unsigned)N && (!prm.in_place || s != n)) atomicAdd(&cnt[s], 1);
    }
    __syncthreads();
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
        if ((unsigned)s < (unsigned)N && (!prm.in_place || s != n))
            dsts[start[s] + atomicAdd(&fill[s], 1)] = n;
    }
    __syncthreads();

    // ---- byte offsets of this thread's vectors inside a block
    int64_t voff[kKvUnroll];
    bool valid[kKvUnroll];
#pragma unroll
    for (int i = 0; i < kKvUnroll; ++i) {
        const uint64_t v = (uint64_t)chunk * kKvChunkVec + (uint64_t)i * kThreads + tid;
        valid[i] = v < prm.vecs;
        const uint64_t g = v / prm.vps, w = v - g * prm.vps;
        voff[i] = (int64_t)g * prm.seg_stride + (int64_t)w * 16;
    }
    const int64_t pbase = o * prm.outer_stride + (int64_t)p * prm.prompt_stride;
    for (int k = 0; k < nsrc; ++k) {
        const int s = srcs[k];
        const char *sb = prm.src + pbase + (int64_t)s * prm.particle_stride;
        uint4 r[kKvUnroll];
#pragma unroll
        for (int i = 0; i < kKvUnroll; ++i)
            if (valid[i]) r[i] = ld_stream(sb + voff[i]);
        const int c = cnt[s], st0 = start[s];
        for (int q = 0; q < c; ++q) {
            char *db = prm.dst + pbase + (int64_t)dsts[st0 + q] * prm.particle_stride;
#pragma unroll
            for (int i = 0; i < kKvUnroll; ++i)
                if (valid[i]) st_stream(db + voff[i], r[i]);
        }
    }
}

}  // namespace smcsd
