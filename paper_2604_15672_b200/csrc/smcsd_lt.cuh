// smcsd_lt.cuh -- the latency tail (LT) of small steps: S2-S7 by one CTA per prompt that runs
// BESIDE K1 instead of after it.
//
// Why: a single-prompt step (cfg2: 64 MB of logits, ~15 us of K1) is latency-bound after K1.
// The two-kernel path (K1 -> k_tail) waits for K1's grid to complete and flush (~1 us), then
// runs S2 (one dependent L2 round trip), the terms, a cluster barrier, S3 and a one-shot S4-S7
// whose code is fetched cold (profiles/r02b_trace_step.txt: ~8 us after K1's last CTA).
//
// How: K1 (LT mode, prm.lt_words != null) triggers its dependents right after its own
// griddepcontrol.wait, so k_lt becomes resident next to K1's streaming CTAs (128 threads,
// <= 80 registers, ~13 KB of shared memory: it fits beside K1's 6 CTAs per SM).  K1 publishes
// each (row, segment) item {m, s} as ONE 8-byte relaxed gpu-scope store into lt_words (a
// zeroed array; a written word is never zero: m finite => s >= 1, an empty segment is
// {-inf, 0}), so the data is its own flag -- no fence, counter or grid completion on the path.
// k_lt reads its inputs (tokens, t_d from the logits, logw_prev, the Philox uniforms) while K1
// streams, then walks its prompt's rows in item order, one row per thread, 128 rows per pass
// (k_tail's exact 4-lane merge order, so every output is bit-identical to the two-kernel path):
// it polls the row's words (ld.relaxed.gpu), zeroes them for the next step, merges, takes ell
// and -- as soon as a particle's draft rows are in -- its S3 sum.  Only the last pass, the last
// particles' S3 and S4-S7 remain when K1's last item lands.  S4-S7 is warp_tail
// (smcsd_warp_tail.cuh, lane per particle, two warps); with -DSMCSD_LT_DRY it also runs once
// "dry" at the start (same code, stores off) as an instruction warm-up.  At its exit k_lt waits for K1's grid (long finished by then) and re-arms
// K1's work counter.
//
// Readings: every arithmetic step is k_tail's (S2 4-lane merge, ell, terms, S3 in j order,
// S4 sequential fp64 prefix in particle order (G6), systematic / multinomial ancestors
// a_n = #{m : C_m <= u_n}, the tie count = #{m : |u_n - C_m| <= 2^-40} (G7), the slot plan
// (G14), S7 reset); PAPER.md:316-331 (Alg. 1), PAPER.md:116 (Eq. 1a).
#pragma once
#include "smcsd_kernels.cuh"

namespace smcsd {

constexpr int kLtThreads = 128;
constexpr int kLtMaxN = 32;            // lane per particle in S4-S7
constexpr int kLtMaxRows = 1024;       // 2 N K
constexpr int kLtMaxParts = 16;        // segments per row (V <= 131072): one row per thread
#ifndef SMCSD_LT_MAXP
#define SMCSD_LT_MAXP 148
#endif
constexpr int kLtMaxP = SMCSD_LT_MAXP; // prompts per call (one CTA each, one per SM beside K1)

struct LtSmem {
    WtSmem w;                          // S4-S7 (smcsd_warp_tail.cuh)
    double ell[kLtMaxRows];            // ell of every row (target rows, then draft rows)
    double term[kLtMaxRows / 2];       // S3 terms, [j][n]
    float x[kLtMaxRows];               // t_d = inv_temp z_d log2(e) (-inf: row not read)
    uint8_t code[kLtMaxRows];          // 0 valid row, 1 not read (j >= k_n or bad k_n), 2 bad token
    float lam[kLtMaxN];                // lam' after S3
    float prev[kLtMaxN];               // logw_prev
    int kn[kLtMaxN];                   // k_n
    uint32_t st;                       // status bits of the prompt
};

__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const void *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Wait until every part word of a row is written (nonzero); returns true on timeout (kXTimeoutNs:
// the missing parts become neutral {-inf, 0} and the caller raises ST_EXCHANGE).
__device__ __forceinline__ bool lt_poll_row(const unsigned long long *w0, int64_t seg_stride, int nparts,
                                            unsigned long long (&w)[kLtMaxParts]) {
    bool pending = false;
#pragma unroll
    for (int i = 0; i < kLtMaxParts; ++i) {
        w[i] = i < nparts ? ld_relaxed_gpu_u64(w0 + i * seg_stride) : 0x00000000FF800000ull;
        pending |= w[i] == 0ull;
    }
    if (!pending) return false;
    const uint64_t t0 = globaltimer_ns();
    for (;;) {
        pending = false;
#pragma unroll
        for (int i = 0; i < kLtMaxParts; ++i) {
            if (w[i] == 0ull) {
                w[i] = ld_relaxed_gpu_u64(w0 + i * seg_stride);
                pending |= w[i] == 0ull;
            }
        }
        if (!pending) return false;
        if (globaltimer_ns() - t0 > kXTimeoutNs) {
#pragma unroll
            for (int i = 0; i < kLtMaxParts; ++i)
                if (w[i] == 0ull) w[i] = 0x00000000FF800000ull;
            return true;
        }
    }
}

// S2 of one row from its (<= 16) part words, bit-identical to k_tail's 4-lane merge: "lane" l
// takes parts 4l .. 4l+3 (max, then the fma sum in part order); the lanes combine as k_tail's
// xor-2 / xor-1 butterfly does: M = max of all, S = (S0' + S2') + (S1' + S3') with
// Sl' = Sl 2^(Ml - M).  Parts >= nparts are neutral {-inf, 0} and change nothing.
__device__ __forceinline__ void lt_merge_row(const unsigned long long (&w)[kLtMaxParts], float &Mo, float &So) {
    float Ml[4], Sl[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < 4; ++k) m = fmaxf(m, __uint_as_float((uint32_t)w[4 * l + k]));
        float sacc = 0.0f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float pm = __uint_as_float((uint32_t)w[4 * l + k]), ps = __uint_as_float((uint32_t)(w[4 * l + k] >> 32));
            sacc = __fmaf_rn(ps, pm == m ? 1.0f : ex2_approx(pm - m), sacc);
        }
        Ml[l] = m;
        Sl[l] = sacc;
    }
    const float M = fmaxf(fmaxf(Ml[0], Ml[2]), fmaxf(Ml[1], Ml[3]));
    float Sp[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) Sp[l] = __fmul_rn(Sl[l], Ml[l] == M ? 1.0f : ex2_approx(Ml[l] - M));
    Mo = M;
    So = __fadd_rn(__fadd_rn(Sp[0], Sp[2]), __fadd_rn(Sp[1], Sp[3]));
}

// grid = P (one CTA per prompt), block = kLtThreads, launched with PDL right behind K1 (LT mode).
__global__ void __launch_bounds__(kLtThreads, 8) k_lt(const __grid_constant__ Params prm, int resample_mode) {
    constexpr int kRowsPerThread = kLtMaxRows / kLtThreads;
    __shared__ __align__(16) LtSmem ls;
    const int tid = threadIdx.x, lane = tid & 31;
    const int p = blockIdx.x;
    const int N = prm.N, K = prm.K, NK = N * K, rows = 2 * NK, nparts = prm.nseg;
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2400);                // resident
    // ---- inputs (complete before K1 passed its griddepcontrol.wait, i.e. before this launch).
    // Memory is saturated by K1's stream now, so every load is issued before any is used:
    // k_n and the token of each of this thread's rows (r = tid + 128 i), then t_d from the logits.
    if (tid == 0) {
        ls.st = 0u;
        ls.w.a = WtArgs{prm.logw_out, prm.wnorm, prm.lse, prm.ess, prm.ancestors, prm.offspring,
                        prm.slot_src, prm.n_ties, prm.resampled, prm.eta, prm.N, prm.scheme};
        ls.w.st = 0u;
    }
    if (tid < N) {                                               // read by S3 (after a barrier)
        const int64_t pn = (int64_t)p * N + tid;
        ls.kn[tid] = prm.n_drafted ? __ldcg(prm.n_drafted + pn) : K;
        ls.prev[tid] = prm.logw_prev ? __ldcg(prm.logw_prev + pn) : (float)(-log((double)N));
    }
    {
        int kn_r[kRowsPerThread];
        int64_t d_r[kRowsPerThread];
#pragma unroll
        for (int i = 0; i < kRowsPerThread; ++i) {
            const int r = tid + kLtThreads * i;
            kn_r[i] = -1;
            d_r[i] = -1;
            if (r < rows) {
                const int model = r >= NK, q = r - model * NK, n = q / K, j = q - n * K;
                const int64_t pn = (int64_t)p * N + n;
                kn_r[i] = prm.n_drafted ? __ldcg(prm.n_drafted + pn) : K;
                d_r[i] = __ldcg(prm.tokens + pn * K + j);
            }
        }
        float x_r[kRowsPerThread];
#pragma unroll
        for (int i = 0; i < kRowsPerThread; ++i) {
            const int r = tid + kLtThreads * i;
            x_r[i] = -INFINITY;
            if (r < rows) {
                const int model = r >= NK, q = r - model * NK, n = q / K, j = q - n * K;
                const int kn = kn_r[i];
                const int64_t d = d_r[i];
                uint8_t code = 1;
                if (kn >= 0 && kn <= K && j < kn) {
                    if (d < 0 || d >= prm.V) {
                        code = 2;
                    } else {
                        code = 0;
                        x_r[i] = load_x(prm, model, (int64_t)p * N + n, j, d);
                    }
                }
                ls.code[r] = code;
            }
        }
#pragma unroll
        for (int i = 0; i < kRowsPerThread; ++i)
            if (tid + kLtThreads * i < rows) ls.x[tid + kLtThreads * i] = x_r[i];   // own rows only
    }
    // this lane's uniform (weight-independent, k_tail's tail_uniform) and fl32(-ln N)
    const double u = tid < 32 && resample_mode ? tail_uniform(prm, p, lane) : 0.0;
    const float reset = (float)(-log((double)N));
#ifdef SMCSD_LT_DRY
    __syncthreads();
    if (tid < 64) warp_tail<1>(tid >> 5, p, 1, 1, ls.lam, u, 0.0, reset, ls.w);   // instruction warm-up, no stores
#endif
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2401);                // inputs (+ warm-up) done

    // ---- S2 + ell, one row per thread, kLtThreads rows per pass in item order (target rows,
    // then draft rows).  A draft row's thread also forms the pair's S3 term when the target
    // row was in an earlier pass (else right after this pass's barrier).  S3 for each particle
    // once its draft rows are in.
    // K1's words are segment-major: part i of global row g at lt_words[i * total_rows + g]
    const int64_t total_rows = (int64_t)prm.P * rows;
    unsigned long long *words = prm.lt_words + (int64_t)p * rows;
    uint32_t st = 0;
    bool late = false;
    int n_done = 0;
    for (int r0 = 0; r0 < rows; r0 += kLtThreads) {
        const int r = r0 + tid;
        bool defer = false;
        double ell = 0.0;
        int term_at = -1;                                       // term_s index of this row's pair
        if (r < rows) {
            unsigned long long w[kLtMaxParts];
#ifdef SMCSD_TRACE
            if (p == 0 && r == rows - 1) g_trace[2490] = clock64();
#endif
            late |= lt_poll_row(words + r, total_rows, nparts, w);
#ifdef SMCSD_TRACE
            if (p == 0 && r == rows - 1) g_trace[2491] = clock64();
#endif
#pragma unroll
            for (int i = 0; i < kLtMaxParts; ++i)
                if (i < nparts) __stcg(words + i * total_rows + r, 0ull);   // zero for the next step
            float M, S;
            lt_merge_row(w, M, S);
            const int code = ls.code[r];
            if (code == 1) {
                ell = 0.0;
            } else if (code == 2) {
                st |= ST_BAD_TOKEN;
                ell = qnan;
            } else if (!isfinite(M) || !isfinite(S)) {
                st |= ST_NONFINITE;
                ell = qnan;
            } else {
                // ell = (x - m - log2 s) * ln 2  (natural log of the softmax at d); s in [1, V]
                ell = __dmul_rn(__dsub_rn(__dsub_rn((double)ls.x[r], (double)M), (double)log2f(S)), kLn2);
            }
            ls.ell[r] = ell;
            const int model = r >= NK, q = r - model * NK;
            float *outp = model == 0 ? prm.logp_tok : prm.logq_tok;
            if (outp) outp[(int64_t)p * NK + q] = (float)ell;
            if (model == 1 && code != 1) {                      // a pair S3 sums (j < k_n)
                const int n = q / K, j = q - n * K;
                term_at = j * N + n;                            // [j][n]: S3 reads conflict-free
                defer = q >= r0;                                // target row in this pass
            }
#ifdef SMCSD_TRACE
            if (p == 0 && r == rows - 1) g_trace[2492] = clock64();
#endif
        }
        // S3 term of a pair: alpha ell^p - ell^q (NaN marks an invalid pair; flag raised above)
        auto term_of = [&](double lp, double lq) {
            if (isnan(lp) || isnan(lq)) return qnan;
            if (lq == -INFINITY) {
                st |= ST_NOT_ABSCONT;
                return qnan;
            }
            return __dsub_rn(__dmul_rn(prm.alpha, lp), lq);
        };
        if (term_at >= 0 && !defer) ls.term[term_at] = term_of(ls.ell[r - NK], ell);
        __syncthreads();
        if (r0 + NK < min(r0 + kLtThreads, rows)) {             // some pair had both rows here
            if (defer) ls.term[term_at] = term_of(ls.ell[r - NK], ell);
            __syncthreads();
        }
#ifdef SMCSD_TRACE
        if (tid == 0 && p == 0 && r0 + kLtThreads >= rows) g_trace[2493] = clock64();
#endif
        // S3 for the particles whose K draft rows are all in: lam' = fl32(prev + sum_j term_j)
        const int rows_done = min(rows, r0 + kLtThreads);
        const int n_ready = rows_done > NK ? min(N, (rows_done - NK) / K) : 0;
        if (tid >= n_done && tid < n_ready) {
            const int n = tid;
            const int64_t pn = (int64_t)p * N + n;
            int kn = ls.kn[n];
            bool bad = false;
            uint32_t st3 = 0;
            if (kn < 0 || kn > K) {
                st3 |= ST_BAD_TOKEN;
                bad = true;
                kn = 0;
            }
            double delta = 0.0;
            for (int j = 0; j < kn; ++j) delta = __dadd_rn(delta, ls.term[j * N + n]);
            if (isnan(delta)) bad = true;                      // an invalid pair (flag raised in S2)
            const float prev = ls.prev[n];
            if (isnan(prev) || prev == INFINITY) {
                st3 |= ST_NONFINITE;
                bad = true;
            }
            const float lam = bad ? -INFINITY : (float)__dadd_rn((double)prev, delta);
            ls.lam[n] = lam;
            if (prm.logw_pre) prm.logw_pre[pn] = lam;
            if (!resample_mode) prm.logw_out[pn] = lam;
            st |= st3;
        }
        n_done = n_ready;
#ifdef SMCSD_TRACE
        if (tid == 0 && p == 0 && r0 / kLtThreads < 64) g_trace[2410 + r0 / kLtThreads] = gtimer();
#endif
    }
    if (late) st |= ST_EXCHANGE;
    if (st) atomicOr(&ls.st, st);
    __syncthreads();
    if (tid == 0 && p == 0) { SMCSD_TRACE_AT(2402); SMCSD_CLK_AT(2494); }   // S2 + S3 done
    if (tid < 64) warp_tail<1>(tid >> 5, p, resample_mode, 0, ls.lam, u, 0.0, reset, ls.w);
    __syncthreads();
    if (tid == 0) prm.status[p] = ls.st | ls.w.st;
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2403);                // S4-S7 done
    if (tid == 0) {
        // K1's grid is complete (its last items are long consumed): re-arm its work counter;
        // after a timeout, clear words a late K1 item may have written since
        pdl_wait();
        if (p == 0) *prm.work_ctr = 0u;
    }
    if (__syncthreads_or(late)) {
        for (int i = tid; i < rows * nparts; i += kLtThreads) words[(i / rows) * total_rows + i % rows] = 0ull;
    }
}

}  // namespace smcsd
