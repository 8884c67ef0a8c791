// smcsd_tail_small.cuh -- k_tail_small: the polling cluster tail of small steps sized to run
// BESIDE K1 (S2-S7 of smcsd_step / smcsd_weights when the polling tail applies, N <= 32).
//
// k_tail's chunk CTAs (256 threads, 64 registers, 38 KB of shared memory) cannot be resident
// next to K1's six 288-thread CTAs per SM, so they start only as K1's CTAs exit and run their
// one-shot code cold after K1's last item.  k_tail_small is the same computation in CTAs that
// fit in what K1 leaves free on an SM (128 threads at <= 64 registers: one warp per SM
// sub-partition; ~7 KB of shared memory): 16 (particle, position) pairs per CTA with 4 lanes per
// row, or 32 with 2 lanes per row for N K up to 512, a prompt's CTAs one thread-block cluster
// (<= 16), N <= 64.  S3 runs in the chunk CTAs when K divides 16, else in
// the finisher from the terms the chunks push to it.  K1 launches it at once (polling tail), so its CTAs
// are resident from the start of K1's stream: they read their inputs while K1 runs, poll K1's
// {m, s} words once K1's work counter shows every item claimed, and the finishing CTA runs
// S4-S7 (warp_tail) once every chunk has pushed its lam' over DSMEM.
//
// Arithmetic and order are k_tail's (so the outputs are bit-identical): S2 4-lane merge of a
// row's 16 parts (lane l4: parts 4 l4 .. 4 l4 + 3, then the xor-2 / xor-1 butterfly), ell =
// (x - m - log2 s) ln 2, term = alpha ell^p - ell^q, S3 in j order, S4-S7 warp_tail.
// PAPER.md:316-331 (Alg. 1), PAPER.md:116 (Eq. 1a).
#pragma once
#include "smcsd_kernels.cuh"

namespace smcsd {

constexpr int kTsThreads = 128;
constexpr int kTsMaxChunks = 16;              // CTAs per prompt (one cluster, non-portable size)
constexpr int kTsMaxPairs = 32 * kTsMaxChunks;
constexpr int kTsMaxN = 64;                   // warp_tail<2>

// LPR = lanes per row: 4 (16 pairs = 32 rows per CTA, N K <= 256) or 2 (32 pairs = 64 rows per
// CTA, N K <= 512).  With 2 lanes each lane merges the parts of two of the 4 "virtual" lanes
// (l and l + 2) and the lanes combine exactly as the 4-lane butterfly does: bit-identical.
// grid = P x chunks (cluster = chunks <= 16, N <= 64), block = kTsThreads.
// H = particles per lane in S4-S7: 1 (N <= 32) or 2 (N <= 64), one warp_tail instance per kernel.
template <int LPR, int H>
__global__ void __launch_bounds__(kTsThreads, 8) k_tail_small(const __grid_constant__ Params prm, int resample_mode,
                                                           int chunks) {
    constexpr int kTsPairs = kTsThreads / (2 * LPR);
    __shared__ float4 rs[2 * kTsPairs];
    __shared__ double term_s[kTsPairs];
    __shared__ float s_lam[kTsMaxN];                            // finisher: every particle's lam'
    __shared__ double s_term[kTsMaxPairs];                      // finisher (S3 there): every pair's term
    __shared__ uint32_t s_flags[16];                            // finisher: every chunk's status bits
    __shared__ __align__(16) WtSmem wts;
    const int tid = threadIdx.x, lane = tid & 31;
    const int N = prm.N, K = prm.K, NK = N * K, rows = 2 * NK;
    const int p = blockIdx.x / chunks, c = blockIdx.x - p * chunks;
    const int q0 = c * kTsPairs, nq = min(kTsPairs, NK - q0);
    // finishing CTA: the last chunk, whose rows are K1's last items (its barrier wait is short;
    // chunk 0 measured 0.1 us slower, and an instruction warm-up of S4-S7 by the finisher's
    // warps -- before its rows arrive or while it waits at the barrier -- 0.5-0.9 us slower:
    // profiles/r02c_ab_tail_small.txt)
    const unsigned fin = (unsigned)(chunks - 1);
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    unsigned crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    // phase 1 of the cluster barrier: DSMEM may be written once every CTA has started
    asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
    if (tid == 0 && blockIdx.x == 0) SMCSD_TRACE_AT(2048);      // resident

    // ---- inputs (complete before K1 launched this grid): pair lane q of warp 0 holds both
    // rows of its pair -- k_n, the token, t_d of the target and the draft row -- and, at j = 0,
    // the particle's lam_prev; warp 0 of the finisher the particles' uniforms
    int kn = 0, j = 0;
    int64_t pn = 0, d = -1;
    float xp = -INFINITY, xq = -INFINITY, prev = 0.0f;
    if (tid < nq) {
        const int q = q0 + tid, n = q / K;
        j = q - n * K;
        pn = (int64_t)p * N + n;
        kn = drafted_len(prm, pn);
        d = prm.tokens[pn * K + j];
        if (kn >= 0 && kn <= K && j < kn && d >= 0 && d < prm.V) {
            xp = load_x(prm, 0, pn, j, d);
            xq = load_x(prm, 1, pn, j, d);
        }
        if (j == 0) prev = prm.logw_prev ? prm.logw_prev[pn] : (float)(-log((double)N));
    }
    // S3 runs in the chunk when whole particles fit in it (K divides 16); otherwise the chunks
    // push their terms to the finisher, whose warp 0 (lane n = particle n) sums them
    const bool s3_fin = (kTsPairs % K) != 0;                    // uniform
    int kn_f0 = 0, kn_f1 = 0;
    float prev_f0 = 0.0f, prev_f1 = 0.0f;
    if (s3_fin && crank == fin && tid < 32) {
        const float nl = (float)(-log((double)N));
        const int64_t pf = (int64_t)p * N + tid;
        if (tid < N) {
            kn_f0 = drafted_len(prm, pf);
            prev_f0 = prm.logw_prev ? prm.logw_prev[pf] : nl;
        }
        if (H == 2 && tid + 32 < N) {
            kn_f1 = drafted_len(prm, pf + 32);
            prev_f1 = prm.logw_prev ? prm.logw_prev[pf + 32] : nl;
        }
    }
    double u0 = 0.0, u1 = 0.0;
    float reset = 0.0f;
    if (crank == fin && tid < 64) {
        if (tid == 0) {
            wts.a = WtArgs{prm.logw_out, prm.wnorm, prm.lse, prm.ess, prm.ancestors, prm.offspring,
                           prm.slot_src, prm.n_ties, prm.resampled, prm.eta, prm.N, prm.scheme};
            wts.st = 0u;
        }
        if (resample_mode && tid < 32) {
            u0 = tail_uniform(prm, p, lane);
            if (H == 2) u1 = tail_uniform(prm, p, lane + 32);
        }
        reset = (float)(-log((double)N));
    }

    // ---- gate: one thread watches K1's work counter (sleeping ~1 us between reads) until every
    // K1 item is claimed; only then do the CTA's lanes poll their words.  Polls in flight beside
    // K1's stream slow it (profiles/r02j_ab_poll_shape_rejected.txt); the gate took cfg2 -0.1 us
    // and N = 64 -0.3 us (profiles/r02j_ab_tail_small_gate.txt).  Bounded like the polls.
    if (tid == 0 && prm.work_ctr) {
        const uint64_t g0 = globaltimer_ns();
        while (*reinterpret_cast<volatile unsigned *>(prm.work_ctr) < prm.gate_ctr && globaltimer_ns() - g0 < kXTimeoutNs)
            __nanosleep(1000);
    }
    __syncthreads();
    // ---- S2: 4 lanes per row, 32 rows (16 target, 16 draft), polling K1's words
    bool late = false;
    {
        // lane li of a row merges virtual lanes v = li + LPR g (g < 4 / LPR): parts 4v .. 4v + 3
        constexpr int kV = 4 / LPR;
        const int li = tid & (LPR - 1), lr = tid / LPR, qq = lr & (kTsPairs - 1);
        float Mv[kV], Sv[kV];
#pragma unroll
        for (int g = 0; g < kV; ++g) {
            Mv[g] = -INFINITY;
            Sv[g] = 0.0f;
        }
        if (qq < nq) {
            const int64_t grow = (int64_t)p * rows + (int64_t)(lr / kTsPairs) * NK + q0 + qq;
            float4 t[4 * kV];
            late = lt_take<kV>(prm.lt_words, 2ll * prm.P * NK, grow, 4 * li, 4 * LPR, prm.nparts, t);
#pragma unroll
            for (int g = 0; g < kV; ++g) {
#pragma unroll
                for (int k = 0; k < 4; ++k) Mv[g] = fmaxf(Mv[g], t[4 * g + k].x);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    Sv[g] = __fmaf_rn(t[4 * g + k].y, t[4 * g + k].x == Mv[g] ? 1.0f : ex2_approx(t[4 * g + k].x - Mv[g]), Sv[g]);
            }
        }
        // the 4-lane butterfly: M = max of all; S = (S0' + S2') + (S1' + S3'), Sv' = Sv 2^(Mv - M)
        float M = kV == 2 ? fmaxf(Mv[0], Mv[kV - 1]) : fmaxf(Mv[0], __shfl_xor_sync(0xffffffffu, Mv[0], 2));
        M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
        float S;
        if (kV == 2) {
            S = __fadd_rn(__fmul_rn(Sv[0], Mv[0] == M ? 1.0f : ex2_approx(Mv[0] - M)),
                          __fmul_rn(Sv[kV - 1], Mv[kV - 1] == M ? 1.0f : ex2_approx(Mv[kV - 1] - M)));
        } else {
            S = __fmul_rn(Sv[0], Mv[0] == M ? 1.0f : ex2_approx(Mv[0] - M));
            S = __fadd_rn(S, __shfl_xor_sync(0xffffffffu, S, 2));
        }
        S = __fadd_rn(S, __shfl_xor_sync(0xffffffffu, S, 1));
        if (li == 0) rs[lr] = make_float4(M, S, -INFINITY, 0.0f);
    }
    const int any_late = __syncthreads_or(late);
    if (tid == 0 && blockIdx.x == 0) SMCSD_TRACE_AT(2053);      // chunk 0 S2 done
    if (tid == 0 && p == 0 && crank == fin) SMCSD_TRACE_AT(2054);   // finisher: its rows merged
    asm volatile("barrier.cluster.wait;" ::: "memory");         // phase 1 complete

    // ---- ell of both rows, the S3 term, S3 of whole particles (warp 0, lane = pair)
    double ellp = 0.0, ellq = 0.0;
    float lam = 0.0f;
    if (tid < 32) {
        uint32_t st = tid == 0 && any_late ? ST_EXCHANGE : 0u;
        double term = 0.0;
        if (tid < nq) {
            const bool valid = kn >= 0 && kn <= K && j < kn;
            double e2[2];
#pragma unroll
            for (int mdl = 0; mdl < 2; ++mdl) {
                const float4 m = rs[mdl * kTsPairs + tid];
                double ell;
                if (!valid) {
                    ell = 0.0;
                } else if (d < 0 || d >= prm.V) {
                    st |= ST_BAD_TOKEN;
                    ell = qnan;
                } else if (!isfinite(m.x) || !isfinite(m.y)) {
                    st |= ST_NONFINITE;
                    ell = qnan;
                } else {
                    ell = __dmul_rn(__dsub_rn(__dsub_rn((double)(mdl ? xq : xp), (double)m.x), (double)log2f(m.y)), kLn2);
                }
                e2[mdl] = ell;
            }
            ellp = e2[0];
            ellq = e2[1];
            if (valid) {
                if (isnan(ellp) || isnan(ellq)) {
                    term = qnan;
                } else if (ellq == -INFINITY) {
                    st |= ST_NOT_ABSCONT;
                    term = qnan;
                } else {
                    term = __dsub_rn(__dmul_rn(prm.alpha, ellp), ellq);
                }
            }
            if (s3_fin) st_cluster_f64(&s_term[q0 + tid], fin, term);
            else term_s[tid] = term;
        }
        __syncwarp();
        if (!s3_fin && tid < nq && j == 0) {
            // S3: lam' = fl32(prev + sum_{j < k_n} term_j) in j order
            int kk = kn;
            bool bad = false;
            if (kk < 0 || kk > K) {
                st |= ST_BAD_TOKEN;
                bad = true;
                kk = 0;
            }
            double delta = 0.0;
            for (int jj = 0; jj < kk; ++jj) delta = __dadd_rn(delta, term_s[tid + jj]);
            if (isnan(delta)) bad = true;
            if (isnan(prev) || prev == INFINITY) {
                st |= ST_NONFINITE;
                bad = true;
            }
            lam = bad ? -INFINITY : (float)__dadd_rn((double)prev, delta);
            st_cluster_f32(&s_lam[(q0 + tid) / K], fin, lam);
        }
        st = __reduce_or_sync(0xffffffffu, st);
        if (tid == 0) st_cluster_u32(&s_flags[crank], fin, st);
        if (tid == 0 && p == 0 && crank == fin) SMCSD_TRACE_AT(2055);   // finisher: its S3 done
    }
    // ---- completion: the cluster barrier (release / acquire at cluster scope) hands every
    // chunk's lam' and bits to the finisher; this chunk's output stores go after the arrive
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
    if (tid < nq) {
        if (prm.logp_tok) prm.logp_tok[pn * K + j] = (float)ellp;
        if (prm.logq_tok) prm.logq_tok[pn * K + j] = (float)ellq;
        if (j == 0 && !s3_fin) {
            if (prm.logw_pre) prm.logw_pre[pn] = lam;
            if (!resample_mode) prm.logw_out[pn] = lam;
        }
    }
    asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
    if (crank != fin) {
        x_tail_rearm(prm);
        pdl_trigger();
        return;
    }
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2050);               // finisher past the barrier
#ifndef SMCSD_TS_LATE_TRIGGER
    // The next kernel (the next step's K1, or the KV reindex) may launch now: its CTAs set up
    // beside this one while S4-S7 runs, and its griddepcontrol.wait still waits for this grid.
    pdl_trigger();
#endif
    uint32_t f = 0;
    if (tid == 64)
        for (int r = 0; r < chunks; ++r) f |= s_flags[r];
    if (s3_fin) {
        // S3 here: lam'_n = fl32(prev_n + sum_{j < k_n} term_{nK + j}) in j order
        if (tid < 32) {
            uint32_t st3 = 0;
            auto s3 = [&](int n, int kk, float pv) {
                bool bad = false;
                if (kk < 0 || kk > K) {
                    st3 |= ST_BAD_TOKEN;
                    bad = true;
                    kk = 0;
                }
                double delta = 0.0;
                for (int jj = 0; jj < kk; ++jj) delta = __dadd_rn(delta, s_term[n * K + jj]);
                if (isnan(delta)) bad = true;
                if (isnan(pv) || pv == INFINITY) {
                    st3 |= ST_NONFINITE;
                    bad = true;
                }
                const float lm = bad ? -INFINITY : (float)__dadd_rn((double)pv, delta);
                s_lam[n] = lm;
                const int64_t pf = (int64_t)p * N + n;
                if (prm.logw_pre) prm.logw_pre[pf] = lm;
                if (!resample_mode) prm.logw_out[pf] = lm;
            };
            if (tid < N) s3(tid, kn_f0, prev_f0);
            if (H == 2 && tid + 32 < N) s3(tid + 32, kn_f1, prev_f1);
            st3 = __reduce_or_sync(0xffffffffu, st3);
            if (tid == 0 && st3) wts.st |= st3;                 // (role 1 sets only ST_DEGENERATE, later)
        }
        if (tid < 64) asm volatile("bar.sync 1, 64;" ::: "memory");     // s_lam for warp 1
    }
    if (tid < 64) warp_tail<H>(tid >> 5, p, resample_mode, 0, s_lam, u0, u1, reset, wts);
    __syncthreads();
    if (tid == 64) prm.status[p] = f | wts.st;
    if (tid == 0 && p == 0) SMCSD_TRACE_AT(2052);               // S4-S7 done
    x_tail_rearm(prm);
    pdl_trigger();
}

}  // namespace smcsd
