/*
 * smcsd_oracle.c -- plain, slow, single-threaded fp64 CPU oracle for the SMC-SD
 * verification hot path (arxiv 2604.15672, "Sequential Monte Carlo Speculative Decoding").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2604_15672_b200/, libsmcsd.so) never calls, links or imports it, and this
 * file shares no source, header, table or constant generator with csrc/.
 *
 * Every function follows the paper's definitions in the paper's order, with no
 * blocking, fusion or reordering.  Citations are PAPER.md line numbers (LaTeX source
 * in /root/reference) plus the algorithm / equation they fall in; readings of
 * ambiguous passages are the G-numbers listed in DESIGN.md section 3.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC -lm
 * (-ffp-contract=off: no fused multiply-add, so every fp64 op is one IEEE rounding.)
 * A second, timing-only build adds -fopenmp (liboracle_omp.so): the row pass of S1+S2 and the
 * KV copy planes run on several threads; every row / block is computed exactly as above, so
 * its outputs are bit-identical (tests/test_oracle_weights.py checks it).
 *
 * Pinned by tests/test_oracle_*.py (see DESIGN.md section 4 for the pin table).
 * Parity unpinned: nothing here.  Multi-round composition (R rounds of weights, resample, bonus,
 * reindex) is pinned statistically by SMC's unbiasedness identity in tests/test_oracle_rounds.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Timing-only build (liboracle_omp.so, -fopenmp): threads for the row-parallel S1+S2 pass
 * and the KV copy planes.  The plain build (liboracle.so) is single-threaded. */
int orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* Status bits (the ABI contract, retyped here from DESIGN.md section 2; no shared header). */
#define ORC_ST_DEGENERATE  1u  /* every log-weight of the prompt is -inf           */
#define ORC_ST_NOT_ABSCONT 2u  /* log q(d) = -inf at a drafted token, p << q violated */
#define ORC_ST_BAD_TOKEN   4u  /* drafted token outside [0,V), or n_drafted outside [0,K]         */
#define ORC_ST_NONFINITE   8u  /* NaN / +inf logit or log-weight, or a row whose max is -inf       */

/* ------------------------------------------------------------------------------------ */
/* Philox4x32-10 counter-based generator (Salmon et al., SC'11; the Random123 reference  */
/* algorithm).  Not in the paper: reading G5/G10 in DESIGN.md (counter-based uniforms,   */
/* north star).  Multipliers and Weyl key increments are the published constants.       */
/* ------------------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {            /* key schedule: bump the key before rounds 2..10 */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------------------ */
/* Decode one logit.  dtype 0 = fp32, 1 = bf16 (the top 16 bits of an fp32).  Both       */
/* decodes are exact in fp64.                                                             */
/* ------------------------------------------------------------------------------------ */
static double decode_logit(const void *row, int dtype, int64_t v)
{
    if (dtype == 1) {
        uint16_t bits16 = ((const uint16_t *)row)[v];
        uint32_t bits32 = (uint32_t)bits16 << 16;
        float f;
        memcpy(&f, &bits32, sizeof f);
        return (double)f;
    }
    return (double)((const float *)row)[v];
}

/* ------------------------------------------------------------------------------------ */
/* S1 over a column range.  For y_v = tau * z_v (temperature, reading G9):               */
/*   m = max_v y_v,  s = sum_v exp(y_v - m) (ascending v),  x = y_d if d is in range.    */
/* This is the log-sum-exp decomposition of the next-token conditional                    */
/* p(y|x) = p(xy)/p(x) (Eq. 1a) for a softmax-parameterised model.          */
/* `row` points at column v_begin; d_local = d - v_begin.  Returns 1 when a NaN or +inf   */
/* logit is present.  When every y is -inf, m = -inf and s = 0.                          */
/* ------------------------------------------------------------------------------------ */
static int row_stats_range(const void *row, int dtype, int64_t v_len, double tau,
                           int64_t d_local, double *m_out, double *s_out, double *x_out)
{
    int bad = 0;
    double m = -INFINITY;
    for (int64_t v = 0; v < v_len; ++v) {
        double z = decode_logit(row, dtype, v);
        if (isnan(z) || z == INFINITY) bad = 1;
        double y = tau * z;
        if (y > m) m = y;
    }
    double s = 0.0;
    if (m != -INFINITY && !bad) {
        for (int64_t v = 0; v < v_len; ++v) {
            double y = tau * decode_logit(row, dtype, v);
            s = s + exp(y - m);
        }
    }
    double x = -INFINITY;
    if (d_local >= 0 && d_local < v_len) x = tau * decode_logit(row, dtype, d_local);
    *m_out = m;
    *s_out = s;
    *x_out = x;
    return bad;
}

/* S1+S2 for a whole row: ell = y_d - m - ln s, the log-softmax at the drafted token,   */
/* i.e. log p(d_j | x d_<j) of Alg. 1 line "Score".  Sets *flag to       */
/* ORC_ST_NONFINITE when the row has a NaN/+inf logit or its max is -inf.               */
double orc_row_logprob(const void *row, int dtype, int64_t V, double tau, int64_t d, uint32_t *flag)
{
    double m, s, x;
    int bad = row_stats_range(row, dtype, V, tau, d, &m, &s, &x);
    *flag = 0;
    if (bad || m == -INFINITY) {
        *flag = ORC_ST_NONFINITE;
        return NAN;
    }
    return x - m - log(s);
}

/* TP reference pieces (north star: vocab-sharded logits, per-row max/sum-exp exchange).
 * orc_row_partial: S1 on the shard of columns [v_begin, v_begin+v_len) -> (m, s, x),
 * natural-log domain.  orc_combine_partials: merge G shards in rank order,
 * M = max m_g, S = sum_g s_g exp(m_g - M), X = max_g x_g, ell = X - M - ln S.        */
int orc_row_partial(const void *row_shard, int dtype, int64_t v_begin, int64_t v_len,
                    double tau, int64_t d, double out3[3])
{
    return row_stats_range(row_shard, dtype, v_len, tau, d - v_begin, &out3[0], &out3[1], &out3[2]);
}

double orc_combine_partials(const double *parts /*[G][3]*/, int G, int64_t row_stride3,
                            uint32_t *flag)
{
    double M = -INFINITY, X = -INFINITY;
    for (int g = 0; g < G; ++g) {
        const double *pg = parts + (int64_t)g * row_stride3;
        if (pg[0] > M) M = pg[0];
        if (pg[2] > X) X = pg[2];
    }
    *flag = 0;
    if (M == -INFINITY || isnan(M) || M == INFINITY) {
        *flag = ORC_ST_NONFINITE;
        return NAN;
    }
    double S = 0.0;
    for (int g = 0; g < G; ++g) {
        const double *pg = parts + (int64_t)g * row_stride3;
        if (pg[0] == -INFINITY) continue;
        S = S + pg[1] * exp(pg[0] - M);
    }
    return X - M - log(S);
}

/* ------------------------------------------------------------------------------------ */
/* S4: normalise + ESS (Alg. 1 lines "normalize" / "effective sample size",             */
/* PAPER.md:323-324; Eq. 3), in log space.              */
/* From fp32 log-weights lam[0..N): M = max lam; e_n = exp(lam_n - M);                  */
/* P_m = sum_{i<=m} e_i (sequential, reading G6); S = P_{N-1}; lse = M + ln S;          */
/* ESS = S^2 / sum_n e_n^2 (sequential).  Returns 1 when degenerate (M = -inf).         */
/* ------------------------------------------------------------------------------------ */
static int s4_normalise(const float *lam, int N, double *e, double *Pcum,
                        double *S_out, double *lse_out, double *ess_out)
{
    double M = -INFINITY;
    for (int n = 0; n < N; ++n)
        if ((double)lam[n] > M) M = (double)lam[n];
    if (M == -INFINITY) return 1;
    for (int n = 0; n < N; ++n) e[n] = exp((double)lam[n] - M);
    double acc = 0.0;
    for (int m = 0; m < N; ++m) {
        acc = acc + e[m];
        Pcum[m] = acc;
    }
    double S = Pcum[N - 1];
    double sumsq = 0.0;
    for (int n = 0; n < N; ++n) {
        double sq = e[n] * e[n];
        sumsq = sumsq + sq;
    }
    *S_out = S;
    *lse_out = M + log(S);
    *ess_out = (S * S) / sumsq;
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* smcsd_weights oracle: S1-S4 for P prompts.                                            */
/* Row (prompt p, particle n, draft position j) of a logits tensor lives at              */
/*   base + ((p*N + n)*rows_per_particle + j)*ld   (elements).                           */
/* S3 (Alg. 1 "Reweight"; power weight PAPER.md:1418, reading G11):        */
/*   Delta_n = sum_{j<k_n} (alpha*ell^p_j - ell^q_j) in fp64, bonus row excluded          */
/*   (PAPER.md:1168); lam'_n = fl32(lam_prev_n + Delta_n).                                */
/* A particle with an invalid row (bad token, non-finite row, q(d)=0) gets lam' = -inf  */
/* and its prompt's status bit is set (reading G13).                                     */
/* logp_tok/logq_tok (optional, [P][N][K] fp64): ell per row; 0 for rows j >= k_n, NaN   */
/* for invalid rows.  wnorm (optional [P][N] fp64): e_n / S.                              */
/* ------------------------------------------------------------------------------------ */
/* Pass 1 of orc_weights: S1+S2 of every scored row (p, n, j < k_n).  Rows are independent,
 * so the timing-only build (liboracle_omp.so, -fopenmp) runs them on several threads; the
 * plain build ignores the pragma.  Each row's arithmetic is the same either way.
 * code[row]: -1 unread (j >= k_n or invalid k_n), 0 ok, 1 bad token, 2 non-finite row,
 * 3 q(d) = 0. */
static void s12_rows(const void *logits_p, int64_t ld_p, int rpp_p, const void *logits_q,
                     int64_t ld_q, int rpp_q, int dtype, const int32_t *tokens,
                     const int32_t *n_drafted, int P, int N, int K, int64_t V, double tau_p,
                     double tau_q, double *lp_out, double *lq_out, int *code)
{
    size_t esz = dtype == 1 ? 2 : 4;
    int64_t rows = (int64_t)P * N * K;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < rows; ++r) {
        int64_t pn = r / K;
        int j = (int)(r - pn * K);
        int k_n = n_drafted ? n_drafted[pn] : K;
        if (k_n < 0 || k_n > K) k_n = 0;
        double lp = 0.0, lq = 0.0;
        int c = -1;
        if (j < k_n) {
            int64_t d = tokens[pn * K + j];
            if (d < 0 || d >= V) {
                c = 1;
                lp = NAN;
                lq = NAN;
            } else {
                const char *rp = (const char *)logits_p + ((pn * rpp_p + j) * ld_p) * (int64_t)esz;
                const char *rq = (const char *)logits_q + ((pn * rpp_q + j) * ld_q) * (int64_t)esz;
                uint32_t fp, fq;
                lp = orc_row_logprob(rp, dtype, V, tau_p, d, &fp);
                lq = orc_row_logprob(rq, dtype, V, tau_q, d, &fq);
                c = (fp | fq) ? 2 : (lq == -INFINITY ? 3 : 0);
            }
        }
        lp_out[r] = lp;
        lq_out[r] = lq;
        code[r] = c;
    }
}

void orc_weights(const void *logits_p, int64_t ld_p, int rpp_p,
                 const void *logits_q, int64_t ld_q, int rpp_q, int dtype,
                 const int32_t *tokens, const int32_t *n_drafted, const float *logw_prev,
                 int P, int N, int K, int64_t V, double alpha, double tau_p, double tau_q,
                 float *logw_out, double *logp_tok, double *logq_tok,
                 double *lse_out, double *ess_out, double *wnorm, uint32_t *status,
                 double *scratch /* 2*N doubles */)
{
    int64_t rows = (int64_t)P * N * K;
    double *lp_all = logp_tok ? logp_tok : (double *)malloc((size_t)rows * sizeof(double));
    double *lq_all = logq_tok ? logq_tok : (double *)malloc((size_t)rows * sizeof(double));
    int *code = (int *)malloc((size_t)(rows > 0 ? rows : 1) * sizeof(int));
    s12_rows(logits_p, ld_p, rpp_p, logits_q, ld_q, rpp_q, dtype, tokens, n_drafted, P, N, K, V,
             tau_p, tau_q, lp_all, lq_all, code);
    for (int p = 0; p < P; ++p) {
        uint32_t st = 0;
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            int k_n = n_drafted ? n_drafted[pn] : K;
            int bad = 0;
            if (k_n < 0 || k_n > K) {
                st |= ORC_ST_BAD_TOKEN;
                bad = 1;
                k_n = 0;
            }
            double delta = 0.0;
            for (int j = 0; j < k_n; ++j) {
                int64_t r = pn * K + j;
                if (code[r] == 1) {
                    st |= ORC_ST_BAD_TOKEN;
                    bad = 1;
                } else if (code[r] == 2) {
                    st |= ORC_ST_NONFINITE;
                    bad = 1;
                } else if (code[r] == 3) {
                    st |= ORC_ST_NOT_ABSCONT;
                    bad = 1;
                } else {
                    delta = delta + (alpha * lp_all[r] - lq_all[r]);
                }
            }
            float prev = logw_prev ? logw_prev[pn] : (float)(-log((double)N));
            if (isnan(prev) || prev == INFINITY) {
                st |= ORC_ST_NONFINITE;
                bad = 1;
            }
            logw_out[pn] = bad ? -INFINITY : (float)((double)prev + delta);
        }
        /* S4 on the fp32 log-weights just stored */
        double S, lse, ess;
        double *e = scratch, *Pc = scratch + N;
        if (s4_normalise(logw_out + (int64_t)p * N, N, e, Pc, &S, &lse, &ess)) {
            st |= ORC_ST_DEGENERATE;
            if (lse_out) lse_out[p] = -INFINITY;
            if (ess_out) ess_out[p] = 0.0;
            if (wnorm) for (int n = 0; n < N; ++n) wnorm[(int64_t)p * N + n] = 0.0;
        } else {
            if (lse_out) lse_out[p] = lse;
            if (ess_out) ess_out[p] = ess;
            if (wnorm) for (int n = 0; n < N; ++n) wnorm[(int64_t)p * N + n] = e[n] / S;
        }
        if (status) status[p] = st;
    }
    free(code);
    if (!logq_tok) free(lq_all);
    if (!logp_tok) free(lp_all);
}

/* ------------------------------------------------------------------------------------ */
/* smcsd_resample oracle: S4-S7 for P prompts from fp32 log-weights.                    */
/* S5: resample iff ESS < eta (strict; reading G3).                        */
/* S6, scheme 0 = systematic (north star; reading G1) by inverse CDF:      */
/*   U = word0(Philox4x32-10(key=(seed_lo,seed_hi), ctr=(step_lo,step_hi,prompt,0)))     */
/*       * 2^-32   (or uniforms[p] * 2^-32 when the override is given),                  */
/*   C_m = P_m / S,  u_n = (n + U) / N,  a_n = #{m : C_m <= u_n}                         */
/* S6, scheme 1 = multinomial, as Alg. 1 prints it (a_n ~ Cat(wbar) i.i.d.): */
/*   u_n = word (n mod 4) of Philox(key, ctr=(step_lo,step_hi,prompt, 1 + floor(n/4)))   */
/*       * 2^-32 (or uniforms[p*N + n] * 2^-32), a_n = #{m : C_m <= u_n} (same CDF).      */
/*   (= min{m : u_n < C_m}; zero-weight particles are never chosen),        */
/*   o_m = #{n : a_n = m},  ties = #{(n,m) : |u_n - C_m| <= 2^-40} (reading G7).          */
/*   In-place slot plan (reading G14): survivors keep their slot; the list E of extra    */
/*   copies (m repeated o_m - 1 times, ascending m) fills the dead slots D (o_m = 0,      */
/*   ascending): slot_src[D_i] = E_i, slot_src[m] = m for survivors.                      */
/* S7: after a resample every log-weight is reset to fl32(-ln N) (G8).     */
/* Without a resample: ancestors = identity, offspring = 1, lam kept.                    */
/* Degenerate prompt: lse = -inf, ESS = 0, identity ancestry, resampled = 0.             */
/* NaN / +inf input log-weights are flagged NONFINITE and treated as -inf (G13).         */
/* ------------------------------------------------------------------------------------ */
void orc_resample(const float *logw, int P, int N, int64_t prompt_base, double eta,
                  int scheme, uint64_t seed, uint64_t step, const uint32_t *uniforms,
                  int32_t *ancestors, int32_t *offspring, int32_t *slot_src, float *logw_out,
                  uint8_t *resampled, double *ess_out, double *lse_out, int32_t *n_ties,
                  uint32_t *status, double *wnorm, double *cdf_out,
                  double *scratch /* 4*N doubles */, int32_t *iscratch /* 3*N ints */)
{
    const double two_m32 = 1.0 / 4294967296.0;
    const double tie_delta = 1.0 / 1099511627776.0; /* 2^-40 */
    float *lam = (float *)(iscratch + 0);          /* reuse int scratch as float storage */
    int32_t *a = iscratch + N;
    int32_t *o = iscratch + 2 * N;
    double *e = scratch, *Pc = scratch + N, *C = scratch + 2 * N, *u = scratch + 3 * N;
    float reset = (float)(-log((double)N));

    for (int p = 0; p < P; ++p) {
        uint32_t st = 0;
        const float *lw = logw + (int64_t)p * N;
        for (int n = 0; n < N; ++n) {
            float v = lw[n];
            if (isnan(v) || v == INFINITY) {
                st |= ORC_ST_NONFINITE;
                v = -INFINITY;
            }
            lam[n] = v;
        }
        double S, lse, ess;
        int degenerate = s4_normalise(lam, N, e, Pc, &S, &lse, &ess);
        int do_resample = 0;
        int ties = 0;
        if (degenerate) {
            st |= ORC_ST_DEGENERATE;
            lse = -INFINITY;
            ess = 0.0;
        } else {
            do_resample = ess < eta;
        }
        if (do_resample) {
            uint64_t prompt = (uint64_t)(prompt_base + p);
            uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
            for (int m = 0; m < N; ++m) C[m] = Pc[m] / S;
            if (scheme == 0) {
                double U;
                if (uniforms) {
                    U = (double)uniforms[p] * two_m32;
                } else {
                    uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)prompt, 0u};
                    uint32_t r[4];
                    orc_philox4x32_10(ctr, key, r);
                    U = (double)r[0] * two_m32;
                }
                for (int n = 0; n < N; ++n) u[n] = ((double)n + U) / (double)N;
            } else {
                for (int n = 0; n < N; ++n) {
                    if (uniforms) {
                        u[n] = (double)uniforms[(int64_t)p * N + n] * two_m32;
                    } else {
                        uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)prompt,
                                           1u + (uint32_t)(n / 4)};
                        uint32_t r[4];
                        orc_philox4x32_10(ctr, key, r);
                        u[n] = (double)r[n % 4] * two_m32;
                    }
                }
            }
            for (int n = 0; n < N; ++n) {
                int count = 0;
                for (int m = 0; m < N; ++m)
                    if (C[m] <= u[n]) count++;
                a[n] = count;
            }
            for (int m = 0; m < N; ++m) o[m] = 0;
            for (int n = 0; n < N; ++n) o[a[n]]++;
            for (int n = 0; n < N; ++n)
                for (int m = 0; m < N; ++m)
                    if (fabs(u[n] - C[m]) <= tie_delta) ties++;
            if (ancestors) for (int n = 0; n < N; ++n) ancestors[(int64_t)p * N + n] = a[n];
            if (offspring) for (int m = 0; m < N; ++m) offspring[(int64_t)p * N + m] = o[m];
            if (slot_src) {
                /* E: extra copies, ascending source; D: dead slots, ascending. */
                int32_t *plan = slot_src + (int64_t)p * N;
                int n_dead = 0;
                for (int m = 0; m < N; ++m) plan[m] = m;
                /* walk the dead slots and the extra list in step */
                int src = 0, left = 0;
                for (int m = 0; m < N; ++m) {
                    if (o[m] != 0) continue;
                    while (left == 0) {         /* advance to the next source with an extra copy */
                        if (o[src] >= 2) left = o[src] - 1;
                        if (left == 0) src++;
                    }
                    plan[m] = src;
                    n_dead++;
                    left--;
                    if (left == 0) src++;
                }
                (void)n_dead;
            }
            for (int n = 0; n < N; ++n) logw_out[(int64_t)p * N + n] = reset;
            if (cdf_out) for (int m = 0; m < N; ++m) cdf_out[(int64_t)p * N + m] = C[m];
        } else {
            for (int n = 0; n < N; ++n) {
                if (ancestors) ancestors[(int64_t)p * N + n] = n;
                if (offspring) offspring[(int64_t)p * N + n] = 1;
                if (slot_src) slot_src[(int64_t)p * N + n] = n;
                logw_out[(int64_t)p * N + n] = lam[n];
            }
            if (cdf_out) for (int m = 0; m < N; ++m)
                cdf_out[(int64_t)p * N + m] = degenerate ? 0.0 : Pc[m] / S;
        }
        if (wnorm) for (int n = 0; n < N; ++n)
            wnorm[(int64_t)p * N + n] = degenerate ? 0.0 : e[n] / S;
        if (resampled) resampled[p] = (uint8_t)do_resample;
        if (ess_out) ess_out[p] = ess;
        if (lse_out) lse_out[p] = lse;
        if (n_ties) n_ties[p] = ties;
        if (status) status[p] = st;
    }
}

/* ------------------------------------------------------------------------------------ */
/* PowerSMC weights (NEXT #4; App. F): K = 1, no bonus token, target and */
/* draft the same model; a particle's importance weight is w = sum_x p(x | prefix)^alpha    */
/* (PAPER.md:1426), here with p = softmax(tau * z) of the particle's row j = 0:              */
/*   log p_v = y_v - m - ln sum_u exp(y_u - m),  log w = ln sum_v exp(alpha * log p_v),      */
/*   lam' = fl32(lam_prev + log w),  then S4 (normalise, ESS) exactly as in orc_weights.      */
/* inc (optional [P][N] fp64) receives log w.                                                */
/* ------------------------------------------------------------------------------------ */
void orc_powersmc_weights(const void *logits, int64_t ld, int rpp, int dtype, const float *logw_prev,
                          int P, int N, int64_t V, double alpha, double tau, float *logw_out,
                          double *inc, double *lse_out, double *ess_out, double *wnorm,
                          uint32_t *status, double *scratch /* 2*N doubles */)
{
    size_t esz = dtype == 1 ? 2 : 4;
    for (int p = 0; p < P; ++p) {
        uint32_t st = 0;
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            const char *row = (const char *)logits + (pn * rpp) * ld * (int64_t)esz;
            double m, s, x;
            int bad = row_stats_range(row, dtype, V, tau, -1, &m, &s, &x);
            double lw = NAN;
            if (bad || m == -INFINITY) {
                st |= ORC_ST_NONFINITE;
                bad = 1;
            } else {
                double lse = m + log(s);
                double w = 0.0;
                for (int64_t v = 0; v < V; ++v) {
                    double logp = tau * decode_logit(row, dtype, v) - lse;
                    w = w + exp(alpha * logp);
                }
                lw = log(w);
            }
            if (inc) inc[pn] = lw;
            float prev = logw_prev ? logw_prev[pn] : (float)(-log((double)N));
            if (isnan(prev) || prev == INFINITY) { st |= ORC_ST_NONFINITE; bad = 1; }
            logw_out[pn] = bad ? -INFINITY : (float)((double)prev + lw);
        }
        double S, lse, ess;
        double *e = scratch, *Pc = scratch + N;
        if (s4_normalise(logw_out + (int64_t)p * N, N, e, Pc, &S, &lse, &ess)) {
            st |= ORC_ST_DEGENERATE;
            if (lse_out) lse_out[p] = -INFINITY;
            if (ess_out) ess_out[p] = 0.0;
            if (wnorm) for (int n = 0; n < N; ++n) wnorm[(int64_t)p * N + n] = 0.0;
        } else {
            if (lse_out) lse_out[p] = lse;
            if (ess_out) ess_out[p] = ess;
            if (wnorm) for (int n = 0; n < N; ++n) wnorm[(int64_t)p * N + n] = e[n] / S;
        }
        if (status) status[p] = st;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Terminal selection: "one complete sequence is sampled from the       */
/* terminal normalized weights" -- one draw per prompt by the same inverse CDF with          */
/* u = word0(Philox(key, ctr=(step_lo,step_hi,prompt, 0xFFFFFFFF))) * 2^-32 (or the override  */
/* uniforms[p]).  Degenerate prompt: selected = -1, status DEGENERATE.                       */
/* ------------------------------------------------------------------------------------ */
void orc_select(const float *logw, int P, int N, int64_t prompt_base, uint64_t seed, uint64_t step,
                const uint32_t *uniforms, int32_t *selected, uint32_t *status,
                double *scratch /* 2*N doubles */)
{
    const double two_m32 = 1.0 / 4294967296.0;
    for (int p = 0; p < P; ++p) {
        uint32_t st = 0;
        const float *lw = logw + (int64_t)p * N;
        double M = -INFINITY;
        for (int n = 0; n < N; ++n) {
            double v = lw[n];
            if (isnan(v) || v == INFINITY) { st |= ORC_ST_NONFINITE; v = -INFINITY; }
            if (v > M) M = v;
        }
        if (M == -INFINITY) {
            selected[p] = -1;
            status[p] = st | ORC_ST_DEGENERATE;
            continue;
        }
        double *Pc = scratch;
        double acc = 0.0;
        for (int m = 0; m < N; ++m) {
            double v = lw[m];
            if (isnan(v) || v == INFINITY) v = -INFINITY;
            acc = acc + exp(v - M);
            Pc[m] = acc;
        }
        double u;
        if (uniforms) {
            u = (double)uniforms[p] * two_m32;
        } else {
            uint64_t prompt = (uint64_t)(prompt_base + p);
            uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)prompt, 0xFFFFFFFFu};
            uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
            uint32_t r[4];
            orc_philox4x32_10(ctr, key, r);
            u = (double)r[0] * two_m32;
        }
        int count = 0;
        for (int m = 0; m < N; ++m)
            if (Pc[m] / acc <= u) count++;
        selected[p] = count;
        status[p] = st;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Bonus token (NEXT #2; Alg. 1 line "sample bonus token x+ ~ p(. | x, y)";   */
/* PAPER.md:330 appends it; weight-neutral).  Reading G22: an    */
/* exact draw from softmax(tau z) of the target row j = k_n (k_n = n_drafted or K) by a      */
/* two-level sampler with counter-based uniforms.  The segment width `seg` is a parameter   */
/* of the reading (any width gives an exact draw; the product path uses 8192 and the tests  */
/* pin this oracle at 8192 and 4096):                                                       */
/*   1. segment masses w_i = sum_{v in seg i} exp(tau z_v - M), M = max_v tau z_v, segments  */
/*      of `seg` columns [seg i, min(V, seg (i+1))); W = sum_i w_i (left to right);           */
/*   2. U = word0(Philox(key = seed, ctr = (step_lo, step_hi, prompt, 2^31 + 2^20 n))) 2^-32; */
/*      a = #{i : C_i / W <= U}, C_i = w_0 + ... + w_i  (inverse CDF, as in S6);              */
/*   3. Gumbel-max inside segment a: for column v = seg a + 4 q + k, word k of                */
/*      Philox(ctr = (step_lo, step_hi, prompt, 2^31 + 2^20 n + 1 + q)) gives                  */
/*      u_v = (word + 1/2) 2^-32, E_v = -ln u_v (= -log1p(-(1 - u_v)) for u_v >= 1/2),        */
/*      g_v = -ln E_v; x+ = argmax_v (tau z_v + g_v), smallest v on equal keys.               */
/* P(x+ = v) = (w_a / W) (exp(tau z_v - M) / w_a) = softmax(tau z)_v, exactly.                */
/* Near-tie diagnostics (optional, the test tolerance for rounding-order near-ties, G7):      */
/*   seg_margin[pn] = min_i |C_i / W - U| (boundary i* attains it),                           */
/*   key_margin[pn] = key(x+) - second-best key in segment a, second[pn] = that column,      */
/*   alt[pn] = the Gumbel-max column of the segment on the other side of boundary i*         */
/*             (i* if C_i* / W <= U, else i* + 1; -1 when that segment does not exist).       */
/* Invalid k_n: -1 and BAD_TOKEN; NaN / +inf logit or an all -inf row: -1 and NONFINITE.      */
/* ------------------------------------------------------------------------------------ */
static int64_t gumbel_max_segment(const char *row, int dtype, int64_t V, double tau, int64_t seg,
                                  int64_t a, const uint32_t key[2], const uint32_t ctr_hi[3],
                                  uint32_t stream, double *best_out, double *second_out,
                                  int64_t *second_col)
{
    const double two_m32 = 1.0 / 4294967296.0;
    int64_t v0 = a * seg;
    int64_t nv = V - v0 < seg ? V - v0 : seg;
    double best = -INFINITY, second = -INFINITY;
    int64_t arg = -1, arg2 = -1;
    uint32_t ctr[4] = {ctr_hi[0], ctr_hi[1], ctr_hi[2], 0u}, r[4] = {0, 0, 0, 0};
    for (int64_t i = 0; i < nv; ++i) {
        if (i % 4 == 0) {
            ctr[3] = stream + 1u + (uint32_t)(i / 4);
            orc_philox4x32_10(ctr, key, r);
        }
        uint32_t w = r[i % 4];
        double E;
        if (w < 0x80000000u) E = -log(((double)w + 0.5) * two_m32);
        else E = -log1p(-(((double)(0xFFFFFFFFu - w) + 0.5) * two_m32));
        double k = tau * decode_logit(row, dtype, v0 + i) - log(E);
        if (k > best) { second = best; arg2 = arg; best = k; arg = v0 + i; }
        else if (k > second) { second = k; arg2 = v0 + i; }
    }
    *best_out = best;
    *second_out = second;
    *second_col = arg2;
    return arg;
}

void orc_bonus(const void *logits_p, int64_t ld, int rpp, int dtype, const int32_t *n_drafted,
               int P, int N, int K, int64_t V, double tau, uint64_t seed, uint64_t step,
               int64_t prompt_base, int64_t seg, int32_t *bonus, double *seg_margin,
               double *key_margin, int32_t *second, int32_t *alt, uint32_t *status)
{
    const double two_m32 = 1.0 / 4294967296.0;
    size_t esz = dtype == 1 ? 2 : 4;
    int64_t nseg = (V + seg - 1) / seg;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int p = 0; p < P; ++p) {
        uint32_t st = 0;
        uint32_t prompt = (uint32_t)(uint64_t)(prompt_base + p);
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            bonus[pn] = -1;
            if (seg_margin) seg_margin[pn] = INFINITY;
            if (key_margin) key_margin[pn] = INFINITY;
            if (second) second[pn] = -1;
            if (alt) alt[pn] = -1;
            int kn = n_drafted ? n_drafted[pn] : K;
            if (kn < 0 || kn > K) { st |= ORC_ST_BAD_TOKEN; continue; }
            const char *row = (const char *)logits_p + (pn * rpp + kn) * ld * (int64_t)esz;
            /* step 1: M, segment masses */
            double M = -INFINITY;
            int bad = 0;
            for (int64_t v = 0; v < V; ++v) {
                double y = tau * decode_logit(row, dtype, v);
                if (isnan(y) || y == INFINITY) bad = 1;
                else if (y > M) M = y;
            }
            if (bad || M == -INFINITY) { st |= ORC_ST_NONFINITE; continue; }
            double W = 0.0, C[8192];
            if (nseg > 8192) { st |= ORC_ST_NONFINITE; continue; }
            for (int64_t i = 0; i < nseg; ++i) {
                double w = 0.0;
                int64_t e = (i + 1) * seg < V ? (i + 1) * seg : V;
                for (int64_t v = i * seg; v < e; ++v)
                    w = w + exp(tau * decode_logit(row, dtype, v) - M);
                W = W + w;
                C[i] = W;
            }
            /* step 2: segment by inverse CDF */
            uint32_t stream = 0x80000000u + ((uint32_t)n << 20);
            uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), prompt, stream};
            uint32_t r[4];
            orc_philox4x32_10(ctr, key, r);
            double U = (double)r[0] * two_m32;
            int64_t a = 0, inear = 0;
            double mg = INFINITY;
            for (int64_t i = 0; i < nseg; ++i) {
                double c = C[i] / W;
                if (c <= U) a++;
                if (fabs(c - U) < mg) { mg = fabs(c - U); inear = i; }
            }
            if (a >= nseg) a = nseg - 1;     /* U < 1 = C_last / W: unreachable up to rounding */
            /* step 3: Gumbel-max inside segment a */
            double best, sec, b2, s2;
            int64_t col2, col2b;
            int64_t arg = gumbel_max_segment(row, dtype, V, tau, seg, a, key, ctr, stream,
                                             &best, &sec, &col2);
            bonus[pn] = (int32_t)arg;
            if (seg_margin) seg_margin[pn] = mg;
            if (key_margin) key_margin[pn] = best - sec;
            if (second) second[pn] = (int32_t)col2;
            if (alt) {
                int64_t b = C[inear] / W <= U ? inear : inear + 1;
                if (b >= 0 && b < nseg)
                    alt[pn] = (int32_t)gumbel_max_segment(row, dtype, V, tau, seg, b, key, ctr,
                                                          stream, &b2, &s2, &col2b);
            }
        }
        if (status) status[p] = st;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Paged KV reindex (NEXT #1; Sec. 3.3 Obs. 2: "resampling by copying page */
/* metadata and incrementing the reference counts"; SPEC.md:466-474 resample_pages).        */
/* table[p][n][0 .. n_pages[p][n]) lists particle n's KV pages.  After the call particle n   */
/* holds its ancestor's list: table_dst[p][n][i] = table_src[p][a_n][i], n_pages_dst[p][n] = */
/* n_pages_src[p][a_n] (slots i >= n_pages_dst are set to -1); refcount[pg] += #references   */
/* in the new lists - #references in the old lists; freed[pg] = 1 for every page referenced */
/* by an old list whose refcount is now 0 (0 for the other old-list pages).  No KV content   */
/* moves.  Ids outside [0, num_pages) or ancestors outside [0, N) flag ST_BAD_PAGE (16) and  */
/* are skipped.                                                                               */
/* ------------------------------------------------------------------------------------ */
#define ORC_ST_BAD_PAGE 16u
void orc_kv_reindex_paged(const int32_t *table_src, const int32_t *n_pages_src, int32_t *table_dst,
                          int32_t *n_pages_dst, int32_t *refcount, uint8_t *freed,
                          const int32_t *src_index, int P, int N, int max_pages, int num_pages,
                          uint32_t *status)
{
    for (int p = 0; p < P; ++p) status[p] = 0;
    for (int p = 0; p < P; ++p) {
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            int a = src_index[pn];
            int len = 0;
            if (a < 0 || a >= N) {
                status[p] |= ORC_ST_BAD_PAGE;
            } else {
                len = n_pages_src[(int64_t)p * N + a];
                if (len < 0 || len > max_pages) { status[p] |= ORC_ST_BAD_PAGE; len = 0; }
            }
            for (int i = 0; i < max_pages; ++i) {
                int32_t pg = -1;
                if (i < len) {
                    pg = table_src[((int64_t)p * N + a) * max_pages + i];
                    if (pg < 0 || pg >= num_pages) { status[p] |= ORC_ST_BAD_PAGE; pg = -1; }
                    else refcount[pg] += 1;
                }
                table_dst[pn * max_pages + i] = pg;
            }
            n_pages_dst[pn] = len;
        }
    }
    for (int p = 0; p < P; ++p)
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            int len = n_pages_src[pn];
            if (len < 0 || len > max_pages) { status[p] |= ORC_ST_BAD_PAGE; continue; }
            for (int i = 0; i < len; ++i) {
                int32_t pg = table_src[pn * max_pages + i];
                if (pg < 0 || pg >= num_pages) { status[p] |= ORC_ST_BAD_PAGE; continue; }
                refcount[pg] -= 1;
            }
        }
    if (freed)
        for (int p = 0; p < P; ++p)
            for (int n = 0; n < N; ++n) {
                int64_t pn = (int64_t)p * N + n;
                int len = n_pages_src[pn];
                if (len < 0 || len > max_pages) continue;
                for (int i = 0; i < len; ++i) {
                    int32_t pg = table_src[pn * max_pages + i];
                    if (pg < 0 || pg >= num_pages) continue;
                    freed[pg] = (uint8_t)(refcount[pg] == 0);
                }
            }
}

/* ------------------------------------------------------------------------------------ */
/* Paged append with copy-on-write (NEXT #1, the other half of the paper's mechanism:       */
/* PAPER.md:488-490, Sec. 3.3 Obs. 2 -- duplicated particles share their ancestor's pages;   */
/* SPEC.md:466-470 append_tokens: "fills the particle's last page if it has exclusive        */
/* ownership (refcount 1); otherwise performs copy-on-write of the partial tail page ...,    */
/* then allocates fresh pages"; full pages are immutable and never copied).  Reading G24.    */
/* Particles are processed one at a time in (p, n) order; particle n appends n_new tokens:  */
/*   f = seq_len mod page_size (tokens in a partial tail page; 0 = no partial page);        */
/*   if n_new > 0, f > 0 and refcount[tail] > 1: copy-on-write -- a fresh page c takes the   */
/*     tail's f filled tokens (cow_src/dst/tokens record it), refcount[tail] -= 1,           */
/*     refcount[c] = 1, the table's last entry becomes c;                                    */
/*   the tail's free slots take the first new tokens, then fresh pages (refcount 1) are      */
/*   appended for the rest; every fresh page is the LOWEST-id page with refcount 0;         */
/*   slot_mapping[p][n][j] = page * page_size + offset of new token j (-1 for j >= n_new);   */
/*   seq_len += n_new, n_pages updated.                                                      */
/* The call is all-or-nothing: if any particle's state is invalid (page id out of range or   */
/* with refcount < 1, n_pages != ceil(seq_len / page_size), n_new < 0 or > max_new, or the   */
/* list would exceed max_pages) its prompt gets ORC_ST_BAD_PAGE; if the pool has fewer free  */
/* pages than the call needs every prompt gets ORC_ST_OUT_OF_PAGES; then *result = 1,        */
/* nothing changes and the copy list reads "none" (-1, -1, 0).  No page is freed here.        */
/* ------------------------------------------------------------------------------------ */
#define ORC_ST_OUT_OF_PAGES 128u
static int lowest_free(const int32_t *refcount, int num_pages, int from)
{
    for (int pg = from; pg < num_pages; ++pg)
        if (refcount[pg] == 0) return pg;
    return -1;
}

void orc_kv_append_paged(int32_t *table, int32_t *n_pages, int32_t *seq_len, int32_t *refcount,
                         const int32_t *n_new, int P, int N, int max_pages, int num_pages,
                         int page_size, int max_new, int32_t *slot_mapping, int32_t *cow_src,
                         int32_t *cow_dst, int32_t *cow_tokens, uint32_t *status, int32_t *result)
{
    int ok = 1;
    int64_t need_total = 0;
    /* simulated refcounts of the tails for the copy-on-write decisions (sequential order) */
    for (int p = 0; p < P; ++p) {
        status[p] = 0;
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            int len = seq_len[pn], np_ = n_pages[pn], add = n_new[pn];
            int bad = len < 0 || np_ < 0 || np_ > max_pages || add < 0 || add > max_new ||
                      np_ != (len + page_size - 1) / page_size;
            for (int i = 0; !bad && i < np_; ++i) {
                int pg = table[pn * max_pages + i];
                if (pg < 0 || pg >= num_pages || refcount[pg] < 1) bad = 1;
            }
            if (!bad) {
                int f = len % page_size;
                int room = f ? page_size - f : 0;
                int fresh = add > room ? (add - room + page_size - 1) / page_size : 0;
                if (np_ + fresh > max_pages) bad = 1;
            }
            if (bad) { status[p] |= ORC_ST_BAD_PAGE; ok = 0; }
        }
    }
    if (ok) {
        /* pages the call needs, in the sequential semantics */
        int32_t *rc = (int32_t *)malloc((size_t)num_pages * sizeof(int32_t));
        memcpy(rc, refcount, (size_t)num_pages * sizeof(int32_t));
        for (int64_t pn = 0; pn < (int64_t)P * N; ++pn) {
            int len = seq_len[pn], add = n_new[pn];
            if (add == 0) continue;
            int f = len % page_size;
            int room = f ? page_size - f : 0;
            if (f && rc[table[pn * max_pages + n_pages[pn] - 1]] > 1) {
                rc[table[pn * max_pages + n_pages[pn] - 1]] -= 1;
                need_total += 1;
            }
            need_total += add > room ? (add - room + page_size - 1) / page_size : 0;
        }
        free(rc);
        int64_t free_pages = 0;
        for (int pg = 0; pg < num_pages; ++pg) free_pages += refcount[pg] == 0;
        if (need_total > free_pages) {
            for (int p = 0; p < P; ++p) status[p] |= ORC_ST_OUT_OF_PAGES;
            ok = 0;
        }
    }
    *result = ok ? 0 : 1;
    if (!ok) {
        for (int64_t pn = 0; pn < (int64_t)P * N; ++pn) {   /* the copy list reads "none" */
            cow_src[pn] = -1;
            cow_dst[pn] = -1;
            cow_tokens[pn] = 0;
        }
        return;
    }
    int cursor = 0;                    /* pages below it are all in use (lowest-id allocation) */
    for (int p = 0; p < P; ++p)
        for (int n = 0; n < N; ++n) {
            int64_t pn = (int64_t)p * N + n;
            int32_t *row = table + pn * max_pages;
            int len = seq_len[pn], add = n_new[pn];
            int f = len % page_size;
            cow_src[pn] = -1;
            cow_dst[pn] = -1;
            cow_tokens[pn] = 0;
            for (int j = 0; j < max_new; ++j) slot_mapping[pn * max_new + j] = -1;
            if (add == 0) continue;
            if (f && refcount[row[n_pages[pn] - 1]] > 1) {           /* copy-on-write */
                int t = row[n_pages[pn] - 1];
                int c = lowest_free(refcount, num_pages, cursor);
                cursor = c + 1;
                refcount[t] -= 1;
                refcount[c] = 1;
                row[n_pages[pn] - 1] = c;
                cow_src[pn] = t;
                cow_dst[pn] = c;
                cow_tokens[pn] = f;
            }
            for (int j = 0; j < add; ++j) {
                int pos = len + j;                                   /* token position */
                int pi = pos / page_size, off = pos % page_size;
                if (pi >= n_pages[pn]) {                             /* a fresh page */
                    int c = lowest_free(refcount, num_pages, cursor);
                    cursor = c + 1;
                    refcount[c] = 1;
                    row[pi] = c;
                    n_pages[pn] = pi + 1;
                }
                slot_mapping[pn * max_new + j] = row[pi] * page_size + off;
            }
            seq_len[pn] = len + add;
        }
}

/* The content copies of orc_kv_append_paged's copy-on-write list for one KV pool: for every  */
/* particle with cow_dst >= 0 and every plane o (e.g. L x {K, V}), the first cow_tokens       */
/* tokens of page cow_src are copied to page cow_dst:                                          */
/*   base + o*plane_stride + page*page_stride + [0, tokens * token_bytes)   (bytes).          */
void orc_paged_cow_copy(void *pool, int64_t n_planes, int64_t plane_stride, int64_t page_stride,
                        int64_t token_bytes, const int32_t *cow_src, const int32_t *cow_dst,
                        const int32_t *cow_tokens, int64_t count)
{
    for (int64_t i = 0; i < count; ++i) {
        if (cow_dst[i] < 0) continue;
        for (int64_t o = 0; o < n_planes; ++o)
            memcpy((char *)pool + o * plane_stride + (int64_t)cow_dst[i] * page_stride,
                   (const char *)pool + o * plane_stride + (int64_t)cow_src[i] * page_stride,
                   (size_t)(cow_tokens[i] * token_bytes));
    }
}

/* ------------------------------------------------------------------------------------ */
/* S8/S9: reindex per-particle state to the ancestor's (Alg. 1: x^(n) <- x^(a_n) d^(a_n) */
/* x+_(a_n)).  Block (o, p, n) = seg_count segments of seg_bytes bytes at  */
/* base + o*outer_stride + p*prompt_stride + n*particle_stride + s*seg_stride.           */
/* Out-of-place (dst != src): dst block n <- src block src_index[n] for every n.         */
/* In-place (dst == src): for every n with src_index[n] != n, block n <- block           */
/* src_index[n] (the slot plan guarantees sources are never destinations).              */
/* Invalid index policy (reading G23): an entry outside [0, N) is skipped     */
/* (destination untouched) and flags ORC_ST_BAD_INDEX in status[p]; in place, an entry   */
/* whose source is itself a destination (src_index[s] != s) makes the plan not           */
/* hazard-free: the prompt is flagged and none of its blocks is copied.                  */
/* ------------------------------------------------------------------------------------ */
#define ORC_ST_BAD_INDEX 64u
void orc_kv_reindex(void *dst, const void *src, int64_t n_outer, int64_t outer_stride,
                    int64_t prompt_stride, int64_t particle_stride, int64_t seg_count,
                    int64_t seg_bytes, int64_t seg_stride, const int32_t *src_index, int P, int N,
                    uint32_t *status)
{
    int in_place = (dst == src);
    for (int p = 0; p < P; ++p) {
        const int32_t *idx = src_index + (int64_t)p * N;
        int oob = 0, hazard = 0;
        for (int n = 0; n < N; ++n) {
            int s = idx[n];
            if (s < 0 || s >= N) oob = 1;
            else if (s != n && idx[s] != s) hazard = 1;
        }
        if (status) status[p] = (oob || (in_place && hazard)) ? ORC_ST_BAD_INDEX : 0u;
        if (in_place && hazard) continue;
#pragma omp parallel for schedule(static)
        for (int64_t o = 0; o < n_outer; ++o)
            for (int n = 0; n < N; ++n) {
                int s = idx[n];
                if (s < 0 || s >= N) continue;
                if (in_place && s == n) continue;
                for (int64_t g = 0; g < seg_count; ++g) {
                    char *d = (char *)dst + o * outer_stride + p * prompt_stride + n * particle_stride + g * seg_stride;
                    const char *sp = (const char *)src + o * outer_stride + p * prompt_stride + (int64_t)s * particle_stride + g * seg_stride;
                    memcpy(d, sp, (size_t)seg_bytes);
                }
            }
    }
}
