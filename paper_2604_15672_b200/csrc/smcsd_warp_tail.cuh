// smcsd_warp_tail.cuh -- S4-S7 of one prompt with N <= 32 particles as two warp-synchronous
// routines, lane n = particle n (the small-N tail of k_tail and of the latency tail k_lt).
//
// The general S4-S7 (normalise_resample: one lane runs the prefix, a binary search per
// particle, shared-memory atomics for the offspring, loops per lane) is a long chain of
// dependent steps; with N <= 32 every per-particle quantity lives in one register of one lane
// and the tail becomes a short chain with its off-path outputs on a second warp:
//   role 0 (warp 0): S5-S7 -- M, e, the prefix P_m, C_m = P_m / S, a_n, ties, offspring, the
//                    in-place slot plan, S7 writes;
//   role 1 (warp 1): the S4 outputs -- ESS, lse, normalised weights (and the degenerate flag),
//                    recomputing M, e and the sums in the same order (bit-identical values).
// Arithmetic and order are those of normalise_resample (so the outputs are bit-identical):
// M = max lam (order-free); e_n = exp(lam_n - M) in fp64; P_m and sum e^2 sequentially in
// particle order (reading G6); ESS = S^2 / sum e^2; lse = M + ln S; C_m = P_m / S;
// a_n = #{m : C_m <= u_n} (capped at N - 1); ties = #{(n, m) : |u_n - C_m| <= 2^-40}
// (reading G7: the run of C values around u_n's boundary is exactly this set, C being
// nondecreasing); slot plan G14 (dead slots o_m = 0 in ascending m take the extra copies,
// source m repeated o_m - 1 times in ascending m).  PAPER.md:316-331 (Alg. 1, lines 9-14).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "smcsd_device.cuh"

namespace smcsd {

// What S4-S7 writes, copied to shared memory once (the routines are noinline: reading the
// kernel parameters through a pointer would be generic loads, re-issued after every store).
struct WtArgs {
    float *logw_out, *wnorm;
    double *lse, *ess;
    int32_t *ancestors, *offspring, *slot_src, *n_ties;
    uint8_t *resampled;
    double eta;
    int N, scheme;
};

struct WtSmem {
    WtArgs a;
    alignas(16) double eb[2][32];   // e of each role (16-byte broadcast reads), then C (role 0)
    alignas(16) int ib[32];         // a_n
    int ex[32];                // source of the i-th extra copy
    uint32_t st;               // ST_DEGENERATE (role 1); the caller ORs it into the status
};

__device__ __forceinline__ int wt_key(float f) {              // order-preserving float -> int
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7fffffff;
}
__device__ __forceinline__ float wt_unkey(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// Every lane: the sequential sums over e_0 .. e_{N-1} (zeros beyond N) read from eb, and
// P_lane.  Broadcast 16-byte shared loads, 8 particles per step.
__device__ __forceinline__ void wt_prefix(const double *eb, int N, int lane, double &S, double &sq, double &Pm) {
    const int N8 = (N + 7) & ~7;
    double acc = 0.0, q = 0.0, pm = 0.0;
    for (int m0 = 0; m0 < N8; m0 += 8) {
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = reinterpret_cast<const double2 *>(eb)[(m0 >> 1) + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double em = (k & 1) ? v[k >> 1].y : v[k >> 1].x;
            acc = __dadd_rn(acc, em);
            q = __dadd_rn(q, __dmul_rn(em, em));
            pm = m0 + k == lane ? acc : pm;
        }
    }
    S = acc;
    sq = q;
    Pm = pm;
}

// role 0 / role 1 of S4-S7 for prompt p (see the file comment).  lam: this lane's lam' (any
// value on lanes >= N); u: this lane's uniform (role 0); reset = fl32(-ln N).  dry != 0 runs the
// same instructions with every global store off (instruction warm-up).  Both roles must be
// called (by two different warps); the caller synchronises them before reading ws.st.
__device__ __noinline__ void warp_tail(int role, int p, int resample_mode, int dry, float lam, double u,
                                       float reset, WtSmem &ws) {
    const unsigned FULL = 0xffffffffu;
    const WtArgs A = ws.a;                                      // registers from here on
    const int N = A.N, lane = threadIdx.x & 31;
    const bool act = lane < N, out = !dry;
    const int64_t pn = (int64_t)p * N + lane;
    if (role == 0 && !resample_mode) return;
    if (role == 0) SMCSD_PHASE(0);
    // ---- S4: M = max lam (order-free: one warp reduction on order-preserving keys)
    const float Mf = wt_unkey(__reduce_max_sync(FULL, wt_key(act ? lam : -INFINITY)));
    if (Mf == -INFINITY) {                                      // degenerate prompt
        if (role == 0) {
            if (act && out) {
                A.ancestors[pn] = lane;
                if (A.offspring) A.offspring[pn] = 1;
                if (A.slot_src) A.slot_src[pn] = lane;
                A.logw_out[pn] = lam;
            }
            if (lane == 0 && out) {
                A.resampled[p] = 0;
                if (A.n_ties) A.n_ties[p] = 0;
            }
        } else {
            if (act && out && A.wnorm) A.wnorm[pn] = 0.0f;
            if (lane == 0 && out) {
                ws.st |= ST_DEGENERATE;
                if (A.lse) A.lse[p] = -INFINITY;
                if (A.ess) A.ess[p] = 0.0;
            }
        }
        return;
    }
    const double M = (double)Mf;
    // (lanes >= N take exp(0) and their divisions use S / S, so no lane sends the fp64
    // routines down their special-operand slow paths)
    const double e = exp(act ? __dsub_rn((double)lam, M) : 0.0);
    double *eb = ws.eb[role];
    eb[lane] = act ? e : 0.0;
    __syncwarp();
    double S, sq, Pm;
    wt_prefix(eb, N, lane, S, sq, Pm);
    if (role == 1) {
        // ---- S4 outputs, off the ancestors' path
        if (A.ess || dry) {
            const double ess = __ddiv_rn(__dmul_rn(S, S), sq);
            if (lane == 0 && out && A.ess) A.ess[p] = ess;
        }
        if (A.wnorm || dry) {
            const float wn = (float)__ddiv_rn(e, act ? S : e);
            if (act && out) A.wnorm[pn] = wn;
        }
        if (A.lse || dry) {
            const double l = __dadd_rn(M, log(S));
            if (lane == 0 && out) A.lse[p] = l;
        }
        __syncwarp();
        return;
    }
    if (role == 0) SMCSD_PHASE(1);
    // ---- S5: resample iff ESS < eta (ESS is finite: S >= 1, sum e^2 >= 1, so eta = +inf
    // always resamples and the division is skipped)
    const bool do_res = dry || A.eta == (double)INFINITY || __ddiv_rn(__dmul_rn(S, S), sq) < A.eta;
    if (!do_res) {
        if (act && out) {
            A.ancestors[pn] = lane;
            if (A.offspring) A.offspring[pn] = 1;
            if (A.slot_src) A.slot_src[pn] = lane;
            A.logw_out[pn] = lam;
        }
        if (lane == 0 && out) {
            A.resampled[p] = 0;
            if (A.n_ties) A.n_ties[p] = 0;
        }
        __syncwarp();
        return;
    }
    // ---- S6: C_m = P_m / S; a_n = #{m : C_m <= u_n}; ties |u_n - C_m| <= 2^-40
    const double Cq = __ddiv_rn(act ? Pm : S, S);
    __syncwarp();                                               // every lane is done with e
    eb[lane] = act ? Cq : (double)INFINITY;                    // +inf never counts
    __syncwarp();
    if (role == 0) SMCSD_PHASE(2);
    const double tie = 9.094947017729282379150390625e-13;      // 2^-40
    const int N8 = (N + 7) & ~7;
    int a = 0, ties = 0;
    for (int m0 = 0; m0 < N8; m0 += 8) {
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = reinterpret_cast<const double2 *>(eb)[(m0 >> 1) + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double Cm = (k & 1) ? v[k >> 1].y : v[k >> 1].x;
            a += Cm <= u;
            ties += fabs(__dsub_rn(u, Cm)) <= tie;
        }
    }
    a = act ? min(a, N - 1) : -1;                               // a < N always (C_{N-1} = 1 > u)
    ties = act ? ties : 0;
    ws.ib[lane] = a;
    __syncwarp();
    if (role == 0) SMCSD_PHASE(3);
    // offspring o_m = #{n : a_n = m} (a = -1 beyond N never matches)
    int o = 0;
    for (int n0 = 0; n0 < N8; n0 += 8) {
        const int4 v0 = reinterpret_cast<const int4 *>(ws.ib)[n0 >> 2];
        const int4 v1 = reinterpret_cast<const int4 *>(ws.ib)[(n0 >> 2) + 1];
        o += (v0.x == lane) + (v0.y == lane) + (v0.z == lane) + (v0.w == lane) +
             (v1.x == lane) + (v1.y == lane) + (v1.z == lane) + (v1.w == lane);
    }
    o = act ? o : 0;
    // ---- in-place slot plan (G14)
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool dead = act && o == 0;
    const int d_rank = __popc(__ballot_sync(FULL, dead) & lt_mask);
    if (A.scheme == 0) {
        // systematic: a is nondecreasing in n, so the copies of m are consecutive particles and
        // every particle after the first of its run is an extra copy -- the extras in particle
        // order are the extras in ascending source order
        const int ap = __shfl_up_sync(FULL, a, 1);
        const bool isx = act && lane > 0 && a == ap;
        const int xr = __popc(__ballot_sync(FULL, isx) & lt_mask);
        if (isx) ws.ex[xr] = a;
    } else {
        // multinomial: scan of the extra counts, source m written o_m - 1 times
        const int extra = o > 1 ? o - 1 : 0;
        int xx = extra;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int xv = __shfl_up_sync(FULL, xx, s);
            if (lane >= s) xx += xv;
        }
        for (int c = 0, x_pos = xx - extra; c < extra; ++c) ws.ex[x_pos + c] = lane;
    }
    __syncwarp();
    const int slot = dead ? ws.ex[d_rank] : lane;
    ties = __reduce_add_sync(FULL, ties);
    if (role == 0) SMCSD_PHASE(4);
    if (act && out) {                                           // S7
        A.ancestors[pn] = a;
        if (A.offspring) A.offspring[pn] = o;
        if (A.slot_src) A.slot_src[pn] = slot;
        A.logw_out[pn] = reset;
    }
    if (lane == 0 && out) {
        A.resampled[p] = 1;
        if (A.n_ties) A.n_ties[p] = ties;
    }
    __syncwarp();                                               // ws reused by the next call
    if (role == 0) SMCSD_PHASE(5);
}

}  // namespace smcsd
