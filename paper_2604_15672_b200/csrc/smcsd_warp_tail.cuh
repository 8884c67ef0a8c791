// smcsd_warp_tail.cuh -- S4-S7 of one prompt with N <= 64 particles as two warp-synchronous
// routines, lane l = particles l (and l + 32) (the small-N tail of k_tail and k_tail_small).
//
// The general S4-S7 (normalise_resample: one lane runs the prefix, a binary search per
// particle, shared-memory atomics for the offspring, loops per lane) is a long chain of
// dependent steps; with N <= 64 every per-particle quantity lives in a register of one lane (two
// particles per lane above 32) and the tail becomes a short chain with its off-path outputs on a
// second warp:
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
#include <type_traits>
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
    alignas(16) double eb[2][64];   // e of each role (16-byte broadcast reads), then C (role 0)
    double pb[64];                  // role 0: the prefix sums P_m
    alignas(16) int ib[64];         // a_n
    int ex[64];                     // source of the i-th extra copy
    uint32_t st;                    // ST_DEGENERATE (role 1); the caller ORs it into the status
};

__device__ __forceinline__ int wt_key(float f) {              // order-preserving float -> int
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7fffffff;
}
__device__ __forceinline__ float wt_unkey(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// role 0 / role 1 of S4-S7 for prompt p (see the file comment), H particles per lane: lane l
// holds particles l and l + 32 (H = 2, N <= 64) or l (H = 1, N <= 32).  lam: the prompt's lam'
// in shared memory (entries >= N are not read); u0 / u1: the uniforms of this lane's particles
// (role 0); reset = fl32(-ln N).  dry != 0 runs the same instructions with every global store
// off (instruction warm-up).  Both roles must be called (by two different warps); the caller
// synchronises them before reading ws.st.
template <int H>
__device__ __noinline__ void warp_tail(int role, int p, int resample_mode, int dry, const float *lam_s,
                                       double u0, double u1, float reset, WtSmem &ws) {
    const unsigned FULL = 0xffffffffu;
    const WtArgs A = ws.a;                                      // registers from here on
    const int N = A.N, lane = threadIdx.x & 31;
    const bool out = !dry;
    bool act[H];
    float lam[H];
    int64_t pn[H];
    const double u[2] = {u0, u1};
#pragma unroll
    for (int h = 0; h < H; ++h) {
        act[h] = lane + 32 * h < N;
        lam[h] = act[h] ? (dry ? 0.0f : lam_s[lane + 32 * h]) : -INFINITY;
        pn[h] = (int64_t)p * N + lane + 32 * h;
    }
    if (role == 0 && !resample_mode) return;
    if (role == 0) SMCSD_PHASE(0);
    // ---- S4: M = max lam (order-free: one warp reduction on order-preserving keys)
    int key = wt_key(lam[0]);
    if (H == 2) key = max(key, wt_key(lam[H - 1]));
    const float Mf = wt_unkey(__reduce_max_sync(FULL, key));
    if (Mf == -INFINITY) {                                      // degenerate prompt
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if (!act[h] || !out) continue;
            if (role == 0) {
                A.ancestors[pn[h]] = lane + 32 * h;
                if (A.offspring) A.offspring[pn[h]] = 1;
                if (A.slot_src) A.slot_src[pn[h]] = lane + 32 * h;
                A.logw_out[pn[h]] = lam[h];
            } else if (A.wnorm) {
                A.wnorm[pn[h]] = 0.0f;
            }
        }
        if (lane == 0 && out) {
            if (role == 0) {
                A.resampled[p] = 0;
                if (A.n_ties) A.n_ties[p] = 0;
            } else {
                ws.st |= ST_DEGENERATE;
                if (A.lse) A.lse[p] = -INFINITY;
                if (A.ess) A.ess[p] = 0.0;
            }
        }
        return;
    }
    const double M = (double)Mf;
    // (inactive particles take exp(0) and their divisions use S / S, so no lane sends the fp64
    // routines down their special-operand slow paths)
    double e[H];
    double *eb = ws.eb[role];
#pragma unroll
    for (int h = 0; h < H; ++h) {
        e[h] = exp(act[h] ? __dsub_rn((double)lam[h], M) : 0.0);
        eb[lane + 32 * h] = act[h] ? e[h] : 0.0;
    }
    if (H == 1) eb[lane + 32] = 0.0;                            // (N8 may reach past 32: never with H = 1)
    __syncwarp();
    // sequential fp64 sums over e_0 .. e_{N-1} in particle order (reading G6), run by every
    // lane from 16-byte broadcast shared loads.  Role 0 records each P_m in shared memory (one
    // store; lane l then reads P_l, P_{l+32}) and skips sum e^2 when eta = +inf (S5 does not
    // read it); role 1 needs sum e^2 (ESS) but not P.
    const int N8 = (N + 7) & ~7;
    double S, sq = 0.0, Pm[H];
    auto sums = [&](auto cap_t, auto sq_t) {
        constexpr bool kCap = decltype(cap_t)::value, kSq = decltype(sq_t)::value;
        double acc = 0.0, q = 0.0;
        for (int m0 = 0; m0 < N8; m0 += 8) {
            double2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = reinterpret_cast<const double2 *>(eb)[(m0 >> 1) + k];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double em = (k & 1) ? v[k >> 1].y : v[k >> 1].x;
                acc = __dadd_rn(acc, em);
                if (kSq) q = __dadd_rn(q, __dmul_rn(em, em));
                if (kCap) ws.pb[m0 + k] = acc;
            }
        }
        S = acc;
        sq = q;
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (role == 1) sums(F_{}, T_{});
    else if (A.eta == (double)INFINITY && !dry) sums(T_{}, F_{});
    else sums(T_{}, T_{});
    if (role == 0) {
        __syncwarp();
#pragma unroll
        for (int h = 0; h < H; ++h) Pm[h] = ws.pb[lane + 32 * h];
    }
    if (role == 1) {
        // ---- S4 outputs, off the ancestors' path
        if (A.ess || dry) {
            const double ess = __ddiv_rn(__dmul_rn(S, S), sq);
            if (lane == 0 && out && A.ess) A.ess[p] = ess;
        }
        if (A.wnorm || dry) {
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const float wn = (float)__ddiv_rn(e[h], act[h] ? S : e[h]);
                if (act[h] && out) A.wnorm[pn[h]] = wn;
            }
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
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if (act[h] && out) {
                A.ancestors[pn[h]] = lane + 32 * h;
                if (A.offspring) A.offspring[pn[h]] = 1;
                if (A.slot_src) A.slot_src[pn[h]] = lane + 32 * h;
                A.logw_out[pn[h]] = lam[h];
            }
        }
        if (lane == 0 && out) {
            A.resampled[p] = 0;
            if (A.n_ties) A.n_ties[p] = 0;
        }
        __syncwarp();
        return;
    }
    // ---- S6: C_m = P_m / S; a_n = #{m : C_m <= u_n}; ties |u_n - C_m| <= 2^-40
    double Cq[H];
#pragma unroll
    for (int h = 0; h < H; ++h) Cq[h] = __ddiv_rn(act[h] ? Pm[h] : S, S);
    __syncwarp();                                               // every lane is done with e
#pragma unroll
    for (int h = 0; h < H; ++h) eb[lane + 32 * h] = act[h] ? Cq[h] : (double)INFINITY;   // +inf never counts
    if (H == 1) eb[lane + 32] = (double)INFINITY;
    __syncwarp();
    if (role == 0) SMCSD_PHASE(2);
    const double tie = 9.094947017729282379150390625e-13;      // 2^-40
    int a[H], o[H], ties = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) a[h] = 0;
    // outputs nobody asked for are not computed: the tie count without n_ties, the offspring and
    // the slot plan without offspring / slot_src (uniform)
    const bool need_ties = A.n_ties != nullptr || dry, need_plan = A.offspring != nullptr || A.slot_src != nullptr || dry;
    if (H == 1) {
        // N <= 32: every lane compares its u with all C (broadcast 16-byte reads)
        for (int m0 = 0; m0 < N8; m0 += 8) {
            double2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = reinterpret_cast<const double2 *>(eb)[(m0 >> 1) + k];
            if (need_ties) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double Cm = (k & 1) ? v[k >> 1].y : v[k >> 1].x;
                    a[0] += Cm <= u[0];
                    ties += act[0] && fabs(__dsub_rn(u[0], Cm)) <= tie;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) a[0] += ((k & 1) ? v[k >> 1].y : v[k >> 1].x) <= u[0];
            }
        }
    } else {
        // 32 < N <= 64: branchless binary search of the 64 entries of C (entries >= N are +inf,
        // C is nondecreasing), both particles' searches interleaved; then the tie run around
        // the boundary (an O(log N) chain instead of 2 x N broadcast compares per lane)
        int lo[H];
#pragma unroll
        for (int h = 0; h < H; ++h) lo[h] = 0;
#pragma unroll
        for (int st = 32; st >= 1; st >>= 1) {
#pragma unroll
            for (int h = 0; h < H; ++h) lo[h] += eb[lo[h] + st - 1] <= u[h] ? st : 0;
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
            a[h] = lo[h];
            if (act[h] && need_ties) {
                for (int m = lo[h] - 1; m >= 0 && fabs(__dsub_rn(u[h], eb[m])) <= tie; --m) ++ties;
                for (int m = lo[h]; m < N && fabs(__dsub_rn(u[h], eb[m])) <= tie; ++m) ++ties;
            }
        }
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
        a[h] = act[h] ? min(a[h], N - 1) : -1;                  // a < N always (C_{N-1} = 1 > u)
        if (H == 1) ws.ib[lane + 32 * h] = a[h];
        else ws.ib[lane + 32 * h] = 0;
        o[h] = 0;
    }
    if (H == 1) ws.ib[lane + 32] = -1;
    __syncwarp();
    if (role == 0) SMCSD_PHASE(3);
    if (!need_plan) {
        ties = __reduce_add_sync(FULL, ties);
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if (act[h] && out) {                                // S7
                A.ancestors[pn[h]] = a[h];
                A.logw_out[pn[h]] = reset;
            }
        }
        if (lane == 0 && out) {
            A.resampled[p] = 1;
            if (A.n_ties) A.n_ties[p] = ties;
        }
        __syncwarp();
        return;
    }
    // offspring o_m = #{n : a_n = m}
    if (H == 1) {
        // broadcast reads of a (a = -1 beyond N never matches)
        for (int n0 = 0; n0 < N8; n0 += 8) {
            const int4 v0 = reinterpret_cast<const int4 *>(ws.ib)[n0 >> 2];
            const int4 v1 = reinterpret_cast<const int4 *>(ws.ib)[(n0 >> 2) + 1];
            o[0] += (v0.x == lane) + (v0.y == lane) + (v0.z == lane) + (v0.w == lane) +
                    (v1.x == lane) + (v1.y == lane) + (v1.z == lane) + (v1.w == lane);
        }
    } else {
        // shared-memory counts
#pragma unroll
        for (int h = 0; h < H; ++h)
            if (act[h]) atomicAdd(&ws.ib[a[h]], 1);
        __syncwarp();
#pragma unroll
        for (int h = 0; h < H; ++h) o[h] = ws.ib[lane + 32 * h];
    }
    // ---- in-place slot plan (G14): ranks over the particle order l, then l + 32
    const unsigned lt_mask = (1u << lane) - 1u;
    bool dead[H];
    int d_rank[H];
    {
        int base = 0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            o[h] = act[h] ? o[h] : 0;
            dead[h] = act[h] && o[h] == 0;
            const unsigned b = __ballot_sync(FULL, dead[h]);
            d_rank[h] = base + __popc(b & lt_mask);
            base += __popc(b);
        }
    }
    if (A.scheme == 0) {
        // systematic: a is nondecreasing in n, so the copies of m are consecutive particles and
        // every particle after the first of its run is an extra copy -- the extras in particle
        // order are the extras in ascending source order
        int base = 0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            int ap = __shfl_up_sync(FULL, a[h], 1);
            if (h == 1) {
                const int last0 = __shfl_sync(FULL, a[0], 31);
                if (lane == 0) ap = last0;
            }
            const bool isx = act[h] && (lane > 0 || h > 0) && a[h] == ap;
            const unsigned b = __ballot_sync(FULL, isx);
            if (isx) ws.ex[base + __popc(b & lt_mask)] = a[h];
            base += __popc(b);
        }
    } else {
        // multinomial: scan of the extra counts, source m written o_m - 1 times
        int base = 0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const int extra = o[h] > 1 ? o[h] - 1 : 0;
            int xx = extra;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const int xv = __shfl_up_sync(FULL, xx, s);
                if (lane >= s) xx += xv;
            }
            for (int c = 0, x_pos = base + xx - extra; c < extra; ++c) ws.ex[x_pos + c] = lane + 32 * h;
            base += __shfl_sync(FULL, xx, 31);
        }
    }
    __syncwarp();
    ties = __reduce_add_sync(FULL, ties);
    if (role == 0) SMCSD_PHASE(4);
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int slot = dead[h] ? ws.ex[d_rank[h]] : lane + 32 * h;
        if (act[h] && out) {                                    // S7
            A.ancestors[pn[h]] = a[h];
            if (A.offspring) A.offspring[pn[h]] = o[h];
            if (A.slot_src) A.slot_src[pn[h]] = slot;
            A.logw_out[pn[h]] = reset;
        }
    }
    if (lane == 0 && out) {
        A.resampled[p] = 1;
        if (A.n_ties) A.n_ties[p] = ties;
    }
    __syncwarp();                                               // ws reused by the next call
    if (role == 0) SMCSD_PHASE(5);
}

}  // namespace smcsd
