// smcsd_api.cu -- extern "C" entry points of libsmcsd.so (declared in include/smcsd.h):
// synchronous argument validation, workspace carve-up, launch configuration.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>
#include <cuda_runtime.h>

#include "smcsd.h"
#include "smcsd_kernels.cuh"
#include "smcsd_paged.cuh"
#include "smcsd_tail_small.cuh"
#include "smcsd_kv_tma.cuh"

using namespace smcsd;

namespace {

constexpr double kLog2e = 1.442695040888963407359924681001892137;
constexpr int64_t kLateClaimItemsPerCta = 32;

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

struct WsLayout {
    size_t ctr, pctr, pst, parts, ell, lam, e, c, rowstat, words, total;
};

WsLayout ws_layout(int P, int N, int K, int64_t v_len) {
    WsLayout L{};
    const size_t rows = 2ull * (size_t)P * (size_t)N * (size_t)K;
    const size_t nseg = (size_t)cdiv(v_len < 1 ? 1 : v_len, kSeg);
    size_t off = 0;
    L.ctr = off;      off += 256;
    L.pctr = off;     off += align256((size_t)P * sizeof(unsigned));
    L.pst = off;      off += align256((size_t)P * sizeof(uint32_t));
    L.parts = off;    off += align256((rows + (size_t)P * N) * nseg * sizeof(float4));  // + bonus rows
    L.ell = off;      off += align256(rows * sizeof(double));
    L.lam = off;      off += align256((size_t)P * N * sizeof(float));
    L.e = off;        off += align256((size_t)P * N * sizeof(double));
    L.c = off;        off += align256((size_t)P * N * sizeof(double));
    L.rowstat = off;  off += align256(rows * sizeof(float4));
    L.words = off;    off += align256(rows * nseg * sizeof(unsigned long long));   // LT words
    L.total = off;
    return L;
}

void bind_workspace(Params &prm, void *ws, const WsLayout &L) {
    char *b = static_cast<char *>(ws);
    prm.part_ws = reinterpret_cast<float4 *>(b + L.parts);
    prm.ell_ws = reinterpret_cast<double *>(b + L.ell);
    prm.lam_ws = reinterpret_cast<float *>(b + L.lam);
    prm.e_ws = reinterpret_cast<double *>(b + L.e);
    prm.c_ws = reinterpret_cast<double *>(b + L.c);
    prm.rowstat_ws = reinterpret_cast<float4 *>(b + L.rowstat);
    prm.work_ctr = reinterpret_cast<unsigned *>(b + L.ctr);
    prm.prompt_ctr = reinterpret_cast<unsigned *>(b + L.pctr);
    prm.st_ws = reinterpret_cast<uint32_t *>(b + L.pst);
    prm.xctr = reinterpret_cast<unsigned *>(b + L.ctr + 64);
    prm.lt_words = nullptr;                     // set by tail_mode() for the polling tails
}


bool valid_temp(float t) { return std::isfinite(t) && t > 0.0f; }

// Validation shared by weights / step / partial.  Returns SMCSD_OK or SMCSD_EINVAL.
smcsd_rc check_logits(const void *lp, int64_t ld_p, int rpp_p, const void *lq, int64_t ld_q,
                      int rpp_q, int dtype, const int32_t *tokens, int P, int N, int K,
                      int64_t v_len) {
    if (!lp || !lq || !tokens) return SMCSD_EINVAL;
    if (P < 1 || N < 1 || K < 1 || v_len < 1) return SMCSD_EINVAL;
    if (dtype != SMCSD_F32 && dtype != SMCSD_BF16) return SMCSD_EINVAL;
    const int64_t vec = dtype == SMCSD_BF16 ? 8 : 4;
    if (ld_p < v_len || ld_q < v_len || ld_p % vec || ld_q % vec) return SMCSD_EINVAL;
    if (rpp_p < K || rpp_q < K) return SMCSD_EINVAL;
    if (!aligned16(lp) || !aligned16(lq)) return SMCSD_EINVAL;
    const int64_t items = 2ll * P * N * K * cdiv(v_len, kSeg);
    if (items >= (1ll << 31)) return SMCSD_EINVAL;
    return SMCSD_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel may start while its
// predecessor in the stream drains; it calls griddepcontrol.wait before touching that
// predecessor's outputs.
template <typename... KArgs, typename... Args>
smcsd_rc launch_pdl_b(void (*kernel)(KArgs...), unsigned grid, size_t smem, cudaStream_t st,
                      unsigned block, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...) == cudaSuccess
               ? SMCSD_OK : SMCSD_ECUDA;
}

// PDL launch with a 1-D thread-block cluster of `cluster` CTAs (grid a multiple of it).
template <typename... KArgs, typename... Args>
smcsd_rc launch_pdl_cluster(void (*kernel)(KArgs...), unsigned grid, unsigned cluster, cudaStream_t st,
                            Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...) == cudaSuccess
               ? SMCSD_OK : SMCSD_ECUDA;
}

template <typename... KArgs, typename... Args>
smcsd_rc launch_pdl_2d(void (*kernel)(KArgs...), dim3 grid, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...) == cudaSuccess
               ? SMCSD_OK : SMCSD_ECUDA;
}

template <typename... KArgs, typename... Args>
smcsd_rc launch_pdl(void (*kernel)(KArgs...), unsigned grid, size_t smem, cudaStream_t st,
                    Args &&...args) {
    return launch_pdl_b(kernel, grid, smem, st, (unsigned)kThreads, std::forward<Args>(args)...);
}

// K1 persistent grid: SMs x resident CTAs (shared-memory ring), capped by the work items.
// Resident CTAs of K1 variant <DT, PW, XP> on the current device (SMs x CTAs per SM; cached,
// with the kernel's shared-memory attributes set on first use), or 0 on a CUDA error.
template <int DT, int PW, bool XP = false>
int k1_ctas() {
    static int ctas[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    if (ctas[dev] == 0) {
        const size_t smem = rowstats_smem_bytes<DT, XP>();
        int occ = 0, sms = 0;
        if (cudaFuncSetAttribute(k_rowstats<DT, PW, XP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            cudaFuncSetAttribute(k_rowstats<DT, PW, XP>, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rowstats<DT, PW, XP>, kK1Threads, smem) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || occ < 1)
            return 0;
        ctas[dev] = occ * sms;
    }
    return ctas[dev];
}

template <int DT, int PW, bool XP = false>
smcsd_rc launch_rowstats_dt(const Params &prm, int64_t items, cudaStream_t st) {
    const int ctas = k1_ctas<DT, PW, XP>();
    if (ctas == 0) return SMCSD_ECUDA;
    const size_t smem = rowstats_smem_bytes<DT, XP>();
    const int64_t grid = items < ctas ? items : ctas;
    // latency-bound streams (<= kLateClaimItemsPerCta items per CTA) claim items late
    // (profiles/r02v_ab_late_claim.txt: cfg2 -0.3 us; long streams +1-3 % with it, so not there)
    Params p2 = prm;
    p2.late_claim = items <= kLateClaimItemsPerCta * grid;
    return launch_pdl_b(k_rowstats<DT, PW, XP>, (unsigned)grid, smem, st, (unsigned)kK1Threads, p2);
}

// K2 tail: one CTA per 32 (particle, position) pairs of each prompt (k_tail), or one CTA per
// prompt with the rows' statistics in the workspace for N > kTailMaxN (k_tail_large).
// One-time (per device) opt-in to the dynamic shared memory the K2 kernels stage through.
smcsd_rc ensure_tail_attrs() {
    static bool attr_set[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SMCSD_ECUDA;
    if (!attr_set[dev]) {
        if (cudaFuncSetAttribute(k_tail_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailStageBytes) != cudaSuccess)
            return SMCSD_ECUDA;
        // clusters of up to 16 chunk CTAs (non-portable size; 4 SMs at 4 CTAs per SM)
        if (cudaFuncSetAttribute(k_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            return SMCSD_ECUDA;
        attr_set[dev] = true;
    }
    return SMCSD_OK;
}

// Polling tail, N <= 64, N K <= 512 pairs (<= 16 CTAs of 16 or 32 pairs per prompt), no bonus rows:
// k_tail_small (smcsd_tail_small.cuh), resident beside K1 from the start of its stream.
#ifndef SMCSD_NO_TAIL_SMALL
int g_tail_small = 1;
#else
int g_tail_small = 0;
#endif

smcsd_rc launch_tail_small(const Params &prm, int resample_mode, int chunks, cudaStream_t st) {
    static bool attr_set[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SMCSD_ECUDA;
    if (!attr_set[dev]) {
        // the SM configuration K1's CTAs run under must admit these CTAs beside them
        for (auto *k : {k_tail_small<4, 1>, k_tail_small<4, 2>, k_tail_small<2, 1>, k_tail_small<2, 2>})
            if (cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess ||
                cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
                return SMCSD_ECUDA;
        attr_set[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(prm.P * chunks));
    cfg.blockDim = dim3(kTsThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)chunks;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const int64_t nk = (int64_t)prm.N * prm.K;
    const bool l4 = nk <= 16ll * kTsMaxChunks, h1 = prm.N <= 32;
    auto *k = l4 ? (h1 ? k_tail_small<4, 1> : k_tail_small<4, 2>) : (h1 ? k_tail_small<2, 1> : k_tail_small<2, 2>);
    // the CTAs poll K1's words only once K1's work counter shows every item claimed (gate_ctr)
    Params p2 = prm;
    const int64_t ctas = prm.dtype == SMCSD_BF16 ? k1_ctas<1, 0>() : k1_ctas<0, 0>();
    const int64_t items = prm.main_items + prm.bonus_items, k1_grid = items < ctas ? items : ctas;
    p2.gate_ctr = (unsigned)(items - k1_grid);
    return cudaLaunchKernelEx(&cfg, k, p2, resample_mode, chunks) == cudaSuccess ? SMCSD_OK : SMCSD_ECUDA;
}

smcsd_rc launch_tail(const Params &prm, int resample_mode, cudaStream_t st) {
    if (ensure_tail_attrs() != SMCSD_OK) return SMCSD_ECUDA;
    if (prm.N > kTailMaxN) return launch_pdl(k_tail_large, (unsigned)prm.P, kTailStageBytes, st, prm);
    if (g_tail_small && prm.lt_words && !prm.bonus_tok && prm.x_from_logits && prm.N <= kTsMaxN && prm.nseg <= 16) {
        // 16 pairs per CTA (4 lanes per row) up to N K = 256, else 32 (2 lanes per row)
        const int64_t nk = (int64_t)prm.N * prm.K;
        const int cs = (int)cdiv(nk, nk <= 16ll * kTsMaxChunks ? 16 : 32);
        if (cs <= kTsMaxChunks && (int64_t)prm.P * cs < (1ll << 31)) return launch_tail_small(prm, resample_mode, cs, st);
    }
    const int chunks = (int)cdiv((int64_t)prm.N * prm.K, kPairsPerCta);
    const int bonus_ctas = prm.bonus_tok ? prm.N : 0;
    const int64_t grid = (int64_t)prm.P * chunks + (int64_t)prm.P * bonus_ctas;
    if (grid >= (1ll << 31)) return SMCSD_EINVAL;
    // one prompt's chunk CTAs as one thread-block cluster (up to 16): their completion is a
    // cluster barrier instead of the per-prompt counter.  Bonus CTAs (after all chunk CTAs)
    // must fill whole clusters of their own: P * N a multiple of chunks.
#ifndef SMCSD_NO_CLUSTER_TAIL
    const bool cl = chunks >= 2 && chunks <= 16 && (bonus_ctas == 0 || ((int64_t)prm.P * prm.N) % chunks == 0);
#else
    const bool cl = false;
#endif
    if (cl) return launch_pdl_cluster(k_tail, (unsigned)grid, (unsigned)chunks, st, prm, resample_mode, chunks, bonus_ctas, 1);
    return launch_pdl(k_tail, (unsigned)grid, 0, st, prm, resample_mode, chunks, bonus_ctas, 0);
}

#ifndef SMCSD_NO_POLL_TAIL
int g_poll_tail = 1;                             // smcsd_set_poll_tail
#else
int g_poll_tail = 0;
#endif

// Tail modes of smcsd_step / smcsd_weights:
//   TAIL_POLL  -- K1 publishes {m, s} words (prm.lt_words) and launches its dependents at once;
//                 the tail (k_tail_small when it applies, else k_tail) polls the words instead
//                 of waiting for K1's grid (no bonus rows, at most 16 segments per row);
//   TAIL_WAIT  -- k_tail behind griddepcontrol.wait on K1's float4 partials (every other call).
enum TailMode { TAIL_WAIT = 0, TAIL_POLL = 1 };

TailMode tail_mode(Params &prm, void *ws, const WsLayout &L) {
    prm.lt_words = nullptr;
    const bool common = !prm.bonus_tok && !prm.xpeer && prm.x_from_logits && prm.n_models == 2;
    TailMode m = TAIL_WAIT;
    if (common && g_poll_tail && prm.nseg <= 16 && prm.N <= kTailMaxN &&
             prm.main_items <= kLateClaimItemsPerCta * (int64_t)(prm.dtype == SMCSD_BF16 ? k1_ctas<1, 0>() : k1_ctas<0, 0>()))
        m = TAIL_POLL;                   // latency-bound steps only (cfg4-sized streams: +10 us)
    if (m != TAIL_WAIT) prm.lt_words = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + L.words);
    return m;
}


template <int PW>
smcsd_rc launch_rowstats_pw(const Params &prm, int dtype, int64_t items, cudaStream_t st) {
    return dtype == SMCSD_BF16 ? launch_rowstats_dt<1, PW>(prm, items, st)
                               : launch_rowstats_dt<0, PW>(prm, items, st);
}

// power: 0 = plain row statistics; otherwise PowerSMC's second sum, with integer alpha in
// 1..4 taken by repeated multiplication of the first sum's ex2 (see pow_acc), half-integer
// alpha in 0.5..3.5 from one ex2 of t/2 (see half_pow), any other alpha by a second exp.
smcsd_rc launch_rowstats(const Params &prm, int dtype, int64_t items, cudaStream_t st,
                         bool power = false) {
    if (prm.xpeer)                                             // S10 fused exchange
        return dtype == SMCSD_BF16 ? launch_rowstats_dt<1, 0, true>(prm, items, st)
                                   : launch_rowstats_dt<0, 0, true>(prm, items, st);
    if (!power) return launch_rowstats_pw<0>(prm, dtype, items, st);
    const float a = prm.alpha_f;
    if (a == 1.0f) return launch_rowstats_pw<1>(prm, dtype, items, st);
    if (a == 2.0f) return launch_rowstats_pw<2>(prm, dtype, items, st);
    if (a == 3.0f) return launch_rowstats_pw<3>(prm, dtype, items, st);
    if (a == 4.0f) return launch_rowstats_pw<4>(prm, dtype, items, st);
    if (a == 0.5f) return launch_rowstats_pw<10>(prm, dtype, items, st);     // half-integer:
    if (a == 1.5f) return launch_rowstats_pw<11>(prm, dtype, items, st);     // one ex2 per element
    if (a == 2.5f) return launch_rowstats_pw<12>(prm, dtype, items, st);
    if (a == 3.5f) return launch_rowstats_pw<13>(prm, dtype, items, st);
    return launch_rowstats_pw<-1>(prm, dtype, items, st);
}

// Magic multiplier for division by d (1 <= d < 2^31): x / d == (x * mg) >> (32 + sh) for
// every x < 2^31, with sh = ceil(log2 d) and mg = ceil(2^(32+sh) / d) < 2^33.
void set_magic(int d, unsigned long long &mg, int &sh) {
    sh = 0;
    while ((1ll << sh) < d) ++sh;
    const unsigned __int128 num = (unsigned __int128)1 << (32 + sh);
    mg = (unsigned long long)((num + (unsigned)d - 1) / (unsigned)d);
}

// Common Params for the logits entry points.
Params logits_params(const void *lp, int64_t ld_p, int rpp_p, const void *lq, int64_t ld_q,
                     int rpp_q, const int32_t *tokens, const int32_t *n_drafted, int P, int N,
                     int K, int64_t V, int64_t v_begin, int64_t v_len, float tp, float tq) {
    Params prm;
    std::memset(&prm, 0, sizeof prm);
    prm.lp = static_cast<const char *>(lp); prm.ld_p = ld_p; prm.rpp_p = rpp_p;
    prm.lq = static_cast<const char *>(lq); prm.ld_q = ld_q; prm.rpp_q = rpp_q;
    prm.tokens = tokens; prm.n_drafted = n_drafted;
    prm.P = P; prm.N = N; prm.K = K; prm.V = V;
    prm.v_begin = v_begin; prm.v_len = v_len;
    prm.nseg = (int)cdiv(v_len, kSeg);
    prm.c_p = (float)((double)tp * kLog2e);
    prm.c_q = (float)((double)tq * kLog2e);
    prm.alpha = 1.0;
    set_magic(prm.nseg, prm.mg_nseg, prm.sh_nseg);
    set_magic(K, prm.mg_K, prm.sh_K);
    set_magic(N, prm.mg_N, prm.sh_N);
    prm.x_from_logits = 1;
    prm.n_models = 2;
    prm.alpha_f = 1.0f;
    prm.main_items = 2ll * P * N * K * prm.nseg;
    prm.bonus_items = 0;
    return prm;
}

}  // namespace

extern "C" {

size_t smcsd_workspace_bytes(int P, int N, int K, int64_t v_len) {
    if (P < 1 || N < 1 || K < 1) return 0;
    return ws_layout(P, N, K, v_len).total;
}

smcsd_rc smcsd_workspace_init(void *workspace, size_t workspace_bytes, void *stream) {
    if (!workspace) return SMCSD_EINVAL;
    return cudaMemsetAsync(workspace, 0, workspace_bytes, as_stream(stream)) == cudaSuccess
               ? SMCSD_OK : SMCSD_ECUDA;
}

smcsd_rc smcsd_weights(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                       const void *logits_q, int64_t ld_q, int rows_per_particle_q, int dtype,
                       const int32_t *tokens, const int32_t *n_drafted, const float *logw_prev,
                       int P, int N, int K, int64_t V, float alpha, float inv_temp_p,
                       float inv_temp_q, float *logw_out, float *logp_tok, float *logq_tok,
                       double *lse_out, double *ess_out, float *wnorm_out, uint32_t *status,
                       void *workspace, size_t workspace_bytes, void *stream) {
    smcsd_rc rc = check_logits(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, dtype, tokens, P, N, K, V);
    if (rc != SMCSD_OK) return rc;
    if (!logw_out || !status || !workspace) return SMCSD_EINVAL;
    if (!(std::isfinite(alpha) && alpha > 0.0f) || !valid_temp(inv_temp_p) || !valid_temp(inv_temp_q))
        return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, K, V);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    Params prm = logits_params(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, tokens, n_drafted, P, N, K, V, 0, V,
                               inv_temp_p, inv_temp_q);
    prm.alpha = (double)alpha;
    prm.dtype = dtype;
    prm.logw_prev = logw_prev;
    prm.logw_out = logw_out; prm.logp_tok = logp_tok; prm.logq_tok = logq_tok;
    prm.lse = lse_out; prm.ess = ess_out; prm.wnorm = wnorm_out; prm.status = status;
    bind_workspace(prm, workspace, L);
    prm.parts = prm.part_ws; prm.part_row_stride = prm.nseg; prm.part_seg_stride = 1;
    prm.nparts = prm.nseg;
    const int64_t items = 2ll * P * N * K * prm.nseg;
    cudaStream_t st = as_stream(stream);
    const TailMode tm = tail_mode(prm, workspace, L);
    rc = launch_rowstats(prm, dtype, items, st);
    if (rc != SMCSD_OK) return rc;
    (void)tm;
    return launch_tail(prm, 0, st);
}

smcsd_rc smcsd_resample(const float *logw, int P, int N, int64_t prompt_base, float eta,
                        int scheme, uint64_t seed, uint64_t step, const uint32_t *uniforms,
                        int32_t *ancestors, int32_t *offspring, int32_t *slot_src,
                        float *logw_out, uint8_t *resampled, double *ess_out, double *lse_out,
                        float *wnorm_out, int32_t *n_ties, uint32_t *status, void *stream) {
    if (!logw || !ancestors || !logw_out || !resampled || !status) return SMCSD_EINVAL;
    if (P < 1 || N < 1 || N > kTailMaxN || std::isnan(eta)) return SMCSD_EINVAL;
    if (scheme != SMCSD_SYSTEMATIC && scheme != SMCSD_MULTINOMIAL) return SMCSD_EINVAL;
    Params prm;
    std::memset(&prm, 0, sizeof prm);
    prm.P = P; prm.N = N;
    prm.logw_prev = logw;
    prm.eta = (double)eta; prm.seed = seed; prm.step = step; prm.prompt_base = prompt_base;
    prm.uniforms = uniforms; prm.scheme = scheme;
    prm.ancestors = ancestors; prm.offspring = offspring; prm.slot_src = slot_src;
    prm.logw_out = logw_out; prm.resampled = resampled; prm.ess = ess_out; prm.lse = lse_out;
    prm.wnorm = wnorm_out; prm.n_ties = n_ties; prm.status = status;
    return launch_pdl(k_resample, (unsigned)P, 0, as_stream(stream), prm);
}

smcsd_rc smcsd_step(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                    const void *logits_q, int64_t ld_q, int rows_per_particle_q, int dtype,
                    const int32_t *tokens, const int32_t *n_drafted, const float *logw_prev,
                    int P, int N, int K, int64_t V, float alpha, float inv_temp_p,
                    float inv_temp_q, float eta, int scheme, uint64_t seed, uint64_t step,
                    int64_t prompt_base, const uint32_t *uniforms, float *logw_out,
                    float *logw_pre, float *logp_tok, float *logq_tok, double *lse_out,
                    double *ess_out, float *wnorm_out, uint32_t *status, int32_t *ancestors,
                    int32_t *offspring, int32_t *slot_src, uint8_t *resampled, int32_t *n_ties,
                    int32_t *bonus_tok, void *workspace, size_t workspace_bytes, void *stream) {
    smcsd_rc rc = check_logits(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, dtype, tokens, P, N, K, V);
    if (rc != SMCSD_OK) return rc;
    if (!logw_out || !status || !ancestors || !resampled || !workspace) return SMCSD_EINVAL;
    if (bonus_tok && (rows_per_particle_p < K + 1 || cdiv(V, kSeg) > kBonusMaxSeg ||
                      (2ll * K + 1) * P * N * cdiv(V, kSeg) >= (1ll << 31)))
        return SMCSD_EINVAL;
    if (N > kTailMaxN || std::isnan(eta)) return SMCSD_EINVAL;
    if (!(std::isfinite(alpha) && alpha > 0.0f) || !valid_temp(inv_temp_p) || !valid_temp(inv_temp_q))
        return SMCSD_EINVAL;
    if (scheme != SMCSD_SYSTEMATIC && scheme != SMCSD_MULTINOMIAL) return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, K, V);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    // logw_prev may alias logw_out: the tail reads lam_prev[n] before any S7 write.
    Params prm = logits_params(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, tokens, n_drafted, P, N, K, V, 0, V,
                               inv_temp_p, inv_temp_q);
    prm.alpha = (double)alpha;
    prm.dtype = dtype;
    prm.logw_prev = logw_prev;
    prm.eta = (double)eta; prm.seed = seed; prm.step = step; prm.prompt_base = prompt_base;
    prm.uniforms = uniforms; prm.scheme = scheme;
    prm.logw_out = logw_out; prm.logw_pre = logw_pre; prm.logp_tok = logp_tok;
    prm.logq_tok = logq_tok; prm.lse = lse_out; prm.ess = ess_out; prm.wnorm = wnorm_out;
    prm.status = status; prm.ancestors = ancestors; prm.offspring = offspring;
    prm.slot_src = slot_src; prm.resampled = resampled; prm.n_ties = n_ties;
    prm.bonus_tok = bonus_tok;
    if (bonus_tok) prm.bonus_items = (long long)P * N * prm.nseg;
    bind_workspace(prm, workspace, L);
    prm.parts = prm.part_ws; prm.part_row_stride = prm.nseg; prm.part_seg_stride = 1;
    prm.nparts = prm.nseg;
    cudaStream_t st = as_stream(stream);
    const TailMode tm = tail_mode(prm, workspace, L);
    rc = launch_rowstats(prm, dtype, prm.main_items + prm.bonus_items, st);
    if (rc != SMCSD_OK) return rc;
    (void)tm;
    return launch_tail(prm, 1, st);
}

smcsd_rc smcsd_weights_partial(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                               const void *logits_q, int64_t ld_q, int rows_per_particle_q,
                               int dtype, const int32_t *tokens, const int32_t *n_drafted,
                               int P, int N, int K, int64_t v_begin, int64_t v_len,
                               float inv_temp_p, float inv_temp_q, float *partials,
                               void *workspace, size_t workspace_bytes, void *stream) {
    smcsd_rc rc = check_logits(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, dtype, tokens, P, N, K, v_len);
    if (rc != SMCSD_OK) return rc;
    if (!partials || !workspace || v_begin < 0 || !aligned16(partials)) return SMCSD_EINVAL;
    if (!valid_temp(inv_temp_p) || !valid_temp(inv_temp_q)) return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, K, v_len);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    Params prm = logits_params(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, tokens, n_drafted, P, N, K,
                               v_begin + v_len, v_begin, v_len, inv_temp_p, inv_temp_q);
    prm.partials_out = reinterpret_cast<float4 *>(partials);
    prm.dtype = dtype;
    bind_workspace(prm, workspace, L);
    prm.parts = prm.part_ws; prm.part_row_stride = prm.nseg; prm.part_seg_stride = 1;
    prm.nparts = prm.nseg;
    cudaStream_t st = as_stream(stream);
    rc = launch_rowstats(prm, dtype, 2ll * P * N * K * prm.nseg, st);
    if (rc != SMCSD_OK) return rc;
    const int64_t grid = (int64_t)P * cdiv(2ll * N * K, kMergeRowsPerCta);
    if (grid >= (1ll << 31)) return SMCSD_EINVAL;
    return launch_pdl(k_merge_rows, (unsigned)grid, 0, st, prm);
}

smcsd_rc smcsd_weights_combine(const float *gathered, int G, const int32_t *tokens,
                               const int32_t *n_drafted, const float *logw_prev, int P, int N,
                               int K, int64_t V, float alpha, float *logw_out, float *logp_tok,
                               float *logq_tok, double *lse_out, double *ess_out,
                               float *wnorm_out, uint32_t *status, void *workspace,
                               size_t workspace_bytes, void *stream) {
    if (!gathered || !tokens || !logw_out || !status || !workspace) return SMCSD_EINVAL;
    if (G < 1 || P < 1 || N < 1 || K < 1 || V < 1 || N > kTailMaxN) return SMCSD_EINVAL;
    if (!(std::isfinite(alpha) && alpha > 0.0f) || !aligned16(gathered)) return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, K, 1);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    Params prm;
    std::memset(&prm, 0, sizeof prm);
    prm.tokens = tokens; prm.n_drafted = n_drafted; prm.logw_prev = logw_prev;
    prm.P = P; prm.N = N; prm.K = K; prm.V = V; prm.alpha = (double)alpha;
    prm.logw_out = logw_out; prm.logp_tok = logp_tok; prm.logq_tok = logq_tok;
    prm.lse = lse_out; prm.ess = ess_out; prm.wnorm = wnorm_out; prm.status = status;
    bind_workspace(prm, workspace, L);
    prm.parts = reinterpret_cast<const float4 *>(gathered);
    prm.part_row_stride = 1;
    prm.part_seg_stride = 2ll * P * N * K;
    prm.nparts = G;
    return launch_tail(prm, 0, as_stream(stream));
}

smcsd_rc smcsd_partials_rescale(const float *partials, const float *max_partials, float *out,
                                int64_t rows, void *stream) {
    if (!partials || !max_partials || !out || rows < 1) return SMCSD_EINVAL;
    if (!aligned16(partials) || !aligned16(max_partials) || !aligned16(out)) return SMCSD_EINVAL;
    const int64_t grid = std::min<int64_t>(cdiv(rows, kThreads), 4 * 148);
    k_partials_rescale<<<(unsigned)grid, kThreads, 0, as_stream(stream)>>>(
        reinterpret_cast<const float4 *>(partials), reinterpret_cast<const float4 *>(max_partials),
        reinterpret_cast<float4 *>(out), rows);
    return cudaGetLastError() == cudaSuccess ? SMCSD_OK : SMCSD_ECUDA;
}

smcsd_rc smcsd_kv_reindex_multi(const smcsd_kv_tensor *tensors, int n_tensors,
                                const int32_t *src_index, int P, int N, uint32_t *status,
                                void *stream) {
    if (!tensors || !src_index || n_tensors < 1 || n_tensors > kMaxKvTensors) return SMCSD_EINVAL;
    if (P < 1 || N < 1 || N > kTailMaxN) return SMCSD_EINVAL;
    KvParams prm;
    std::memset(&prm, 0, sizeof prm);
    prm.idx = src_index; prm.P = P; prm.N = N; prm.n_tensors = n_tensors; prm.status = status;
    // bulk-copy kernel (smcsd_kv_tma.cuh) for N <= 256
#ifndef SMCSD_NO_KV_TMA
    const bool use_tma = N <= kKvTmaMaxN;
#else
    const bool use_tma = false;
#endif
    int64_t items = 0;
    for (int k = 0; k < n_tensors; ++k) {
        const smcsd_kv_tensor &a = tensors[k];
        if (!a.dst || !a.src) return SMCSD_EINVAL;
        if (a.n_outer < 1 || a.seg_count < 1 || a.seg_bytes < 16) return SMCSD_EINVAL;
        if (!aligned16(a.dst) || !aligned16(a.src)) return SMCSD_EINVAL;
        if ((a.seg_bytes | a.outer_stride | a.prompt_stride | a.particle_stride | a.seg_stride) & 15)
            return SMCSD_EINVAL;
        if (a.outer_stride < 0 || a.prompt_stride < 0 || a.particle_stride < 0 || a.seg_stride < 0)
            return SMCSD_EINVAL;
        const uint64_t vps = (uint64_t)a.seg_bytes / 16;
        if (vps >= (1ull << 32)) return SMCSD_EINVAL;
        KvTensor &t = prm.t[k];
        t.dst = static_cast<char *>(a.dst);
        t.src = static_cast<const char *>(a.src);
        t.outer_stride = a.outer_stride; t.prompt_stride = a.prompt_stride;
        t.particle_stride = a.particle_stride; t.seg_stride = a.seg_stride;
        t.vps = (uint32_t)vps;
        t.in_place = a.dst == a.src;
        prm.any_in_place |= t.in_place;
        t.vecs = (uint64_t)a.seg_count * vps;
        t.nchunks = use_tma ? (int64_t)a.seg_count * cdiv(a.seg_bytes, kKvTmaChunk)
                            : (int64_t)cdiv((int64_t)t.vecs, kKvChunkVec);
        items += a.n_outer * P * t.nchunks;
        if (items >= (1ll << 31)) return SMCSD_EINVAL;
        t.item_end = items;
    }
    if (use_tma) {
        static bool attr_set[64] = {false};
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SMCSD_ECUDA;
        if (!attr_set[dev]) {
            if (cudaFuncSetAttribute(k_kv_reindex_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kKvTmaBufs * kKvTmaChunk) != cudaSuccess ||
                cudaFuncSetAttribute(k_kv_reindex_tma_w, cudaFuncAttributeMaxDynamicSharedMemorySize, kKvTmaBufs * kKvTmaChunk) != cudaSuccess)
                return SMCSD_ECUDA;
            attr_set[dev] = true;
        }
#ifndef SMCSD_NO_KV_TMA_WARP
        if (N <= 32)
            return launch_pdl_b(k_kv_reindex_tma_w, (unsigned)items, kKvTmaBufs * kKvTmaChunk, as_stream(stream), 32u, prm);
#endif
        return launch_pdl(k_kv_reindex_tma, (unsigned)items, kKvTmaBufs * kKvTmaChunk, as_stream(stream), prm);
    }
    return launch_pdl(k_kv_reindex, (unsigned)items, 0, as_stream(stream), prm);
}

smcsd_rc smcsd_kv_reindex(void *dst, const void *src, int64_t n_outer, int64_t outer_stride,
                          int64_t prompt_stride, int64_t particle_stride, int64_t seg_count,
                          int64_t seg_bytes, int64_t seg_stride, const int32_t *src_index,
                          int P, int N, uint32_t *status, void *stream) {
    const smcsd_kv_tensor t = {dst, src, n_outer, outer_stride, prompt_stride, particle_stride,
                               seg_count, seg_bytes, seg_stride};
    return smcsd_kv_reindex_multi(&t, 1, src_index, P, N, status, stream);
}

smcsd_rc smcsd_select(const float *logw, int P, int N, int64_t prompt_base, uint64_t seed,
                      uint64_t step, const uint32_t *uniforms, int32_t *selected, uint32_t *status,
                      void *workspace, size_t workspace_bytes, void *stream) {
    if (!logw || !selected || !status || !workspace || P < 1 || N < 1) return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, 1, 1);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    Params prm;
    std::memset(&prm, 0, sizeof prm);
    prm.P = P; prm.N = N; prm.K = 1;
    prm.logw_prev = logw; prm.prompt_base = prompt_base; prm.seed = seed; prm.step = step;
    prm.uniforms = uniforms; prm.selected = selected; prm.status = status;
    bind_workspace(prm, workspace, L);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)P);
    cfg.blockDim = dim3(32);
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_select, prm) == cudaSuccess ? SMCSD_OK : SMCSD_ECUDA;
}

smcsd_rc smcsd_kv_reindex_paged(const int32_t *table_src, const int32_t *n_pages_src,
                                int32_t *table_dst, int32_t *n_pages_dst, int32_t *refcount,
                                uint8_t *freed, const int32_t *src_index, int P, int N,
                                int max_pages, int num_pages, uint32_t *status, void *stream) {
    if (!table_src || !n_pages_src || !table_dst || !n_pages_dst || !refcount || !src_index)
        return SMCSD_EINVAL;
    if (P < 1 || N < 1 || max_pages < 1 || num_pages < 1) return SMCSD_EINVAL;
    if (table_src == table_dst || n_pages_src == n_pages_dst) return SMCSD_EINVAL;
    PagedParams q;
    q.table_src = table_src; q.n_src = n_pages_src; q.idx = src_index;
    q.table_dst = table_dst; q.n_dst = n_pages_dst; q.refcount = refcount;
    q.freed = freed; q.status = status;
    q.P = P; q.N = N; q.max_pages = max_pages; q.num_pages = num_pages;
    cudaStream_t st = as_stream(stream);
    if ((int64_t)N * max_pages >= (1ll << 31) || P > 65535) return SMCSD_EINVAL;
    if (status && cudaMemsetAsync(status, 0, (size_t)P * sizeof(uint32_t), st) != cudaSuccess) return SMCSD_ECUDA;
    const dim3 grid((unsigned)cdiv((int64_t)N * max_pages, kThreads), (unsigned)P);
    smcsd_rc rc = launch_pdl_2d(k_paged_gather, grid, st, q);
    if (rc != SMCSD_OK || !freed) return rc;
    return launch_pdl_2d(k_paged_freed, grid, st, q);
}

size_t smcsd_kv_append_workspace_bytes(int P, int N, int num_pages, int max_pages) {
    if (P < 1 || N < 1 || num_pages < 1 || max_pages < 1) return 0;
    const size_t chunks = (size_t)cdiv(num_pages, kFreeChunk);
    return align256(2 * (size_t)num_pages * 4) + align256(chunks * 4) + align256((size_t)P * N * 4) +
           align256((size_t)P * N * (size_t)(max_pages + 1) * 4);
}

smcsd_rc smcsd_kv_append_paged(int32_t *table, int32_t *n_pages, int32_t *seq_len, int32_t *refcount,
                               const int32_t *n_new, int P, int N, int max_pages, int num_pages,
                               int page_size, int max_new, int32_t *slot_mapping, int32_t *cow_src,
                               int32_t *cow_dst, int32_t *cow_tokens, uint32_t *status,
                               int32_t *result, const smcsd_kv_pool *pools, int n_pools,
                               void *workspace, size_t workspace_bytes, void *stream) {
    if (!table || !n_pages || !seq_len || !refcount || !n_new || !slot_mapping || !cow_src ||
        !cow_dst || !cow_tokens || !status || !result || !workspace)
        return SMCSD_EINVAL;
    if (P < 1 || N < 1 || max_pages < 1 || num_pages < 1 || page_size < 1 || max_new < 1)
        return SMCSD_EINVAL;
    if ((int64_t)num_pages * page_size >= (1ll << 31) || (int64_t)P * N >= (1 << 24)) return SMCSD_EINVAL;
    if (n_pools < 0 || n_pools > kMaxPools || (n_pools > 0 && !pools)) return SMCSD_EINVAL;
    if (workspace_bytes < smcsd_kv_append_workspace_bytes(P, N, num_pages, max_pages) || !aligned16(workspace))
        return SMCSD_EINVAL;
    AppendParams q;
    std::memset(&q, 0, sizeof q);
    q.table = table; q.n_pages = n_pages; q.seq_len = seq_len; q.refcount = refcount; q.n_new = n_new;
    q.P = P; q.N = N; q.max_pages = max_pages; q.num_pages = num_pages; q.page_size = page_size;
    q.max_new = max_new; q.slot_mapping = slot_mapping; q.cow_src = cow_src; q.cow_dst = cow_dst;
    q.cow_tokens = cow_tokens; q.status = status; q.result = result;
    q.nchunks = (int)cdiv(num_pages, kFreeChunk);
    char *b = static_cast<char *>(workspace);
    q.cnt = reinterpret_cast<int32_t *>(b);
    q.last = q.cnt + num_pages;
    b += align256(2 * (size_t)num_pages * 4);
    q.chunk_free = reinterpret_cast<int32_t *>(b);  b += align256((size_t)q.nchunks * 4);
    q.need = reinterpret_cast<int32_t *>(b);        b += align256((size_t)P * N * 4);
    q.alloc = reinterpret_cast<int32_t *>(b);
    q.max_alloc = (int64_t)P * N * (max_pages + 1);
    q.n_pools = n_pools;
    int64_t planes = 0;
    for (int k = 0; k < n_pools; ++k) {
        const smcsd_kv_pool &a = pools[k];
        if (!a.base || !aligned16(a.base) || a.n_planes < 1 || a.token_bytes < 16) return SMCSD_EINVAL;
        if ((a.plane_stride | a.page_stride | a.token_bytes) & 15) return SMCSD_EINVAL;
        if (a.plane_stride < 0 || a.page_stride < (int64_t)page_size * a.token_bytes) return SMCSD_EINVAL;
        planes += a.n_planes;
        q.pool[k] = KvPool{static_cast<char *>(a.base), a.plane_stride, a.page_stride, a.token_bytes, planes};
    }
    q.total_planes = planes;
    cudaStream_t st = as_stream(stream);
    smcsd_rc rc = launch_pdl(k_append_count, (unsigned)q.nchunks, 0, st, q);
    if (rc != SMCSD_OK) return rc;
    rc = launch_pdl(k_append_plan, 1u, 0, st, q);
    if (rc != SMCSD_OK || planes == 0) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P * N), (unsigned)cdiv(planes, kCowPlanesPerCta));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cdiv(planes, kCowPlanesPerCta) > 65535) return SMCSD_EINVAL;
    return cudaLaunchKernelEx(&cfg, k_append_cow, q) == cudaSuccess ? SMCSD_OK : SMCSD_ECUDA;
}

smcsd_rc smcsd_powersmc_weights(const void *logits, int64_t ld, int rows_per_particle, int dtype,
                                const float *logw_prev, int P, int N, int64_t V, float alpha,
                                float inv_temp, float *logw_out, float *log_inc, double *lse_out,
                                double *ess_out, float *wnorm_out, uint32_t *status,
                                void *workspace, size_t workspace_bytes, void *stream) {
    smcsd_rc rc = check_logits(logits, ld, rows_per_particle, logits, ld, rows_per_particle, dtype,
                               reinterpret_cast<const int32_t *>(logits), P, N, 1, V);
    if (rc != SMCSD_OK) return rc;
    if (!logw_out || !status || !workspace || N > kTailMaxN) return SMCSD_EINVAL;
    if (!(std::isfinite(alpha) && alpha > 0.0f) || !valid_temp(inv_temp)) return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, 1, V);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    Params prm = logits_params(logits, ld, rows_per_particle, logits, ld, rows_per_particle,
                               nullptr, nullptr, P, N, 1, V, 0, V, inv_temp, inv_temp);
    prm.n_models = 1;
    prm.main_items = (long long)P * N * prm.nseg;
    prm.alpha_f = alpha;
    prm.dtype = dtype;
    prm.logw_prev = logw_prev;
    prm.logw_out = logw_out; prm.logp_tok = log_inc;
    prm.lse = lse_out; prm.ess = ess_out; prm.wnorm = wnorm_out; prm.status = status;
    bind_workspace(prm, workspace, L);
    cudaStream_t st = as_stream(stream);
    rc = launch_rowstats(prm, dtype, (int64_t)P * N * prm.nseg, st, true);
    if (rc != SMCSD_OK) return rc;
    return launch_pdl(k_power_tail, (unsigned)P, 0, st, prm);
}

size_t smcsd_tp_exchange_bytes(int P, int N, int K, int G, int xnseg) {
    if (P < 1 || N < 1 || K < 1 || G < 1 || G > kXMaxG || xnseg < 1) return 0;
    return kXFlagBytes + 2 * x_half_elems(2 * P * N * K, G, xnseg) * sizeof(float4);
}

smcsd_rc smcsd_tp_exchange_init(void *xbuf, size_t xbuf_bytes, void *stream) {
    if (!xbuf || !aligned16(xbuf) || xbuf_bytes < (size_t)kXFlagBytes) return SMCSD_EINVAL;
    const size_t n = (xbuf_bytes - kXFlagBytes) / sizeof(float4);
    k_xinit<<<(unsigned)std::max<size_t>(1, std::min<size_t>(1184, cdiv((int64_t)n, 256))), 256, 0,
              as_stream(stream)>>>(static_cast<char *>(xbuf), n);
    return cudaGetLastError() == cudaSuccess ? SMCSD_OK : SMCSD_ECUDA;
}

// An IPC handle names a whole cudaMalloc allocation and opens at its base; a tensor from a
// caching allocator may sit at an offset inside it.  The exported bytes are the handle plus
// that offset (found with the driver's cuMemGetAddressRange, fetched through the runtime).
struct IpcBlob {
    cudaIpcMemHandle_t h;
    uint64_t offset;
};

size_t smcsd_ipc_handle_bytes(void) { return sizeof(IpcBlob); }

smcsd_rc smcsd_ipc_export(const void *dev_ptr, void *handle_out) {
    if (!dev_ptr || !handle_out) return SMCSD_EINVAL;
    using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return SMCSD_ECUDA;
    unsigned long long base = 0;
    size_t size = 0;
    if (reinterpret_cast<GetRange>(fn)(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
        return SMCSD_ECUDA;
    IpcBlob b;
    std::memset(&b, 0, sizeof b);
    if (cudaIpcGetMemHandle(&b.h, reinterpret_cast<void *>(base)) != cudaSuccess) return SMCSD_ECUDA;
    b.offset = reinterpret_cast<unsigned long long>(dev_ptr) - base;
    std::memcpy(handle_out, &b, sizeof b);
    return SMCSD_OK;
}

smcsd_rc smcsd_ipc_open(const void *handle, void **dev_ptr_out) {
    if (!handle || !dev_ptr_out) return SMCSD_EINVAL;
    IpcBlob b;
    std::memcpy(&b, handle, sizeof b);
    void *base = nullptr;
    if (cudaIpcOpenMemHandle(&base, b.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return SMCSD_ECUDA;
    *dev_ptr_out = static_cast<char *>(base) + b.offset;
    return SMCSD_OK;
}

smcsd_rc smcsd_ipc_close(void *dev_ptr, const void *handle) {
    if (!dev_ptr || !handle) return SMCSD_EINVAL;
    IpcBlob b;
    std::memcpy(&b, handle, sizeof b);
    return cudaIpcCloseMemHandle(static_cast<char *>(dev_ptr) - b.offset) == cudaSuccess ? SMCSD_OK : SMCSD_ECUDA;
}

smcsd_rc smcsd_tp_step(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                       const void *logits_q, int64_t ld_q, int rows_per_particle_q, int dtype,
                       const int32_t *tokens, const int32_t *n_drafted, const float *logw_prev,
                       int P, int N, int K, int64_t V, int64_t v_begin, int64_t v_len,
                       float alpha, float inv_temp_p, float inv_temp_q, float eta, int scheme,
                       uint64_t seed, uint64_t step, int64_t prompt_base, const uint32_t *uniforms,
                       int rank, int G, int xnseg, uint32_t epoch, void *const *xpeer,
                       void *xlocal, float *logw_out, float *logw_pre, float *logp_tok,
                       float *logq_tok, double *lse_out, double *ess_out, float *wnorm_out,
                       uint32_t *status, int32_t *ancestors, int32_t *offspring,
                       int32_t *slot_src, uint8_t *resampled, int32_t *n_ties,
                       void *workspace, size_t workspace_bytes, void *stream) {
    smcsd_rc rc = check_logits(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, dtype, tokens, P, N, K, v_len);
    if (rc != SMCSD_OK) return rc;
    if (!logw_out || !status || !ancestors || !resampled || !workspace || !xpeer || !xlocal)
        return SMCSD_EINVAL;
    if (N > kTailMaxN || std::isnan(eta) || v_begin < 0 || v_begin + v_len > V) return SMCSD_EINVAL;
    if (G < 1 || G > kXMaxG || rank < 0 || rank >= G || !aligned16(xlocal)) return SMCSD_EINVAL;
    if (xnseg < cdiv(v_len, kSeg) || (int64_t)G * xnseg > 4096) return SMCSD_EINVAL;
    if (!(std::isfinite(alpha) && alpha > 0.0f) || !valid_temp(inv_temp_p) || !valid_temp(inv_temp_q))
        return SMCSD_EINVAL;
    if (scheme != SMCSD_SYSTEMATIC && scheme != SMCSD_MULTINOMIAL) return SMCSD_EINVAL;
    const WsLayout L = ws_layout(P, N, K, v_len);
    if (workspace_bytes < L.total || !aligned16(workspace)) return SMCSD_EINVAL;
    Params prm = logits_params(logits_p, ld_p, rows_per_particle_p, logits_q, ld_q,
                               rows_per_particle_q, tokens, n_drafted, P, N, K, V, v_begin, v_len,
                               inv_temp_p, inv_temp_q);
    prm.alpha = (double)alpha;
    prm.dtype = dtype;
    prm.logw_prev = logw_prev;
    prm.eta = (double)eta; prm.seed = seed; prm.step = step; prm.prompt_base = prompt_base;
    prm.uniforms = uniforms; prm.scheme = scheme;
    prm.logw_out = logw_out; prm.logw_pre = logw_pre; prm.logp_tok = logp_tok;
    prm.logq_tok = logq_tok; prm.lse = lse_out; prm.ess = ess_out; prm.wnorm = wnorm_out;
    prm.status = status; prm.ancestors = ancestors; prm.offspring = offspring;
    prm.slot_src = slot_src; prm.resampled = resampled; prm.n_ties = n_ties;
    bind_workspace(prm, workspace, L);
    prm.xpeer = reinterpret_cast<char *const *>(xpeer);
    prm.xlocal = static_cast<char *>(xlocal);                  // K1 reads the device epoch here
    prm.xrank = rank; prm.xG = G; prm.xnseg = xnseg; prm.xepoch = epoch;
    cudaStream_t st = as_stream(stream);
    rc = launch_rowstats(prm, dtype, prm.main_items, st);         // S1 + push (S10)
    if (rc != SMCSD_OK) return rc;
    // S2-S7 over the G * xnseg parts of every row, after every rank's flag reaches epoch
    Params t = prm;
    t.xpeer = nullptr;
    t.xlocal = static_cast<char *>(xlocal);
    t.x_from_logits = 0;
    const int rows = 2 * P * N * K;
    // explicit epoch: the host picks the parity half; device epoch (0): the tail adds
    // (epoch & 1) * xhalf itself
    t.xhalf = (int64_t)x_half_elems(rows, G, xnseg);
    t.parts = reinterpret_cast<const float4 *>(static_cast<char *>(xlocal) + kXFlagBytes) +
              (epoch ? (epoch & 1u) * x_half_elems(rows, G, xnseg) : 0);
    t.part_row_stride = (int64_t)G * xnseg;
    t.part_seg_stride = 1;
    t.nparts = G * xnseg;
    return launch_tail(t, 1, st);
}

const char *smcsd_strerror(smcsd_rc rc) {
    switch (rc) {
        case SMCSD_OK: return "ok";
        case SMCSD_EINVAL: return "invalid argument";
        case SMCSD_ECUDA: return "CUDA launch or runtime error";
        case SMCSD_ENOSYS: return "not implemented in this build";
    }
    return "unknown smcsd_rc";
}

int smcsd_set_small_tail(int enable) {
    const int prev = g_tail_small;
    g_tail_small = enable != 0;
    return prev;
}

int smcsd_set_poll_tail(int enable) {
    const int prev = g_poll_tail;
    g_poll_tail = enable != 0;
    return prev;
}


const char *smcsd_version(void) { return "smcsd 0.1 sm_100a"; }

#ifdef SMCSD_TRACE
SMCSD_API int smcsd_trace_read(unsigned long long *host, int n) {
    return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * (n > 4096 ? 4096 : n)) == cudaSuccess ? 0 : 2;
}
#endif

}  // extern "C"
