/*
 * smcsd.h -- C ABI of libsmcsd.so, the B200 (sm_100a) verification hot path of
 * Sequential Monte Carlo Speculative Decoding (arxiv 2604.15672; PAPER.md = its LaTeX
 * source, cited by line number).
 *
 * One SMC-SD round (Alg. 1) after the target forward pass:
 *   S1/S2  score:     ell^p_j = log p(d_j | x d_<j), ell^q_j = log q(d_j | x d_<j) from logits
 *                     (Alg. 1 "Score"; Eq. 1a)
 *   S3     reweight:  lam'_n = lam_n + sum_{j<k_n} (alpha ell^p_j - ell^q_j)
 *                     (Alg. 1 "Reweight"; power target PAPER.md:1418)
 *   S4     normalise, ESS = (sum w)^2 / sum w^2   (Eq. 3)
 *   S5-S7  if ESS < eta: draw ancestors, reset weights to 1/N
 *   S8/S9  x^(n) <- x^(a_n): per-particle KV cache and token history reindex
 *   S10    (tensor parallel) per-row max / sum-exp exchange across vocab shards (north star)
 * Readings of the paper where it is silent (G1..G18) are listed in DESIGN.md section 3; the
 * ones that shape this ABI are cited inline.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless marked "host".  Every call only enqueues work on
 *    `stream` (a cudaStream_t passed as void*, NULL = legacy default stream): no call
 *    synchronises, allocates or frees.  All buffers are caller-owned.
 *  - Layouts are row-major.  Logit row (prompt p, particle n, draft position j) of a logits
 *    tensor starts at element  base + ((p*N + n)*rows_per_particle + j)*ld ; the first V
 *    elements are read, and the buffer must hold  P*N*rows_per_particle*ld  elements.
 *    Base pointers must be 16-byte aligned and ld a multiple of 16 bytes (8 bf16 / 4 fp32).
 *  - Synchronous argument errors return SMCSD_EINVAL and enqueue nothing.  A failed launch
 *    returns SMCSD_ECUDA.  There is no CPU fallback and no silent layout fallback.
 *  - Data-dependent conditions cannot be returned synchronously; they are written to
 *    status[p] (uint32 per prompt, overwritten by each call) as SMCSD_ST_* bits.  A particle
 *    with an invalid row (bad token, non-finite row, q(d) = 0) gets lam' = -inf and the
 *    prompt is flagged (reading G13).
 *  - Ancestor indices are local to the prompt (0..N-1).  Philox counters use the GLOBAL
 *    prompt index prompt_base + p, so prompt-sharded (data-parallel) runs are bit-identical
 *    to a single-GPU run.
 *  - The library keeps no global state beyond a per-device cache of kernel attributes and
 *    occupancy (set on first use).  A workspace may not be shared by concurrent calls.
 */
#ifndef SMCSD_H
#define SMCSD_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SMCSD_API __attribute__((visibility("default")))
#else
#define SMCSD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SMCSD_OK = 0,
    SMCSD_EINVAL = 1,   /* invalid argument (synchronous; nothing enqueued)          */
    SMCSD_ECUDA = 2,    /* a CUDA launch / runtime call failed                       */
    SMCSD_ENOSYS = 3    /* valid request that this build does not implement          */
} smcsd_rc;

typedef enum { SMCSD_F32 = 0, SMCSD_BF16 = 1 } smcsd_dtype;

/* Resampling scheme.  Systematic is the north star's choice (reading G1); multinomial is the
 * paper's literal draw a_n ~ Cat(wbar) i.i.d. (Alg. 1) with
 * u_n = word (n mod 4) of Philox(key = seed, ctr = (step_lo, step_hi, prompt, 1 + n/4)). */
typedef enum { SMCSD_SYSTEMATIC = 0, SMCSD_MULTINOMIAL = 1 } smcsd_scheme;

/* Per-prompt status bits (asynchronous, data-dependent). */
#define SMCSD_ST_DEGENERATE  1u  /* every log-weight of the prompt is -inf           */
#define SMCSD_ST_NOT_ABSCONT 2u  /* q(d) = 0 at a drafted token: p << q violated     */
#define SMCSD_ST_BAD_TOKEN   4u  /* drafted token outside [0,V), or n_drafted outside [0,K]         */
#define SMCSD_ST_NONFINITE   8u  /* NaN/+inf logit or log-weight, or a row whose max is -inf        */
#define SMCSD_ST_BAD_PAGE   16u  /* paged reindex: page id or ancestor out of range (entry skipped) */
#define SMCSD_ST_EXCHANGE   32u  /* smcsd_tp_step: a peer's partials did not arrive within 20 s;   */
                                 /* polling tails: K1's words of a row did not arrive within 20 s  */
#define SMCSD_ST_BAD_INDEX  64u  /* kv reindex: src_index entry outside [0,N) (entry skipped), or an
                                    in-place index that is both a source and a destination (the
                                    prompt's in-place copies skipped)                              */

/* Segment length (elements) of the fixed in-row split used by every logit row (G17). */
#define SMCSD_SEGMENT 8192

/* Bytes of device workspace needed by smcsd_weights / smcsd_step / smcsd_weights_partial /
 * smcsd_weights_combine for P prompts, N particles, K drafted tokens and v_len vocabulary
 * columns per row (V, or the shard width for the partial call). */
SMCSD_API size_t smcsd_workspace_bytes(int P, int N, int K, int64_t v_len);

/* Zero a workspace (enqueued).  Required after allocation AND whenever the workspace is next
 * used with a different (P, N, K, v_len): the kernels keep per-prompt completion counters and
 * status words inside the workspace at shape-dependent offsets and leave them zero on exit,
 * so a workspace stays valid across calls and CUDA-graph replays of one shape, but a new
 * shape may place its counters over an earlier shape's data.  (The Python binding's
 * Workspace does this re-zeroing on shape change.) */
SMCSD_API smcsd_rc smcsd_workspace_init(void *workspace, size_t workspace_bytes, void *stream);

/* S1-S4.
 *  logits_p: target logits, rows_per_particle_p >= K (K+1 when the bonus row is present; the
 *            bonus row is never read: it cancels in the weight).
 *  logits_q: draft logits, rows_per_particle_q >= K.  dtype: SMCSD_F32 or SMCSD_BF16 (both).
 *  tokens:   [P][N][K] int32 drafted tokens d_j (global vocabulary ids).
 *  n_drafted:[P][N] int32 drafted length k_n in [0,K] (EOS inside a block, reading G10), or
 *            NULL for k_n = K.  Rows j >= k_n are not read.
 *  logw_prev:[P][N] fp32 prior log-weights lam_n, or NULL for -ln N.  May alias logw_out.
 *  alpha:    power-target exponent (1 = plain SMC-SD), > 0.
 *  inv_temp_p/q: inverse temperatures applied to logits before the log-softmax (G9), > 0.
 *  Outputs (NULL allowed except logw_out and status):
 *    logw_out [P][N] fp32 lam'_n;  logp_tok/logq_tok [P][N][K] fp32 ell (0 for j >= k_n,
 *    NaN for invalid rows);  lse_out [P] fp64 log sum_n exp(lam'_n);  ess_out [P] fp64;
 *    wnorm_out [P][N] fp32 normalised weights;  status [P].
 *  Any N >= 1 is accepted (N > 1024 uses a slower serial normalisation). */
SMCSD_API smcsd_rc smcsd_weights(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                       const void *logits_q, int64_t ld_q, int rows_per_particle_q,
                       int dtype, const int32_t *tokens, const int32_t *n_drafted,
                       const float *logw_prev, int P, int N, int K, int64_t V,
                       float alpha, float inv_temp_p, float inv_temp_q,
                       float *logw_out, float *logp_tok, float *logq_tok,
                       double *lse_out, double *ess_out, float *wnorm_out, uint32_t *status,
                       void *workspace, size_t workspace_bytes, void *stream);

/* S4-S7 from fp32 log-weights, N <= 1024.
 *  eta:       resample iff ESS < eta (strict); +INFINITY forces, 0 never.
 *  seed/step: Philox4x32-10 key and counter high words: U = word0(Philox(key = seed,
 *             ctr = (step_lo, step_hi, prompt_base + p, 0))) * 2^-32 (reading G5).
 *  uniforms:  optional raw 32-bit words replacing the Philox draws (tests), or NULL:
 *             [P] for SMCSD_SYSTEMATIC, [P][N] for SMCSD_MULTINOMIAL.
 *  Ancestors: C_m = P_m / S (fp64 sequential prefix), a_n = #{m : C_m <= u_n} with
 *  u_n = (n + U)/N (systematic; ancestors ascending) or u_n i.i.d. (multinomial; draw order);
 *  offspring o_m; slot_src = the in-place plan (survivors keep their
 *  slot, dead slots take the extra copies in ascending order; reading G14); n_ties counts
 *  pairs |u_n - C_m| <= 2^-40 (reading G7).  Without a resample: identity, o = 1, lam kept.
 *  logw_out [P][N]: fl32(-ln N) after a resample, else lam.  May alias logw.
 *  Outputs other than ancestors, logw_out, resampled and status may be NULL. */
SMCSD_API smcsd_rc smcsd_resample(const float *logw, int P, int N, int64_t prompt_base, float eta,
                        int scheme, uint64_t seed, uint64_t step, const uint32_t *uniforms,
                        int32_t *ancestors, int32_t *offspring, int32_t *slot_src,
                        float *logw_out, uint8_t *resampled, double *ess_out, double *lse_out,
                        float *wnorm_out, int32_t *n_ties, uint32_t *status, void *stream);

/* Fused S1-S7 in one enqueue (one launch: row statistics + last-CTA-per-prompt tail), the
 * performance path.  Arguments as smcsd_weights + smcsd_resample; N <= 1024.
 *  logw_pre [P][N] (optional): lam' before the S7 reset -- the exact fp32 values the
 *  resampling consumed (staged parity).  logw_out receives the S7 output.
 *  bonus_tok [P][N] (optional, NEXT #2; "sample bonus token x+ ~ p"): when
 *  non-NULL the target's row j = k_n (rows_per_particle_p >= K + 1) is streamed in the same
 *  K1 pass and bonus_tok[p][n] receives one exact draw from softmax(inv_temp_p * z) of that
 *  row (reading G22: segment by inverse CDF, then Gumbel-max, Philox counters
 *  (step, prompt_base + p, 2^31 + 2^20 n + i)).  Indexed by the particle BEFORE resampling
 *  (append it, then reindex the history with the ancestors).  -1 with
 *  NONFINITE (NaN / +inf / all -inf row) or BAD_TOKEN (k_n outside [0, K]).  V <= 2^21.
 *  The bonus row does not enter the weights (it cancels). */
SMCSD_API smcsd_rc smcsd_step(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                    const void *logits_q, int64_t ld_q, int rows_per_particle_q,
                    int dtype, const int32_t *tokens, const int32_t *n_drafted,
                    const float *logw_prev, int P, int N, int K, int64_t V,
                    float alpha, float inv_temp_p, float inv_temp_q,
                    float eta, int scheme, uint64_t seed, uint64_t step, int64_t prompt_base,
                    const uint32_t *uniforms,
                    float *logw_out, float *logw_pre, float *logp_tok, float *logq_tok,
                    double *lse_out, double *ess_out, float *wnorm_out, uint32_t *status,
                    int32_t *ancestors, int32_t *offspring, int32_t *slot_src,
                    uint8_t *resampled, int32_t *n_ties, int32_t *bonus_tok,
                    void *workspace, size_t workspace_bytes, void *stream);

/* S1 on this rank's vocabulary shard (tensor-parallel, north star).  Row pointers address
 * only the shard: logits_* row r holds columns [v_begin, v_begin + v_len) of the full row
 * (ld >= v_len).  tokens are GLOBAL ids.  partials: [P][2][N][K][4] fp32 per row
 * {m, s, x, 0} in the log2 domain of the scaled logits t = inv_temp * z * log2(e):
 *   m = max t over the shard, s = sum 2^(t - m), x = t_d if d is in the shard else -inf.
 * Rows are ordered (prompt, model p then q, particle, position).  Rows j >= k_n hold
 * {-inf, 0, -inf, 0}. */
SMCSD_API smcsd_rc smcsd_weights_partial(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
                               const void *logits_q, int64_t ld_q, int rows_per_particle_q,
                               int dtype, const int32_t *tokens, const int32_t *n_drafted,
                               int P, int N, int K, int64_t v_begin, int64_t v_len,
                               float inv_temp_p, float inv_temp_q, float *partials,
                               void *workspace, size_t workspace_bytes, void *stream);

/* S2-S4 after the exchange: gathered = [G][P][2][N][K][4] (the all_gather_into_tensor layout
 * of G smcsd_weights_partial outputs in rank order).  Shards are merged in rank order, so
 * every rank obtains bit-identical results.  V (full vocabulary) is used for the token range
 * check.  Outputs as smcsd_weights.  workspace: smcsd_workspace_bytes(P, N, K, 1) bytes. */
SMCSD_API smcsd_rc smcsd_weights_combine(const float *gathered, int G, const int32_t *tokens,
                               const int32_t *n_drafted, const float *logw_prev,
                               int P, int N, int K, int64_t V, float alpha,
                               float *logw_out, float *logp_tok, float *logq_tok,
                               double *lse_out, double *ess_out, float *wnorm_out,
                               uint32_t *status, void *workspace, size_t workspace_bytes,
                               void *stream);

/* S10 in the all-reduce form of the north star ("NCCL over NVLink all-reduces the per-row
 * max/sum-exp"), the alternative to the rank-ordered all-gather above:
 *   1. smcsd_weights_partial on each rank -> partials [rows][4] {m, s, x, 0};
 *   2. all_reduce(MAX) of a copy of the partials -> max_partials (fields 0 and 2 used: M, X);
 *   3. this call: out[r] = {M_r, s_r 2^(m_r - M_r), X_r, 0} (rows = 2 P N K; device, 16-byte
 *      aligned; out may alias partials);
 *   4. all_reduce(SUM) of field 1 of out across ranks -> {M, S, X} per row;
 *   5. smcsd_weights_combine with G = 1.
 * Every rank ends with the same weights (the collectives give every rank the same values) but
 * S is summed in NCCL's order, not rank order, so it need not be bit-identical to the
 * unsharded result (the all-gather path is).  Enqueued on stream; EINVAL on null/misaligned. */
SMCSD_API smcsd_rc smcsd_partials_rescale(const float *partials, const float *max_partials, float *out,
                                          int64_t rows, void *stream);

/* S8/S9: reindex per-particle state blocks (dense analogue of the paged
 * pointer copy of PAPER.md:489).  Block (o, p, n), o < n_outer (e.g. L*2 layer K/V planes),
 * is seg_count segments of seg_bytes bytes at
 *   base + o*outer_stride + p*prompt_stride + n*particle_stride + s*seg_stride   (bytes),
 * e.g. the filled rows [0, seq_len) of each KV head (reading G12).
 *  dst != src (out of place): dst block n <- src block src_index[n] for every n
 *                             (src_index = ancestors).
 *  dst == src (in place):     block n <- block src_index[n] where src_index[n] != n
 *                             (src_index = slot_src; precondition: no index is both a source
 *                             and a destination, which slot_src guarantees).
 * Copies are bitwise (16-byte integer vectors; NaN payloads survive) and source-major: each
 * source chunk is read once and written to all of its destinations.  seg_bytes, all strides
 * and both base pointers must be multiples of 16; N <= 1024.
 *  status [P] (optional, device): SMCSD_ST_BAD_INDEX when prompt p's src_index holds an entry
 *  outside [0, N) (that destination is left untouched) or, in place, an index that is both a
 *  source and a destination (the prompt's in-place copies are skipped); 0 otherwise.  The index
 *  values live on the device, so this cannot be a synchronous error. */
SMCSD_API smcsd_rc smcsd_kv_reindex(void *dst, const void *src, int64_t n_outer, int64_t outer_stride,
                          int64_t prompt_stride, int64_t particle_stride, int64_t seg_count,
                          int64_t seg_bytes, int64_t seg_stride, const int32_t *src_index,
                          int P, int N, uint32_t *status, void *stream);

/* S8/S9 over several state tensors in ONE launch, with one src_index: e.g. per-layer K and V
 * tensors of a serving engine (dst[], src[], n_tensors) plus the token history.
 * tensors: HOST array of n_tensors (1..256) descriptors, read during the call (caller keeps
 * ownership; not retained).  Each tensor has its own geometry, with the meaning and the
 * alignment rules of smcsd_kv_reindex above; dst == src selects in-place per tensor.  Tensors
 * must not overlap each other.  smcsd_kv_reindex(...) is this call with n_tensors = 1. */
typedef struct {
    void *dst;                    /* device base of the destination blocks            */
    const void *src;              /* device base of the source blocks (== dst: in place) */
    int64_t n_outer, outer_stride, prompt_stride, particle_stride;   /* bytes */
    int64_t seg_count, seg_bytes, seg_stride;                        /* bytes */
} smcsd_kv_tensor;
SMCSD_API smcsd_rc smcsd_kv_reindex_multi(const smcsd_kv_tensor *tensors, int n_tensors,
                                          const int32_t *src_index, int P, int N, uint32_t *status,
                                          void *stream);

/* Terminal selection: "one complete sequence is sampled from the terminal
 * normalized weights".  selected[p] = #{m : C_m <= u} with u = word0(Philox(key = seed,
 * ctr = (step_lo, step_hi, prompt_base + p, 0xFFFFFFFF))) * 2^-32 (or uniforms[p]); -1 and
 * SMCSD_ST_DEGENERATE when every weight is -inf.  workspace: smcsd_workspace_bytes(P, N, 1, 1). */
SMCSD_API smcsd_rc smcsd_select(const float *logw, int P, int N, int64_t prompt_base, uint64_t seed,
                                uint64_t step, const uint32_t *uniforms, int32_t *selected,
                                uint32_t *status, void *workspace, size_t workspace_bytes,
                                void *stream);

/* Paged (pointer) KV reindex -- the paper's own resampling mechanism (PAPER.md:488-490,
 * Sec. 3.3 Obs. 2: "copying page metadata and incrementing the reference counts").
 * table_*: [P][N][max_pages] int32 page ids; n_pages_*: [P][N] int32 list lengths.
 *   table_dst[p][n][i] = table_src[p][a_n][i] for i < n_pages_src[p][a_n], -1 beyond;
 *   n_pages_dst[p][n] = n_pages_src[p][a_n];   (a = src_index, local to the prompt)
 *   refcount[pg] += #references in the new lists - #references in the old lists (exact int);
 *   freed (optional, [num_pages] u8): 1 for old-list pages whose refcount reached 0, else 0
 *   (pages no old list references are untouched).
 * No KV content moves; a partially filled tail page shared after resampling is copied on
 * the next append (engine-level copy-on-write, outside this call).  src and dst tables must
 * not alias.  Out-of-range ids are skipped and flagged SMCSD_ST_BAD_PAGE in status[p]. */
SMCSD_API smcsd_rc smcsd_kv_reindex_paged(const int32_t *table_src, const int32_t *n_pages_src,
                                          int32_t *table_dst, int32_t *n_pages_dst,
                                          int32_t *refcount, uint8_t *freed,
                                          const int32_t *src_index, int P, int N, int max_pages,
                                          int num_pages, uint32_t *status, void *stream);

/* Paged append with copy-on-write (NEXT #1; Sec. 3.3 Obs. 2: resampling
 * shares the ancestor's pages, so the first write after a resample must not land in a page
 * another particle sees; SPEC.md:466-470 append_tokens; reading G24).  Defined sequentially in
 * (p, n) order; particle n appends n_new[p][n] tokens (e.g. its K + 1 new tokens):
 *   f = seq_len mod page_size (filled tokens of a partial tail page, 0 = none);
 *   if n_new > 0, f > 0 and refcount[tail] > 1 (shared, e.g. after smcsd_kv_reindex_paged):
 *     copy-on-write -- a fresh page c receives the tail's f filled tokens (only those: full
 *     pages are immutable and never copied), refcount[tail] -= 1, refcount[c] = 1, and c
 *     replaces the tail in the particle's table;  otherwise the tail is filled in place;
 *   fresh pages (refcount 1) take the remaining tokens; every fresh page is the LOWEST-id page
 *   whose refcount is 0 (the free pool is the set of refcount-0 pages: smcsd_kv_reindex_paged
 *   releases pages by bringing their refcount to 0);
 *   slot_mapping[p][n][j] = page * page_size + offset where new token j's KV goes (-1 for
 *   j >= n_new, up to max_new); seq_len += n_new; n_pages updated.
 * table [P][N][max_pages], n_pages / seq_len / n_new [P][N], refcount [num_pages] (device,
 * int32, updated in place).  cow_src / cow_dst / cow_tokens [P][N]: the copy-on-write list
 * (-1 / -1 / 0 where none).  pools: HOST array of n_pools (0..64) KV pool descriptors whose
 * copy-on-write content is copied on the device (bytes: plane o of page g starts at
 * base + o * plane_stride + g * page_stride, token t at + t * token_bytes; all multiples of 16).
 * All-or-nothing: if any particle's state is invalid (page id outside [0, num_pages) or with
 * refcount < 1, n_pages != ceil(seq_len / page_size), n_new outside [0, max_new], more than
 * max_pages pages) its prompt gets SMCSD_ST_BAD_PAGE; if fewer pages are free than the call
 * needs every prompt gets SMCSD_ST_OUT_OF_PAGES; then *result (device int32) = 1, nothing is
 * modified, no content is copied, the copy list reads "none" (-1 / -1 / 0) and slot_mapping
 * is not written.  *result = 0 on success.
 * workspace: smcsd_kv_append_workspace_bytes(P, N, num_pages, max_pages) bytes, zeroed once
 * (smcsd_workspace_init) -- the call leaves it zeroed.  num_pages * page_size < 2^31. */
typedef struct {
    void *base;
    int64_t n_planes, plane_stride, page_stride, token_bytes;
} smcsd_kv_pool;
#define SMCSD_ST_OUT_OF_PAGES 128u
SMCSD_API size_t smcsd_kv_append_workspace_bytes(int P, int N, int num_pages, int max_pages);
SMCSD_API smcsd_rc smcsd_kv_append_paged(int32_t *table, int32_t *n_pages, int32_t *seq_len,
                                         int32_t *refcount, const int32_t *n_new, int P, int N,
                                         int max_pages, int num_pages, int page_size, int max_new,
                                         int32_t *slot_mapping, int32_t *cow_src, int32_t *cow_dst,
                                         int32_t *cow_tokens, uint32_t *status, int32_t *result,
                                         const smcsd_kv_pool *pools, int n_pools, void *workspace,
                                         size_t workspace_bytes, void *stream);

/* PowerSMC weights (App. F): K = 1, no bonus token, draft = target.  Row 0
 * of each particle (rows_per_particle >= 1) gives p = softmax(inv_temp * z) and the weight
 * increment log w = ln sum_v p_v^alpha; lam' = fl32(lam_prev + log w), then
 * S4.  Resample with smcsd_resample.  log_inc (optional, [P][N] fp32) receives log w.
 * alpha = 1 gives log w = 0 exactly.  workspace: smcsd_workspace_bytes(P, N, 1, V); N <= 1024. */
SMCSD_API smcsd_rc smcsd_powersmc_weights(const void *logits, int64_t ld, int rows_per_particle,
                                          int dtype, const float *logw_prev, int P, int N,
                                          int64_t V, float alpha, float inv_temp,
                                          float *logw_out, float *log_inc, double *lse_out,
                                          double *ess_out, float *wnorm_out, uint32_t *status,
                                          void *workspace, size_t workspace_bytes, void *stream);

/* ---- S10 fused into K1: tensor-parallel step over peer memory (NVLink P2P) -------------------
 * The north star's vocab-sharded config: every rank holds columns [v_begin, v_begin + v_len)
 * of every logit row.  Instead of partial -> NCCL all_gather -> combine, K1 itself pushes each
 * (row, segment) partial straight into every rank's exchange buffer through peer mappings, as
 * two 8-byte words {m, s} and {x_d, 1} (st.relaxed.sys: single-copy atomic, and both words are
 * nonzero whenever written).  There is no fence, flag or collective: each rank's tail polls
 * the words of its rows itself (ld.relaxed.sys; bounded: 20 s -> SMCSD_ST_EXCHANGE), zeroes
 * them after reading, and merges the G * xnseg parts of each row in rank order -- the global
 * column order -- so every rank computes identical weights, ancestors and resets (same Philox
 * counters).  Two launches per step, like smcsd_step.
 *
 * Exchange buffer (one per rank, caller-allocated, 16-byte aligned, smcsd_tp_exchange_bytes):
 * 256 B of control words then two parity halves (epoch & 1) of [2*P*N*K][G*xnseg] 16-byte
 * slots.  Initialise once with smcsd_tp_exchange_init (all zero = nothing written), share it
 * with smcsd_ipc_export / smcsd_ipc_open (plumbing; the handles travel over torch.distributed).
 * xnseg >= ceil(v_len / SMCSD_SEGMENT) on every rank (the same value everywhere); a rank with
 * fewer segments fills its unused slots with neutral parts.
 * epoch: 0 = device-resident epoch (recommended): each rank's buffer holds the last epoch it
 *   completed, advanced by the tail's last CTA, so the call can be captured in a CUDA graph
 *   and replayed (every replay is the next epoch).  >= 1 = explicit host epoch, +1 per call,
 *   identical on every rank; then a captured graph would replay a stale epoch and must not be
 *   used.  Do not mix the two modes on one buffer.  A rank may run at most one step ahead of
 *   another: it writes the other parity half, which every reader has zeroed before (its K1 of
 *   step e + 2 needs our pushes of step e + 1, made after our tail of step e finished). */
SMCSD_API size_t smcsd_tp_exchange_bytes(int P, int N, int K, int G, int xnseg);
SMCSD_API smcsd_rc smcsd_tp_exchange_init(void *xbuf, size_t xbuf_bytes, void *stream);
/* CUDA IPC plumbing.  smcsd_ipc_export writes smcsd_ipc_handle_bytes() opaque host bytes naming
 * the device address dev_ptr: the IPC handle of its whole allocation plus dev_ptr's offset in
 * it (so tensors from a caching allocator work).  smcsd_ipc_open maps a peer's bytes (peer
 * access enabled lazily) and returns the same address in this process; smcsd_ipc_close(ptr,
 * the same bytes) unmaps it. */
SMCSD_API size_t smcsd_ipc_handle_bytes(void);
SMCSD_API smcsd_rc smcsd_ipc_export(const void *dev_ptr, void *handle_out);
SMCSD_API smcsd_rc smcsd_ipc_open(const void *handle, void **dev_ptr_out);
SMCSD_API smcsd_rc smcsd_ipc_close(void *dev_ptr, const void *handle);
/* S1 + S10 + S2-S7 on this rank's shard.  Arguments as smcsd_step, plus
 *  v_begin/v_len: this rank's columns (logits rows hold only them; tokens are global ids);
 *  rank, G (1..32), xnseg, epoch: see above;  xpeer: DEVICE array [G] of every rank's exchange buffer
 *  as mapped in this process (xpeer[rank] == xlocal);  xlocal: this rank's buffer.
 *  Workspace: smcsd_workspace_bytes(P, N, K, v_len).  N <= 1024, G <= 32. */
SMCSD_API smcsd_rc smcsd_tp_step(const void *logits_p, int64_t ld_p, int rows_per_particle_p,
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
                       void *workspace, size_t workspace_bytes, void *stream);

/* Polling tail switch (process-wide; default 1 = on).  With it on, smcsd_step and smcsd_weights
 * calls without the bonus token, with at most 16 segments per row (V <= 131072) and N <= 1024
 * let K1 publish each (row, segment) {m, s} as one 8-byte word and launch the tail at once; the
 * tail polls those words instead of waiting for K1's grid to complete and flush (results are
 * bit-identical).  The words live in the workspace and are zero between calls (the tail clears
 * them); after a call that returned an error, re-initialise the workspace.  0 restores the
 * wait-for-K1 tail (A/B timing, tests).  Not synchronised with calls in flight on other host
 * threads.  Returns the previous setting. */
SMCSD_API int smcsd_set_poll_tail(int enable);

/* Small-tail switch (process-wide; default 1 = on).  Among the polling-tail calls, those with
 * N <= 64 and N*K <= 512 run the tail as 128-thread CTAs (16 or 32 pairs each, one
 * cluster per prompt) that fit beside K1's CTAs and are resident from the start of K1's stream
 * (paper_2604_15672_b200/csrc/smcsd_tail_small.cuh); results are bit-identical.  0 uses the
 * 256-thread tail for them.  Returns the previous setting. */
SMCSD_API int smcsd_set_small_tail(int enable);

/* Human-readable name of a return code (static storage). */
SMCSD_API const char *smcsd_strerror(smcsd_rc rc);

/* Library build identifier, e.g. "smcsd 0.1 sm_100a" (static storage). */
SMCSD_API const char *smcsd_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SMCSD_H */
