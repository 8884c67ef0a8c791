// smcsd_kv_tma.cuh -- K3 (S8/S9 source-major block gather) with bulk asynchronous copies.
//
// k_kv_reindex moves every 16-byte vector through registers: 256 threads x 4 loads of a 16 KB
// chunk per source, then the stores to each destination.  Here one thread per CTA drives the
// copy engine instead: cp.async.bulk loads a chunk of a source (up to kKvTmaChunk bytes of one
// segment) into shared memory (mbarrier, complete_tx), and cp.async.bulk stores it from there to
// every destination; eight buffers, so the next sources' loads are in flight while the current
// one's stores drain.  The copy plan and the ST_BAD_INDEX policy are k_kv_reindex's.
#pragma once
#include "smcsd_kernels.cuh"

namespace smcsd {

#ifndef SMCSD_KV_TMA_CHUNK
#define SMCSD_KV_TMA_CHUNK 4096
#endif
constexpr int kKvTmaChunk = SMCSD_KV_TMA_CHUNK;             // bytes per chunk (within one segment)
#ifndef SMCSD_KV_TMA_BUFS
#define SMCSD_KV_TMA_BUFS 8
#endif
constexpr int kKvTmaBufs = SMCSD_KV_TMA_BUFS;               // chunk buffers (loads in flight + 1)
constexpr int kKvTmaMaxN = 256;                              // particles (plan arrays in smem)

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src_smem, uint32_t bytes) {
#ifdef SMCSD_KV_TMA_EVICT_FIRST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 :: "l"(dst), "r"(smem_u32(src_smem)), "r"(bytes), "l"(pol) : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
#endif
}
// global -> shared bulk load (k_kv_reindex_tma's sources), optionally with an L2 evict-first hint
__device__ __forceinline__ void bulk_g2s_kv(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
#ifdef SMCSD_KV_TMA_EVICT_FIRST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
#else
    bulk_g2s(dst, src, bytes, bar);
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory"); }

// grid = sum over tensors of n_outer * P * seg_count * ceil(seg_bytes / kKvTmaChunk) (item_end
// holds the prefix; nchunks = chunks per block), block = kThreads, dynamic smem = 2 chunks.
__global__ void __launch_bounds__(kThreads) k_kv_reindex_tma(const __grid_constant__ KvParams prm) {
    extern __shared__ __align__(128) char kbuf[];                // [kKvTmaBufs][kKvTmaChunk]
    __shared__ __align__(8) uint64_t full[kKvTmaBufs];
    __shared__ int cnt[kKvTmaMaxN], start[kKvTmaMaxN], fill[kKvTmaMaxN], dsts[kKvTmaMaxN], srcs[kKvTmaMaxN];
    __shared__ int wtot[kWarps + 1];
    __shared__ int s_bad;
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
    if (tid == 0) {
        for (int b = 0; b < kKvTmaBufs; ++b) mbar_init(&full[b], 1);
        fence_mbar_init();
        s_bad = 0;
    }
    pdl_wait();                                                // src_index from the tail kernel

    // ---- copy plan for prompt p (k_kv_reindex's): destinations grouped by source
    for (int n = tid; n < N; n += kThreads) {
        cnt[n] = 0;
        srcs[n] = idx[n];
    }
    __syncthreads();
    int bad = 0;
    for (int n = tid; n < N; n += kThreads) {
        const int s = srcs[n];
        if ((unsigned)s >= (unsigned)N) bad |= 1;
        else if (s != n && srcs[s] != s) bad |= 2;
        if ((unsigned)s < (unsigned)N && (!in_place || s != n)) atomicAdd(&cnt[s], 1);
    }
    if (bad) atomicOr(&s_bad, bad);
    __syncthreads();
    const int pbad = s_bad;
    if (prm.status && lo == 0 && o == 0 && chunk == 0 && tid == 0)
        prm.status[p] = ((pbad & 1) || ((pbad & 2) && prm.any_in_place)) ? ST_BAD_INDEX : 0u;
    if (in_place && (pbad & 2)) return;
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
    if (tid != 0) return;

    // ---- this chunk: segment g, bytes [off, off + len) of it
    const int64_t cps = ((int64_t)T.vps * 16 + kKvTmaChunk - 1) / kKvTmaChunk;   // chunks per segment
    const int64_t g = chunk / cps;
    const int64_t off = (chunk - g * cps) * kKvTmaChunk;
    const uint32_t len = (uint32_t)min((int64_t)kKvTmaChunk, (int64_t)T.vps * 16 - off);
    const int64_t base = o * T.outer_stride + (int64_t)p * T.prompt_stride + g * T.seg_stride + off;
    // kKvTmaBufs buffers: the loads of sources k+1 .. k+B-1 are in flight while source k's
    // stores drain (one bulk group per source)
    auto load = [&](int k) {
        const int b = k % kKvTmaBufs;
        mbar_arrive_expect_tx(&full[b], len);
        bulk_g2s_kv(kbuf + b * kKvTmaChunk, T.src + base + (int64_t)srcs[k] * T.particle_stride, len, &full[b]);
    };
    for (int k = 0; k < kKvTmaBufs - 1 && k < nsrc; ++k) load(k);
    for (int k = 0; k < nsrc; ++k) {
        const int b = k % kKvTmaBufs;
        if (k + kKvTmaBufs - 1 < nsrc) {
            // its buffer was last read by the stores of source k - 1 (the newest group)
            bulk_wait_read<0>();
            load(k + kKvTmaBufs - 1);
        }
        mbar_wait(&full[b], (uint32_t)((k / kKvTmaBufs) & 1));
        const int s = srcs[k], c = cnt[s], st0 = start[s];
        for (int q = 0; q < c; ++q)
            bulk_s2g(T.dst + base + (int64_t)dsts[st0 + q] * T.particle_stride, kbuf + b * kKvTmaChunk, len);
        bulk_commit();
    }
    bulk_wait_read<0>();                                       // (smem must outlive the stores' reads)
}

// The same copy with N <= 32 and one warp per CTA: lane n = particle n builds the plan with warp
// votes and shared-memory counts (no block barriers), lane 0 drives the copy.  For small N the
// per-CTA plan is what a CTA mostly does besides waiting on the copy engine; a warp builds it in
// a few dozen instructions and more CTAs fit on an SM.
__global__ void __launch_bounds__(32) k_kv_reindex_tma_w(const __grid_constant__ KvParams prm) {
    extern __shared__ __align__(128) char kbuf[];                // [kKvTmaBufs][kKvTmaChunk]
    __shared__ __align__(8) uint64_t full[kKvTmaBufs];
    __shared__ int cnt[32], start[32], dsts[32], srcs[32];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x, N = prm.N;
    int lo = 0, hi = prm.n_tensors - 1;
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
    if (lane == 0) {
        for (int b = 0; b < kKvTmaBufs; ++b) mbar_init(&full[b], 1);
        fence_mbar_init();
    }
    cnt[lane] = 0;
    pdl_wait();                                                // src_index from the tail kernel
    // ---- copy plan (k_kv_reindex's): lane n holds src_index[n]
    const bool act = lane < N;
    const int s = act ? prm.idx[(int64_t)p * N + lane] : -1;
    const bool inr = act && (unsigned)s < (unsigned)N;
    const int s_of_s = __shfl_sync(FULL, s, inr ? s : 0);      // src_index[s]
    int bad = 0;
    if (act && !inr) bad |= 1;
    if (inr && s != lane && s_of_s != s) bad |= 2;             // source s is itself overwritten
    bad = __reduce_or_sync(FULL, bad);
    if (prm.status && lo == 0 && o == 0 && chunk == 0 && lane == 0)
        prm.status[p] = ((bad & 1) || ((bad & 2) && prm.any_in_place)) ? ST_BAD_INDEX : 0u;
    if (in_place && (bad & 2)) return;
    const bool valid = inr && (!in_place || s != lane);
    __syncwarp();
    if (valid) atomicAdd(&cnt[s], 1);
    __syncwarp();
    const int c = cnt[lane];
    const unsigned lt = (1u << lane) - 1u;
    const unsigned has = __ballot_sync(FULL, c > 0);
    const int nsrc = __popc(has);
    if (c > 0) srcs[__popc(has & lt)] = lane;
    int x = c;                                                 // inclusive scan of the counts
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL, x, d);
        if (lane >= d) x += y;
    }
    start[lane] = x - c;
    const unsigned grp = __match_any_sync(FULL, valid ? s : -1 - lane);
    const int st_s = __shfl_sync(FULL, x - c, valid ? s : 0);  // start[s]
    __syncwarp();
    if (valid) dsts[st_s + __popc(grp & lt)] = lane;
    __syncwarp();
    if (lane != 0) return;

    const int64_t cps = ((int64_t)T.vps * 16 + kKvTmaChunk - 1) / kKvTmaChunk;   // chunks per segment
    const int64_t g = chunk / cps;
    const int64_t off = (chunk - g * cps) * kKvTmaChunk;
    const uint32_t len = (uint32_t)min((int64_t)kKvTmaChunk, (int64_t)T.vps * 16 - off);
    const int64_t base = o * T.outer_stride + (int64_t)p * T.prompt_stride + g * T.seg_stride + off;
    auto load = [&](int k) {
        const int b = k % kKvTmaBufs;
        mbar_arrive_expect_tx(&full[b], len);
        bulk_g2s_kv(kbuf + b * kKvTmaChunk, T.src + base + (int64_t)srcs[k] * T.particle_stride, len, &full[b]);
    };
    for (int k = 0; k < kKvTmaBufs - 1 && k < nsrc; ++k) load(k);
    for (int k = 0; k < nsrc; ++k) {
        const int b = k % kKvTmaBufs;
        if (k + kKvTmaBufs - 1 < nsrc) {
            bulk_wait_read<0>();
            load(k + kKvTmaBufs - 1);
        }
        mbar_wait(&full[b], (uint32_t)((k / kKvTmaBufs) & 1));
        const int sk = srcs[k], ck = cnt[sk], s0 = start[sk];
        for (int q = 0; q < ck; ++q)
            bulk_s2g(T.dst + base + (int64_t)dsts[s0 + q] * T.particle_stride, kbuf + b * kKvTmaChunk, len);
        bulk_commit();
    }
    bulk_wait_read<0>();
}

}  // namespace smcsd
