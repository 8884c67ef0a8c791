// smcsd_paged.cuh -- K6: paged append with copy-on-write (NEXT #1, the second half of the
// paper's pointer mechanism; Sec. 3.3 Obs. 2: resampled particles share their
// ancestor's pages; SPEC.md:466-470 append_tokens; reading G24 in DESIGN.md).
//
// The operation is defined sequentially in (p, n) order (the oracle, orc_kv_append_paged): a
// particle appending to a partially filled tail page that another particle still references
// (refcount > 1) first copies the page's filled tokens to a fresh page (copy-on-write); fresh
// pages are the lowest-id pages with refcount 0.  It is computed here without a sequential
// scan:
//   * copy-on-write decision: appender i (in order) of a shared tail t sees refcount R_t - i,
//     so it copies iff i < R_t - 1.  Only the LAST appender can keep t, and only when every
//     owner of t appends (k_t == R_t).  So an order-free count k_t (atomicAdd) and the last
//     appender's index (atomicMax) decide every particle exactly;
//   * page allocation: no page is freed by an append, so the sequential "lowest free page"
//     choices are the first `total` free pages in ascending id order, handed out in (p, n)
//     order by an exclusive scan of each particle's page need.
// Kernels: k_append_count (grid over 4096-page chunks: free pages per chunk), k_append_plan
// (one CTA: validation, decisions, scan, collection of the free ids from the chunks that hold
// them, table / refcount / slot-mapping updates), k_append_cow (the content copies: only the
// filled tokens of each copied tail page, 16-byte vectors, every KV pool plane).
#pragma once
#include "smcsd_kernels.cuh"

namespace smcsd {

constexpr uint32_t ST_OUT_OF_PAGES = 128u;
constexpr int kFreeChunk = 1024;                // pages per free-count chunk (4 per thread)
constexpr int kMaxPools = 64;                   // KV pool descriptors per call
constexpr int kCowPlanesPerCta = 2;

struct KvPool {
    char *base;
    int64_t plane_stride, page_stride, token_bytes;
    int64_t plane_end;                          // exclusive prefix of planes over pools
};

struct AppendParams {
    int32_t *table, *n_pages, *seq_len, *refcount;
    const int32_t *n_new;
    int P, N, max_pages, num_pages, page_size, max_new;
    int32_t *slot_mapping, *cow_src, *cow_dst, *cow_tokens;
    uint32_t *status;
    int32_t *result;
    // workspace (zero at entry; the plan leaves cnt / last zero again)
    int32_t *cnt, *last;                        // [num_pages]: appenders of a shared tail, last+1
    int32_t *chunk_free;                        // [nchunks]
    int32_t *need;                              // [P*N] page need -> exclusive offsets (bit 30: cow)
    int32_t *alloc;                             // [max_alloc] allocated page ids, in order
    int nchunks;
    int64_t max_alloc;
    int n_pools;
    int64_t total_planes;
    KvPool pool[kMaxPools];
};

__global__ void __launch_bounds__(kThreads) k_append_count(const __grid_constant__ AppendParams q) {
    __shared__ int red[kWarps];
    pdl_wait();                                 // refcounts may come from the reindex before
    const int base = blockIdx.x * kFreeChunk;
    int c = 0;
    int v[kFreeChunk / kThreads];
#pragma unroll
    for (int u = 0; u < kFreeChunk / kThreads; ++u) {          // all loads first
        const int pg = base + u * kThreads + threadIdx.x;
        v[u] = pg < q.num_pages ? __ldcg(&q.refcount[pg]) : 1;
    }
#pragma unroll
    for (int u = 0; u < kFreeChunk / kThreads; ++u) c += v[u] == 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kWarps; ++w) t += red[w];
        q.chunk_free[blockIdx.x] = t;
    }
    pdl_trigger();
}

// Page need of particle pn (fresh pages for the tokens past the tail's room).
__device__ __forceinline__ int append_fresh(int len, int add, int page) {
    const int f = len % page, room = f ? page - f : 0;
    return add > room ? (add - room + page - 1) / page : 0;
}

__global__ void __launch_bounds__(kThreads) k_append_plan(const __grid_constant__ AppendParams q) {
    __shared__ int wtot[kWarps + 1];
    __shared__ int s_bad;
    __shared__ long long s_free;
    __shared__ int s_scan[kThreads];
    const int tid = threadIdx.x;
    const int PN = q.P * q.N, MP = q.max_pages, page = q.page_size;
    pdl_wait();
    if (tid == 0) { s_bad = 0; s_free = 0; }
    for (int p = tid; p < q.P; p += kThreads) q.status[p] = 0u;
    __syncthreads();
    // ---- 1. validation; appenders of a partial tail count themselves on the tail page.  The
    // page ids of every list are checked over (particle, slot) pairs, so the loads of a long
    // list are independent (not one dependent chain per particle).
    constexpr int kU = 8;                                      // entries in flight per thread
    for (int64_t e0 = tid; e0 < (int64_t)PN * MP; e0 += (int64_t)kU * kThreads) {
        int pg[kU], rc[kU], pnv[kU];
        bool chk[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t e = e0 + (int64_t)u * kThreads;
            chk[u] = false;
            pnv[u] = 0;
            pg[u] = -1;
            if (e < (int64_t)PN * MP) {
                const int pn = (int)(e / MP), i = (int)(e - (int64_t)pn * MP);
                const int np = q.n_pages[pn];
                pnv[u] = pn;
                chk[u] = i < np && np <= MP;
                pg[u] = chk[u] ? q.table[e] : -1;
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            rc[u] = chk[u] && pg[u] >= 0 && pg[u] < q.num_pages ? __ldcg(&q.refcount[pg[u]]) : 1;
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (chk[u] && (pg[u] < 0 || pg[u] >= q.num_pages || rc[u] < 1)) {
                atomicOr(&q.status[pnv[u] / q.N], ST_BAD_PAGE);
                s_bad = 1;
            }
    }
    __syncthreads();
    for (int pn = tid; pn < PN; pn += kThreads) {
        const int len = q.seq_len[pn], np = q.n_pages[pn], add = q.n_new[pn];
        bool bad = len < 0 || np < 0 || np > MP || add < 0 || add > q.max_new ||
                   np != (int)(((long long)len + page - 1) / page) ||
                   (__ldcg(&q.status[pn / q.N]) & ST_BAD_PAGE) != 0;
        if (!bad && np + append_fresh(len, add, page) > MP) bad = true;
        if (bad) {
            atomicOr(&q.status[pn / q.N], ST_BAD_PAGE);
            s_bad = 1;
        } else if (add > 0 && len % page) {
            const int t = q.table[(int64_t)pn * MP + np - 1];
            atomicAdd(&q.cnt[t], 1);
            atomicMax(&q.last[t], pn + 1);
        }
    }
    for (int c = tid; c < q.nchunks; c += kThreads) atomicAdd((unsigned long long *)&s_free, (unsigned long long)q.chunk_free[c]);
    __syncthreads();
    const bool bad_any = s_bad != 0;
    // ---- 2. copy-on-write decisions and page needs (sequential semantics, see the header)
    for (int pn = tid; pn < PN; pn += kThreads) {
        int need = 0;
        if (!bad_any) {
            const int len = q.seq_len[pn], np = q.n_pages[pn], add = q.n_new[pn];
            if (add > 0) {
                need = append_fresh(len, add, page);
                if (len % page) {
                    const int t = q.table[(int64_t)pn * MP + np - 1];
                    const bool keep = __ldcg(&q.cnt[t]) == __ldcg(&q.refcount[t]) &&
                                      __ldcg(&q.last[t]) == pn + 1;
                    if (!keep) need += 1 | (1 << 30);
                }
            }
        }
        q.need[pn] = need;
    }
    __syncthreads();
    // exclusive scan of the needs (cow bit kept aside)
    long long total = 0;
    for (int base = 0; base < PN; base += kThreads) {
        const int pn = base + tid;
        const int raw = pn < PN ? q.need[pn] : 0;
        s_scan[tid] = raw & ~(1 << 30);
        __syncthreads();
        const int tot = block_exclusive_scan(s_scan, kThreads, wtot);
        if (pn < PN) q.need[pn] = (int)(total + s_scan[tid]) | (raw & (1 << 30));
        total += tot;
        __syncthreads();
    }
    // ---- 3. all-or-nothing: invalid state or too few free pages change nothing
    if (bad_any || total > s_free || total > q.max_alloc) {
        for (int pn = tid; pn < PN; pn += kThreads) {
            const int len = q.seq_len[pn], np = q.n_pages[pn], add = q.n_new[pn];
            if (np >= 1 && np <= MP && len > 0 && add > 0 && len % page) {
                const int t = q.table[(int64_t)pn * MP + np - 1];
                if (t >= 0 && t < q.num_pages) { q.cnt[t] = 0; q.last[t] = 0; }
            }
        }
        if (!bad_any)
            for (int p = tid; p < q.P; p += kThreads) q.status[p] |= ST_OUT_OF_PAGES;
        for (int pn = tid; pn < PN; pn += kThreads) {           // no copy-on-write to run
            q.cow_src[pn] = -1;
            q.cow_dst[pn] = -1;
            q.cow_tokens[pn] = 0;
        }
        if (tid == 0) *q.result = 1;
        pdl_trigger();
        return;
    }
    // ---- 4. the first `total` free pages in ascending id order, from the chunks holding them
    long long got = 0;
    for (int c = 0; c < q.nchunks && got < total; ++c) {
        const int fc = q.chunk_free[c];
        if (fc == 0) continue;
        for (int b0 = 0; b0 < kFreeChunk && got < total; b0 += kThreads) {
            const int pg = c * kFreeChunk + b0 + tid;
            const int fr = pg < q.num_pages && __ldcg(&q.refcount[pg]) == 0;
            s_scan[tid] = fr;
            __syncthreads();
            const int tot = block_exclusive_scan(s_scan, kThreads, wtot);
            if (fr && got + s_scan[tid] < total) q.alloc[got + s_scan[tid]] = pg;
            got += tot;
            __syncthreads();
        }
    }
    __syncthreads();
    // ---- 5. apply, particle by particle (disjoint rows; refcount updates are atomics)
    for (int pn = tid; pn < PN; pn += kThreads) {
        const int len = q.seq_len[pn], add = q.n_new[pn];
        int np = q.n_pages[pn];
        int32_t *row = q.table + (int64_t)pn * MP;
        int32_t *slots = q.slot_mapping + (int64_t)pn * q.max_new;
        int cs = -1, cd = -1, ct = 0;
        if (add > 0) {
            int off = q.need[pn] & ~(1 << 30);
            const bool cow = (q.need[pn] >> 30) & 1;
            if (len % page) {
                const int t = row[np - 1];
                q.cnt[t] = 0;                   // step 2 has read it: leave the workspace zero
                q.last[t] = 0;
                if (cow) {
                    cd = q.alloc[off++];
                    cs = t;
                    ct = len % page;
                    atomicSub(&q.refcount[t], 1);
                    q.refcount[cd] = 1;
                    row[np - 1] = cd;
                }
            }
            for (int j = 0; j < add; ++j) {
                const int pos = len + j, pi = pos / page;
                if (pi >= np) {
                    const int c = q.alloc[off++];
                    q.refcount[c] = 1;
                    row[pi] = c;
                    np = pi + 1;
                }
                slots[j] = row[pi] * page + pos % page;
            }
            q.seq_len[pn] = len + add;
            q.n_pages[pn] = np;
        }
        for (int j = add > 0 ? add : 0; j < q.max_new; ++j) slots[j] = -1;
        q.cow_src[pn] = cs;
        q.cow_dst[pn] = cd;
        q.cow_tokens[pn] = ct;
    }
    if (tid == 0) *q.result = 0;
    pdl_trigger();
}

// Content of each copied tail page: the first cow_tokens tokens of every plane of every pool.
// grid = (P*N, ceil(total_planes / kCowPlanesPerCta)).
__global__ void __launch_bounds__(kThreads) k_append_cow(const __grid_constant__ AppendParams q) {
    pdl_wait();
    const int pn = blockIdx.x;
    const int cd = q.cow_dst[pn];
    if (cd < 0 || *q.result != 0) return;
    const int cs = q.cow_src[pn], ct = q.cow_tokens[pn];
    const int64_t pl0 = (int64_t)blockIdx.y * kCowPlanesPerCta;
    const int npl = (int)min((int64_t)kCowPlanesPerCta, q.total_planes - pl0);
    // every plane of this CTA copies the same token range: (plane, vector) pairs flattened so a
    // thread keeps 4 independent 16-byte loads in flight
    const char *srcp[kCowPlanesPerCta];
    char *dstp[kCowPlanesPerCta];
    int64_t nv[kCowPlanesPerCta];
    int64_t tot = 0;
#pragma unroll
    for (int u = 0; u < kCowPlanesPerCta; ++u) {
        nv[u] = 0; srcp[u] = nullptr; dstp[u] = nullptr;
        if (u < npl) {
            const int64_t pl = pl0 + u;
            int k = 0;
            while (q.pool[k].plane_end <= pl) ++k;
            const KvPool &P_ = q.pool[k];
            const int64_t o = pl - (k ? q.pool[k - 1].plane_end : 0);
            nv[u] = (int64_t)ct * P_.token_bytes / 16;
            srcp[u] = P_.base + o * P_.plane_stride + (int64_t)cs * P_.page_stride;
            dstp[u] = P_.base + o * P_.plane_stride + (int64_t)cd * P_.page_stride;
            tot += nv[u];
        }
    }
    for (int64_t b = threadIdx.x; b < tot; b += 4 * kThreads) {
        uint4 r[4];
        char *dp[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            int64_t v = b + (int64_t)w * kThreads;
            dp[w] = nullptr;
            if (v < tot) {
                int u = 0;
                while (v >= nv[u]) { v -= nv[u]; ++u; }
                r[w] = ld_stream(srcp[u] + v * 16);
                dp[w] = dstp[u] + v * 16;
            }
        }
#pragma unroll
        for (int w = 0; w < 4; ++w)
            if (dp[w]) st_stream(dp[w], r[w]);
    }
}

}  // namespace smcsd
