// ubench_tail.cu -- cycle-level timing of the K2 tail phases in one CTA (cfg2 shapes), run
// REPS times inside a single kernel so cold (first pass) and warm costs separate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2604_15672_b200/csrc -o /tmp/ubt scripts/ubench_tail.cu && /tmp/ubt
#include <cstdio>
#include <vector>
__device__ long long g_phase[16];
#define SMCSD_PHASE(i) do { if (threadIdx.x == 0) g_phase[(i)] = clock64(); } while (0)
#include "smcsd_kernels.cuh"

using namespace smcsd;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int REPS = 4;

__global__ void __launch_bounds__(kThreads) k_probe(const __grid_constant__ Params prm, long long *clk) {
    __shared__ TailSmem sh;
    extern __shared__ float4 dyn[];
    float4 *stage = dyn, *rowstat = dyn + kThreads * kStagePitch;
    const int tid = threadIdx.x;
    for (int r = 0; r < REPS; ++r) {
        __syncthreads();
        long long t0 = clock64();
        // (a) one dependent L2 load chain of 16 independent loads per thread (uncoalesced rows)
        tail_rowstats(prm, 0, rowstat, stage);
        __syncthreads();
        long long t1 = clock64();
        tail_scores(prm, 0, rowstat, sh.e, &sh.st, -INFINITY);
        __syncthreads();
        long long t2 = clock64();
        for (int n = tid; n < prm.N; n += kThreads) sh.lam[n] = -1.0f - n * 0.01f;
        if (tid == 0) tail_prologue(prm, 0, sh);
        __syncthreads();
        normalise_resample(prm, 0, true, sh);
        __syncwarp();
        __syncthreads();
        long long t3 = clock64();
        // (b) raw L2 latency: thread 0 dependent chain of 8 loads
        float acc = 0.f;
        if (tid == 0) {
            const float4 *q = prm.parts;
            int idx = 0;
            for (int i = 0; i < 8; ++i) {
                float4 v = __ldcg(q + idx);
                acc += v.y;
                idx = ((int)v.w & 1) + i * 97;
            }
        }
        __syncthreads();
        long long t4 = clock64();
        if (tid == 0) {
            clk[r * 5 + 0] = t1 - t0;
            clk[r * 5 + 1] = t2 - t1;
            clk[r * 5 + 2] = t3 - t2;
            clk[r * 5 + 3] = t4 - t3;
            clk[r * 5 + 4] = (long long)acc;
            if (r == REPS - 1)
                for (int i = 0; i < 9; ++i) clk[40 + i] = g_phase[i] - t2;
        }
    }
}

int main() {
    const int P = 1, N = 16, K = 8, nseg = 16;
    const int rows = 2 * N * K;
    std::vector<float4> hp((size_t)rows * nseg);
    for (size_t i = 0; i < hp.size(); ++i) hp[i] = make_float4(1.0f + (i % 7) * 0.1f, 100.0f + i % 13, (i % nseg == 3) ? 0.5f : -INFINITY, 0.f);
    std::vector<int> htok(P * N * K, 3 * 8192 + 5);
    float4 *parts; int *tok; double *ell; float *lw, *wn; int *anc, *off, *slot, *nt; unsigned char *res;
    double *lse, *ess; unsigned *st; long long *clk;
    CK(cudaMalloc(&parts, hp.size() * 16));
    CK(cudaMemcpy(parts, hp.data(), hp.size() * 16, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&tok, htok.size() * 4));
    CK(cudaMemcpy(tok, htok.data(), htok.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&ell, 1 << 20)); CK(cudaMalloc(&lw, 4096)); CK(cudaMalloc(&wn, 4096));
    CK(cudaMalloc(&anc, 4096)); CK(cudaMalloc(&off, 4096)); CK(cudaMalloc(&slot, 4096)); CK(cudaMalloc(&nt, 64));
    CK(cudaMalloc(&res, 64)); CK(cudaMalloc(&lse, 64)); CK(cudaMalloc(&ess, 64)); CK(cudaMalloc(&st, 64));
    CK(cudaMalloc(&clk, 8 * 64));
    Params prm{};
    prm.tokens = tok; prm.P = P; prm.N = N; prm.K = K; prm.V = 128256; prm.v_len = 128256; prm.nseg = nseg;
    prm.alpha = 1.0; prm.eta = INFINITY; prm.seed = 1; prm.step = 2;
    prm.logw_out = lw; prm.wnorm = wn; prm.lse = lse; prm.ess = ess; prm.status = st;
    prm.ancestors = anc; prm.offspring = off; prm.slot_src = slot; prm.n_ties = nt; prm.resampled = res;
    prm.parts = parts; prm.part_row_stride = nseg; prm.part_seg_stride = 1; prm.nparts = nseg;
    prm.ell_ws = ell;
    for (int launch = 0; launch < 3; ++launch) {
        const int smem = (int)(kTailStageBytes + rows * 16);
        CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_probe<<<1, kThreads, smem>>>(prm, clk);
        CK(cudaDeviceSynchronize());
        long long h[REPS * 5];
        CK(cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost));
        long long ph[9];
        CK(cudaMemcpy(ph, clk + 40, sizeof ph, cudaMemcpyDeviceToHost));
        printf("S4-S7 phase clocks:");
        for (int i = 0; i < 9; ++i) printf(" %lld", ph[i]);
        printf("   (0 start, 1 max, 2 exp, 3 serial, 4 bcast+wnorm, 5 Cdiv, 6 search, 7 plan, 8 end)\n");
        for (int r = 0; r < REPS; ++r)
            printf("launch %d rep %d: S2a %lld  S2b+S3 %lld  S4-S7 %lld  8-dep-L2 %lld cycles\n", launch, r,
                   h[r * 5], h[r * 5 + 1], h[r * 5 + 2], h[r * 5 + 3]);
    }
    return 0;
}
