// ubench_lt_prof.cu -- lt_finish called 2000 times back to back by one warp (dry: no stores), for
// ncu source-level stall sampling of the S4-S7 warp routine.
#include <cstdio>
#include "smcsd_lt.cuh"
using namespace smcsd;

__global__ void k(int N, int reps, float *logw, double *lse, double *ess, float *wnorm, int32_t *anc,
                  int32_t *off, int32_t *slot, int32_t *ties, uint8_t *res) {
    __shared__ WtSmem ls;
    __shared__ float lam_s[64];
    const int lane = threadIdx.x;
    if (lane == 0) {
        ls.st = 0;
        ls.a = WtArgs{logw, wnorm, lse, ess, anc, off, slot, ties, res, (double)INFINITY, N, 0};
    }
    __syncwarp();
    const double u = (lane + 0.37) / N;
    float lam = lane < N ? -0.1f * lane + 0.05f * (lane % 3) : -INFINITY;
    for (int r = 0; r < reps; ++r) {
        lam_s[lane] = lam;
        __syncwarp();
        warp_tail<1>(0, 0, 1, r != reps - 1, lam_s, u, 0.0, -2.77f, ls);
        lam += 1e-7f;
    }
}

int main() {
    float *logw, *wnorm; double *lse, *ess; int32_t *anc, *off, *slot, *ties; uint8_t *res;
    cudaMalloc(&logw, 4096); cudaMalloc(&wnorm, 4096); cudaMalloc(&lse, 64); cudaMalloc(&ess, 64);
    cudaMalloc(&anc, 4096); cudaMalloc(&off, 4096); cudaMalloc(&slot, 4096); cudaMalloc(&ties, 64);
    cudaMalloc(&res, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<1, 32>>>(16, 10, logw, lse, ess, wnorm, anc, off, slot, ties, res);
    cudaEventRecord(a);
    k<<<1, 32>>>(16, 2000, logw, lse, ess, wnorm, anc, off, slot, ties, res);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("N=16: %.1f ns per lt_finish (warm, 2000 calls)\n", ms * 1e6 / 2000);
}
