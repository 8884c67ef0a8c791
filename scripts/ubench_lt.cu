// ubench_lt.cu -- warm latency of warp_tail (S4-S7 for N <= 32, two warps), no other
// load on the GPU: phase clocks of the 3rd back-to-back call.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DSMCSD_TRACE -I include -I paper_2604_15672_b200/csrc scripts/ubench_lt.cu -o /tmp/ubench_lt
#include <cstdio>
#include "smcsd_lt.cuh"
using namespace smcsd;

__global__ void k(int N, float *logw, double *lse, double *ess, float *wnorm, int32_t *anc, int32_t *off,
                  int32_t *slot, int32_t *ties, uint8_t *res, long long *out) {
    __shared__ WtSmem ls;
    __shared__ float lam_s[64];
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        ls.st = 0;
        ls.a = WtArgs{logw, wnorm, lse, ess, anc, off, slot, ties, res, (double)INFINITY, N, 0};
    }
    __syncwarp();
    const double u = (lane + 0.37) / N;
    const float lam = lane < N ? -0.1f * lane + 0.05f * (lane % 3) : -INFINITY;
    for (int r = 0; r < 4; ++r) {
        const long long t0 = clock64();
        lam_s[lane] = lam;
        __syncthreads();
        warp_tail<1>(threadIdx.x >> 5, 0, 1, 0, lam_s, u, 0.0, -2.77f, ls);
        __syncthreads();
        const long long t1 = clock64();
        if (threadIdx.x == 0) {
            out[r] = t1 - t0;
            for (int i = 0; i < 8; ++i) out[8 + 8 * r + i] = g_trace[2300 + i] - g_trace[2300];
        }
    }
}

int main() {
    float *logw, *wnorm; double *lse, *ess; int32_t *anc, *off, *slot, *ties; uint8_t *res; long long *o;
    cudaMalloc(&logw, 4096); cudaMalloc(&wnorm, 4096); cudaMalloc(&lse, 64); cudaMalloc(&ess, 64);
    cudaMalloc(&anc, 4096); cudaMalloc(&off, 4096); cudaMalloc(&slot, 4096); cudaMalloc(&ties, 64);
    cudaMalloc(&res, 64); cudaMalloc(&o, 1024);
    for (int N : {4, 16, 32}) {
        k<<<1, 64>>>(N, logw, lse, ess, wnorm, anc, off, slot, ties, res, o);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
        long long h[40];
        cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
        printf("N=%2d total per call:", N);
        for (int r = 0; r < 4; ++r) printf(" %lld", h[r]);
        printf("  | last call phases:");
        for (int i = 1; i < 6; ++i) printf(" %lld", h[8 + 24 + i]);
        printf("\n");
    }
}
