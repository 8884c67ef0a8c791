// ubench_fp64.cu -- single-thread latency of FP64 ops used by the resampling tail.
#include <cstdio>
#include <cmath>
__global__ void k(double x0, long long *out, double *sink) {
    double x = x0; long long t0, t1;
    t0 = clock64(); for (int i = 0; i < 256; ++i) x = __dadd_rn(x, 1e-9); t1 = clock64(); out[0] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) x = __dmul_rn(x, 1.0000001); t1 = clock64(); out[1] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < 64; ++i) x = __ddiv_rn(x, 1.0000001) + 1e-12; t1 = clock64(); out[2] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < 64; ++i) x = exp(-x) + 0.5; t1 = clock64(); out[3] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < 64; ++i) x = log(x + 2.0); t1 = clock64(); out[4] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < 64; ++i) x = log2(x + 2.0); t1 = clock64(); out[5] = t1 - t0;
    float f = (float)x;
    t0 = clock64(); for (int i = 0; i < 256; ++i) f = f * 1.0001f + 1e-7f; t1 = clock64(); out[6] = t1 - t0;
    t0 = clock64(); for (int i = 0; i < 256; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f)); f = y * 0.5f; } t1 = clock64(); out[7] = t1 - t0;
    sink[0] = x + f;
}
int main() {
    long long *o; double *s; cudaMalloc(&o, 64 * 8); cudaMalloc(&s, 8);
    for (int r = 0; r < 2; ++r) { k<<<1, 1>>>(0.5, o, s); cudaDeviceSynchronize(); }
    long long h[8]; cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
    printf("DADD %.1f  DMUL %.1f  DDIV %.1f  exp %.1f  log %.1f  log2 %.1f  FFMA %.1f  MUFU.EX2+FMUL %.1f cycles/op\n",
           h[0] / 256., h[1] / 256., h[2] / 64., h[3] / 64., h[4] / 64., h[5] / 64., h[6] / 256., h[7] / 256.);
}
