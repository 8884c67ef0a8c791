/* examples/c_abi_step.c -- the C ABI of libsmcsd.so used from plain C (no Python, no torch):
 * device buffers from the CUDA runtime, one smcsd_step (S1-S7) and one in-place
 * smcsd_kv_reindex (S8), checked against closed forms.
 *   gcc -std=c11 -O2 -I include -I /usr/local/cuda/include examples/c_abi_step.c \
 *       -L paper_2604_15672_b200 -lsmcsd -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2604_15672_b200 -lm -o c_abi_step && ./c_abi_step
 * Case 1: target and draft logits bitwise equal => every block weight is exactly 1 (Delta = 0,
 *         SPEC.md:201), so lam' = -ln N, ESS = N exactly, systematic ancestors = identity.
 * Case 2: particle 2's draft differs => ESS < N; the ancestors are non-decreasing, offspring
 *         sum to N, the slot plan is a permutation of them, and the in-place KV reindex leaves
 *         block n equal to the original block slot_src[n]. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include "smcsd.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)
#define RC(x) do { smcsd_rc r_ = (x); if (r_ != SMCSD_OK) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, smcsd_strerror(r_)); return 1; } } while (0)
#define EXPECT(c) do { if (!(c)) { fprintf(stderr, "check failed: %s (line %d)\n", #c, __LINE__); return 1; } } while (0)

enum { P = 1, N = 4, K = 2, V = 8, LD = 8, L = 1, H = 1, S = 4, D = 4 };

static int run_case(int perturb, void *ws, size_t wsb) {
    float hp[P * N * K * LD], hq[P * N * K * LD];
    int32_t htok[P * N * K];
    for (int r = 0; r < P * N * K; ++r)
        for (int v = 0; v < LD; ++v) hp[r * LD + v] = hq[r * LD + v] = 0.25f * (float)((v * 5 + r) % 7);
    for (int i = 0; i < P * N * K; ++i) htok[i] = (3 + i) % V;
    if (perturb)                                           /* particle 2: draft prefers another token */
        for (int j = 0; j < K; ++j) hq[(2 * K + j) * LD + 6] += 3.0f;
    float *dp, *dq, *dlogw, *dpre; int32_t *dtok, *danc, *doff, *dslot, *dties;
    double *dlse, *dess; uint32_t *dst; uint8_t *dres;
    CK(cudaMalloc((void **)&dp, sizeof hp)); CK(cudaMalloc((void **)&dq, sizeof hq));
    CK(cudaMalloc((void **)&dtok, sizeof htok));
    CK(cudaMalloc((void **)&dlogw, P * N * sizeof(float))); CK(cudaMalloc((void **)&dpre, P * N * sizeof(float)));
    CK(cudaMalloc((void **)&danc, P * N * 4)); CK(cudaMalloc((void **)&doff, P * N * 4));
    CK(cudaMalloc((void **)&dslot, P * N * 4)); CK(cudaMalloc((void **)&dties, P * 4));
    CK(cudaMalloc((void **)&dlse, P * 8)); CK(cudaMalloc((void **)&dess, P * 8));
    CK(cudaMalloc((void **)&dst, P * 4)); CK(cudaMalloc((void **)&dres, P));
    CK(cudaMemcpy(dp, hp, sizeof hp, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dq, hq, sizeof hq, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dtok, htok, sizeof htok, cudaMemcpyHostToDevice));
    RC(smcsd_step(dp, LD, K, dq, LD, K, SMCSD_F32, dtok, NULL, NULL, P, N, K, V, 1.0f, 1.0f, 1.0f,
                  INFINITY, SMCSD_SYSTEMATIC, 0x5EED5EEDull, 7ull, 0, NULL, dlogw, dpre, NULL, NULL,
                  dlse, dess, NULL, dst, danc, doff, dslot, dres, dties, NULL, ws, wsb, NULL));
    CK(cudaDeviceSynchronize());
    float logw[N], pre[N]; int32_t anc[N], off[N], slot[N]; double ess; uint32_t st; uint8_t res;
    CK(cudaMemcpy(logw, dlogw, sizeof logw, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pre, dpre, sizeof pre, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(anc, danc, sizeof anc, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(off, doff, sizeof off, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(slot, dslot, sizeof slot, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&ess, dess, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&res, dres, 1, cudaMemcpyDeviceToHost));
    const float reset = (float)(-log((double)N));
    EXPECT(st == 0 && res == 1);
    int sum = 0;
    for (int n = 0; n < N; ++n) {
        EXPECT(logw[n] == reset);                          /* S7 reset */
        EXPECT(anc[n] >= 0 && anc[n] < N && (n == 0 || anc[n] >= anc[n - 1]));
        sum += off[n];
    }
    EXPECT(sum == N);
    if (!perturb) {
        for (int n = 0; n < N; ++n) EXPECT(pre[n] == reset && anc[n] == n && off[n] == 1 && slot[n] == n);
        EXPECT(ess == (double)N);
    } else {
        EXPECT(ess < (double)N && ess >= 1.0);
        EXPECT(pre[2] != reset);
    }
    /* S8: in-place KV reindex with the slot plan; block n must equal the original block slot[n] */
    const int blk = H * S * D, tot = L * 2 * P * N * blk;
    float hkv[L * 2 * P * N * H * S * D], out[L * 2 * P * N * H * S * D];
    for (int i = 0; i < tot; ++i) hkv[i] = (float)i;
    float *dkv;
    CK(cudaMalloc((void **)&dkv, sizeof hkv));
    CK(cudaMemcpy(dkv, hkv, sizeof hkv, cudaMemcpyHostToDevice));
    const int64_t e = 4;
    RC(smcsd_kv_reindex(dkv, dkv, L * 2, P * N * blk * e, N * blk * e, blk * e, H, S * D * e, S * D * e,
                        dslot, P, N, dst, NULL));
    CK(cudaMemcpy(out, dkv, sizeof out, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost));
    EXPECT(st == 0);                               /* slot plan is valid: no SMCSD_ST_BAD_INDEX */
    for (int o = 0; o < L * 2; ++o)
        for (int n = 0; n < N; ++n)
            EXPECT(memcmp(out + (o * N + n) * blk, hkv + (o * N + slot[n]) * blk, blk * sizeof(float)) == 0);
    cudaFree(dp); cudaFree(dq); cudaFree(dtok); cudaFree(dlogw); cudaFree(dpre); cudaFree(danc);
    cudaFree(doff); cudaFree(dslot); cudaFree(dties); cudaFree(dlse); cudaFree(dess); cudaFree(dst);
    cudaFree(dres); cudaFree(dkv);
    printf("case %d: ESS %.6f ancestors %d %d %d %d slot_src %d %d %d %d\n", perturb, ess, anc[0], anc[1],
           anc[2], anc[3], slot[0], slot[1], slot[2], slot[3]);
    return 0;
}

int main(void) {
    printf("%s\n", smcsd_version());
    const size_t wsb = smcsd_workspace_bytes(P, N, K, V);
    void *ws;
    CK(cudaMalloc(&ws, wsb));
    RC(smcsd_workspace_init(ws, wsb, NULL));
    if (run_case(0, ws, wsb) || run_case(1, ws, wsb)) return 1;
    cudaFree(ws);
    printf("c abi ok\n");
    return 0;
}
