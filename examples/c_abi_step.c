/* Plain-C use of the q8 C ABI (include/q8.h) -- no Python, no torch: allocate device buffers with the
 * CUDA runtime, run 8-bit AdamW steps on a flat buffer, then check one documented property of the
 * result: at t = 1 from the zero state every parameter moves by about -lr * sign(g) (bias-corrected
 * Adam, G8; |dw| = lr * |g| / (|g| + eps) up to rounding), decayed first (AdamW, G10).
 *
 *   build:  gcc -O2 -I include examples/c_abi_step.c -L paper_2110_02861_b200 -lq8 \
 *               -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2110_02861_b200 \
 *               -o /tmp/c_abi_step
 *   run:    /tmp/c_abi_step [n]          (prints "c_abi_step ok ..." and exits 0 on success) */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "q8.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 2; } } while (0)
#define Q8(x) do { q8_status s_ = (x); if (s_ != Q8_OK) { fprintf(stderr, "%s: %d %s\n", #x, (int)s_, q8_last_error()); return 3; } } while (0)

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1000003;
    const int64_t nb = (n + 2047) / 2048;
    float* hp = malloc(n * sizeof(float));
    float* hg = malloc(n * sizeof(float));
    float* out = malloc(n * sizeof(float));
    uint32_t seed = 12345u;
    for (int64_t i = 0; i < n; ++i) {  /* a small LCG: parameters ~ U(-0.02, 0.02), grads ~ U(-1e-3, 1e-3) */
        seed = seed * 1664525u + 1013904223u;
        hp[i] = ((float)(seed >> 8) / 16777216.0f - 0.5f) * 0.04f;
        seed = seed * 1664525u + 1013904223u;
        hg[i] = ((float)(seed >> 8) / 16777216.0f - 0.5f) * 2e-3f;
    }
    float *p, *g, *a1, *a2;
    uint8_t *s1, *s2;
    CK(cudaMalloc((void**)&p, n * 4)); CK(cudaMalloc((void**)&g, n * 4));
    CK(cudaMalloc((void**)&s1, n)); CK(cudaMalloc((void**)&s2, n));
    CK(cudaMalloc((void**)&a1, nb * 4)); CK(cudaMalloc((void**)&a2, nb * 4));
    CK(cudaMemcpy(p, hp, n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(g, hg, n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(s1, 0, n)); CK(cudaMemset(s2, 0, n));  /* all-zero codes + absmax: the initial state */
    CK(cudaMemset(a1, 0, nb * 4)); CK(cudaMemset(a2, 0, nb * 4));
    const q8_hparams hpar = {1e-3, 0.9, 0.999, 1e-8, 0.01, 1};
    Q8(q8_optim8bit_step(Q8_ADAMW, p, g, Q8_F32, s1, s2, a1, a2, n, 2048, &hpar, 1, NULL));
    CK(cudaMemcpy(out, p, n * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    const double decay = 1.0 - 1e-3 * 0.01;
    for (int64_t i = 0; i < n; ++i) {
        const double want = (double)hp[i] * decay - 1e-3 * hg[i] / (fabs(hg[i]) + 1e-8);
        if (fabs(out[i] - want) > 1e-6 * fabs(want) + 1e-9) ++bad;
    }
    /* and a second step through the same buffers (t = 2) must run cleanly */
    Q8(q8_optim8bit_step(Q8_ADAMW, p, g, Q8_F32, s1, s2, a1, a2, n, 2048, &hpar, 2, NULL));
    CK(cudaDeviceSynchronize());
    /* argument validation is synchronous and documented */
    if (q8_optim8bit_step(Q8_ADAMW, p, g, Q8_F32, s1, s2, a1, a2, n, 1024, &hpar, 1, NULL) != Q8_ERR_UNSUPPORTED) ++bad;
    printf("c_abi_step %s: %s, n=%lld, %lld mismatches\n", bad ? "FAILED" : "ok", q8_version(), (long long)n, (long long)bad);
    cudaFree(p); cudaFree(g); cudaFree(s1); cudaFree(s2); cudaFree(a1); cudaFree(a2);
    free(hp); free(hg); free(out);
    return bad ? 1 : 0;
}
