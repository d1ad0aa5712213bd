// microbenchmark: throughput of VIMNMX.U32 (predicated min/max), FMNMX and SHFL.BFLY per SM
#include <cstdio>
#include <cstdint>
template <int OP>
__global__ void kern(uint32_t* out, int iters) {
    uint32_t a[8];
    float f[8];
    const bool lo = threadIdx.x & 1;
    for (int i = 0; i < 8; i++) { a[i] = threadIdx.x * 7919u + i * 104729u; f[i] = __uint_as_float(a[i] >> 2); }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0) a[i] = lo ? min(a[i], a[(i + 1) & 7]) : max(a[i], a[(i + 3) & 7]);
            if (OP == 1) f[i] = lo ? fminf(f[i], f[(i + 1) & 7]) : fmaxf(f[i], f[(i + 3) & 7]);
            if (OP == 2) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 15));
            if (OP == 3) a[i] = a[i] ^ (a[(i + 1) & 7] + 3u);
        }
    }
    uint32_t s = 0;
    for (int i = 0; i < 8; i++) s += a[i] + __float_as_uint(f[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint32_t* out;
    cudaMalloc(&out, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"VIMNMX.U32 (pred)", "FMNMX (pred)", "SHFL.BFLY", "LOP3+IADD"};
    int iters = 20000;
    for (int op = 0; op < 4; op++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            if (op == 0) kern<0><<<148 * 4, 512>>>(out, iters);
            if (op == 1) kern<1><<<148 * 4, 512>>>(out, iters);
            if (op == 2) kern<2><<<148 * 4, 512>>>(out, iters);
            if (op == 3) kern<3><<<148 * 4, 512>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double ops = 148.0 * 4 * 512 * iters * 8;  // thread-ops
            int clk;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            if (rep) printf("%-20s %.3f ms  %.1f thread-ops/clk/SM (at %d MHz max)\n", names[op], ms,
                            ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
