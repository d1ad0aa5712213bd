// micro: where does the time between two CUDA events around ONE persistent 148 x 512 launch go?
// Each case: an L2 flush as the bench does it (256 MB memset, then a 256 MB read kernel), optionally a
// "primer" kernel, then ev0 / kernel / ev1.  Cases vary the parameter size (1 KB vs 24 KB), the dynamic
// shared memory (0 vs 223 KB: the SM's L1/shared carveout differs from the flush kernels'), and whether
// the primer (same smem config as the timed kernel) ran just before ev0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/lf tools/micro/launch_floor.cu && /tmp/lf
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct Blob { long long v[N]; };
template <int N> __global__ void k(const __grid_constant__ Blob<N> b, long long* out) {
    extern __shared__ char sm[];
    if (threadIdx.x == 0 && b.v[blockIdx.x % N] == 12345) { sm[0] = 1; out[0] = sm[1]; }
}
__global__ void rd(const int4* p, size_t n, int* out) {
    int4 acc = {0, 0, 0, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        int4 v = p[i]; acc.x ^= v.x; acc.y ^= v.y;
    }
    if (acc.x == 0x7fffffff && acc.y == 1) out[0] = 1;
}
template <int N> float run(int mode, int smem, int primer_smem, void* big, void* big2, long long* out) {
    Blob<N> b = {};
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0; const int it = 40;
    for (int i = 0; i < it + 5; ++i) {
        if (mode >= 1) {
            cudaMemsetAsync(big, i, 256 << 20);
            rd<<<148 * 4, 512>>>((const int4*)big2, (256u << 20) / 16, (int*)out);
        }
        if (primer_smem >= 0) k<1><<<148, 512, primer_smem>>>(Blob<1>{}, out);
        cudaEventRecord(e0);
        if (mode != 2) k<N><<<148, 512, smem>>>(b, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) tot += ms;
    }
    return tot / it * 1000.f;
}
int main() {
    void *big, *big2; cudaMalloc(&big, 256 << 20); cudaMalloc(&big2, 256 << 20); cudaMemset(big2, 0, 256 << 20);
    long long* out; cudaMalloc(&out, 8);
    const int S = 223 * 1024;
    printf("events only (flush before)                : %6.2f us\n", run<128>(2, 0, -1, big, big2, out));
    printf("param  1 KB smem   0, idle               : %6.2f us\n", run<128>(0, 0, -1, big, big2, out));
    printf("param  1 KB smem   0, after flush        : %6.2f us\n", run<128>(1, 0, -1, big, big2, out));
    printf("param  1 KB smem 223, after flush        : %6.2f us\n", run<128>(1, S, -1, big, big2, out));
    printf("param 24 KB smem   0, after flush        : %6.2f us\n", run<3072>(1, 0, -1, big, big2, out));
    printf("param 24 KB smem 223, after flush        : %6.2f us\n", run<3072>(1, S, -1, big, big2, out));
    printf("param 24 KB smem 223, flush+primer(223)  : %6.2f us\n", run<3072>(1, S, S, big, big2, out));
    printf("param  1 KB smem 223, flush+primer(223)  : %6.2f us\n", run<128>(1, S, S, big, big2, out));
    printf("param 24 KB smem 223, flush+primer(0)    : %6.2f us\n", run<3072>(1, S, 0, big, big2, out));
    printf("param 24 KB smem 223, idle               : %6.2f us\n", run<3072>(0, S, -1, big, big2, out));
    return 0;
}
