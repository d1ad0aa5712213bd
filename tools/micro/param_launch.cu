// micro: what does the launch of a persistent kernel cost between CUDA events?  An empty 148 x 512
// kernel timed with events around each launch (after a 256 MB memset, as the bench's L2 flush), with a
// 1 KB vs a 24 KB __grid_constant__ parameter and with 0 vs 223 KB of dynamic shared memory.
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct Blob { long long v[N]; };
template <int N> __global__ void k(const __grid_constant__ Blob<N> b, long long* out) {
    extern __shared__ char sm[];
    if (threadIdx.x == 0 && b.v[blockIdx.x % N] == 12345) { sm[0] = 1; out[0] = sm[1]; }
}
template <int N> float run(bool flush, int smem, void* big, long long* out) {
    Blob<N> b = {};
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0; const int it = 50;
    for (int i = 0; i < it + 5; ++i) {
        if (flush) cudaMemsetAsync(big, i, 256 << 20);
        cudaEventRecord(e0);
        k<N><<<148, 512, smem>>>(b, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) tot += ms;
    }
    return tot / it * 1000.f;
}
int main() {
    void* big; cudaMalloc(&big, 256 << 20); long long* out; cudaMalloc(&out, 8);
    const int S = 223 * 1024;
    printf("param 1 KB,  smem 0     : %.2f us idle, %.2f us after memset\n", run<128>(false, 0, big, out), run<128>(true, 0, big, out));
    printf("param 24 KB, smem 0     : %.2f us idle, %.2f us after memset\n", run<3072>(false, 0, big, out), run<3072>(true, 0, big, out));
    printf("param 1 KB,  smem 223 KB: %.2f us idle, %.2f us after memset\n", run<128>(false, S, big, out), run<128>(true, S, big, out));
    printf("param 24 KB, smem 223 KB: %.2f us idle, %.2f us after memset\n", run<3072>(false, S, big, out), run<3072>(true, S, big, out));
    return 0;
}
