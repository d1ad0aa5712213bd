// micro: does the size of a __grid_constant__ kernel parameter cost launch time on the device?
// empty persistent-style kernel (148 CTAs x 512 threads) with a 1 KB vs a 24 KB parameter struct,
// timed with events around each launch, back to back and after a 256 MB memset.
#include <cstdio>
#include <cuda_runtime.h>
template <int N> struct Blob { long long v[N]; };
template <int N> __global__ void k(const __grid_constant__ Blob<N> b, long long* out) {
    if (threadIdx.x == 0 && b.v[blockIdx.x % N] == 12345) out[0] = 1;
}
template <int N> float run(bool flush, void* big, long long* out) {
    Blob<N> b = {};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0; const int it = 50;
    for (int i = 0; i < it + 5; ++i) {
        if (flush) cudaMemsetAsync(big, i, 256 << 20);
        cudaEventRecord(e0);
        k<N><<<148, 512>>>(b, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (i >= 5) tot += ms;
    }
    return tot / it * 1000.f;
}
int main() {
    void* big; cudaMalloc(&big, 256 << 20); long long* out; cudaMalloc(&out, 8);
    printf("param 1 KB : %.2f us (after memset %.2f us)\n", run<128>(false, big, out), run<128>(true, big, out));
    printf("param 24 KB: %.2f us (after memset %.2f us)\n", run<3072>(false, big, out), run<3072>(true, big, out));
    return 0;
}
