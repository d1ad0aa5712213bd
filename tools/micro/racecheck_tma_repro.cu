// Minimal reproducer: compute-sanitizer racecheck reports a write-after-read
// hazard between generic shared-memory loads and a later TMA bulk copy (cp.async.bulk) into the same
// buffer even when every read is ordered before the copy by a full __syncthreads() plus
// fence.proxy.async -- i.e. the report does not depend on the stage hand-off protocol the step kernel
// uses (per-warp count-out with an acq_rel shared atomic; mode 0 here), it appears with a CTA barrier
// too (mode 1).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o racecheck_tma_repro
// racecheck_tma_repro.cu ; run: compute-sanitizer --tool racecheck ./racecheck_tma_repro <mode>.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void stream_kernel(const float* __restrict__ src, float* __restrict__ out, int blocks, int mode) {
    __shared__ alignas(128) float stage[1024];
    __shared__ alignas(8) unsigned long long bar;
    __shared__ unsigned cnt;
    const unsigned sb = smem_u32(stage), bb = smem_u32(&bar), cb = smem_u32(&cnt);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
        cnt = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int b) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(4096u) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sb),
                     "l"(src + b * 1024), "r"(4096u), "r"(bb)
                     : "memory");
    };
    if (threadIdx.x == 0) issue(0);
    float acc = 0.f;
    for (int b = 0; b < blocks; ++b) {
        asm volatile(
            "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(bb),
            "r"(b & 1)
            : "memory");
        for (int i = threadIdx.x; i < 1024; i += blockDim.x) acc += stage[i];   // generic reads of the stage
        if (mode == 0) {  // step-kernel protocol: each warp counts itself out, the last one re-arms the stage
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                unsigned old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cb) : "memory");
                if (old % (blockDim.x / 32) == blockDim.x / 32 - 1 && b + 1 < blocks) issue(b + 1);
            }
        } else {          // a full CTA barrier orders every read before the copy
            __syncthreads();
            if (threadIdx.x == 0 && b + 1 < blocks) issue(b + 1);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0, blocks = 4;
    float *src, *out;
    cudaMalloc(&src, blocks * 4096);
    cudaMalloc(&out, 128 * sizeof(float));
    cudaMemset(src, 0, blocks * 4096);
    stream_kernel<<<1, 128>>>(src, out, blocks, mode);
    const cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d (%s): %s\n", mode, mode == 0 ? "per-warp count-out" : "__syncthreads", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
