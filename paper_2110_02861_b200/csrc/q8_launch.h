// q8_launch.h -- internal: launchers for the step kernels, instantiated per gradient dtype
// in step_inst.cu (compiled once per dtype, in parallel) and called by q8_api.cu.
#pragma once

#include <cuda_runtime.h>

#include "q8_kernels.cuh"

namespace q8 {

struct LaunchCtx {
    const float* tabs;
    int sms;
    cudaStream_t stream;
    int search;  // SEARCH_BUCKET or SEARCH_EYTZINGER
    int nsub;    // 2, 3 or 4 sub-blocks per CTA
    int subt;    // threads per sub-block (128 or 256); 0 = default for the gradient dtype
};

constexpr int kMultiMaxT = 384;

// Launch the fused step for gradient dtype g<N> (0 fp32, 1 fp16, 2 bf16); exactly one of
// single / multi is non-NULL.  Returns the launch error (cudaSuccess if ok).
cudaError_t launch_step_g0(int kind, const StepParams<1>* single, const StepParams<kMultiMaxT>* multi,
                           const LaunchCtx& ctx);
cudaError_t launch_step_g1(int kind, const StepParams<1>* single, const StepParams<kMultiMaxT>* multi,
                           const LaunchCtx& ctx);
cudaError_t launch_step_g2(int kind, const StepParams<1>* single, const StepParams<kMultiMaxT>* multi,
                           const LaunchCtx& ctx);

// Opt a kernel into `smem` bytes of dynamic shared memory (once per kernel and thread).
cudaError_t ensure_smem(const void* fn, int smem);

}  // namespace q8
