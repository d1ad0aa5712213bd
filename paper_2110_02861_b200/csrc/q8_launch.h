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
    int plan = 0;  // multi-tensor plan launch (mixed 32-bit states, shared-memory / device scalars)
};

constexpr int kMultiMaxT = 384;
// Layer-wise lists of at most kSmallMaxT tensors launch with a half-size descriptor table: the kernel
// parameters are copied at every launch (~0.05 us per KB, DESIGN 12b), and a LARS step is two launches.
constexpr int kSmallMaxT = 192;

// Launch the fused step for gradient dtype g<N> (0 fp32, 1 fp16, 2 bf16); exactly one of
// single / multi is non-NULL.  Returns the launch error (cudaSuccess if ok).
cudaError_t launch_step_g0(int kind, const StepParams<1>* single, const StepParams<kMultiMaxT>* multi,
                           const LaunchCtx& ctx);
cudaError_t launch_step_g1(int kind, const StepParams<1>* single, const StepParams<kMultiMaxT>* multi,
                           const LaunchCtx& ctx);
cudaError_t launch_step_g2(int kind, const StepParams<1>* single, const StepParams<kMultiMaxT>* multi,
                           const LaunchCtx& ctx);

// Plan launch (the PLAN instantiation of the fused step) with the 192-entry descriptor table, for plans of
// <= kSmallMaxT non-empty tensors.
cudaError_t launch_plan_small_g0(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx);
cudaError_t launch_plan_small_g1(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx);
cudaError_t launch_plan_small_g2(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx);

// Layer-wise step (LAMB / LARS) for gradient dtype g<N>: norms pass, per-tensor scale pass
// (writes scale[0 .. P.num_tensors)), fused step; partial holds P.total_blocks entries; count holds
// P.num_tensors block counters, zero on entry and on return (LARS: the scales come from its norms pass).
cudaError_t launch_layerwise_g0(int kind, const StepParams<kMultiMaxT>& P, const LaunchCtx& ctx, double2* partial,
                                float* scale, unsigned int* count, double lr, double eta, double wd);
cudaError_t launch_layerwise_g1(int kind, const StepParams<kMultiMaxT>& P, const LaunchCtx& ctx, double2* partial,
                                float* scale, unsigned int* count, double lr, double eta, double wd);
cudaError_t launch_layerwise_g2(int kind, const StepParams<kMultiMaxT>& P, const LaunchCtx& ctx, double2* partial,
                                float* scale, unsigned int* count, double lr, double eta, double wd);
cudaError_t launch_layerwise_g0(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx, double2* partial,
                                float* scale, unsigned int* count, double lr, double eta, double wd);
cudaError_t launch_layerwise_g1(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx, double2* partial,
                                float* scale, unsigned int* count, double lr, double eta, double wd);
cudaError_t launch_layerwise_g2(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx, double2* partial,
                                float* scale, unsigned int* count, double lr, double eta, double wd);

// Fused ZeRO-1 step (MODE_ZERO) for gradient dtype g<N> with exactly `grid` CTAs (identical on
// every rank: the cross-rank barrier pairs CTA i with CTA i).
cudaError_t launch_zero_g0(int kind, const StepParams<1>& P, const LaunchCtx& ctx, int grid);
cudaError_t launch_zero_g1(int kind, const StepParams<1>& P, const LaunchCtx& ctx, int grid);
cudaError_t launch_zero_g2(int kind, const StepParams<1>& P, const LaunchCtx& ctx, int grid);

// Opt a kernel into `smem` bytes of dynamic shared memory (once per kernel and thread).
cudaError_t ensure_smem(const void* fn, int smem);

}  // namespace q8
