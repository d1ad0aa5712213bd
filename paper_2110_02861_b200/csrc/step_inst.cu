// step_inst.cu -- instantiates and launches the fused step kernels for ONE gradient dtype
// (Q8_GDT = 0 fp32, 1 fp16, 2 bf16); build.py compiles this file once per dtype in parallel.
#include <algorithm>
#include <cstdlib>

#include "q8_launch.h"
#include "q8_layerwise.cuh"
#include "q8_step_kernel.cuh"

#ifndef Q8_GDT
#error "compile with -DQ8_GDT=0|1|2"
#endif

namespace q8 {
namespace {

// Grid of a persistent step launch: one CTA per SM, fewer when there are fewer blocks than sub-blocks.
int64_t persistent_grid(int64_t work_blocks, int nsub, int sms) {
    const int64_t grid = (work_blocks + nsub - 1) / nsub;
    return grid > sms ? sms : grid;
}

template <typename Kern, typename... Args>
cudaError_t persistent(Kern fn, int nsub, int subt, int64_t work_blocks, const LaunchCtx& ctx, const Args&... args) {
    const int smem = step_smem_bytes(nsub, Q8_GDT);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = persistent_grid(work_blocks, nsub, ctx.sms);
    fn<<<static_cast<unsigned>(grid), nsub * subt, smem, ctx.stream>>>(args...);
    return cudaGetLastError();
}

// The same launch as a programmatic dependent launch: the kernel may start while the previous kernel on
// the stream drains (it must execute griddepcontrol.wait before consuming that kernel's results).
template <typename... KArgs, typename... Args>
cudaError_t persistent_pdl(void (*fn)(KArgs...), int nsub, int subt, int64_t work_blocks, const LaunchCtx& ctx,
                           const Args&... args) {
    const int smem = step_smem_bytes(nsub, Q8_GDT);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (work_blocks + nsub - 1) / nsub;
    if (grid > ctx.sms) grid = ctx.sms;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(nsub * subt);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = ctx.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, args...);
}

// Sub-block size: 128 threads x 16 elements for 16-bit gradients (4 sub-blocks, 16 warps per
// SM: the per-block overhead is amortized over more elements), 256 x 8 for fp32 gradients (their
// 20 KB stages allow only 3 sub-blocks, so more warps per sub-block).  Q8_SUBT overrides.
template <int KIND, int MAXT, int SUBT>
cudaError_t launch_kind_t(const StepParams<MAXT>& P, const LaunchCtx& ctx) {
    constexpr int G = Q8_GDT;
    if (ctx.search == SEARCH_EYTZINGER)  // reference variant: one configuration
        return persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_EYTZINGER, 3, SUBT>, 3, SUBT, P.total_blocks,
                          ctx, P, ctx.tabs);
    switch (ctx.nsub) {
        case 2: return persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, 2, SUBT>, 2, SUBT,
                                  P.total_blocks, ctx, P, ctx.tabs);
        case 4:
            if constexpr (G != G_F32)
                return persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, 4, SUBT>, 4, SUBT,
                                  P.total_blocks, ctx, P, ctx.tabs);
            [[fallthrough]];
        default: return persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, 3, SUBT>, 3, SUBT,
                                   P.total_blocks, ctx, P, ctx.tabs);
    }
}

template <int KIND, int MAXT>
cudaError_t launch_kind(const StepParams<MAXT>& P, const LaunchCtx& ctx) {
    if constexpr (MAXT > 1) {
        if (ctx.plan) {  // plans: the default configuration only
            constexpr int G = Q8_GDT;
            constexpr int NS = G == G_F32 ? 3 : 4;
            constexpr int SUBT = G == G_F32 ? 256 : 128;
            return persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, NS, SUBT, MODE_STEP, true>, NS, SUBT,
                              P.total_blocks, ctx, P, ctx.tabs);
        }
    }
    const int subt = ctx.subt ? ctx.subt : (Q8_GDT == G_F32 ? 256 : 128);
    return subt == 128 ? launch_kind_t<KIND, MAXT, 128>(P, ctx) : launch_kind_t<KIND, MAXT, 256>(P, ctx);
}

template <int MAXT>
cudaError_t launch_any(int kind, const StepParams<MAXT>& P, const LaunchCtx& ctx) {
    switch (kind) {
        case KIND_ADAM:
            return P.s.wd != 0.0f ? launch_kind<KIND_ADAM | KIND_L2, MAXT>(P, ctx) : launch_kind<KIND_ADAM, MAXT>(P, ctx);
        case KIND_ADAMW: return launch_kind<KIND_ADAMW, MAXT>(P, ctx);
        case KIND_MOMENTUM:
            return P.s.wd != 0.0f ? launch_kind<KIND_MOMENTUM | KIND_L2, MAXT>(P, ctx)
                                  : launch_kind<KIND_MOMENTUM, MAXT>(P, ctx);
        default: return cudaErrorInvalidValue;
    }
}

// Layer-wise kinds (LAMB, LARS): norms -> per-tensor scale -> fused step, default configuration.
template <int KIND, int MAXT>
cudaError_t launch_layerwise_t(const StepParams<MAXT>& P, const LaunchCtx& ctx, double2* partial,
                               float* scale, unsigned int* count, double lr, double eta, double wd) {
    constexpr int G = Q8_GDT;
    constexpr int NS = G == G_F32 ? 3 : 4;
    constexpr int SUBT = G == G_F32 ? 256 : 128;
    if (P.total_blocks == 0) {  // only empty tensors: their scale is still defined (lr)
        layer_scale_kernel<KIND, MAXT><<<P.num_tensors, kScaleThreads, 0, ctx.stream>>>(P, partial, scale, lr, eta, wd,
                                                                                        0);
        return cudaGetLastError();
    }
    cudaError_t e;
    // LARS as ONE cooperative launch (MODE_LARSF: norms, grid barrier, scales, grid barrier, step) when
    // Q8_LARS_ONE_LAUNCH=1.  Measured slower than the three launches below on ResNet-50 (0.121 vs
    // 0.110 ms): the persistent 16-warp CTAs hide the norms pass's load latency worse
    // than the many small CTAs of lars_norms_kernel, and each grid barrier adds a tail.
    static const bool one_launch = [] {
        const char* v = std::getenv("Q8_LARS_ONE_LAUNCH");
        return v && std::atoi(v) == 1;
    }();
    if constexpr (KIND == KIND_LARS) if (one_launch) {
        const auto fn = optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, NS, SUBT, MODE_LARSF>;
        const int smem = step_smem_bytes(NS, G);
        e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(P.lw.gbar, 0, 2 * sizeof(unsigned int), ctx.stream);
        if (e != cudaSuccess) return e;
        int64_t grid = (P.total_blocks + NS - 1) / NS;
        if (grid > ctx.sms) grid = ctx.sms;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(NS * SUBT);
        cfg.dynamicSmemBytes = static_cast<size_t>(smem);
        cfg.stream = ctx.stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, fn, P, ctx.tabs);
    }
    if constexpr (KIND == KIND_LAMB) {
        e = persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, NS, SUBT, MODE_NORMS>, NS, SUBT,
                       P.total_blocks, ctx, P, ctx.tabs);
    } else {
        static int occ = [] {
            int o = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, lars_norms_kernel<G, MAXT>, kThreads, 0) !=
                    cudaSuccess || o < 1)
                o = 1;
            return o;
        }();
        // norms + per-tensor scales in one pass, then the step as a dependent launch (q8_layerwise.cuh)
        const int64_t g1 = std::min<int64_t>(P.total_blocks, static_cast<int64_t>(ctx.sms) * occ);
        lars_norms_kernel<G, MAXT><<<static_cast<unsigned>(g1), kThreads, 0, ctx.stream>>>(P, count, scale);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        return persistent_pdl(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, NS, SUBT>, NS, SUBT,
                              P.total_blocks, ctx, P, ctx.tabs);
    }
    if (e != cudaSuccess) return e;
    // LAMB (the only kind that gets here): the norms pass wrote one partial per warp per tensor segment of
    // each of its grid * NS sub-blocks, in the slot of the segment's last block
    const int64_t nsubs = persistent_grid(P.total_blocks, NS, ctx.sms) * NS;
    lamb_scale_kernel<MAXT><<<P.num_tensors, kScaleThreads, 0, ctx.stream>>>(P, partial, scale, lr, SUBT / 32,
                                                                                  nsubs);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return persistent(optim8bit_step_kernel<KIND, G, MAXT, SEARCH_BUCKET, NS, SUBT>, NS, SUBT, P.total_blocks,
                      ctx, P, ctx.tabs);
}

}  // namespace

#define Q8_CAT2(a, b) a##b
#define Q8_CAT(a, b) Q8_CAT2(a, b)
namespace {
template <int KIND>
cudaError_t launch_plan_small_kind(const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx) {
    constexpr int G = Q8_GDT;
    constexpr int NS = G == G_F32 ? 3 : 4;
    constexpr int SUBT = G == G_F32 ? 256 : 128;
    return persistent(optim8bit_step_kernel<KIND, G, kSmallMaxT, SEARCH_BUCKET, NS, SUBT, MODE_STEP, true>, NS, SUBT,
                      P.total_blocks, ctx, P, ctx.tabs);
}
}  // namespace

cudaError_t Q8_CAT(launch_plan_small_g, Q8_GDT)(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx) {
    switch (kind) {
        case KIND_ADAM:
            return P.s.wd != 0.0f ? launch_plan_small_kind<KIND_ADAM | KIND_L2>(P, ctx) : launch_plan_small_kind<KIND_ADAM>(P, ctx);
        case KIND_ADAMW: return launch_plan_small_kind<KIND_ADAMW>(P, ctx);
        case KIND_MOMENTUM:
            return P.s.wd != 0.0f ? launch_plan_small_kind<KIND_MOMENTUM | KIND_L2>(P, ctx)
                                  : launch_plan_small_kind<KIND_MOMENTUM>(P, ctx);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t Q8_CAT(launch_step_g, Q8_GDT)(int kind, const StepParams<1>* single,
                                          const StepParams<kMultiMaxT>* multi, const LaunchCtx& ctx) {
    return single ? launch_any<1>(kind, *single, ctx) : launch_any<kMultiMaxT>(kind, *multi, ctx);
}

}  // namespace q8

namespace q8 {
cudaError_t Q8_CAT(launch_layerwise_g, Q8_GDT)(int kind, const StepParams<kMultiMaxT>& P, const LaunchCtx& ctx,
                                               double2* partial, float* scale, unsigned int* count, double lr,
                                               double eta, double wd) {
    if (kind == KIND_LAMB) return launch_layerwise_t<KIND_LAMB, kMultiMaxT>(P, ctx, partial, scale, count, lr, eta, wd);
    if (kind == KIND_LARS) return launch_layerwise_t<KIND_LARS, kMultiMaxT>(P, ctx, partial, scale, count, lr, eta, wd);
    return cudaErrorInvalidValue;
}
cudaError_t Q8_CAT(launch_layerwise_g, Q8_GDT)(int kind, const StepParams<kSmallMaxT>& P, const LaunchCtx& ctx,
                                               double2* partial, float* scale, unsigned int* count, double lr,
                                               double eta, double wd) {
    if (kind == KIND_LAMB) return launch_layerwise_t<KIND_LAMB, kSmallMaxT>(P, ctx, partial, scale, count, lr, eta, wd);
    if (kind == KIND_LARS) return launch_layerwise_t<KIND_LARS, kSmallMaxT>(P, ctx, partial, scale, count, lr, eta, wd);
    return cudaErrorInvalidValue;
}
}  // namespace q8

namespace q8 {
namespace {
template <int KIND>
cudaError_t launch_zero_t(const StepParams<1>& P, const LaunchCtx& ctx, int grid) {
    constexpr int G = Q8_GDT;
    constexpr int NS = G == G_F32 ? 3 : 4;
    constexpr int SUBT = G == G_F32 ? 256 : 128;
    const auto fn = optim8bit_step_kernel<KIND, G, 1, SEARCH_BUCKET, NS, SUBT, MODE_ZERO>;
    const int smem = step_smem_bytes(NS, G);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(fn), smem);
    if (e != cudaSuccess) return e;
    // Cooperative launch: the runtime guarantees (or refuses with
    // cudaErrorCooperativeLaunchTooLarge) that every CTA of this grid is resident at once, so CTA i
    // can never wait at the cross-rank flag barrier behind a CTA of its own rank that has no SM.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(NS * SUBT);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = ctx.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, P, ctx.tabs);
}
}  // namespace

cudaError_t Q8_CAT(launch_zero_g, Q8_GDT)(int kind, const StepParams<1>& P, const LaunchCtx& ctx, int grid) {
    switch (kind) {
        case KIND_ADAM:
            return P.s.wd != 0.0f ? launch_zero_t<KIND_ADAM | KIND_L2>(P, ctx, grid) : launch_zero_t<KIND_ADAM>(P, ctx, grid);
        case KIND_ADAMW: return launch_zero_t<KIND_ADAMW>(P, ctx, grid);
        case KIND_MOMENTUM:
            return P.s.wd != 0.0f ? launch_zero_t<KIND_MOMENTUM | KIND_L2>(P, ctx, grid)
                                  : launch_zero_t<KIND_MOMENTUM>(P, ctx, grid);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace q8
