// q8_layerwise.cuh -- the two extra passes of the layer-wise (trust-ratio) 8-bit optimizers,
// LAMB and LARS (the paper benchmarks both, T5 P:366-367).  Readings L1-L4:
// DESIGN.md section 3.
//
// A layer-wise step needs per-tensor norms before any parameter can move, so it is three
// stream-ordered launches per chunk of <= 384 tensors:
//   1. layer_norms_kernel   per 2048-block partial sums (binary64) of w^2 and of x^2, where
//                           x = u (LAMB: the update direction from the fp32 post-update states,
//                           computed exactly as pass 3 computes it) or x = g (LARS); no writes
//                           besides the partials (16 B per block)
//   2. layer_scale_kernel   one warp per tensor: sums its partials in a fixed order, then the
//                           tensor's scale a = RN(lr * ratio) (binary64 ratio, L3)
//   3. optim8bit_step_kernel<KIND_LAMB / KIND_LARS>  the fused step with the tensor's scale
// HBM traffic per parameter with bf16 grads: LAMB 8 B (pass 1) + 14 B (pass 3); LARS 6 B + 12 B.
#pragma once

#include "q8_kernels.cuh"

namespace q8 {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int KIND, int GDT, int MAXT>
__global__ void __launch_bounds__(kThreads) layer_norms_kernel(const __grid_constant__ StepParams<MAXT> P,
                                                               const float* __restrict__ tabs,
                                                               double2* __restrict__ partial) {
    static_assert(KIND == KIND_LAMB || KIND == KIND_LARS, "layer-wise kinds only");
    __shared__ float Qs[256], Qu[256];
    __shared__ double red[2][kWarps];
    const int tid = threadIdx.x;
    if constexpr (KIND == KIND_LAMB) {
        Qs[tid] = tabs[kTabQs + tid];
        Qu[tid] = tabs[kTabQu + tid];
        __syncthreads();
    }
    const StepScalars S = P.s;
    for (int64_t gb = blockIdx.x; gb < P.total_blocks; gb += gridDim.x) {
        const int ti = find_tensor<MAXT>(P, gb);
        const TensorDesc& T = P.t[ti];
        const int64_t b = gb - P.block_start[ti];
        const int64_t base = b * kBlock;
        const bool full = base + kBlock <= T.n;
        const float N1 = KIND == KIND_LAMB ? T.a1[b] : 0.0f;
        const float N2 = KIND == KIND_LAMB ? T.a2[b] : 0.0f;
        double sw = 0.0, sx = 0.0;
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int i0 = c * (kThreads * kVec) + tid * kVec;
            float w[kVec], g[kVec];
            uint32_t k1 = 0, k2 = 0;
            if (full) {
                const float4 pv = *reinterpret_cast<const float4*>(T.p + base + i0);
                w[0] = pv.x; w[1] = pv.y; w[2] = pv.z; w[3] = pv.w;
                load_g4<GDT>(T.g, base + i0, g);
                if constexpr (KIND == KIND_LAMB) {
                    k1 = *reinterpret_cast<const uint32_t*>(T.s1 + base + i0);
                    k2 = *reinterpret_cast<const uint32_t*>(T.s2 + base + i0);
                }
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) {
                    const bool ok = base + i0 + e < T.n;
                    w[e] = ok ? T.p[base + i0 + e] : 0.0f;
                    g[e] = ok ? load_g1<GDT>(T.g, base + i0 + e) : 0.0f;
                    if constexpr (KIND == KIND_LAMB) {
                        k1 |= (ok ? static_cast<uint32_t>(T.s1[base + i0 + e]) : 0u) << (8 * e);
                        k2 |= (ok ? static_cast<uint32_t>(T.s2[base + i0 + e]) : 0u) << (8 * e);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
                if (!full && base + i0 + e >= T.n) continue;
                sw += static_cast<double>(w[e]) * static_cast<double>(w[e]);  // exact product
                if constexpr (KIND == KIND_LARS) {
                    sx += static_cast<double>(g[e]) * static_cast<double>(g[e]);
                } else {
                    // the update direction of pass 3, bit for bit: dequantize, Eq.2 (G9),
                    // d = m / (sqrt(r) + eps_hat), u = c d + wd w (L1)
                    float m = __fmul_rn(Qs[(k1 >> (8 * e)) & 0xffu], N1);
                    float r = __fmul_rn(Qu[(k2 >> (8 * e)) & 0xffu], N2);
                    m = __fadd_rn(__fmul_rn(S.beta1, m), __fmul_rn(S.omb1, g[e]));
                    r = __fadd_rn(__fmul_rn(S.beta2, r), __fmul_rn(S.omb2, __fmul_rn(g[e], g[e])));
                    const float d = __fdiv_rn(m, __fadd_rn(__fsqrt_rn(r), S.eps_hat));
                    const float u = __fadd_rn(__fmul_rn(S.step_size, d), __fmul_rn(S.wd, w[e]));
                    sx += static_cast<double>(u) * static_cast<double>(u);
                }
            }
        }
        sw = warp_sum_f64(sw);
        sx = warp_sum_f64(sx);
        if ((tid & 31) == 0) {
            red[0][tid >> 5] = sw;
            red[1][tid >> 5] = sx;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, x = 0.0;
            for (int k = 0; k < kWarps; ++k) {
                a += red[0][k];
                x += red[1][k];
            }
            partial[gb] = make_double2(a, x);
        }
        __syncthreads();
    }
}

// One warp per tensor of the launch: ||w|| and ||x|| from its block partials (fixed summation
// order: lane-strided, then a butterfly), then the fp32 scale (L1-L3):
//   LAMB  a = RN(lr * (||w|| / ||u||))                    (1 when either norm is 0)
//   LARS  a = RN(lr * (eta ||w|| / (||g|| + wd ||w||)))   (lr when either norm is 0)
template <int KIND, int MAXT>
__global__ void __launch_bounds__(32) layer_scale_kernel(const __grid_constant__ StepParams<MAXT> P,
                                                         const double2* __restrict__ partial, float* __restrict__ scale,
                                                         double lr, double eta, double wd) {
    const int t = blockIdx.x, lane = threadIdx.x;
    double sw = 0.0, sx = 0.0;
    for (int64_t b = P.block_start[t] + lane; b < P.block_start[t + 1]; b += 32) {
        const double2 v = partial[b];
        sw += v.x;
        sx += v.y;
    }
    sw = warp_sum_f64(sw);
    sx = warp_sum_f64(sx);
    if (lane == 0) {
        const double wn = sqrt(sw), xn = sqrt(sx);
        double f = 1.0;
        if (wn > 0.0 && xn > 0.0) f = KIND == KIND_LAMB ? wn / xn : eta * wn / (xn + wd * wn);
        scale[t] = static_cast<float>(lr * f);
    }
}

}  // namespace q8
