// q8_step32_kernel.cuh -- the 32-bit-state optimizer step: the paper keeps
// the Stable Embedding layer's optimizer states in 32 bits ("This is the only layer that uses
// 32-bit optimizer states", S3.3 P:124-125).  Same fp32 update as the fused 8-bit step (Eq.1/2,
// G8-G12, identical operation order), states m, r stored as fp32 -- no quantization.
// TensorDesc is reused with s1 / s2 holding the fp32 m / r arrays.
#pragma once

#include "q8_kernels.cuh"

namespace q8 {

template <int KIND, int GDT, int MAXT>
__global__ void __launch_bounds__(kThreads) optim32bit_step_kernel(const __grid_constant__ StepParams<MAXT> P) {
    constexpr bool kTwo = (KIND != KIND_MOMENTUM);
    const StepScalars S = P.s;
    const int tid = threadIdx.x;
    int ti = 0;
    for (int64_t gb = blockIdx.x; gb < P.total_blocks; gb += gridDim.x) {
        ti = find_tensor<MAXT>(P, gb, ti);
        const TensorDesc& T = P.t[ti];
        const int64_t base = (gb - P.block_start[ti]) * kBlock;
        float* __restrict__ m = reinterpret_cast<float*>(T.s1) + base;
        float* __restrict__ r = kTwo ? reinterpret_cast<float*>(T.s2) + base : nullptr;
        float* __restrict__ p = T.p + base;
        const bool full = base + kBlock <= T.n;
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int i0 = c * (kThreads * kVec) + tid * kVec;
            float w[kVec], g[kVec], mm[kVec], rr[kVec];
            if (full) {
                const float4 pv = ld_stream_f4(p + i0), mv = ld_stream_f4(m + i0);
                const float4 rv = kTwo ? ld_stream_f4(r + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
                w[0] = pv.x; w[1] = pv.y; w[2] = pv.z; w[3] = pv.w;
                mm[0] = mv.x; mm[1] = mv.y; mm[2] = mv.z; mm[3] = mv.w;
                rr[0] = rv.x; rr[1] = rv.y; rr[2] = rv.z; rr[3] = rv.w;
                load_g4<GDT>(T.g, base + i0, g);
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) {
                    const bool ok = base + i0 + e < T.n;
                    w[e] = ok ? p[i0 + e] : 0.f;
                    mm[e] = ok ? m[i0 + e] : 0.f;
                    rr[e] = (ok && kTwo) ? r[i0 + e] : 0.f;
                    g[e] = ok ? load_g1<GDT>(T.g, base + i0 + e) : 0.f;
                }
            }
#pragma unroll
            for (int e = 0; e < kVec; ++e) update_element<KIND>(S, w[e], g[e], mm[e], rr[e]);
            if (full) {
                st_stream_f4(p + i0, make_float4(w[0], w[1], w[2], w[3]));
                st_stream_f4(m + i0, make_float4(mm[0], mm[1], mm[2], mm[3]));
                if (kTwo) st_stream_f4(r + i0, make_float4(rr[0], rr[1], rr[2], rr[3]));
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) {
                    if (base + i0 + e < T.n) {
                        p[i0 + e] = w[e];
                        m[i0 + e] = mm[e];
                        if (kTwo) r[i0 + e] = rr[e];
                    }
                }
            }
        }
    }
}

}  // namespace q8
