// q8_codec.cuh -- the stand-alone block-wise codec kernels (a8) besides the quantizer
// (q8_quant_kernel.cuh): dequantize, the tensor-wise absmax of Eq.3 and the non-finite
// gradient count.  Included by q8_api.cu only.
#pragma once

#include "q8_kernels.cuh"

namespace q8 {

// ---------------------------------------------------------------------------- codec kernels

// Tensor-wise absmax N = max |T| (Eq.3; the "reduction over the entire tensor" that
// block-wise quantization avoids): per-CTA REDUX/shared reduction, then one atomicMax
// per CTA on the float bits (non-negative floats order like unsigned integers).  *out must be
// 0 on entry.
__global__ void __launch_bounds__(kThreads) tensor_absmax_kernel(const float* __restrict__ x, int64_t n,
                                                                 unsigned int* __restrict__ out) {
    __shared__ unsigned int red[kWarps];
    float mx = 0.0f;
    const int64_t n4 = n / 4;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * kThreads) {
        const float4 v = ld_stream_f4(x + 4 * i);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    if (blockIdx.x == 0 && threadIdx.x < n - 4 * n4) mx = fmaxf(mx, fabsf(x[4 * n4 + threadIdx.x]));
    const unsigned int w = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x < 32) {
        const unsigned int v = __reduce_max_sync(0xffffffffu, threadIdx.x < kWarps ? red[threadIdx.x] : 0u);
        if (threadIdx.x == 0) atomicMax(out, v);
    }
}

// Block-wise dequantization: out = Q[code] * N_b -- a8.  TW: N = absmax[0] for all.
template <bool TW>
__global__ void __launch_bounds__(kThreads) dequantize_blockwise_kernel(const float* __restrict__ code,
                                                                        const uint8_t* __restrict__ codes,
                                                                        const float* __restrict__ absmax,
                                                                        float* __restrict__ out, int64_t n,
                                                                        int64_t nblocks) {
    __shared__ float sQ[256];
    const int tid = threadIdx.x;
    sQ[tid] = code[tid];
    __syncthreads();
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int64_t base = b * kBlock;
        const bool full = base + kBlock <= n;
        const float N = absmax[TW ? 0 : b];
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            if (full) {
                const uint32_t cc = ld_stream_u32(codes + i0);
                st_stream_f4(out + i0, make_float4(__fmul_rn(sQ[cc & 0xffu], N), __fmul_rn(sQ[(cc >> 8) & 0xffu], N),
                                                   __fmul_rn(sQ[(cc >> 16) & 0xffu], N),
                                                   __fmul_rn(sQ[cc >> 24], N)));
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e)
                    if (i0 + e < n) out[i0 + e] = __fmul_rn(sQ[codes[i0 + e]], N);
            }
        }
    }
}

// Non-finite gradient count (failure detection: non-finite gradients are out of contract
// for the step, G13; an AMP-style caller checks before stepping).  Bit tests on the raw encodings:
// fp32 exponent 0xff, fp16 0x1f, bf16 0xff (NaN or +-inf).  16-byte vector loads, one 64-bit
// atomic per CTA.
template <int GDT>
__global__ void __launch_bounds__(kThreads) count_nonfinite_kernel(const void* __restrict__ g, int64_t n,
                                                                   unsigned long long* __restrict__ out) {
    __shared__ unsigned int red[kWarps];
    constexpr int kPer = GDT == G_F32 ? 4 : 8;  // elements per 16-byte load
    unsigned int cnt = 0;
    const int64_t nv = n / kPer;
    const uint4* gv = static_cast<const uint4*>(g);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; i < nv;
         i += static_cast<int64_t>(gridDim.x) * kThreads) {
        const uint4 v = __ldcs(gv + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if constexpr (GDT == G_F32) {
                cnt += ((w[k] & 0x7f800000u) == 0x7f800000u);
            } else {
                const uint32_t m = GDT == G_F16 ? 0x7c00u : 0x7f80u;
                cnt += ((w[k] & m) == m) + (((w[k] >> 16) & m) == m);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < n - nv * kPer) {  // the tail (< kPer elements)
        const int64_t i = nv * kPer + threadIdx.x;
        if constexpr (GDT == G_F32) {
            cnt += ((static_cast<const uint32_t*>(g)[i] & 0x7f800000u) == 0x7f800000u);
        } else {
            const uint32_t m = GDT == G_F16 ? 0x7c00u : 0x7f80u;
            cnt += ((static_cast<const uint16_t*>(g)[i] & m) == m);
        }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int k = 0; k < kWarps; ++k) s += red[k];
        if (s) atomicAdd(out, s);
    }
}

}  // namespace q8
