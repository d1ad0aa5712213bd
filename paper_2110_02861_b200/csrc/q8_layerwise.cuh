// q8_layerwise.cuh -- the two extra passes of the layer-wise (trust-ratio) 8-bit optimizers,
// LAMB and LARS (the paper benchmarks both, T5 P:366-367).  Readings L1-L4:
// DESIGN.md section 3.
//
// A layer-wise step needs per-tensor norms before any parameter can move, so it is three
// stream-ordered launches per chunk of <= 384 tensors (LARS: two -- its norms pass also computes the
// scales, lars_norms_kernel below):
//   1. norms pass           partial sums (binary64) of w^2 and of x^2 -- LAMB: one per warp per
//                           run of consecutive blocks of one tensor (segment) that a sub-block steps,
//                           in the slot of the segment's last block --, where
//                           x = u (LAMB: the update direction from the fp32 post-update states,
//                           computed exactly as pass 3 computes it -- the fused step kernel in
//                           MODE_NORMS: same TMA stages, decode and update, no stores) or x = g
//                           (LARS: lars_norms_kernel); no writes besides the partials (16 B/block)
//   2. lamb_scale_kernel    one CTA per tensor: sums its partials in a fixed order, then the
//                           tensor's scale a = RN(lr * ratio) (binary64 ratio, L3)
//   3. optim8bit_step_kernel<KIND_LAMB / KIND_LARS>  the fused step with the tensor's scale
// HBM traffic per parameter with bf16 grads: LAMB 8 B (pass 1) + 14 B (pass 3); LARS 6 B + 12 B.
// LAMB's pass 1 keeps two blocks in flight per sub-block (q8_step_kernel.cuh, stage_part_b).  LARS can
// also run as one cooperative launch (MODE_LARSF in q8_step_kernel.cuh, Q8_LARS_ONE_LAUNCH=1).
#pragma once

#include "q8_kernels.cuh"
#include "q8_step_kernel.cuh"

namespace q8 {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// LARS norms pass with the per-tensor scales folded in (two launches per LARS step instead of three).
// CTA q takes the contiguous block range [q*B/Q, (q+1)*B/Q) of the launch.  Per block: binary64 sums
// of w^2 and g^2 (warp butterflies, then the 8 warps in order: ONE partial per block, partial[block]).
// When the range leaves a tensor (and at its end) thread 0 adds the number of that tensor's blocks it
// summed to the tensor's counter (count[t], zero on entry); the CTA that completes a tensor's count
// sums its partials in a fixed order (thread-strided over blocks, warp butterfly, warps in order --
// reading L3: any fixed order) and writes scale[t] = RN(lr * eta ||w|| / (||g|| + wd ||w||)) (lr when
// a norm is 0, L2), then resets count[t] to 0.  Empty tensors (no blocks) get scale lr.  The kernel
// lets the step launch early (programmatic dependent launch): the step stages its tables and first
// blocks while this pass drains, and waits for it (griddepcontrol.wait) before it reads any scale.
template <int MAXT>
__device__ __forceinline__ void lars_count_tensor(const StepParams<MAXT>& P, int ti, unsigned int seg,
                                                  unsigned int* __restrict__ count, float* __restrict__ scale,
                                                  double (*red)[kWarps], int* last) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        __threadfence();  // this CTA's partials of ti (all written by thread 0) before they are counted
        const unsigned int nb = static_cast<unsigned int>(P.block_start[ti + 1] - P.block_start[ti]);
        *last = atomicAdd(count + ti, seg) + seg == nb;
    }
    __syncthreads();
    if (!*last) return;
    __threadfence();
    double aw = 0.0, ag = 0.0;
    for (int64_t b = P.block_start[ti] + tid; b < P.block_start[ti + 1]; b += kThreads) {
        const double2 v = __ldcg(P.partial + b);
        aw += v.x;
        ag += v.y;
    }
    aw = warp_sum_f64(aw);
    ag = warp_sum_f64(ag);
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = aw;
        red[1][tid >> 5] = ag;
    }
    __syncthreads();
    if (tid == 0) {
        aw = ag = 0.0;
        for (int k = 0; k < kWarps; ++k) {
            aw += red[0][k];
            ag += red[1][k];
        }
        const double wn = sqrt(aw), gn = sqrt(ag);
        double f = 1.0;
        if (wn > 0.0 && gn > 0.0) f = P.lw.eta * wn / (gn + P.lw.wd * wn);
        scale[ti] = static_cast<float>(P.lw.lr * f);
        count[ti] = 0u;
    }
    __syncthreads();  // red and *last are free again
}

template <int GDT, int MAXT>
__global__ void __launch_bounds__(kThreads) lars_norms_kernel(const __grid_constant__ StepParams<MAXT> P,
                                                              unsigned int* __restrict__ count,
                                                              float* __restrict__ scale) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ double red[2][2][kWarps];  // [block parity][w, g][warp]
    __shared__ int last;
    const int tid = threadIdx.x;
    for (int t = blockIdx.x * kThreads + tid; t < P.num_tensors; t += gridDim.x * kThreads)
        if (P.block_start[t + 1] == P.block_start[t]) scale[t] = static_cast<float>(P.lw.lr);
    const int64_t gb0 = static_cast<int64_t>(blockIdx.x) * P.total_blocks / gridDim.x;
    const int64_t gb1 = static_cast<int64_t>(blockIdx.x + 1) * P.total_blocks / gridDim.x;
    if (gb0 >= gb1) return;
    int ti = find_tensor<MAXT>(P, gb0, 0);
    unsigned int seg = 0;  // blocks of tensor ti summed by this CTA
    for (int64_t gb = gb0; gb < gb1; ++gb) {
        if (gb >= P.block_start[ti + 1]) {
            lars_count_tensor<MAXT>(P, ti, seg, count, scale, red[0], &last);
            ti = find_tensor<MAXT>(P, gb, ti);
            seg = 0;
        }
        const TensorDesc& T = P.t[ti];
        const int64_t base = (gb - P.block_start[ti]) * kBlock;
        const bool full = base + kBlock <= T.n;
        double sw = 0.0, sg = 0.0;
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int i0 = c * (kThreads * kVec) + tid * kVec;
            float w[kVec], g[kVec];
            if (full) {
                const float4 pv = *reinterpret_cast<const float4*>(T.p + base + i0);
                w[0] = pv.x; w[1] = pv.y; w[2] = pv.z; w[3] = pv.w;
                load_g4<GDT>(T.g, base + i0, g);
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) {
                    const bool ok = base + i0 + e < T.n;
                    w[e] = ok ? T.p[base + i0 + e] : 0.0f;
                    g[e] = ok ? load_g1<GDT>(T.g, base + i0 + e) : 0.0f;
                }
            }
#pragma unroll
            for (int e = 0; e < kVec; ++e) {  // squares of binary32 values are exact in binary64
                sw = __fma_rn(static_cast<double>(w[e]), static_cast<double>(w[e]), sw);
                sg = __fma_rn(static_cast<double>(g[e]), static_cast<double>(g[e]), sg);
            }
        }
        sw = warp_sum_f64(sw);
        sg = warp_sum_f64(sg);
        const int par = static_cast<int>(gb & 1);  // double-buffered: one barrier per block
        if ((tid & 31) == 0) {
            red[par][0][tid >> 5] = sw;
            red[par][1][tid >> 5] = sg;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int k = 0; k < kWarps; ++k) {
                a += red[par][0][k];
                b += red[par][1][k];
            }
            P.partial[gb] = make_double2(a, b);
        }
        ++seg;
    }
    lars_count_tensor<MAXT>(P, ti, seg, count, scale, red[0], &last);
}

// LAMB: one CTA per tensor of the launch, ||w|| and ||u|| from the norms pass's segment partials.  The
// pass (MODE_NORMS of the step kernel) gives sub-block q of its Q = nsubs sub-blocks the block range
// [q*B/Q, (q+1)*B/Q) and writes, per warp, one partial pair per run of that range inside one tensor,
// in the slot of the run's last block.  Tensor t's blocks [bs, be) meet the ranges q0..q1 (those
// holding bs and be-1); the run of range q ends at min(be, (q+1)*B/Q) - 1.  Fixed summation order:
// thread-strided over q, slots in order, warp butterfly, warps in order (L3); then as below,
//   a = RN(lr * (||w|| / ||u||))   (lr when either norm is 0)
__device__ __forceinline__ int64_t range_start(int64_t q, int64_t B, int64_t Q) { return q * B / Q; }
__device__ __forceinline__ int64_t range_of_block(int64_t x, int64_t B, int64_t Q) {
    int64_t q = x * Q / B;  // within one of the answer; settle it with the kernel's own arithmetic
    while (q + 1 < Q && range_start(q + 1, B, Q) <= x) ++q;
    while (q > 0 && range_start(q, B, Q) > x) --q;
    return q;
}
constexpr int kScaleThreads = 1024;
template <int MAXT>
__global__ void __launch_bounds__(kScaleThreads) lamb_scale_kernel(const __grid_constant__ StepParams<MAXT> P,
                                                                   const double2* __restrict__ partial,
                                                                   float* __restrict__ scale, double lr, int wpb,
                                                                   int64_t nsubs) {
    __shared__ double red[2][kScaleThreads / 32];
    const int t = blockIdx.x, tid = threadIdx.x;
    const int64_t bs = P.block_start[t], be = P.block_start[t + 1], B = P.total_blocks, Q = nsubs;
    double sw = 0.0, sx = 0.0;
    if (be > bs) {
        const int64_t q0 = range_of_block(bs, B, Q), q1 = range_of_block(be - 1, B, Q);
        for (int64_t q = q0 + tid; q <= q1; q += kScaleThreads) {
            const int64_t r0 = range_start(q, B, Q), r1 = range_start(q + 1, B, Q);
            if (r0 == r1) continue;  // an empty range (fewer blocks than sub-blocks)
            const int64_t end = (be < r1 ? be : r1) - 1;
            double2 v[kNormSlots];
#pragma unroll
            for (int k = 0; k < kNormSlots; ++k)
                if (k < wpb) v[k] = partial[end * kNormSlots + k];
#pragma unroll
            for (int k = 0; k < kNormSlots; ++k)
                if (k < wpb) {
                    sw += v[k].x;
                    sx += v[k].y;
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
        sw = sx = 0.0;
        for (int k = 0; k < kScaleThreads / 32; ++k) {
            sw += red[0][k];
            sx += red[1][k];
        }
        const double wn = sqrt(sw), xn = sqrt(sx);
        scale[t] = static_cast<float>(lr * (wn > 0.0 && xn > 0.0 ? wn / xn : 1.0));
    }
}

// One CTA (kThreads) per tensor of the launch: ||w|| and ||x|| from its per-warp block partials
// (wpb of the kNormSlots slots per block; fixed summation order: thread-strided over blocks, slots in
// order, warp butterfly, warps in order), then the fp32 scale (L1-L3):
//   LAMB  a = RN(lr * (||w|| / ||u||))                    (1 when either norm is 0)
//   LARS  a = RN(lr * (eta ||w|| / (||g|| + wd ||w||)))   (lr when either norm is 0)
// (LAMB now uses lamb_scale_kernel above; this per-block form serves the lists with no blocks at all)
template <int KIND, int MAXT>
__global__ void __launch_bounds__(kScaleThreads) layer_scale_kernel(const __grid_constant__ StepParams<MAXT> P,
                                                                    const double2* __restrict__ partial,
                                                                    float* __restrict__ scale, double lr, double eta,
                                                                    double wd, int wpb) {
    __shared__ double red[2][kScaleThreads / 32];
    const int t = blockIdx.x, tid = threadIdx.x;
    double sw = 0.0, sx = 0.0;
    const int64_t b1 = P.block_start[t + 1];
    for (int64_t b = P.block_start[t] + tid; b < b1; b += kScaleThreads) {
        double2 v[kNormSlots];
#pragma unroll
        for (int k = 0; k < kNormSlots; ++k)  // independent loads first, then the sums in slot order
            if (k < wpb) v[k] = partial[b * kNormSlots + k];
#pragma unroll
        for (int k = 0; k < kNormSlots; ++k)
            if (k < wpb) {
                sw += v[k].x;
                sx += v[k].y;
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
        sw = sx = 0.0;
        for (int k = 0; k < kScaleThreads / 32; ++k) {
            sw += red[0][k];
            sx += red[1][k];
        }
        const double wn = sqrt(sw), xn = sqrt(sx);
        double f = 1.0;
        if (wn > 0.0 && xn > 0.0) f = KIND == KIND_LAMB ? wn / xn : eta * wn / (xn + wd * wn);
        scale[t] = static_cast<float>(lr * f);
    }
}

}  // namespace q8
