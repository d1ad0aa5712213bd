// q8_kernels.cuh -- sm_100a kernels of the block-wise dynamic 8-bit optimizer step.
//
// Paper: Dettmers et al. 2021 (arXiv 2110.02861); "P:<line>" = /root/reference/PAPER.md,
// "G<n>" = readings in DESIGN.md section 3.  No tensor cores: nothing on this path is a
// dense contraction; the kernels are HBM-bound streaming kernels whose on-chip limits
// are instruction issue and shared-memory wavefronts.
//
// Work decomposition (all kernels): one CTA processes one 2048-element block at a time
// ("performing normalization independently in each core across this block"),
// grid-striding over blocks so the shared-memory tables are staged once per CTA.
// 256 threads x 8 elements: thread t owns the 4-element groups at block offsets
// c*1024 + 4t (c = 0, 1), so every warp-wide load/store instruction touches one
// contiguous span (512 B of fp32, 128 B of codes): fully coalesced, minimal L1 wavefronts.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace q8 {

constexpr int kBlock = 2048;       // B
constexpr int kThreads = 256;
constexpr int kVec = 4;            // elements per vector group
constexpr int kGroups = kBlock / (kThreads * kVec);  // 2 groups per thread
constexpr int kWarps = kThreads / 32;

enum { KIND_ADAM = 0, KIND_ADAMW = 1, KIND_MOMENTUM = 2 };
enum { G_F32 = 0, G_F16 = 1, G_BF16 = 2 };

// Device-resident immutable tables (built on the host, codebook_host.cpp), as fp32 words:
//   [0,256)     Q_s   signed dynamic tree codebook, ascending
//   [256,512)   E_s   signed thresholds, Eytzinger order (slot 0 unused)
//   [512,768)   Q_u   unsigned dynamic codebook, ascending
//   [768,1024)  E_u   unsigned thresholds, Eytzinger order
//   [1024,1280) S_s   signed thresholds T_k in sorted order, S_s[255] = +inf
//   [1280,1536) S_u   unsigned thresholds, sorted, S_u[255] = +inf
//   [1536,...)  bucket tables (uint8), see "bucketed search" below
constexpr int kTabQs = 0, kTabTs = 256, kTabQu = 512, kTabTu = 768, kTabSs = 1024, kTabSu = 1280;
constexpr int kTabLut = 1536;                     // word offset of the byte tables

// Bucketed search.  The binary search's first seven levels are replaced by
// one table lookup indexed by the leading bits of y, the eighth by a compare:
//   signed:   mag = |y| bits clamped below at 2^-22;  mk = (mag >> 17) - (2^-22 bits >> 17)
//             (exponent + 6 mantissa bits, 1409 buckets over [0, 1]); key = mk + 1536*[y < 0]
//   unsigned: mk = (max(bits, 2^-22 bits) >> 16) - (2^-22 bits >> 16)  (7 mantissa bits, 2817)
// LUT[key] = c0 = the smallest code in the bucket.  Every bucket spans at most two codes
// (verified exhaustively at table-build time), so code = c0 + [y > T_{c0}]  (T sorted).
constexpr uint32_t kMinMagBits = (127u - 22u) << 23;   // 2^-22: below every |threshold| (>= 1.6e-7)
constexpr int kShiftS = 17, kShiftU = 16;
constexpr int kBucketsS = ((0x3f800000 >> kShiftS) - (kMinMagBits >> kShiftS)) + 1;  // 1409
constexpr int kBucketsU = ((0x3f800000 >> kShiftU) - (kMinMagBits >> kShiftU)) + 1;  // 2817
constexpr int kNegOffS = 1536;
constexpr int kLutSBytes = 3072;                   // [0,1409) y >= 0, [1536, 2945) y < 0
constexpr int kLutUBytes = 2944;                   // 2817 used, padded to a multiple of 128
constexpr int kTabBytes = kTabLut * 4 + kLutSBytes + kLutUBytes;
constexpr int kTabFloats = kTabBytes / 4;
constexpr int SEARCH_EYTZINGER = 0, SEARCH_BUCKET = 1;

struct TensorDesc {
    float* p;
    const void* g;
    uint8_t* s1;
    uint8_t* s2;
    float* a1;
    float* a2;
    int64_t n;
};

struct StepScalars {       // all computed on the host in double, rounded once (G8-G10)
    float lr, beta1, beta2, omb1, omb2, step_size, eps_hat, wd, decay;
};

template <int MAXT>
struct StepParams {
    StepScalars s;
    int num_tensors;
    int64_t total_blocks;
    int64_t block_start[MAXT + 1];  // prefix sums of per-tensor block counts
    TensorDesc t[MAXT];
};

// ---------------------------------------------------------------------------- loads

__device__ __forceinline__ float4 ld_stream_f4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st_stream_f4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }
__device__ __forceinline__ uint32_t ld_stream_u32(const uint8_t* p) {
    return __ldcs(reinterpret_cast<const unsigned int*>(p));
}
__device__ __forceinline__ void st_stream_u32(uint8_t* p, uint32_t v) {
    __stcs(reinterpret_cast<unsigned int*>(p), v);
}

// 4 consecutive gradients widened to fp32 (exact for fp16/bf16, G13).
template <int GDT>
__device__ __forceinline__ void load_g4(const void* g, int64_t i, float out[4]) {
    if constexpr (GDT == G_F32) {
        float4 v = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(g) + i));
        out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
    } else {
        uint2 v = __ldcs(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(g) + i));
        if constexpr (GDT == G_F16) {
            float2 a = __half22float2(*reinterpret_cast<__half2*>(&v.x));
            float2 b = __half22float2(*reinterpret_cast<__half2*>(&v.y));
            out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
        } else {
            out[0] = __uint_as_float(v.x << 16);
            out[1] = __uint_as_float(v.x & 0xffff0000u);
            out[2] = __uint_as_float(v.y << 16);
            out[3] = __uint_as_float(v.y & 0xffff0000u);
        }
    }
}

template <int GDT>
__device__ __forceinline__ float load_g1(const void* g, int64_t i) {
    if constexpr (GDT == G_F32) return static_cast<const float*>(g)[i];
    else if constexpr (GDT == G_F16) return __half2float(static_cast<const __half*>(g)[i]);
    else return __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(g)[i]) << 16);
}

// ---------------------------------------------------------------------------- search

// Nearest code via the 8-step branch-free binary search (Eq.3 "via a binary search",
// P:76): descend the Eytzinger-ordered threshold tree, i <- 2i + [y > T[i]].  After 8
// levels i - 256 = #{k : y > T_k} = argmin_j |Q_j - y| with ties to the lower index (G6).
__device__ __forceinline__ uint32_t eytzinger_search(const float* __restrict__ T, float y) {
    uint32_t i = 1;
#pragma unroll
    for (int l = 0; l < 8; ++l) i = 2u * i + (y > T[i] ? 1u : 0u);
    return i - 256u;
}

// Bucketed nearest code: LUT lookup replaces levels 1-7 of the binary
// search, one compare against the sorted threshold T_{c0} is level 8.  Keys are clamped so a
// non-finite y (out of contract) can never index outside the tables.
__device__ __forceinline__ uint32_t bucket_search_signed(const uint8_t* __restrict__ lut,
                                                         const float* __restrict__ T, float y) {
    const uint32_t u = __float_as_uint(y);
    const uint32_t mag = min(max(u & 0x7fffffffu, kMinMagBits), 0x3f800000u);
    const uint32_t key = (mag >> kShiftS) - (kMinMagBits >> kShiftS) + ((u & 0x80000000u) ? kNegOffS : 0u);
    const uint32_t c0 = lut[key];
    return c0 + (y > T[c0] ? 1u : 0u);
}

__device__ __forceinline__ uint32_t bucket_search_unsigned(const uint8_t* __restrict__ lut,
                                                           const float* __restrict__ T, float y) {
    // signed clamp: negative y (sign bit set) joins bucket 0, whose nearest code is Q_u[0] = 0
    const int32_t u = min(max(static_cast<int32_t>(__float_as_uint(y)), static_cast<int32_t>(kMinMagBits)),
                          static_cast<int32_t>(0x3f800000));
    const uint32_t key = (static_cast<uint32_t>(u) >> kShiftU) - (kMinMagBits >> kShiftU);
    const uint32_t c0 = lut[key];
    return c0 + (y > T[c0] ? 1u : 0u);
}

// ---------------------------------------------------------------------------- reduction

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block absmax N_b = max |T_b|.  red is [2][kWarps], double-buffered by
// iteration parity so one __syncthreads per block suffices.
__device__ __forceinline__ float block_max(float v, float* red) {
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = red[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) r = fmaxf(r, red[w]);
    return r;
}

// ---------------------------------------------------------------------------- normalize

// y = x / N in IEEE binary32 (Eq.4's T_bi / N_b; G7).  Block-uniform mode:
//   0: N == 0           -> y = 0 (all elements are 0)
//   1: 2^-70 <= N < 2^126 -> reciprocal-multiply with one Markstein correction,
//      q = x*rcp, e = fma(-q, N, x), y = fma(e, rcp, q), rcp = RN(1/N).  Equals RN(x/N)
//      whenever |x/N| >= 2^-40 (verified on 6.7e7 adversarial pairs); below
//      that every dynamic-table threshold (|T| >= 1.6e-7) is far away, so codes agree.
//   2: otherwise        -> IEEE division
struct Normalizer {
    float N, rcp;
    int mode;
    __device__ __forceinline__ explicit Normalizer(float n) : N(n) {
        mode = (n == 0.0f) ? 0 : ((n >= 0x1p-70f && n < 0x1p126f) ? 1 : 2);
        rcp = (mode == 1) ? __frcp_rn(n) : 0.0f;
    }
    __device__ __forceinline__ float operator()(float x) const {
        if (mode == 1) {
            float q = __fmul_rn(x, rcp);
            float e = __fmaf_rn(-q, N, x);
            return __fmaf_rn(e, rcp, q);
        }
        if (mode == 0) return 0.0f;
        return __fdiv_rn(x, N);
    }
};

// ---------------------------------------------------------------------------- update

// One element of the 32-bit update (Eq.1 / Eq.2), each operator one IEEE RN operation in
// the order the equations write them (G9); identical operation sequence to the oracle.
template <int KIND>
__device__ __forceinline__ void update_element(const StepScalars& s, float& w, float g, float& m, float& r) {
    if constexpr (KIND == KIND_ADAMW) {
        w = __fmul_rn(w, s.decay);                       // decoupled decay (G10)
    } else {
        if (s.wd != 0.0f) g = __fadd_rn(g, __fmul_rn(s.wd, w));  // L2 (G10)
    }
    if constexpr (KIND == KIND_MOMENTUM) {
        m = __fadd_rn(__fmul_rn(s.beta1, m), g);         // Eq.1 m_t = b1 m + g
        w = __fadd_rn(w, -__fmul_rn(s.lr, m));           // w_t = w - a m_t
    } else {
        m = __fadd_rn(__fmul_rn(s.beta1, m), __fmul_rn(s.omb1, g));             // Eq.2 state 1
        r = __fadd_rn(__fmul_rn(s.beta2, r), __fmul_rn(s.omb2, __fmul_rn(g, g)));  // state 2
        w = __fadd_rn(w, -__fmul_rn(s.step_size, __fdiv_rn(m, __fadd_rn(__fsqrt_rn(r), s.eps_hat))));
    }
}

// ---------------------------------------------------------------------------- step kernel

template <int MAXT>
__device__ __forceinline__ int find_tensor(const StepParams<MAXT>& P, int64_t b) {
    if constexpr (MAXT == 1) {
        return 0;
    } else {
        int lo = 0, hi = P.num_tensors - 1;  // largest t with block_start[t] <= b
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (P.block_start[mid] <= b) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
}

// Shared-memory image of the tables one step kernel needs.
template <int SEARCH>
struct StepSmem {
    float qs[256], qu[256];                          // decode tables Q_s, Q_u
    float ts[256], tu[256];                          // thresholds: Eytzinger or sorted order
    uint8_t lut_s[SEARCH == SEARCH_BUCKET ? kLutSBytes : 4];
    uint8_t lut_u[SEARCH == SEARCH_BUCKET ? kLutUBytes : 4];
};

template <int SEARCH, bool kTwo>
__device__ __forceinline__ void stage_step_tables(StepSmem<SEARCH>& sm, const float* __restrict__ tabs) {
    const int tid = threadIdx.x;
    sm.qs[tid] = tabs[kTabQs + tid];
    sm.ts[tid] = tabs[(SEARCH == SEARCH_BUCKET ? kTabSs : kTabTs) + tid];
    if constexpr (kTwo) {
        sm.qu[tid] = tabs[kTabQu + tid];
        sm.tu[tid] = tabs[(SEARCH == SEARCH_BUCKET ? kTabSu : kTabTu) + tid];
    }
    if constexpr (SEARCH == SEARCH_BUCKET) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(tabs + kTabLut);
        uint32_t* dst_s = reinterpret_cast<uint32_t*>(sm.lut_s);
        for (int i = tid; i < kLutSBytes / 4; i += kThreads) dst_s[i] = src[i];
        if constexpr (kTwo) {
            uint32_t* dst_u = reinterpret_cast<uint32_t*>(sm.lut_u);
            for (int i = tid; i < kLutUBytes / 4; i += kThreads) dst_u[i] = src[kLutSBytes / 4 + i];
        }
    }
    __syncthreads();
}

template <int SEARCH>
__device__ __forceinline__ uint32_t nearest_s(const StepSmem<SEARCH>& sm, float y) {
    if constexpr (SEARCH == SEARCH_BUCKET) return bucket_search_signed(sm.lut_s, sm.ts, y);
    else return eytzinger_search(sm.ts, y);
}

template <int SEARCH>
__device__ __forceinline__ uint32_t nearest_u(const StepSmem<SEARCH>& sm, float y) {
    if constexpr (SEARCH == SEARCH_BUCKET) return bucket_search_unsigned(sm.lut_u, sm.tu, y);
    else return eytzinger_search(sm.tu, y);
}

// The fused step (S3; Fig.1): dequantize -> fp32 update -> block absmax ->
// requantize, all in registers; each HBM byte is read once and written once.
template <int KIND, int GDT, int MAXT, int SEARCH>
__global__ void __launch_bounds__(kThreads) optim8bit_step_kernel(const __grid_constant__ StepParams<MAXT> P,
                                                                  const float* __restrict__ tabs) {
    constexpr bool kTwo = (KIND != KIND_MOMENTUM);
    __shared__ __align__(16) StepSmem<SEARCH> sm;
    __shared__ float red[2][2][kWarps];
    const int tid = threadIdx.x;
    stage_step_tables<SEARCH, kTwo>(sm, tabs);
    const StepScalars& S = P.s;

    int parity = 0;
    for (int64_t gb = blockIdx.x; gb < P.total_blocks; gb += gridDim.x, parity ^= 1) {
        const int ti = find_tensor<MAXT>(P, gb);
        const TensorDesc& T = P.t[ti];
        const int64_t b = gb - P.block_start[ti];
        const int64_t base = b * kBlock;
        const bool full = base + kBlock <= T.n;

        float w[kGroups][kVec], g[kGroups][kVec], m[kGroups][kVec], r[kGroups][kVec];
        uint32_t c1[kGroups], c2[kGroups];
        const float N1old = T.a1[b];
        const float N2old = kTwo ? T.a2[b] : 0.0f;

        // ---- load (a2) + dequantize (a3)
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            if (full) {
                float4 pv = ld_stream_f4(T.p + i0);
                w[c][0] = pv.x; w[c][1] = pv.y; w[c][2] = pv.z; w[c][3] = pv.w;
                load_g4<GDT>(T.g, i0, g[c]);
                c1[c] = ld_stream_u32(T.s1 + i0);
                c2[c] = kTwo ? ld_stream_u32(T.s2 + i0) : 0u;
            } else {
                c1[c] = 0u; c2[c] = 0u;
#pragma unroll
                for (int e = 0; e < kVec; ++e) {
                    const bool ok = i0 + e < T.n;
                    w[c][e] = ok ? T.p[i0 + e] : 0.0f;
                    g[c][e] = ok ? load_g1<GDT>(T.g, i0 + e) : 0.0f;
                    c1[c] |= (ok ? static_cast<uint32_t>(T.s1[i0 + e]) : 0u) << (8 * e);
                    if (kTwo) c2[c] |= (ok ? static_cast<uint32_t>(T.s2[i0 + e]) : 0u) << (8 * e);
                }
            }
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
                m[c][e] = __fmul_rn(sm.qs[(c1[c] >> (8 * e)) & 0xffu], N1old);
                r[c][e] = kTwo ? __fmul_rn(sm.qu[(c2[c] >> (8 * e)) & 0xffu], N2old) : 0.0f;
            }
        }

        // ---- fp32 update (a4), element by element in registers
        float mx1 = 0.0f, mx2 = 0.0f;
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
                update_element<KIND>(S, w[c][e], g[c][e], m[c][e], r[c][e]);
                const bool ok = full || (i0 + e < T.n);
                if (!ok) { m[c][e] = 0.0f; r[c][e] = 0.0f; }
                mx1 = fmaxf(mx1, fabsf(m[c][e]));
                if (kTwo) mx2 = fmaxf(mx2, fabsf(r[c][e]));
            }
        }

        // ---- block absmax of the new states (a5)
        float* rb = &red[parity][0][0];
        mx1 = warp_max(mx1);
        if (kTwo) mx2 = warp_max(mx2);
        if ((tid & 31) == 0) {
            rb[tid >> 5] = mx1;
            if (kTwo) rb[kWarps + (tid >> 5)] = mx2;
        }
        __syncthreads();
        float N1 = rb[0], N2 = kTwo ? rb[kWarps] : 0.0f;
#pragma unroll
        for (int k = 1; k < kWarps; ++k) {
            N1 = fmaxf(N1, rb[k]);
            if (kTwo) N2 = fmaxf(N2, rb[kWarps + k]);
        }
        const Normalizer nz1(N1), nz2(N2);

        // ---- normalize + nearest code (a6, Eq.4) and store (a7)
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            uint32_t o1 = 0u, o2 = 0u;
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
                o1 |= nearest_s<SEARCH>(sm, nz1(m[c][e])) << (8 * e);
                if (kTwo) o2 |= nearest_u<SEARCH>(sm, nz2(r[c][e])) << (8 * e);
            }
            if (full) {
                st_stream_f4(T.p + i0, make_float4(w[c][0], w[c][1], w[c][2], w[c][3]));
                st_stream_u32(T.s1 + i0, o1);
                if (kTwo) st_stream_u32(T.s2 + i0, o2);
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) {
                    if (i0 + e < T.n) {
                        T.p[i0 + e] = w[c][e];
                        T.s1[i0 + e] = static_cast<uint8_t>(o1 >> (8 * e));
                        if (kTwo) T.s2[i0 + e] = static_cast<uint8_t>(o2 >> (8 * e));
                    }
                }
            }
        }
        if (tid == 0) {
            T.a1[b] = N1;
            if (kTwo) T.a2[b] = N2;
        }
    }
}

// ---------------------------------------------------------------------------- codec kernels

// In-order rank of Eytzinger node i (1..255) of the perfect 8-level tree.
__device__ __forceinline__ int eytzinger_rank_dev(int i) {
    const int level = 31 - __clz(i);
    const int pos = i - (1 << level);
    return (2 * pos + 1) * (1 << (7 - level)) - 1;
}

// Stage a caller-provided ascending table and derive its Eytzinger thresholds
// T_k = RD((Q_k + Q_{k+1}) / 2): __fadd_rd rounds the exact sum down, the halving is exact.
__device__ __forceinline__ void stage_generic_table(const float* __restrict__ code, float* sQ, float* sT) {
    const int tid = threadIdx.x;
    sQ[tid] = code[tid];
    __syncthreads();
    if (tid >= 1) {
        const int k = eytzinger_rank_dev(tid);
        sT[tid] = __fmul_rn(__fadd_rd(sQ[k], sQ[k + 1]), 0.5f);
    } else {
        sT[0] = __int_as_float(0x7f800000);
    }
    __syncthreads();
}

// Block-wise quantization, Eq.4 -- a8.  IEEE division for y = x / N_b.
__global__ void __launch_bounds__(kThreads) quantize_blockwise_kernel(const float* __restrict__ code,
                                                                      const float* __restrict__ x,
                                                                      float* __restrict__ absmax,
                                                                      uint8_t* __restrict__ codes, int64_t n,
                                                                      int64_t nblocks) {
    __shared__ float sQ[256], sT[256];
    __shared__ float red[2][kWarps];
    stage_generic_table(code, sQ, sT);
    const int tid = threadIdx.x;
    int parity = 0;
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, parity ^= 1) {
        const int64_t base = b * kBlock;
        const bool full = base + kBlock <= n;
        float v[kGroups][kVec];
        float mx = 0.0f;
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            if (full) {
                float4 xv = ld_stream_f4(x + i0);
                v[c][0] = xv.x; v[c][1] = xv.y; v[c][2] = xv.z; v[c][3] = xv.w;
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) v[c][e] = (i0 + e < n) ? x[i0 + e] : 0.0f;
            }
#pragma unroll
            for (int e = 0; e < kVec; ++e) mx = fmaxf(mx, fabsf(v[c][e]));
        }
        const float N = block_max(mx, red[parity]);
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            uint32_t o = 0u;
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
                const float y = (N > 0.0f) ? __fdiv_rn(v[c][e], N) : 0.0f;
                o |= eytzinger_search(sT, y) << (8 * e);
            }
            if (full) {
                st_stream_u32(codes + i0, o);
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e)
                    if (i0 + e < n) codes[i0 + e] = static_cast<uint8_t>(o >> (8 * e));
            }
        }
        if (tid == 0) absmax[b] = N;
    }
}

// Block-wise quantization with the library's own dynamic data type (signed P:90 or unsigned
// P:118): same normalization (Normalizer) and bucketed search as the fused step kernel.
template <bool kSigned>
__global__ void __launch_bounds__(kThreads) quantize_blockwise_dynamic_kernel(const float* __restrict__ tabs,
                                                                              const float* __restrict__ x,
                                                                              float* __restrict__ absmax,
                                                                              uint8_t* __restrict__ codes, int64_t n,
                                                                              int64_t nblocks) {
    __shared__ float sT[256];
    __shared__ __align__(16) uint8_t sLut[kSigned ? kLutSBytes : kLutUBytes];
    __shared__ float red[2][kWarps];
    const int tid = threadIdx.x;
    sT[tid] = tabs[(kSigned ? kTabSs : kTabSu) + tid];
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(tabs + kTabLut) + (kSigned ? 0 : kLutSBytes / 4);
        uint32_t* dst = reinterpret_cast<uint32_t*>(sLut);
        for (int i = tid; i < (kSigned ? kLutSBytes : kLutUBytes) / 4; i += kThreads) dst[i] = src[i];
    }
    __syncthreads();
    int parity = 0;
    for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x, parity ^= 1) {
        const int64_t base = b * kBlock;
        const bool full = base + kBlock <= n;
        float v[kGroups][kVec];
        float mx = 0.0f;
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            if (full) {
                float4 xv = ld_stream_f4(x + i0);
                v[c][0] = xv.x; v[c][1] = xv.y; v[c][2] = xv.z; v[c][3] = xv.w;
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e) v[c][e] = (i0 + e < n) ? x[i0 + e] : 0.0f;
            }
#pragma unroll
            for (int e = 0; e < kVec; ++e) mx = fmaxf(mx, fabsf(v[c][e]));
        }
        const Normalizer nz(block_max(mx, red[parity]));
#pragma unroll
        for (int c = 0; c < kGroups; ++c) {
            const int64_t i0 = base + c * (kThreads * kVec) + tid * kVec;
            uint32_t o = 0u;
#pragma unroll
            for (int e = 0; e < kVec; ++e) {
                const float y = nz(v[c][e]);
                o |= (kSigned ? bucket_search_signed(sLut, sT, y) : bucket_search_unsigned(sLut, sT, y)) << (8 * e);
            }
            if (full) {
                st_stream_u32(codes + i0, o);
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e)
                    if (i0 + e < n) codes[i0 + e] = static_cast<uint8_t>(o >> (8 * e));
            }
        }
        if (tid == 0) absmax[b] = nz.N;
    }
}

// Block-wise dequantization: out = Q[code] * N_b -- a8.
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
        const float N = absmax[b];
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

}  // namespace q8
