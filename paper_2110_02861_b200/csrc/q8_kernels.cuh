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

enum { KIND_ADAM = 0, KIND_ADAMW = 1, KIND_MOMENTUM = 2, KIND_LAMB = 3, KIND_LARS = 4 };
// Kinds with two states (s1 signed, s2 unsigned): the Adam family and LAMB; Momentum and LARS
// keep one (the momentum buffer, signed table).
// Kernel-only flag on KIND_ADAM / KIND_MOMENTUM: the L2 weight-decay term g += wd*w (G10) is on
// (wd != 0).  The launchers pick it from the host hyper-parameters, so the step kernel carries no
// per-element run-time test for it.
constexpr int KIND_L2 = 8;
__host__ __device__ constexpr int kind_base(int kind) { return kind & 7; }
__host__ __device__ constexpr bool two_states(int kind) {
    return kind_base(kind) != KIND_MOMENTUM && kind_base(kind) != KIND_LARS;
}
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
// one lookup in a table indexed directly by the leading bits of y, the eighth by a compare:
//   signed:   key = bits(y) >> 17  (sign, exponent, 6 mantissa bits); 0x6000 keys cover [-1, 1]
//   unsigned: key = max(bits(y) >> 16, 0x3400) (exponent, 7 mantissa bits); keys 0x3400-0x3fff
//             cover [0, 1] (every y < 2^-23 shares bucket 0x3400: all below T_0 = 1.6e-7)
// LUT[key] = c0 = the smallest code of any y in the bucket.  Every bucket spans at most two
// codes (checked exhaustively when the tables are built), so code = c0 + [y > T_{c0}].
constexpr int kShiftS = 17, kShiftU = 16;
constexpr int kLutUKeyMin = 0x3400;
constexpr int kLutSBytes = 0x6000, kLutUBytes = 0x4000 - kLutUKeyMin;
constexpr int kTabBytes = kTabLut * 4 + kLutSBytes + kLutUBytes;
constexpr int kTabFloats = kTabBytes / 4;
constexpr int SEARCH_EYTZINGER = 0, SEARCH_BUCKET = 1;

// One tensor of a launch.  8-bit states: s1/s2 codes, a1/a2 absmax.  In multi-tensor launches a
// tensor with a1 == NULL keeps 32-bit states (the Stable Embedding, S3.3 P:124): s1/s2 then hold
// its fp32 m / r arrays.
struct TensorDesc {
    float* p;
    const void* g;
    uint8_t* s1;
    uint8_t* s2;
    float* a1;
    float* a2;
    int64_t n;
};

struct StepScalars {       // all computed in double and rounded once (G8-G10)
    // step_size: alpha_t for Adam/AdamW; for LAMB the bias-correction factor c alone (L1)
    float lr, beta1, beta2, omb1, omb2, step_size, eps_hat, wd, decay;
    int fast_div;          // eps_hat >= 2^-40: the packed sqrt/div fast path may be used
};

// The fp32 scalars of one update at step t (1-based), from the double hyper-parameters: one
// source for the host (every host-stepped launch) and the device (capturable launches that read t
// from device memory, DeviceStep).  Readings G8 (Kingma & Ba's folded bias correction
// alpha_t = alpha sqrt(1 - b2^t)/(1 - b1^t), eps_hat = eps sqrt(1 - b2^t)), G10 (decay = 1 - lr wd)
// and, for LAMB, L1 (step_size = the bias-correction factor c alone).  Every expression is
// evaluated in binary64 (no contraction: the library is built with -fmad=false) and rounded once.
// Host and device differ only in the pow() implementation (glibc vs CUDA's libdevice, both within
// 1-2 double ulps), which can change an fp32 result only if the double value lies within ~2^-51
// relative of an fp32 rounding boundary; tests/test_gpu_plan.py compares both for t = 1 .. 2^20.
__host__ __device__ inline StepScalars compute_scalars(int kind, double lr, double beta1, double beta2, double eps,
                                                       double wd, int bias_correction, int64_t step) {
    StepScalars s;
    s.lr = static_cast<float>(lr);
    s.beta1 = static_cast<float>(beta1);
    s.beta2 = static_cast<float>(beta2);
    s.omb1 = static_cast<float>(1.0 - beta1);
    s.omb2 = static_cast<float>(1.0 - beta2);
    if (bias_correction) {
        const double bc1 = 1.0 - pow(beta1, static_cast<double>(step));
        const double bc2 = 1.0 - pow(beta2, static_cast<double>(step));
        s.step_size = static_cast<float>(lr * sqrt(bc2) / bc1);
        s.eps_hat = static_cast<float>(eps * sqrt(bc2));
    } else {
        s.step_size = static_cast<float>(lr);
        s.eps_hat = static_cast<float>(eps);
    }
    s.wd = static_cast<float>(wd);
    s.decay = static_cast<float>(1.0 - lr * wd);
    if (kind == 3 /* KIND_LAMB */) {
        s.step_size = bias_correction ? static_cast<float>(sqrt(1.0 - pow(beta2, static_cast<double>(step))) /
                                                           (1.0 - pow(beta1, static_cast<double>(step))))
                                      : 1.0f;
    }
    s.fast_div = (s.eps_hat >= 0x1p-40f && isfinite(s.eps_hat)) ? 1 : 0;
    return s;
}

// Capturable step (q8_plan_step_device): the launch reads t - 1 from *step (device int64) and
// computes its scalars on the device; the last CTA to finish the launch that carries `advance`
// stores t back (a CTA-completion counter, reset to 0 by that CTA), so a whole optimizer step can be
// captured in a CUDA graph and replayed with no host work.
struct DeviceStep {
    int64_t* step = nullptr;  // NULL: host scalars (StepParams::s) are used
    unsigned int* done;    // CTA completion counter, 0 between launches
    int advance;           // this launch stores *step = t at its end
    int kind;
    double lr, beta1, beta2, eps, wd;
    int bias_correction;
};

// Fused ZeRO-1 step over peer memory: every rank's full padded
// gradient and parameter buffers and its signal pad, mapped into this GPU's address space
// (NVLink P2P / CUDA IPC).  Reading Z1: the shard gradient is the rank-order binary32 sum of the
// ranks' gradients divided by world (IEEE; a multiply by the exact reciprocal when world is a
// power of two); the updated shard parameters are written into every rank's buffer.
constexpr int kMaxWorld = 16;
struct ZeroParams {
    const void* g[kMaxWorld];
    float* p[kMaxWorld];
    uint32_t* sig[kMaxWorld];   // [2 phases][world][grid] uint32 flags (epochs)
    float* p_mc;                // NVLS multicast address of the parameter buffers (NULL: W peer stores)
    int64_t off;                // first element of this rank's shard
    int world, rank;
    uint32_t epoch;             // this call's flag value (strictly increasing, >= 1)
    float invw;                 // 1/world (exact when pow2)
    int pow2;
    int64_t pad_;               // keeps the size a multiple of 16 B (the fields after it stay 16-B aligned)
};
static_assert(sizeof(ZeroParams) % 16 == 0, "ZeroParams keeps the step parameters 16-byte aligned");

// LARS in ONE cooperative launch (MODE_LARSF): norms pass, grid barrier, per-tensor scales, grid
// barrier, fused step.  gbar: [count, generation] of the grid barrier (count 0 on entry).
struct LayerwiseFused {
    double lr, eta, wd;
    unsigned int* gbar;
};
static_assert(sizeof(LayerwiseFused) % 16 == 0, "keeps the step parameters 16-byte aligned");

template <int MAXT>
struct StepParams {
    StepScalars s;
    DeviceStep ds;                  // multi-tensor plans only (ds.step NULL otherwise)
    const float* scale;             // LAMB / LARS: per-tensor trust scale RN(lr*ratio) (L1-L3)
    double2* partial;               // LAMB norms pass: per-block (sum w^2, sum u^2)
    LayerwiseFused lw;              // LARS one-launch mode only
    ZeroParams z;                   // fused ZeRO-1 mode only
    int num_tensors;
    int64_t total_blocks;
    int64_t block_start[MAXT + 1];  // prefix sums of per-tensor block counts
    TensorDesc t[MAXT];
};

// The gradient of tensor ti of a launch.
template <int MAXT>
__device__ __forceinline__ const void* grad_of(const StepParams<MAXT>&, const TensorDesc& T, int) {
    return T.g;
}

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
    // mode-1 path only (caller has checked mode == 1 for the whole block)
    __device__ __forceinline__ float fast(float x) const {
        const float q = __fmul_rn(x, rcp);
        const float e = __fmaf_rn(-q, N, x);
        return __fmaf_rn(e, rcp, q);
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

// Tensor of global block b: the largest t with block_start[t] <= b.  `from` is a tensor known to
// start at or before b (grid-stride loops visit blocks in increasing order, so the previous
// answer is one): the common case -- b still inside tensor `from` -- costs one compare instead of
// a dependent binary search over the launch's parameter-space table.
template <int MAXT>
__device__ __forceinline__ int find_tensor(const StepParams<MAXT>& P, int64_t b, int from = 0) {
    if constexpr (MAXT == 1) {
        return 0;
    } else {
        if (from + 1 >= P.num_tensors || P.block_start[from + 1] > b) return from;
        int lo = from + 1, hi = P.num_tensors - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (P.block_start[mid] <= b) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
}

}  // namespace q8
