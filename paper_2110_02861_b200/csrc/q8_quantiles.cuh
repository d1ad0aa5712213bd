// q8_quantiles.cuh -- SRAM-Quantiles (App G) and the quantile data type (App F.2,
// Eq.5) on sm_100a.  Readings Q1-Q5 in DESIGN.md section 3.
//
// "Instead of finding the full eCDF we find the eCDF for a subset of values of the tensor that
// fits into SRAM (about 4096 32-bit values).  Once we found the quantiles for each subset, we
// average the quantiles".  B200 design:
//   * persistent CTAs of 256 threads, each chunk of 4096 values sorted entirely on chip: 16 keys
//     per thread in registers, a bitonic network in its "flip" form (every comparator ascending:
//     for each merge size K a mirror stage e <-> e^(K-1), then half-cleaners e <-> e^j), so no
//     per-stage direction logic.  Comparators whose partners live in the same thread are
//     register min/max; partners in the same warp are exchanged with SHFL (j = 16..256); only
//     the 6 stages with partners in another warp (j >= 512) go through shared memory, double-
//     buffered so each needs one barrier.  Keys are the fp32 values (FMNMX); cross-thread
//     comparators run in signed views so that they too cost one FMNMX per key (see below).
//   * the 257 order statistics floor(j*m/257) (Q1, Q2) are read from the sorted chunk and summed
//     per thread in binary64 registers across the CTA's chunks (Q4); one partial row per CTA.
//   * a one-CTA finalize kernel sums the partial rows in CTA order, divides by the chunk count,
//     rounds once to fp32, and optionally builds the Eq.5 codebook (Q5) on the device.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace q8 {

constexpr int kQChunk = 4096;          // "about 4096 32-bit values", reading Q3
#ifndef Q8_QT_PER
#define Q8_QT_PER 16
#endif
constexpr int kQPer = Q8_QT_PER;       // keys per thread (16 or 32)
constexpr int kQThreads = kQChunk / kQPer;
constexpr int kQQuads = kQPer / 4;
static_assert(kQPer == 16 || kQPer == 32, "16 or 32 keys per thread");
constexpr int kQuantiles = 257;        // Q_X(j/257), j = 0..256 (Eq.5, reading Q1)
constexpr int kQSmemBytes = 2 * kQChunk * 4;  // two 16 KB exchange buffers

// Keys are the fp32 values themselves (zeros canonicalized to +0 on load: -0 and +0 are equal
// values, reading Q2 compares values), compared with FMNMX.  In-thread comparators have
// compile-time roles (one FMNMX per key).  For comparators whose partner is another thread, the
// lower thread keeps the min and the upper the max; to make that ONE instruction on both sides each
// thread holds its keys in a signed "view" v = s*key during such stages (s = +1 lower, -1 upper):
// then both compute v = min(v, -v_partner) (the negation is an FMNMX operand modifier), since for
// the upper thread -min(-a, -b) = max(a, b).  Changing views is an exact multiply by +-1 on the FMA
// pipe, which this kernel otherwise leaves idle.

// word offset of key e = P t + r in an exchange buffer (P = kQPer): thread t's quads are permuted
// so that eight consecutive threads' 16-byte accesses of one quad hit eight distinct bank groups
__device__ __forceinline__ int qslot(int t, int q) {
    return kQPer * t + 4 * (q ^ (kQPer == 16 ? ((t >> 1) & 3) : (t & 7)));
}

__device__ __forceinline__ void q_scale(float (&a)[kQPer], float f) {
#pragma unroll
    for (int r = 0; r < kQPer; r++) a[r] = __fmul_rn(a[r], f);  // f = +-1: exact
}

// ------------------------------------------------------------------ comparator stages
// in-thread half-cleaner, distance J < P (key space)
template <int J>
__device__ __forceinline__ void q_ce_reg(float (&a)[kQPer]) {
#pragma unroll
    for (int r = 0; r < kQPer; r++)
        if (!(r & J)) {
            const float x = a[r], y = a[r | J];
            a[r] = fminf(x, y);
            a[r | J] = fmaxf(x, y);
        }
}

// in-thread mirror stage of merge size K <= P: r <-> r ^ (K-1) (key space)
template <int K>
__device__ __forceinline__ void q_mirror_reg(float (&a)[kQPer]) {
#pragma unroll
    for (int r = 0; r < kQPer; r++)
        if (!(r & (K / 2))) {
            const int p = r ^ (K - 1);
            const float x = a[r], y = a[p];
            a[r] = fminf(x, y);
            a[p] = fmaxf(x, y);
        }
}

// enter the view of a cross-thread stage whose upper side is `upper` (s_cur: the current view)
__device__ __forceinline__ void q_enter(float (&a)[kQPer], float& s_cur, bool upper) {
    const float s_new = upper ? -1.0f : 1.0f;
    q_scale(a, s_cur * s_new);
    s_cur = s_new;
}

// warp half-cleaner: partner lane ^ M (M in 1..16), same register (distance M*P)
template <int M>
__device__ __forceinline__ void q_ce_shfl(float (&a)[kQPer], int lane, float& s_cur) {
    q_enter(a, s_cur, lane & M);
#pragma unroll
    for (int r = 0; r < kQPer; r++) a[r] = fminf(a[r], -__shfl_xor_sync(0xffffffffu, a[r], M));
}

// warp mirror stage of merge size K in (P, 32P]: partner lane ^ (K/P - 1), register P-1-r
template <int K>
__device__ __forceinline__ void q_mirror_shfl(float (&a)[kQPer], int lane, float& s_cur) {
    constexpr int M = K / kQPer - 1;
    q_enter(a, s_cur, lane & (K / (2 * kQPer)));
    float o[kQPer];
#pragma unroll
    for (int r = 0; r < kQPer; r++) o[r] = __shfl_xor_sync(0xffffffffu, a[kQPer - 1 - r], M);
#pragma unroll
    for (int r = 0; r < kQPer; r++) a[r] = fminf(a[r], -o[r]);
}

// cross-warp stage through shared memory: partner thread t ^ T; MIRROR reverses the registers
// (mirror of merge size K: T = K/P - 1, upper bit K/2P).  `buf` alternates between the two
// exchange buffers, so one barrier per stage suffices (a buffer is rewritten only after the
// next stage's barrier, which every thread reaches after its reads of this one).
template <int T, bool MIRROR>
__device__ __forceinline__ void q_stage_smem(float (&a)[kQPer], int t, float* xbuf, int& buf, float& s_cur) {
    q_enter(a, s_cur, MIRROR ? (t & ((T + 1) / 2)) : (t & T));
    float* s = xbuf + buf * kQChunk;
    buf ^= 1;
#pragma unroll
    for (int q = 0; q < kQQuads; q++)
        *reinterpret_cast<float4*>(s + qslot(t, q)) = make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
    __syncthreads();
    const int pt = t ^ T;
    float o[kQPer];
#pragma unroll
    for (int q = 0; q < kQQuads; q++) {
        const float4 v = *reinterpret_cast<const float4*>(s + qslot(pt, q));
        o[4 * q] = v.x;
        o[4 * q + 1] = v.y;
        o[4 * q + 2] = v.z;
        o[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int r = 0; r < kQPer; r++) a[r] = fminf(a[r], -(MIRROR ? o[kQPer - 1 - r] : o[r]));
}

// Per-thread context of the network: the two block-wide exchange buffers (cross-warp stages).
struct QCtx {
    int t, lane;
    float* xbuf;   // 2 x 4096 words
    int buf;
};

// in-register half-cleaners J, J/2, ..., 1 (key space)
template <int J>
__device__ __forceinline__ void q_cleaners_reg(float (&a)[kQPer]) {
    if constexpr (J >= 1) {
        q_ce_reg<J>(a);
        q_cleaners_reg<J / 2>(a);
    }
}

// half-cleaners of distance J, J/2, ..., 1 (key e = P t + r: J < P in registers, J < 32P within
// the warp, else shared memory).  Cross-thread stages run in views; the view is left (back to
// key space) before the first in-register stage.
template <int J>
__device__ __forceinline__ void q_cleaners(float (&a)[kQPer], QCtx& c, float& s_cur) {
    if constexpr (J >= 1) {
        if constexpr (J < kQPer) {
            q_scale(a, s_cur);
            s_cur = 1.0f;
            q_cleaners_reg<J>(a);
        } else {
            if constexpr (J < 32 * kQPer) q_ce_shfl<J / kQPer>(a, c.lane, s_cur);
            else q_stage_smem<J / kQPer, false>(a, c.t, c.xbuf, c.buf, s_cur);
            q_cleaners<J / 2>(a, c, s_cur);
        }
    }
}

// bitonic merges of size K, 2K, ..., 4096 (flip form: mirror stage, then half-cleaners)
// The network sorts the two halves of the chunk (merges up to kQSortK = 2048); the last merge is
// replaced by selection: each wanted order statistic is found by one merge-path binary search over
// the two sorted halves (q_select), which costs ~12 shared loads per quantile instead of the 12
// network stages of the final merge for every key.
#ifndef Q8_QT_SELECT
#define Q8_QT_SELECT 1
#endif
constexpr int kQSortK = Q8_QT_SELECT ? kQChunk / 2 : kQChunk;

template <int K>
__device__ __forceinline__ void q_merges(float (&a)[kQPer], QCtx& c) {
    if constexpr (K <= kQSortK) {
        float s_cur = 1.0f;
        if constexpr (K <= kQPer) q_mirror_reg<K>(a);
        else if constexpr (K <= 32 * kQPer) q_mirror_shfl<K>(a, c.lane, s_cur);
        else q_stage_smem<K / kQPer - 1, true>(a, c.t, c.xbuf, c.buf, s_cur);
        q_cleaners<K / 4>(a, c, s_cur);
        q_merges<2 * K>(a, c);
    }
}

// word of key e in an exchange buffer (the layout q_stage_smem / the publish step write)
__device__ __forceinline__ int qword(int e) { return qslot(e / kQPer, (e % kQPer) >> 2) + (e & 3); }

// The value of rank i (0-based) of the chunk.  Without selection the buffer holds the sorted chunk.
// With it, it holds two ascending runs A = [0, H), B = [H, 2H) (H = kQChunk/2): the element of rank
// i of their merge is the last of the first D = i+1 merged elements; with a = #A-elements among them
// (the merge path: A[a-1] <= B[D-a] and B[D-1-a] < A[a], ties taken from A first) it is
// max(A[a-1], B[D-1-a]).  Equal values make the tie rule irrelevant: the value is unique (Q2).
__device__ __forceinline__ float q_select(const float* s, int i) {
    if constexpr (!Q8_QT_SELECT) {
        return s[qword(i)];
    } else {
        constexpr int H = kQChunk / 2;
        const int D = i + 1;
        int lo = D > H ? D - H : 0, hi = D < H ? D : H;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s[qword(mid)] <= s[qword(H + D - 1 - mid)]) lo = mid + 1;
            else hi = mid;
        }
        const float x = lo > 0 ? s[qword(lo - 1)] : -__int_as_float(0x7f800000);
        const float y = D - lo > 0 ? s[qword(H + D - 1 - lo)] : -__int_as_float(0x7f800000);
        return fmaxf(x, y);
    }
}

// ------------------------------------------------------------------ SRAM-Quantiles pass
// partial[blockIdx.x * 257 + j] = sum over this CTA's chunks c (c = blockIdx.x + k*gridDim.x)
// of the chunk's j-th sample quantile (binary64).
// 4 resident CTAs per SM (64 registers, no spills): the network's pipes (ALU for FMNMX, the
// shared-memory crossbar for SHFL and the exchanges) are co-limits at ~60-70 % each, so more
// warps to hide the SHFL / LDS latency is what pays (measured: 2 CTAs 11.4 ms, 3: 11.0, 4: 10.5).
#ifndef Q8_QT_MINB
#define Q8_QT_MINB 4
#endif
__global__ void __launch_bounds__(kQThreads, Q8_QT_MINB) sram_quantiles_kernel(const float* __restrict__ x, int64_t n,
                                                                    int64_t nchunks, double* __restrict__ partial) {
    extern __shared__ __align__(16) float xbuf[];
    const int t = threadIdx.x, lane = t & 31;
    QCtx ctx;
    ctx.t = t;
    ctx.lane = lane;
    ctx.xbuf = xbuf;
    ctx.buf = 0;
    constexpr int kJ = (kQuantiles + kQThreads - 1) / kQThreads;  // quantiles j = t + k*T per thread
    double acc[kJ];
#pragma unroll
    for (int k = 0; k < kJ; k++) acc[k] = 0.0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const int64_t base = c * kQChunk;
        const int64_t left = n - base;
        const int m = left < kQChunk ? static_cast<int>(left) : kQChunk;
        float a[kQPer];
        // which element lands in which register does not matter (the network sorts the set):
        // coalesced float4 loads, zeros canonicalized (-0 + 0 = +0), the chunk's tail padded
        // with +inf (never selected: every selected index is < m)
#pragma unroll
        for (int q = 0; q < kQQuads; q++) {
            const int e = 4 * (t + kQThreads * q);
            if (e + 4 <= m) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(x + base + e));
                a[4 * q] = __fadd_rn(v.x, 0.0f);
                a[4 * q + 1] = __fadd_rn(v.y, 0.0f);
                a[4 * q + 2] = __fadd_rn(v.z, 0.0f);
                a[4 * q + 3] = __fadd_rn(v.w, 0.0f);
            } else {
#pragma unroll
                for (int i = 0; i < 4; i++)
                    a[4 * q + i] = (e + i < m) ? __fadd_rn(x[base + e + i], 0.0f) : __int_as_float(0x7f800000);
            }
        }
        q_merges<2>(a, ctx);
        // sorted runs of kQSortK: key e = P t + r is a[r] of thread t; publish and read the order
        // statistics
        float* s = xbuf + ctx.buf * kQChunk;
        ctx.buf ^= 1;
#pragma unroll
        for (int q = 0; q < kQQuads; q++)
            *reinterpret_cast<float4*>(s + qslot(t, q)) = make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kJ; k++) {
            const int j = t + k * kQThreads;
            if (j < kQuantiles) {
                const int i = static_cast<int>((static_cast<int64_t>(j) * m) / kQuantiles);  // Q2
                acc[k] += static_cast<double>(q_select(s, i));
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kJ; k++) {
        const int j = t + k * kQThreads;
        if (j < kQuantiles) partial[static_cast<int64_t>(blockIdx.x) * kQuantiles + j] = acc[k];
    }
}

// ------------------------------------------------------------------ finalize (one CTA)
// quantiles[j] = RN32( (sum_b partial[b][j]) / nchunks ) (Q4); if code != NULL also the Eq.5
// quantile data type (Q5): mid_i = (Q_i + Q_{i+1}) * 0.5 in binary64, code_i = RN32(mid_i / max|mid|)
// (all zeros when every midpoint is 0).
__global__ void __launch_bounds__(512) quantiles_finalize_kernel(const double* __restrict__ partial, int nrows,
                                                                 int64_t nchunks, float* __restrict__ quantiles,
                                                                 float* __restrict__ code) {
    __shared__ float q[kQuantiles];
    __shared__ double wmax[16];
    const int j = threadIdx.x;
    if (j < kQuantiles) {
        double s = 0.0;
        for (int b = 0; b < nrows; b++) s += partial[static_cast<int64_t>(b) * kQuantiles + j];
        const float v = static_cast<float>(s / static_cast<double>(nchunks));
        q[j] = v;
        quantiles[j] = v;
    }
    if (code == nullptr) return;
    __syncthreads();
    double mid = 0.0;
    if (j < 256) mid = (static_cast<double>(q[j]) + static_cast<double>(q[j + 1])) * 0.5;
    double m = fabs(mid);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((j & 31) == 0) wmax[j >> 5] = m;
    __syncthreads();
    double M = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); w++) M = fmax(M, wmax[w]);
    if (j < 256) code[j] = M > 0.0 ? static_cast<float>(mid / M) : 0.0f;
}

}  // namespace q8
