// q8_quant_kernel.cuh -- the stand-alone block-wise quantizer (Eq.4 P:105-108,
// Eq.3 P:73-78 for the tensor-wise variant) as a persistent, TMA-pipelined streaming kernel.
//
// Work decomposition: one CTA per SM, NSUB = 4 sub-blocks of 128 threads; a sub-block owns one
// 2048-element block at a time (16 elements per thread, thread t owns elements c*512 + 4t .. +3)
// and grid-strides over the blocks.  Each sub-block has kQStages shared-memory stages of 8 KB fed
// by TMA bulk copies (mbarrier completion), kQStages - 1 blocks ahead of the one being quantized,
// so the HBM latency of the loads is hidden (the previous direct-load kernel reached 44 % of the
// copy peak, latency-bound; BENCH codec line in profiles/).  A stage is released without a
// barrier: each warp counts itself out after reading it and the last one issues the TMA of the
// block kQStages iterations ahead into it.
//
// Tables:
//   BUILTIN  the library's signed / unsigned dynamic type: the step kernel's bucket table and
//            threshold rows (q8_step_kernel.cuh, "Bucketed search"), normalization by the packed
//            Markstein division (IEEE fallback outside its range).
//   GENERIC  a caller table Q[256] (strictly ascending): thresholds T_k = RD((Q_k + Q_{k+1})/2)
//            derived per CTA, Eytzinger order, 32 lane copies per node (conflict-free), the 8-step
//            descent i <- 2i + [y > T_i] (Eq.3 "binary search"); IEEE division y = RN(x/N).
// TW (tensor-wise): N = absmax[0], computed beforehand over the whole tensor; nothing reduced or
// stored per block.
#pragma once

#include "q8_step_kernel.cuh"

namespace q8 {

constexpr int kQNSub = 4, kQSubT = 256, kQStages = 3;
constexpr uint32_t kQBarAddr = 0x7200;                   // [sub][stage] mbarriers
constexpr uint32_t kQCntAddr = kQBarAddr + kQNSub * kQStages * 8;   // [sub][stage] release counters
constexpr uint32_t kQGenSorted = 0x20000;                // GENERIC: 256 rows x 128 B, sorted T_c (T_255 = +inf)
constexpr uint32_t kQGenRows = 0x28000;                  // GENERIC: 256 rows x 128 B (Eytzinger nodes)
constexpr uint32_t kQGenT = kLutUAddr;                   // GENERIC: plain sorted T[256] for the table build (1 KB)
constexpr int kQLutMinBlocksPerCta = 16;                 // GENERIC: build the bucket table only for launches this long
constexpr int kQtSmemBytes = static_cast<int>(0x38000 - kDynBase);
static_assert(kQCntAddr + kQNSub * kQStages * 4 <= 0x8000, "quantizer barriers below the free region");
static_assert(kQNSub * kQStages <= 12, "stages: 8 in 0x10000-0x20000, 4 in 0x30000-0x38000");

// Shared address of stage s of sub-block `sub` (8 KB each).
__device__ __forceinline__ uint32_t q_stage(int sub, int s) {
    const int i = sub * kQStages + s;
    return i < 8 ? 0x10000u + i * 0x2000u : 0x30000u + (i - 8) * 0x2000u;
}

enum { QTAB_BUILTIN = 0, QTAB_GENERIC = 1 };

template <int QTAB, bool kSigned, bool TW>
__global__ void __launch_bounds__(kQNSub * kQSubT, 1)
    quantize_tma_kernel(const float* __restrict__ tabs, const float* __restrict__ code,
                        const float* __restrict__ x, float* __restrict__ absmax, uint8_t* __restrict__ codes,
                        int64_t n, int64_t nblocks) {
    Q8_SUB_CONSTANTS(kQSubT);
    extern __shared__ __align__(128) uint8_t smem[];
    if (smem_addr(smem) != kDynBase) __trap();
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int sub = tid / kSubThreads, stid = tid % kSubThreads;
    const uint32_t lane4 = (tid & 31u) * 4u;
    const uint64_t pol = evict_first_policy();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kQNSub;
    const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kQNSub + sub;

    // ---- barriers, then the first kQStages loads (before the tables, so their latency overlaps)
    if (stid == 0) {
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(kQBarAddr + (sub * kQStages + s) * 8, 1);
            asm volatile("st.shared.u32 [%0], 0;" ::"r"(kQCntAddr + (sub * kQStages + s) * 4) : "memory");
        }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (stid == 0) {
        for (int s = 0; s < kQStages; ++s) {
            const int64_t b = b0 + s * stride;
            if (b < nblocks && (b + 1) * kBlock <= n) {
                const uint32_t bar = kQBarAddr + (sub * kQStages + s) * 8;
                mbar_expect_tx(bar, kBlock * 4);
                bulk_g2s(q_stage(sub, s), x + b * kBlock, kBlock * 4, bar, pol);
            }
        }
    }

    // ---- tables
    if constexpr (QTAB == QTAB_BUILTIN) {
        // threshold rows (sorted order, 32 lane copies of T_c; signed half at +0, unsigned at +128)
        const int src = kSigned ? kTabSs : kTabSu;
        for (int i = tid; i < 256 * 8; i += nthr) {
            const int row = i >> 3, q = i & 7;
            sts_f32x4(kThreshAddr + row * 256 + (kSigned ? 0 : 128) + q * 16, tabs[src + row]);
        }
        const uint4* lut = reinterpret_cast<const uint4*>(tabs + kTabLut);
        if constexpr (kSigned) {  // signed bucket table without the unreachable |y| > 1 hole
            constexpr int h0 = (kLutSHole - kLutSAddr) / 16, h1 = h0 + 0x2000 / 16, n16 = kLutSBytes / 16;
            for (int i = tid; i < n16 - (h1 - h0); i += nthr) {
                const int j = i < h0 ? i : i + (h1 - h0);
                sts_u32x4(kLutSAddr + j * 16, lut[j]);
            }
        } else {
            for (int i = tid; i < kLutUBytes / 16; i += nthr)
                sts_u32x4(kLutUAddr + i * 16, lut[kLutSBytes / 16 + i]);
        }
    }
    // caller table: T_k = RD((Q_k + Q_{k+1})/2) (__fadd_rd rounds the exact sum down, halving is
    // exact), node i of the Eytzinger tree = T_{rank(i)}, 32 lane copies per 128 B row.  gen_fast: no
    // threshold has 0 < |T| <= 2^-39 or T = 0, so the packed Markstein normalization (exactly RN(x/N)
    // for |x/N| >= 2^-40) yields the same codes as the IEEE division: below 2^-39 both
    // values lie on the same side of every threshold.
    //   Long launches also build the step kernel's bucket table for the caller table (signed key layout,
    //   q8_kernels.cuh "Bucketed search": LUT[key] = the code of the bucket's smallest value, from the
    //   sorted thresholds) and check that no bucket spans more than two codes; if one does (a table
    //   with codes closer than 1/64 of their binade), the launch keeps the 8-step descent.
    bool gen_unsafe = false;
    bool gen_lut = QTAB == QTAB_GENERIC && nblocks >= static_cast<int64_t>(kQLutMinBlocksPerCta) * gridDim.x;
    if constexpr (QTAB == QTAB_GENERIC) {
        for (int i = tid; i < 256 * 8; i += nthr) {
            const int node = i >> 3, q = i & 7;
            float t = __int_as_float(0x7f800000);
            if (node >= 1) {
                const int level = 31 - __clz(node);
                const int k = (2 * (node - (1 << level)) + 1) * (1 << (7 - level)) - 1;
                t = __fmul_rn(__fadd_rd(code[k], code[k + 1]), 0.5f);
                gen_unsafe |= fabsf(t) <= 0x1p-39f;
            }
            sts_f32x4(kQGenRows + node * 128 + q * 16, t);
            const float ts = i < 255 * 8 ? __fmul_rn(__fadd_rd(code[i >> 3], code[(i >> 3) + 1]), 0.5f)
                                         : __int_as_float(0x7f800000);
            sts_f32x4(kQGenSorted + (i >> 3) * 128 + q * 16, ts);
            if (q == 0) asm volatile("st.shared.f32 [%0], %1;" ::"r"(kQGenT + (i >> 3) * 4), "f"(ts) : "memory");
        }
        if (gen_lut) {
            __syncthreads();
            bool wide = false;
            constexpr uint32_t kPos = 0x1FC1;  // keys of 0 <= y <= 1 (bits >> 17 <= 0x1FC0), likewise for y < 0
            for (uint32_t i = tid; i < 2 * kPos; i += nthr) {
                const uint32_t key = i < kPos ? i : 0x4000u + (i - kPos);
                const bool neg = key >= 0x4000u;
                const uint32_t mlo = (key << kShiftS) & 0x7fffffffu;
                const uint32_t mhi = min(mlo + (1u << kShiftS) - 1u, 0x3f800000u);
                const float a = __uint_as_float(mlo), bb = __uint_as_float(mhi);
                const float lo = neg ? -bb : a, hi = neg ? -a : bb;  // the bucket's value range
                uint32_t clo = 0, chi = 0;  // #{k : y > T_k}, branch-free binary search over T[0..255]
#pragma unroll
                for (uint32_t st = 128; st; st >>= 1) {
                    clo += lo > lds_f32(kQGenT + (clo + st - 1) * 4) ? st : 0u;
                    chi += hi > lds_f32(kQGenT + (chi + st - 1) * 4) ? st : 0u;
                }
                wide |= chi - clo > 1u;
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(kLutSAddr + key), "r"(clo) : "memory");
            }
            gen_lut = !__syncthreads_or(wide);
        }
    }
    const bool gen_fast = !__syncthreads_or(gen_unsafe);

    const uint32_t red_base = kRedAddr + sub * (2 * 2 * kMaxSubWarps * 4);
    const uint32_t trow = kThreshAddr + lane4 + (kSigned ? 0u : 128u);
    const uint32_t grow = kQGenRows + lane4;
    const uint32_t gsrow = kQGenSorted + lane4;
    const float Ntw = TW ? absmax[0] : 0.0f;
    uint32_t phase_bits = 0;  // bit s: parity of stage s
    int parity = 0;
    int k = 0;
    for (int64_t b = b0; b < nblocks; b += stride, ++k, parity ^= 1) {
        const int s = k % kQStages;
        const uint32_t stg = q_stage(sub, s);
        const uint32_t bar = kQBarAddr + (sub * kQStages + s) * 8;
        const int64_t base = b * kBlock;
        const bool full = base + kBlock <= n;
        float v[kSGroups][kVec];
        float mx = 0.0f;
        if (full) {
            mbar_wait(bar, (phase_bits >> s) & 1u);
            phase_bits ^= 1u << s;
#pragma unroll
            for (int c = 0; c < kSGroups; ++c) {
                const float4 xv = lds_f32x4(stg + (c * (kSubThreads * kVec) + stid * kVec) * 4);
                v[c][0] = xv.x; v[c][1] = xv.y; v[c][2] = xv.z; v[c][3] = xv.w;
            }
            // release the stage: the last warp of the sub-block to read it issues the TMA of the block
            // kQStages iterations ahead into it
            __syncwarp();
            if ((stid & 31) == 0) {
                uint32_t old;
                const uint32_t cnt = kQCntAddr + (sub * kQStages + s) * 4;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(cnt) : "memory");
                if (old % kSubWarps == kSubWarps - 1) {
                    const int64_t bn = b + kQStages * stride;
                    if (bn < nblocks && (bn + 1) * kBlock <= n) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        mbar_expect_tx(bar, kBlock * 4);
                        bulk_g2s(stg, x + bn * kBlock, kBlock * 4, bar, pol);
                    }
                }
            }
        } else {  // the short last block ("n/B blocks"): guarded direct loads
#pragma unroll
            for (int c = 0; c < kSGroups; ++c) {
                const int64_t i0 = base + c * (kSubThreads * kVec) + stid * kVec;
#pragma unroll
                for (int e = 0; e < kVec; ++e) v[c][e] = (i0 + e < n) ? x[i0 + e] : 0.0f;
            }
        }
        float N;
        if constexpr (TW) {
            N = Ntw;
        } else {  // a5: block absmax, REDUX + per-warp partials + the sub-block's named barrier
#pragma unroll
            for (int c = 0; c < kSGroups; ++c)
#pragma unroll
                for (int e = 0; e < kVec; ++e) mx = fmaxf(mx, fabsf(v[c][e]));
            const uint32_t red = red_base + parity * (2 * kSubWarps * 4);
            const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
            if ((stid & 31) == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(red + (stid >> 5) * 4), "r"(wm) : "memory");
            sub_barrier(sub, kSubThreads);
            N = __uint_as_float(__reduce_max_sync(0xffffffffu, lds_u32(red + (stid & (kSubWarps - 1)) * 4)));
        }
        // a6: normalize + nearest code
        uint32_t o[kSGroups];
        if constexpr (QTAB == QTAB_BUILTIN) {
            if (N >= 0x1p-70f && N < 0x1p126f) {  // block-uniform: packed Markstein division
                const float rcp = __frcp_rn(N);
                const f2 rc = pk(rcp, rcp), nN = pk(-N, -N);
#pragma unroll
                for (int c = 0; c < kSGroups; ++c) {
                    uint32_t kk[kVec];
#pragma unroll
                    for (int e = 0; e < kVec; e += 2) {
                        const f2 xx = pk(v[c][e], v[c][e + 1]);
                        const f2 q = fmul2(xx, rc);
                        const f2 y = ffma2(ffma2(q, nN, xx), rc, q);
                        float y0 = lo_of(y), y1 = hi_of(y);
                        if (!kSigned) {  // unsigned table: y < 0 (incl. -0) -> code of +0 (Eq.3)
                            y0 = __int_as_float(max(__float_as_int(y0), 0));
                            y1 = __int_as_float(max(__float_as_int(y1), 0));
                        }
                        kk[e] = nearest_code<SEARCH_BUCKET, !kSigned>(trow, y0);
                        kk[e + 1] = nearest_code<SEARCH_BUCKET, !kSigned>(trow, y1);
                    }
                    o[c] = pack4(kk[0], kk[1], kk[2], kk[3]);
                }
            } else {
                const Normalizer nz(N);
#pragma unroll
                for (int c = 0; c < kSGroups; ++c) {
                    uint32_t kk[kVec];
#pragma unroll
                    for (int e = 0; e < kVec; ++e) {
                        float y = nz(v[c][e]);
                        if (!kSigned) y = __int_as_float(max(__float_as_int(y), 0));
                        kk[e] = nearest_code<SEARCH_BUCKET, !kSigned>(trow, y);
                    }
                    o[c] = pack4(kk[0], kk[1], kk[2], kk[3]);
                }
            }
        } else {
            // all 16 descents advance level by level, so 16 independent shared-load chains are in
            // flight per thread (the search is a chain of 8 dependent loads per element)
            float y[kSGroups * kVec];
            uint32_t i[kSGroups * kVec];
            if (gen_fast && N >= 0x1p-70f && N < 0x1p126f) {  // block-uniform: packed Markstein division
                const float rcp = __frcp_rn(N);
                const f2 rc = pk(rcp, rcp), nN = pk(-N, -N);
#pragma unroll
                for (int c = 0; c < kSGroups; ++c)
#pragma unroll
                    for (int e = 0; e < kVec; e += 2) {
                        const f2 xx = pk(v[c][e], v[c][e + 1]);
                        const f2 q = fmul2(xx, rc);
                        const f2 yy = ffma2(ffma2(q, nN, xx), rc, q);
                        y[c * kVec + e] = lo_of(yy);
                        y[c * kVec + e + 1] = hi_of(yy);
                    }
            } else {
#pragma unroll
                for (int c = 0; c < kSGroups; ++c)
#pragma unroll
                    for (int e = 0; e < kVec; ++e) y[c * kVec + e] = N > 0.0f ? __fdiv_rn(v[c][e], N) : 0.0f;
            }
            if (gen_lut) {  // bucket table + one compare against the sorted thresholds (128-B rows)
#pragma unroll
                for (int c = 0; c < kSGroups; ++c)
                    o[c] = pack4(nearest_code<SEARCH_BUCKET, false, 7>(gsrow, y[c * kVec]),
                                 nearest_code<SEARCH_BUCKET, false, 7>(gsrow, y[c * kVec + 1]),
                                 nearest_code<SEARCH_BUCKET, false, 7>(gsrow, y[c * kVec + 2]),
                                 nearest_code<SEARCH_BUCKET, false, 7>(gsrow, y[c * kVec + 3]));
            } else {
#pragma unroll
                for (int j = 0; j < kSGroups * kVec; ++j) i[j] = 1u;
#pragma unroll
                for (int l = 0; l < 8; ++l)
#pragma unroll
                    for (int j = 0; j < kSGroups * kVec; ++j)
                        i[j] = 2u * i[j] + (y[j] > lds_f32(grow + (i[j] << 7)) ? 1u : 0u);
#pragma unroll
                for (int c = 0; c < kSGroups; ++c)
                    o[c] = pack4(i[c * kVec] - 256u, i[c * kVec + 1] - 256u, i[c * kVec + 2] - 256u, i[c * kVec + 3] - 256u);
            }
        }
        // a7: store
#pragma unroll
        for (int c = 0; c < kSGroups; ++c) {
            const int64_t i0 = base + c * (kSubThreads * kVec) + stid * kVec;
            if (full) {
                st_stream_u32(codes + i0, o[c]);
            } else {
#pragma unroll
                for (int e = 0; e < kVec; ++e)
                    if (i0 + e < n) codes[i0 + e] = static_cast<uint8_t>(o[c] >> (8 * e));
            }
        }
        if (!TW && stid == 0) absmax[b] = N;
    }
}

}  // namespace q8
