// codebook_host.cpp -- host-side construction of the dynamic data types and of the
// Eytzinger-ordered threshold tables the sm_100a kernels search.
//
// Independent of oracle/ (no shared code).  The value formula is the reading G1 of
// P:90 (S2.3 dynamic tree quantization) and P:118 (S3.2 unsigned dynamic quantization):
// decade z in 0..6 (a run of z zero bits), F fraction bits after the indicator bit
// (F = 6 - z signed, 7 - z unsigned), fraction integer f in [0, 2^F):
//     |q| = 10^-z * (0.1 + 0.9 * (f + 1/2) / 2^F) = (2*2^F + 18 f + 9) / (20 * 2^F * 10^z)
// plus the two patterns without an indicator bit, read as 0 and +1 (G1).  The ratio of two
// exactly representable integers is divided once in double and rounded once to fp32 (G2).
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstring>

namespace q8 {

void build_dynamic_codebook(bool is_signed, float out[256]) {
    int k = 0;
    out[k++] = 0.0f;
    out[k++] = 1.0f;
    double pow10 = 1.0;
    for (int z = 0; z < 7; ++z, pow10 *= 10.0) {
        const int F = is_signed ? 6 - z : 7 - z;
        const double L = std::ldexp(1.0, F);
        for (int f = 0; f < (1 << F); ++f) {
            const double num = 2.0 * L + 18.0 * f + 9.0;   // exact integer
            const double den = 20.0 * L * pow10;           // exact integer (< 2^53)
            const float v = static_cast<float>(num / den);
            out[k++] = v;
            if (is_signed) out[k++] = -v;
        }
    }
    std::sort(out, out + 256);
}

// Threshold between codes k and k+1: the exact midpoint (Q_k + Q_{k+1}) / 2 rounded DOWN
// to fp32.  For fp32 y:  y > T_k  <=>  y is strictly closer to Q_{k+1} than to Q_k, so
// #{k : y > T_k} = argmin_j |Q_j - y| with ties to the lower index (Eq.3, G6).
static float midpoint_round_down(float a, float b) {
    const double mid = (static_cast<double>(a) + static_cast<double>(b)) * 0.5;  // exact
    float t = static_cast<float>(mid);
    if (static_cast<double>(t) > mid) t = std::nextafter(t, -INFINITY);
    return t;
}

// In-order rank (0..254) of node i (1..255) of the perfect 8-level binary search tree in
// Eytzinger (BFS) numbering.
int eytzinger_rank(int i) {
    int level = 31 - __builtin_clz(static_cast<unsigned>(i));
    int pos = i - (1 << level);
    return (2 * pos + 1) * (1 << (7 - level)) - 1;
}

// out[0] unused (set to +inf); out[i] = T_{rank(i)} for i = 1..255.  An 8-step descent
// i <- 2i + [y > out[i]] starting at i = 1 ends at 256 + #{k : y > T_k}.
void build_eytzinger_thresholds(const float Q[256], float out[256]) {
    out[0] = INFINITY;
    for (int i = 1; i < 256; ++i) {
        const int k = eytzinger_rank(i);
        out[i] = midpoint_round_down(Q[k], Q[k + 1]);
    }
}

// Sorted thresholds: out[k] = T_k for k = 0..254, out[255] = +inf (so c0 = 255 never moves).
void build_sorted_thresholds(const float Q[256], float out[256]) {
    for (int k = 0; k < 255; ++k) out[k] = midpoint_round_down(Q[k], Q[k + 1]);
    out[255] = INFINITY;
}

static float bits_to_float(uint32_t u) {
    float f;
    std::memcpy(&f, &u, sizeof f);
    return f;
}

// code(y) = #{k : y > T_k}  (= Eq.3 argmin with lower-index ties, see above)
static int code_of(const float T[256], float y) {
    int c = 0;
    while (c < 255 && y > T[c]) ++c;
    return c;
}

// Bucket tables of the bucketed search (q8_kernels.cuh "Bucketed search").  Key k covers the
// fp32 bit patterns [k << shift, (k + 1) << shift) (signed: sign bit included in the key).
// lut[k] = smallest code of any value in [-1, 1] (signed) / [0, 1] (unsigned) in the bucket;
// keys beyond that range are unreachable for a normalized value and hold 255 (positive) or 0
// (negative).  Returns false if some bucket spans more than two codes.
// Keys below key_min are clamped up to key_min by the kernel, so bucket key_min also covers
// every smaller (non-negative) value.  lut[i] belongs to key key_min + i.
bool build_bucket_lut(const float T[256], bool is_signed, int shift, int key_min, int entries, uint8_t* lut) {
    const uint32_t one = 0x3f800000u, width = 1u << shift;
    for (int i = 0; i < entries; ++i) {
        const int k = key_min + i;
        const uint32_t hi_bits = (k == key_min && key_min > 0) ? 0u : static_cast<uint32_t>(k) << shift;
        const bool neg = is_signed && (hi_bits & 0x80000000u);
        const uint32_t mlo = hi_bits & 0x7fffffffu;
        if (mlo > one) {                       // |y| > 1: unreachable
            lut[i] = neg ? 0 : 255;
            continue;
        }
        uint32_t mhi = (static_cast<uint32_t>(k) << shift & 0x7fffffffu) + width - 1u;
        if (mhi > one) mhi = one;
        const float a = bits_to_float(mlo), b = bits_to_float(mhi);
        const float lo = neg ? -b : a, hi = neg ? -a : b;   // the bucket's value range
        const int c_lo = code_of(T, lo), c_hi = code_of(T, hi);
        if (c_hi - c_lo > 1) return false;
        lut[i] = static_cast<uint8_t>(c_lo);
    }
    return true;
}

}  // namespace q8
