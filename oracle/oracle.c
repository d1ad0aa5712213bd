/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path of
 * Dettmers, Lewis, Shleifer & Zettlemoyer, "8-bit Optimizers via Block-wise
 * Quantization" (arXiv 2110.02861) computes.  Citations are to
 * /root/reference/PAPER.md as "P:<line>" (section / equation in brackets) and to
 * the readings "G<n>" listed in DESIGN.md section 3 (taken from SURVEY.md 8(c)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this file.  It shares no code, header, table or constant
 * generator with the CUDA library under paper_2110_02861_b200/; neither side
 * includes or links the other.
 *
 * Compiled with  gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math  so that every
 * float expression written below is one IEEE-754 binary32 round-to-nearest-even
 * operation per operator (no FMA contraction, no reassociation).
 *
 * Parity status of every exported function (pins live in tests/test_oracle_*.py):
 *   oracle_dynamic_codebook   pinned: exact rational closed form, invariants,
 *                              golden hashes (tests/golden/)
 *   oracle_linear_codebook     pinned: even spacing, exact endpoints, symmetry
 *   oracle_nearest_code        pinned: brute-force argmin (numpy) incl. exact ties
 *   oracle_quantize_blockwise  pinned: SPEC worked examples, absmax = np.max|x|,
 *                              half-gap bound, block independence
 *   oracle_dequantize_blockwise pinned: Q[code]*N by numpy
 *   oracle_optim32bit_step     pinned: torch.optim.{Adam,AdamW,SGD} (CPU fp32),
 *                              hand arithmetic S:315/S:324, t=1 closed form
 *   oracle_optim8bit_step      pinned: == 32-bit step + explicit block quantize
 *                              (bit-exact), 8-bit vs 32-bit within quantization
 *                              error over 10 steps
 *   oracle_optim32bit_layerwise_step  (8-bit LAMB / LARS, T5 P:366-367; readings L1-L4)
 *                              pinned: LAMB states == Adam states (bit-exact); LAMB
 *                              p against the unfolded textbook form in float64 and
 *                              |dw| = lr*|w| closed forms; LARS == torch.optim.SGD on
 *                              the trust-scaled gradient (bit-exact), |dw| closed form
 *   oracle_optim8bit_layerwise_step   pinned: == dequantize -> 32-bit layer-wise step
 *                              -> block quantize (bit-exact), 8-bit vs 32-bit within
 *                              quantization error
 *   oracle_exact_quantiles    pinned: closed-form order statistics of permuted integer
 *                              ranges, np.sort indexing, scipy normal ppf (large n)
 *   oracle_sram_quantiles     pinned: == exact quantiles when one chunk holds the tensor;
 *                              constant chunks -> their mean (closed form); permutation
 *                              invariance inside a chunk; close to the normal ppf
 *   oracle_quantile_codebook  pinned: uniform data -> evenly spaced Eq.5 midpoints (closed
 *                              form); symmetry for symmetric quantiles; max |code| = 1
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_ADAM 0
#define ORACLE_ADAMW 1
#define ORACLE_MOMENTUM 2
#define ORACLE_LAMB 3
#define ORACLE_LARS 4

typedef struct {
    double lr;            /* alpha,  Eq.1/Eq.2 */
    double beta1;         /* beta_1 (Momentum: beta of Eq.1) */
    double beta2;         /* beta_2, Adam only */
    double eps;           /* epsilon, Adam only */
    double weight_decay;  /* G10: AdamW decoupled, Adam/Momentum L2 */
    int bias_correction;  /* G8 */
} oracle_hparams;

/* ------------------------------------------------------------------------- */
/* 1. Dynamic (tree) quantization data type -- P:90 [S2.3], P:118 [S3.2], G1/G2 */
/* ------------------------------------------------------------------------- */

static int cmp_float_asc(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

/*
 * Decode one 8-bit pattern of the dynamic data type.
 *
 * "(1) The first bit of the data type is reserved for a sign. (2) The
 * number of subsequent zero bits indicates the magnitude of the exponent. (3)
 * The first bit that is set to one indicates that all following values are
 * reserved for (4) linear quantization."  The exponent is a power of ten
 * (base 10^0 = 1, each zero bit divides by 10, minimum 10^-7: P:400).
 * P:118 (unsigned): the sign bit is re-purposed as a *fixed* extra fraction bit.
 *
 * Reading G1: with z leading zeros and F fraction bits holding integer f, the
 * linear part quantizes the decade (0.1, 1] into 2^F equal bins and takes the
 * bin midpoint:   magnitude = 10^-z * (0.1 + 0.9 * (f + 0.5) / 2^F).
 * The two patterns without an indicator bit become 0 and +1.0 (G1).
 * Evaluated in double, rounded once to binary32 (G2).
 */
static float decode_pattern(int is_signed, unsigned pattern) {
    static const double decade[7] = {1.0, 0.1, 0.01, 1e-3, 1e-4, 1e-5, 1e-6};
    unsigned lead = (pattern >> 7) & 1u;         /* sign bit (signed) or fixed fraction bit (unsigned) */
    unsigned rest = pattern & 0x7fu;                                       /* 7 bits: zeros, indicator, fraction */
    int z = 0;
    while (z < 7 && ((rest >> (6 - z)) & 1u) == 0u) z++;
    if (z == 7) {
        /* no indicator bit: the two special patterns -> 0 and +1.0 (G1) */
        return lead ? 1.0f : 0.0f;
    }
    int nfrac7 = 6 - z;                          /* fraction bits after the indicator */
    unsigned f = rest & ((1u << nfrac7) - 1u);
    int F = nfrac7;
    if (!is_signed) {                            /* fixed bit = one more fraction bit */
        f = (lead << nfrac7) | f;
        F = nfrac7 + 1;
    }
    double L = (double)(1u << F);
    double mag = decade[z] * (0.1 + 0.9 * ((double)f + 0.5) / L);
    double v = (is_signed && lead) ? -mag : mag;
    return (float)v;
}

/* Q^map as an ascending table of 256 binary32 values; codes are indices into it (G4). */
int oracle_dynamic_codebook(int is_signed, float out[256]) {
    for (unsigned p = 0; p < 256; p++) out[p] = decode_pattern(is_signed, p);
    qsort(out, 256, sizeof(float), cmp_float_asc);
    for (int i = 1; i < 256; i++)
        if (!(out[i - 1] < out[i])) return -1;   /* must be 256 distinct values */
    return 0;
}

/*
 * Linear data type (the ablation baseline "without dynamic quantization use linear
 * quantization", T3 caption P:214): 256 evenly spaced values.  Reading L0: the
 * paper gives no formula; 256 evenly spaced values cannot be symmetric AND contain 0, and an
 * optimizer state needs an exact 0 (Eq.2 "r_0 = m_0 = 0"), so the signed type is
 * (i - 127)/128 -- exact 0 at index 127 and +1 at 255, the dynamic type's layout of its
 * specials -- and the unsigned type i/255, i = 0..255; evaluated in double, rounded once.
 */
int oracle_linear_codebook(int is_signed, float out[256]) {
    for (int i = 0; i < 256; i++) {
        double v = is_signed ? (double)(i - 127) / 128.0 : (double)i / 255.0;
        out[i] = (float)v;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 2. Nearest code -- Eq.3: argmin_j |Q_j - T_i/N|, via binary search */
/* ------------------------------------------------------------------------- */

/*
 * Exact difference a - b of two binary32 values as an unevaluated pair s + e of
 * binary64 values: s = RN(a - b), e = the exact rounding error (Knuth's TwoSum
 * of a and -b; every operation binary64 round-to-nearest, no contraction).
 * A binary64 subtraction alone is NOT always exact here: for y = 1e-45 and
 * Q = 1/255 the 2^141 exponent gap loses y entirely.
 */
static void exact_diff(float a, float b, double* s, double* e) {
    double x = (double)a, c = -(double)b;
    double sum = x + c;
    double cv = sum - x;                 /* the part of c that made it into sum */
    double xv = sum - cv;
    *s = sum;
    *e = (x - xv) + (c - cv);
}

/* Is the exact value s1 + e1 smaller than s2 + e2?  (s = RN(s + e), so the
 * s parts order the exact values unless they are equal; then the errors do.) */
static int pair_less(double s1, double e1, double s2, double e2) {
    return s1 < s2 || (s1 == s2 && e1 < e2);
}

/*
 * Returns argmin_{j in 0..255} |Q[j] - y| with ties broken toward the lower
 * index (G6).  Q must be strictly ascending.  As Eq.3 says, the closest value
 * is found "via a binary search": lower_bound finds the first Q[hi] >= y, and
 * the answer is whichever of Q[hi-1], Q[hi] is closer.  The two (non-negative)
 * distances Q[hi] - y and y - Q[hi-1] are compared exactly (exact_diff).
 */
int oracle_nearest_code(const float Q[256], float y) {
    int lo = 0, hi = 256;                        /* lower_bound over Q */
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (Q[mid] < y) lo = mid + 1; else hi = mid;
    }
    if (hi == 0) return 0;
    if (hi == 256) return 255;
    double s_lo, e_lo, s_hi, e_hi;
    exact_diff(y, Q[hi - 1], &s_lo, &e_lo);
    exact_diff(Q[hi], y, &s_hi, &e_hi);
    return pair_less(s_hi, e_hi, s_lo, e_lo) ? hi : hi - 1;   /* tie -> lower index */
}

/* ------------------------------------------------------------------------- */
/* 3. Block-wise quantization -- Eq.4, dequantization P:71          */
/* ------------------------------------------------------------------------- */

/* Number of blocks: ceil(n / B); the last block may be short (G5). */
static int64_t num_blocks(int64_t n, int64_t B) { return (n + B - 1) / B; }

/* N_b = max(|T_b|) */
static float block_absmax(const float* x, int64_t len) {
    float N = 0.0f;
    for (int64_t i = 0; i < len; i++) {
        float a = fabsf(x[i]);
        if (a > N) N = a;
    }
    return N;
}

/* T^Q_bi = argmin_j |Q_j - T_bi / N_b|   (Eq.4).  N_b = 0 means the block is all
 * zeros; its normalized values are taken as 0 (G7). */
static void quantize_block(const float Q[256], const float* x, int64_t len, float* absmax, uint8_t* codes) {
    float N = block_absmax(x, len);
    *absmax = N;
    for (int64_t i = 0; i < len; i++) {
        float y = (N > 0.0f) ? x[i] / N : 0.0f;
        codes[i] = (uint8_t)oracle_nearest_code(Q, y);
    }
}

int oracle_quantize_blockwise(const float Q[256], const float* x, int64_t n, int64_t B,
                              float* absmax, uint8_t* codes) {
    if (n < 0 || B < 1) return -1;
    for (int64_t b = 0; b < num_blocks(n, B); b++) {
        int64_t start = b * B, len = (n - start < B) ? n - start : B;
        quantize_block(Q, x + start, len, absmax + b, codes + start);
    }
    return 0;
}

/* T^D_i = Q^map(T^Q_i) * N, with N = N_b of the element's block. */
int oracle_dequantize_blockwise(const float Q[256], const uint8_t* codes, const float* absmax,
                                int64_t n, int64_t B, float* out) {
    if (n < 0 || B < 1) return -1;
    for (int64_t i = 0; i < n; i++) out[i] = Q[codes[i]] * absmax[i / B];
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 4. Optimizer updates in 32-bit -- Eq.1, Eq.2              */
/* ------------------------------------------------------------------------- */

typedef struct {
    int kind;
    float lr, beta1, beta2, one_minus_beta1, one_minus_beta2;
    float step_size, eps_hat, weight_decay, decay;
} scalars;

/*
 * Host scalars, computed in double and rounded once to binary32 (G8-G10).
 * Bias correction (G8) uses Kingma & Ba's folded form (Adam paper, S2 last
 * paragraph):  alpha_t = alpha*sqrt(1-beta2^t)/(1-beta1^t),
 * eps_hat = eps*sqrt(1-beta2^t); then w -= alpha_t * m/(sqrt(r) + eps_hat).
 */
static scalars make_scalars(int kind, const oracle_hparams* hp, int64_t step) {
    scalars s;
    s.kind = kind;
    s.lr = (float)hp->lr;
    s.beta1 = (float)hp->beta1;
    s.beta2 = (float)hp->beta2;
    s.one_minus_beta1 = (float)(1.0 - hp->beta1);
    s.one_minus_beta2 = (float)(1.0 - hp->beta2);
    if (hp->bias_correction) {
        double bc1 = 1.0 - pow(hp->beta1, (double)step);
        double bc2 = 1.0 - pow(hp->beta2, (double)step);
        s.step_size = (float)(hp->lr * sqrt(bc2) / bc1);
        s.eps_hat = (float)(hp->eps * sqrt(bc2));
    } else {
        s.step_size = (float)hp->lr;
        s.eps_hat = (float)hp->eps;
    }
    s.weight_decay = (float)hp->weight_decay;
    s.decay = (float)(1.0 - hp->lr * hp->weight_decay);
    return s;
}

/*
 * One element of the 32-bit update, in the order Eq.1/Eq.2 write it; every
 * operator is one binary32 rounding (G9).  Weight decay (G10): AdamW scales w
 * by (1 - lr*wd) first (decoupled, Loshchilov & Hutter, cited P:134);
 * Adam and Momentum add wd*w to the gradient (L2) when wd != 0.
 */
static void update_element(const scalars* s, float* w, float g, float* m, float* r) {
    if (s->kind == ORACLE_ADAMW) {
        *w = *w * s->decay;
    } else if (s->weight_decay != 0.0f) {
        g = g + s->weight_decay * *w;
    }
    if (s->kind == ORACLE_MOMENTUM) {
        /* Eq.1: m_t = beta1*m_{t-1} + g_t ;  w_t = w_{t-1} - alpha*m_t.
         * m_0 = g_0 follows from the zero initial state. */
        *m = s->beta1 * *m + g;
        *w = *w - s->lr * *m;
    } else {
        /* Eq.2: m_t = beta1*m + (1-beta1)*g ;  r_t = beta2*r + (1-beta2)*g^2 ;
         *       w_t = w - alpha*m_t/(sqrt(r_t)+eps)   (alpha, eps -> step_size, eps_hat) */
        *m = s->beta1 * *m + s->one_minus_beta1 * g;
        *r = s->beta2 * *r + s->one_minus_beta2 * (g * g);
        *w = *w - s->step_size * (*m / (sqrtf(*r) + s->eps_hat));
    }
}

/* 32-bit optimizer step (states m, r in fp32; r unused for Momentum). */
int oracle_optim32bit_step(int kind, float* p, const float* g, float* m, float* r, int64_t n,
                           const oracle_hparams* hp, int64_t step) {
    if (kind < 0 || kind > 2 || n < 0 || step < 1) return -1;
    scalars s = make_scalars(kind, hp, step);
    float dummy = 0.0f;
    for (int64_t i = 0; i < n; i++)
        update_element(&s, &p[i], g[i], &m[i], kind == ORACLE_MOMENTUM ? &dummy : &r[i]);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 5. 8-bit optimizer step -- S3, Fig.1 caption                */
/*    dequantize -> 32-bit update (Eq.1/2) -> block absmax        */
/*    -> requantize (Eq.4); w uses the 32-bit post-update states (G12).          */
/*    s1 uses the signed data type, s2 (strictly positive) the unsigned (G14).  */
/* ------------------------------------------------------------------------- */

typedef struct {
    int kind;
    float* p;
    const float* g;
    uint8_t* s1;
    uint8_t* s2;
    float* absmax1;
    float* absmax2;
    int64_t n, B, b_begin, b_end;
    const scalars* s;
    const float* Qs;
    const float* Qu;
} step_job;

static void* step_blocks(void* arg) {
    step_job* j = (step_job*)arg;
    float* m = (float*)malloc(sizeof(float) * (size_t)j->B);
    float* r = (float*)malloc(sizeof(float) * (size_t)j->B);
    for (int64_t b = j->b_begin; b < j->b_end; b++) {
        int64_t start = b * j->B, len = (j->n - start < j->B) ? j->n - start : j->B;
        /* dequantize: T^D = Q^map(T^Q) * N_b */
        for (int64_t i = 0; i < len; i++) {
            m[i] = j->Qs[j->s1[start + i]] * j->absmax1[b];
            r[i] = (j->kind == ORACLE_MOMENTUM) ? 0.0f : j->Qu[j->s2[start + i]] * j->absmax2[b];
        }
        /* 32-bit update, element by element */
        for (int64_t i = 0; i < len; i++) update_element(j->s, &j->p[start + i], j->g[start + i], &m[i], &r[i]);
        /* block-wise requantization of the new states (Eq.4) */
        quantize_block(j->Qs, m, len, &j->absmax1[b], j->s1 + start);
        if (j->kind != ORACLE_MOMENTUM) quantize_block(j->Qu, r, len, &j->absmax2[b], j->s2 + start);
    }
    free(m);
    free(r);
    return NULL;
}

/*
 * g is binary32 (16-bit gradients are widened exactly by the caller, G13).
 * Blocks are independent, so nthreads > 1 splits the block range into
 * contiguous pieces; results do not depend on nthreads.
 */
int oracle_optim8bit_step(int kind, float* p, const float* g, uint8_t* s1, uint8_t* s2, float* absmax1,
                          float* absmax2, int64_t n, int64_t B, const oracle_hparams* hp, int64_t step,
                          int nthreads) {
    if (kind < 0 || kind > 2 || n < 0 || B < 1 || step < 1) return -1;
    float Qs[256], Qu[256];
    if (oracle_dynamic_codebook(1, Qs) != 0 || oracle_dynamic_codebook(0, Qu) != 0) return -1;
    scalars s = make_scalars(kind, hp, step);
    int64_t nb = num_blocks(n, B);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    step_job jobs[256];
    for (int t = 0; t < nthreads; t++) {
        step_job j = {kind, p, g, s1, s2, absmax1, absmax2, n, B, nb * t / nthreads, nb * (t + 1) / nthreads,
                      &s, Qs, Qu};
        jobs[t] = j;
    }
    for (int t = 1; t < nthreads; t++) pthread_create(&th[t], NULL, step_blocks, &jobs[t]);
    step_blocks(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 6. Layer-wise (trust-ratio) optimizers: 8-bit LAMB and LARS (T5)  */
/* ------------------------------------------------------------------------- */
/*
 * The paper benchmarks 8-bit LAMB and LARS (T5) but prints no formula for them; they are
 * the textbook algorithms with their states quantized exactly like Adam's / Momentum's
 * (S3: dequantize -> 32-bit update -> requantize).  Readings (L1-L4):
 *
 * L1 LAMB (You et al. 2020, "Large Batch Optimization for Deep Learning", Alg. 2), per
 *    tensor ("layer"):  m, r as Eq.2 (G9 order, no L2 term in g);
 *      d = m / (sqrt(r) + eps_hat);   u = c*d + wd*w   with c = sqrt(1-b2^t)/(1-b1^t)
 *      (the folded bias correction of G8; c = 1 without it);
 *      ratio = ||w|| / ||u|| if both norms > 0, else 1;   w = w - RN(lr*ratio) * u.
 * L2 LARS (You, Gitman & Ginsburg 2017, "Large Batch Training of Convolutional
 *    Networks", Alg. 1), per tensor, momentum state v (signed table):
 *      local = eta * ||w|| / (||g|| + wd*||w||) if ||w|| > 0 and ||g|| > 0, else 1;
 *      v = beta1*v + RN(lr*local) * (g + wd*w);   w = w - v.
 * L3 Norms: ||x|| = sqrt(sum_i x_i^2) over the whole tensor, squares and sum in binary64
 *    (sequential here), ratio / local in binary64, the per-tensor scale rounded once to
 *    binary32.  Norms use the PRE-update w (and, LAMB, the fp32 post-update states).
 * L4 Each fp32 operator above is one IEEE RN operation in the written order (as G9).
 */

static double sum_squares(const float* x, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += (double)x[i] * (double)x[i];
    return s;
}

/* 32-bit layer-wise step over ONE tensor (the layer).  m, r fp32 states (r LAMB only);
 * *scale_out (may be NULL) receives the fp32 per-tensor scale RN(lr*ratio) / RN(lr*local).
 * scale_in (may be NULL) teacher-forces that scale instead of computing it from the norms: the
 * norms are binary64 sums whose order reading L3 leaves open, so two correct implementations may
 * round the scale differently in its last bit; given the same scale every other output is unique. */
int oracle_optim32bit_layerwise_step(int kind, float* p, const float* g, float* m, float* r, int64_t n,
                                     const oracle_hparams* hp, double trust_coeff, int64_t step, float* scale_out,
                                     const float* scale_in) {
    if ((kind != ORACLE_LAMB && kind != ORACLE_LARS) || n < 0 || step < 1) return -1;
    const float beta1 = (float)hp->beta1, wd = (float)hp->weight_decay;
    float a;
    if (kind == ORACLE_LAMB) {
        const float beta2 = (float)hp->beta2;
        const float omb1 = (float)(1.0 - hp->beta1), omb2 = (float)(1.0 - hp->beta2);
        float c = 1.0f, eps_hat = (float)hp->eps;
        if (hp->bias_correction) {
            double bc1 = 1.0 - pow(hp->beta1, (double)step);
            double bc2 = 1.0 - pow(hp->beta2, (double)step);
            c = (float)(sqrt(bc2) / bc1);
            eps_hat = (float)(hp->eps * sqrt(bc2));
        }
        float* u = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
        for (int64_t i = 0; i < n; i++) {
            m[i] = beta1 * m[i] + omb1 * g[i];                 /* Eq.2 state 1 */
            r[i] = beta2 * r[i] + omb2 * (g[i] * g[i]);        /* Eq.2 state 2 */
            float d = m[i] / (sqrtf(r[i]) + eps_hat);
            u[i] = c * d + wd * p[i];                          /* LAMB update direction */
        }
        double wn = sqrt(sum_squares(p, n)), un = sqrt(sum_squares(u, n));
        double ratio = (wn > 0.0 && un > 0.0) ? wn / un : 1.0; /* trust ratio */
        a = scale_in ? *scale_in : (float)(hp->lr * ratio);
        for (int64_t i = 0; i < n; i++) p[i] = p[i] - a * u[i];
        free(u);
    } else {
        double wn = sqrt(sum_squares(p, n)), gn = sqrt(sum_squares(g, n));
        double local = (wn > 0.0 && gn > 0.0) ? trust_coeff * wn / (gn + hp->weight_decay * wn) : 1.0;
        a = scale_in ? *scale_in : (float)(hp->lr * local);
        for (int64_t i = 0; i < n; i++) {
            float t = g[i] + wd * p[i];
            t = a * t;
            m[i] = beta1 * m[i] + t;                           /* v = beta1 v + lr*local*(g + wd w) */
            p[i] = p[i] - m[i];
        }
    }
    if (scale_out) *scale_out = a;
    return 0;
}

/* 8-bit layer-wise step over ONE tensor: dequantize all states, the 32-bit layer-wise
 * step above, block-wise requantization of the new states (Eq.4); s1 signed, s2 unsigned
 * (LAMB only, G14). */
int oracle_optim8bit_layerwise_step(int kind, float* p, const float* g, uint8_t* s1, uint8_t* s2, float* absmax1,
                                    float* absmax2, int64_t n, int64_t B, const oracle_hparams* hp, double trust_coeff,
                                    int64_t step, float* scale_out, const float* scale_in) {
    if ((kind != ORACLE_LAMB && kind != ORACLE_LARS) || n < 0 || B < 1 || step < 1) return -1;
    float Qs[256], Qu[256];
    if (oracle_dynamic_codebook(1, Qs) != 0 || oracle_dynamic_codebook(0, Qu) != 0) return -1;
    size_t bytes = sizeof(float) * (size_t)(n > 0 ? n : 1);
    float* m = (float*)malloc(bytes);
    float* r = (float*)malloc(bytes);
    oracle_dequantize_blockwise(Qs, s1, absmax1, n, B, m);
    if (kind == ORACLE_LAMB) oracle_dequantize_blockwise(Qu, s2, absmax2, n, B, r);
    int rc = oracle_optim32bit_layerwise_step(kind, p, g, m, r, n, hp, trust_coeff, step, scale_out, scale_in);
    if (rc == 0) {
        oracle_quantize_blockwise(Qs, m, n, B, absmax1, s1);
        if (kind == ORACLE_LAMB) oracle_quantize_blockwise(Qu, r, n, B, absmax2, s2);
    }
    free(m);
    free(r);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* 7. Quantile quantization (App F.2, Eq.5) and SRAM-Quantiles      */
/*    (App G)                                                        */
/* ------------------------------------------------------------------------- */

/*
 * Readings (rows Q1-Q5):
 *  Q1  Eq.5: q_i = (Q_X(i/(2^k+1)) + Q_X((i+1)/(2^k+1))) / 2, i = 0..2^k-1, so k = 8
 *      needs the 257 quantiles Q_X(j/257), j = 0..256, as the equation is written (the prose
 *      "2^k+1 equally spaced quantiles over [0,1]" would put them at j/256; we follow the formula).
 *  Q2  sample quantile: "the value at index i = q x n" of the ascending sorted values,
 *      0-based, i = floor(j*m/257) computed exactly in integers for a set of m values.
 *  Q3  SRAM-Quantiles subsets: consecutive chunks of S values ("about 4096 32-bit
 *      values"), the last one possibly short; each chunk's quantiles are found from its own
 *      eCDF (Q2 with its own m).
 *  Q4  "we average the quantiles": arithmetic mean over chunks, every chunk weight 1,
 *      summed in binary64 and rounded once to binary32.  (The paper's atomic averaging has no
 *      fixed order; the oracle sums in chunk order.)
 *  Q5  Eq.5 midpoints in binary64, normalized into [-1, 1] by their largest magnitude (Fig. 6
 *      caption P:427 "normalize them into the range [-1, 1]"), rounded once to binary32.
 */

static int cmp_float_total(const void* a, const void* b) {
    /* ascending by value; -0 before +0 so the order is total (only relevant for the bit of a zero) */
    float x = *(const float*)a, y = *(const float*)b;
    if (x < y) return -1;
    if (x > y) return 1;
    return (signbit(y) != 0) - (signbit(x) != 0);
}

/* Q2 on one set of m values: sort a copy, take index floor(j*m/257) for j = 0..256. */
static void sample_quantiles(const float* x, int64_t m, float* tmp, float out[257]) {
    memcpy(tmp, x, sizeof(float) * (size_t)m);
    qsort(tmp, (size_t)m, sizeof(float), cmp_float_total);
    for (int64_t j = 0; j <= 256; j++) out[j] = tmp[(j * m) / 257];
}

/* The exact sample quantiles of the whole tensor ("The easiest way to find the eCDF is
 * to sort a given tensor"): Q2 with m = n.  n >= 1. */
int oracle_exact_quantiles(const float* x, int64_t n, float out[257]) {
    if (n < 1) return -1;
    float* tmp = (float*)malloc(sizeof(float) * (size_t)n);
    if (!tmp) return -1;
    sample_quantiles(x, n, tmp, out);
    free(tmp);
    return 0;
}

/* SRAM-Quantiles (App G): the quantiles of every S-value chunk (Q3), averaged (Q4).
 * out[j] estimates Q_X(j/257), j = 0..256.  n >= 1, S >= 1. */
int oracle_sram_quantiles(const float* x, int64_t n, int64_t S, float out[257]) {
    if (n < 1 || S < 1) return -1;
    int64_t nchunks = (n + S - 1) / S;
    float* tmp = (float*)malloc(sizeof(float) * (size_t)S);
    if (!tmp) return -1;
    double sum[257];
    float q[257];
    for (int j = 0; j <= 256; j++) sum[j] = 0.0;
    for (int64_t c = 0; c < nchunks; c++) {
        int64_t start = c * S, m = (n - start < S) ? n - start : S;
        sample_quantiles(x + start, m, tmp, q);
        for (int j = 0; j <= 256; j++) sum[j] += (double)q[j];
    }
    for (int j = 0; j <= 256; j++) out[j] = (float)(sum[j] / (double)nchunks);
    free(tmp);
    return 0;
}

/* Quantile data type (Eq.5, Q1/Q5) from the 257 quantiles Q_X(j/257): 256 values in [-1, 1],
 * ascending whenever the quantiles are.  Returns -1 if every midpoint is 0 (no scale). */
int oracle_quantile_codebook(const float quantiles[257], float out[256]) {
    double mid[256], M = 0.0;
    for (int i = 0; i < 256; i++) {
        mid[i] = ((double)quantiles[i] + (double)quantiles[i + 1]) * 0.5;
        if (fabs(mid[i]) > M) M = fabs(mid[i]);
    }
    if (!(M > 0.0)) return -1;
    for (int i = 0; i < 256; i++) out[i] = (float)(mid[i] / M);
    return 0;
}
