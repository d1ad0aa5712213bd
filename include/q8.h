/*
 * q8.h -- C ABI of the B200-native (sm_100a) block-wise dynamic 8-bit optimizer step.
 *
 * Method: Dettmers, Lewis, Shleifer & Zettlemoyer, "8-bit Optimizers via Block-wise
 * Quantization" (arXiv 2110.02861).  "P:<line>" cites /root/reference/PAPER.md;
 * "G<n>" cites the readings in DESIGN.md section 3.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Plain C: pointers, sizes, enums; no torch types.  Link: libq8.so (cudart static).
 *  - "_dev" pointers are CUDA device pointers on the current device; "_host" pointers
 *    are host memory.  The CALLER owns every buffer; the library never allocates on
 *    the hot path.  It owns only immutable internal tables (the two dynamic codebooks
 *    and their search tables), created once per device on first use.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is
 *    enqueued asynchronously; argument validation is synchronous.  Asynchronous CUDA
 *    errors surface at the caller's next synchronisation (CUDA convention).
 *  - Codes are uint8 indices into the ASCENDING 256-entry codebook (G4); block b of a
 *    tensor covers elements [b*B, min((b+1)*B, n)) and has one fp32 absmax N_b;
 *    the last block may be short (G5).  Blocks never span tensors.
 *  - Every call returns a q8_status; on failure q8_last_error() describes why
 *    (thread-local string, valid until the next call on the same thread).
 *  - n == 0 is a valid no-op (empty shards under ZeRO padding are normal).
 *  - Thread-safe and re-entrant: the library holds no mutable state besides its
 *    per-device table cache (guarded by a mutex).
 */
#ifndef Q8_H
#define Q8_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    Q8_OK = 0,
    Q8_ERR_INVALID = -1,      /* bad argument: NULL with n > 0, n < 0, misaligned, bad enum/hparam */
    Q8_ERR_UNSUPPORTED = -2,  /* valid request this build does not implement (blocksize != 2048) */
    Q8_ERR_CUDA = -3          /* a CUDA runtime call or kernel launch failed */
} q8_status;

typedef enum { Q8_F32 = 0, Q8_F16 = 1, Q8_BF16 = 2 } q8_dtype;          /* gradient dtype (G13) */
/* Eq.2, AdamW, Eq.1; the layer-wise LAMB and LARS of T5 are taken only by
 * q8_optim8bit_step_layerwise */
typedef enum { Q8_ADAM = 0, Q8_ADAMW = 1, Q8_MOMENTUM = 2, Q8_LAMB = 3, Q8_LARS = 4 } q8_kind;

/* Optimizer hyper-parameters (host struct, doubles; every derived fp32 scalar is computed
 * in double and rounded once, G8-G10).
 *   lr            alpha of Eq.1/Eq.2, >= 0
 *   beta1         beta_1 of Eq.2; the momentum beta of Eq.1 for Q8_MOMENTUM / Q8_LARS; in [0, 1)
 *   beta2         beta_2 of Eq.2, in [0, 1) (ignored by Q8_MOMENTUM / Q8_LARS)
 *   eps           epsilon of Eq.2, > 0 (ignored by Q8_MOMENTUM / Q8_LARS)
 *   weight_decay  >= 0.  Q8_ADAMW: decoupled, w *= (1 - lr*wd) before the update.
 *                 Q8_ADAM / Q8_MOMENTUM: L2, g += wd*w (G10).  Q8_LAMB / Q8_LARS: L1 / L2
 *   bias_correction  0/1: Kingma & Ba's folded correction alpha_t, eps_hat (G8);
 *                 ignored by Q8_MOMENTUM / Q8_LARS */
typedef struct {
    double lr, beta1, beta2, eps, weight_decay;
    int32_t bias_correction;
} q8_hparams;

/* One tensor of a multi-tensor step (all device pointers; s2/absmax2 may be NULL for
 * Q8_MOMENTUM).  Alignment: p, g, s1, s2 16 B (TMA bulk copies). */
typedef struct {
    float* p;
    const void* g;
    uint8_t* s1;
    uint8_t* s2;
    float* absmax1;
    float* absmax2;
    int64_t n;
} q8_tensor;

/* Fill out_host[256] with the dynamic data type's 256 values in ascending order.
 * is_signed = 1: dynamic tree quantization (S2.3): sign, run of zero bits =
 *                decade exponent, indicator bit, linear fraction; used for state 1.
 * is_signed = 0: dynamic quantization (S3.2): the sign bit re-purposed as a fixed
 *                extra fraction bit; used for the strictly positive state 2.
 * Reading G1/G2: bin-midpoint linear fraction, specials {0, +1}, built in double and
 * rounded once to fp32.  Pure host function.  Errors: INVALID if out_host is NULL. */
q8_status q8_create_dynamic_codebook(int32_t is_signed, float* out_host);

/* Fill out_host[256] with the linear data type: 256 evenly spaced values, signed
 * (is_signed = 1) (i - 127)/128 over [-127/128, 1] with an exact 0 at index 127 (reading L0,
 * zero states must round-trip exactly), unsigned (is_signed = 0) i/255 over [0, 1];
 * computed in double and rounded once.  The paper's ablation baseline "without dynamic quantization use linear quantization"
 * (T3 caption).  Pure host function.  Errors: INVALID if out_host is NULL. */
q8_status q8_create_linear_codebook(int32_t is_signed, float* out_host);

/* Block-wise quantization, Eq.4:
 *   N_b = max_i |x_i| over block b;  y_i = x_i / N_b (IEEE fp32 division; y = 0
 *   when N_b = 0, G7);  codes_i = argmin_j |code_dev[j] - y_i|, ties to the lower index (G6).
 *   x_dev      [n] fp32, 16-B aligned (read)
 *   code_dev   [256] fp32 device table, strictly ascending (read; e.g. a table made by
 *              q8_create_dynamic_codebook and copied to the device)
 *   absmax_dev [ceil(n/B)] fp32 (written)
 *   codes_dev  [n] uint8, 4-B aligned (written)
 *   blocksize  must be 2048 (else UNSUPPORTED, G16). */
q8_status q8_quantize_blockwise(const float* code_dev, const float* x_dev, float* absmax_dev,
                                uint8_t* codes_dev, int64_t n, int32_t blocksize, void* stream);

/* Block-wise quantization with the library's built-in dynamic data type (is_signed = 1:
 * the signed table of q8_create_dynamic_codebook(1); 0: the unsigned one), computed by the
 * same normalization and nearest-code search as q8_optim8bit_step (bucketed search,
 * DESIGN.md 6.2).  Results are identical to q8_quantize_blockwise with that table copied to
 * the device (Eq.4; ties to the lower index).  For is_signed = 0 negative inputs get code 0.
 * Buffers and errors as q8_quantize_blockwise. */
q8_status q8_quantize_blockwise_dynamic(int32_t is_signed, const float* x_dev, float* absmax_dev,
                                        uint8_t* codes_dev, int64_t n, int32_t blocksize, void* stream);

/* Block-wise dequantization: out_i = code_dev[codes_i] * absmax_dev[i / B] (one fp32
 * multiply).  codes_dev [n] uint8 4-B aligned, absmax_dev [ceil(n/B)], out_dev [n] fp32 16-B
 * aligned.  blocksize must be 2048. */
q8_status q8_dequantize_blockwise(const float* code_dev, const uint8_t* codes_dev, const float* absmax_dev,
                                  float* out_dev, int64_t n, int32_t blocksize, void* stream);

/* Tensor-wise quantization, Eq.3: one normalization constant N = max_i |x_i| for
 * the whole tensor (the cross-core reduction that block-wise quantization avoids), then
 * codes_i = argmin_j |code_dev[j] - x_i / N| (IEEE division, ties to the lower index).
 *   absmax_dev [1] fp32 (written: N); other buffers as q8_quantize_blockwise.  Two kernels: a
 *   grid reduction then the search. */
q8_status q8_quantize_tensorwise(const float* code_dev, const float* x_dev, float* absmax_dev,
                                 uint8_t* codes_dev, int64_t n, void* stream);

/* Tensor-wise dequantization: out_i = code_dev[codes_i] * absmax_dev[0]. */
q8_status q8_dequantize_tensorwise(const float* code_dev, const uint8_t* codes_dev, const float* absmax_dev,
                                   float* out_dev, int64_t n, void* stream);

/* SRAM-Quantiles (App G): approximate sample quantiles Q_X(j/257), j = 0..256, of the
 * tensor x -- the 257 quantiles whose Eq.5 midpoints form the quantile data type (App F.2,
 * P:403-416).  "we find the eCDF for a subset of values of the tensor that fits into SRAM (about
 * 4096 32-bit values).  Once we found the quantiles for each subset, we average the quantiles"
 * (P:440).  Readings Q1-Q4: chunks of 4096 consecutive elements (the last may be
 * short), each sorted on chip; chunk quantile j = its sorted value at index floor(j*m/257);
 * the estimate is the mean over chunks, accumulated in binary64 and rounded once to fp32 (the
 * summation order is fixed per device -- deterministic -- but differs from a sequential sum).
 *   x_dev          [n] fp32, 16-B aligned (read); n >= 1 (else INVALID).  NaNs are out of contract.
 *   quantiles_dev  [257] fp32 (written)
 *   code_dev       NULL, or [256] fp32 (written): the quantile data type of Eq.5 (reading Q5),
 *                  RN32(mid_i / max|mid|) with mid_i = (Q_i + Q_{i+1})/2 in binary64 (all zeros if
 *                  every midpoint is 0), usable as code_dev of q8_quantize_blockwise (entries are
 *                  non-decreasing; equal neighbours resolve to the lower index)
 *   workspace_dev  >= q8_quantiles_workspace_bytes(n) bytes, 16-B aligned, caller-owned scratch
 *                  (binary64 partial sums per CTA), not shared with a concurrent call
 * Two stream-ordered launches: the sort/accumulate pass and a one-CTA finalize. */
q8_status q8_estimate_quantiles(const float* x_dev, int64_t n, float* quantiles_dev, float* code_dev,
                                void* workspace_dev, int64_t workspace_bytes, void* stream);

/* Bytes of workspace q8_estimate_quantiles needs for n elements on the current device (host
 * function): 257 * 8 per persistent CTA.  -1 on bad input or no device. */
int64_t q8_quantiles_workspace_bytes(int64_t n);

/* Quantile data type from 257 host quantiles (Eq.5, reading Q5): out_host[i] =
 * RN32(mid_i / max_k |mid_k|), mid_i = (q_i + q_{i+1})/2 in binary64.  Pure host function.
 * Errors: INVALID for NULL buffers or when every midpoint is 0. */
q8_status q8_create_quantile_codebook(const float* quantiles_host, float* out_host);

/* The fused 8-bit optimizer step (S3; Fig.1), in place, for one tensor:
 * for each block b:
 *   1. dequantize  m = Q_s[s1_i] * absmax1[b],  r = Q_u[s2_i] * absmax2[b]
 *   2. update in fp32, element by element in registers: Eq.2 (Q8_ADAM/ADAMW,
 *      bias correction G8, weight decay G10) or Eq.1 (Q8_MOMENTUM); p uses the fp32
 *      post-update states (G12)
 *   3. absmax1[b] = max|m|, absmax2[b] = max|r| over the block
 *   4. requantize s1 = nearest code of m/absmax1[b] in Q_s (signed), s2 likewise in
 *      Q_u (unsigned) (Eq.4, G14)
 * Arguments (device pointers unless noted):
 *   p        [n] fp32 parameters, read-modify-write, 16-B aligned
 *   g        [n] gradients of g_dtype, read, 16-B aligned
 *   s1, s2   [n] uint8 codes (state 1 / state 2), RMW, 16-B aligned; s2 unused (may be
 *            NULL) for Q8_MOMENTUM.  All-zero codes+absmax is the valid initial state.
 *   absmax1, absmax2  [ceil(n/2048)] fp32, RMW; absmax2 unused for Q8_MOMENTUM
 *   blocksize must be 2048; step = t >= 1, the 1-based index of this update (the caller
 *   owns t, as torch's state['step']); hp host pointer.
 * Buffers must not alias each other. */
q8_status q8_optim8bit_step(q8_kind kind, float* p, const void* g, q8_dtype g_dtype, uint8_t* s1,
                            uint8_t* s2, float* absmax1, float* absmax2, int64_t n, int32_t blocksize,
                            const q8_hparams* hp, int64_t step, void* stream);

/* Multi-tensor variant (one launch per up-to-Q8_MAX_TENSORS_PER_LAUNCH tensors): the same
 * step applied to every tensor of tensors_host[num_tensors] (a HOST array of device-pointer
 * descriptors, copied into the launch).  Blocks are per tensor: each tensor's last
 * block may be short.  Tensors with n == 0 are skipped.  Same validation as above, per tensor. */
#define Q8_MAX_TENSORS_PER_LAUNCH 384
q8_status q8_optim8bit_step_multi(q8_kind kind, q8_dtype g_dtype, const q8_tensor* tensors_host,
                                  int32_t num_tensors, int32_t blocksize, const q8_hparams* hp, int64_t step,
                                  void* stream);

/* One tensor of a 32-bit-state step: fp32 states m, r instead of codes + absmax (r unused,
 * may be NULL, for Q8_MOMENTUM).  All device pointers, 16-byte aligned. */
typedef struct {
    float* p;
    const void* g;
    float* m;
    float* r;
    int64_t n;
} q8_tensor32;

/* The same fp32 update as q8_optim8bit_step (Eq.1/Eq.2, G8-G12, identical operation order) with
 * the states kept in 32 bits, over many tensors: the paper keeps the Stable Embedding layer's
 * optimizer states in 32 bits ("the only layer that uses 32-bit optimizer states", S3.3
 * P:124-125).  m, r are read-modify-write fp32 [n]; zero is the initial state.  Validation as
 * q8_optim8bit_step_multi. */
q8_status q8_optim32bit_step_multi(q8_kind kind, q8_dtype g_dtype, const q8_tensor32* tensors_host,
                                   int32_t num_tensors, const q8_hparams* hp, int64_t step, void* stream);

/* Layer-wise (trust-ratio) 8-bit optimizers: 8-bit LAMB and LARS, which the paper benchmarks
 * (T5) without printing their formulas; readings L1-L4, per tensor
 * ("layer") t of tensors_host[num_tensors]:
 *   Q8_LAMB (You et al. 2020, Alg. 2): states m, r as Eq.2 (s1 signed, s2 unsigned),
 *            u = c * m/(sqrt(r) + eps_hat) + wd*w  (c = sqrt(1-b2^t)/(1-b1^t), G8),
 *            w -= RN(lr * ||w||/||u||) * u  (ratio 1 when either norm is 0)
 *   Q8_LARS (You et al. 2017, Alg. 1): momentum state v (s1 signed; s2/absmax2 unused),
 *            v = beta1*v + RN(lr * eta*||w||/(||g|| + wd*||w||)) * (g + wd*w),  w -= v
 *            (the factor is lr when either norm is 0); eta = trust_coefficient > 0
 * Norms are over the whole tensor, of the PRE-update w (and of u from the fp32 post-update
 * states), accumulated in binary64; the per-tensor scale is rounded once to fp32 (L3).  States
 * are dequantized / requantized block-wise exactly as in q8_optim8bit_step.
 * Stream-ordered launches per chunk of Q8_MAX_TENSORS_PER_LAUNCH tensors: LAMB a norms pass (reads
 * w, g and the states), a per-tensor scale pass, the fused step; LARS a norms pass that also computes
 * the scales (the CTA that finishes a tensor's last block sums its partials), then the fused step as a
 * programmatic dependent launch (it stages its tables while the norms pass drains).
 *   workspace_dev  device scratch of at least q8_layerwise_workspace_bytes(tensors, n) bytes,
 *                  16-B aligned, caller-owned; its first Q8_LAYERWISE_SCALE_OFFSET bytes (block
 *                  counters of the LARS norms pass, at a fixed offset for any tensor list) must be
 *                  ZERO before the first call that uses it, and every call leaves them zero again;
 *                  must not be used by another call until this one completes on `stream`.  On
 *                  completion the 4*num_tensors bytes at offset Q8_LAYERWISE_SCALE_OFFSET hold each
 *                  tensor's fp32 scale (float scale[i] for tensors_host[i]; lr for empty tensors)
 *                  -- the trust ratio times lr, a diagnostic output.
 * Other arguments, alignment and errors as q8_optim8bit_step_multi; INVALID also for a kind
 * other than LAMB/LARS, trust_coefficient <= 0 (LARS) or a too-small workspace. */
#define Q8_LAYERWISE_SCALE_OFFSET 1552  /* bytes: 4 * Q8_MAX_TENSORS_PER_LAUNCH counters + 16 */
q8_status q8_optim8bit_step_layerwise(q8_kind kind, q8_dtype g_dtype, const q8_tensor* tensors_host,
                                      int32_t num_tensors, int32_t blocksize, const q8_hparams* hp,
                                      double trust_coefficient, int64_t step, void* workspace_dev,
                                      int64_t workspace_bytes, void* stream);

/* Bytes of workspace q8_optim8bit_step_layerwise needs for these tensors (host function):
 * 4 * Q8_MAX_TENSORS_PER_LAUNCH (per-tensor block counters of the LARS norms pass) + 16 (the grid
 * barrier of the one-launch LARS step) + 4 per tensor (the scales, rounded up to 16) + 128 per
 * 2048-block of the largest launch chunk (binary64 partial norms per warp).  -1 on bad input. */
int64_t q8_layerwise_workspace_bytes(const q8_tensor* tensors_host, int32_t num_tensors);

/* Fused ZeRO-1 step over peer memory: ONE kernel per rank does
 * the reduce-scatter of the gradients, the fused 8-bit step of this rank's shard and the
 * all-gather of the updated parameters, reading and writing the other ranks' buffers directly
 * (NVLink peer access / CUDA IPC mappings), tile by tile, so the transfers overlap the step.
 * The flat buffers of n_pad elements (a multiple of world*2048) are split into world shards of
 * n_pad/world on block boundaries (blocks are independent, so sharding is exact).
 *   g_peers_host[r]   rank r's full gradient buffer (n_pad elements of g_dtype), readable here
 *   p_peers_host[r]   rank r's full fp32 parameter buffer (n_pad), writable here; this rank's own
 *                     shard is read from p_peers_host[rank]
 *   sig_peers_host[r] rank r's signal pad, q8_zero_signal_bytes(world, num_ctas) bytes, zeroed once
 *                     at allocation and then owned by these calls
 *   p_multicast       NULL, or the NVLS multicast address (NVSwitch, e.g. torch symmetric memory's
 *                     multicast_ptr) that maps every rank's parameter buffer: the all-gather is then
 *                     ONE multimem.st per 16 bytes instead of world peer stores (16-B aligned)
 *   s1, s2, absmax1, absmax2  this rank's shard states (n_pad/world codes, n_pad/world/2048 absmax)
 * (the three peer arrays are HOST arrays of device pointers, copied into the launch)
 * Reading Z1: g = (g_0 + ... + g_{world-1}) / world per element -- binary32 adds in rank order,
 * IEEE division; then the step of q8_optim8bit_step on the shard, and every rank's buffer receives
 * the shard's new parameters.  Synchronisation: CTA i of every rank raises its flag (= epoch) in
 * every rank's pad and waits for all ranks' flags before reading gradients, and again after its
 * parameter writes; so when the call completes on `stream`, every rank's gradients have been
 * consumed and this rank's parameter buffer holds all shards.  epoch must start at 1 and grow by
 * one per call (the pads are never reset).  Launch contract: every rank makes the same sequence of
 * calls with the same num_ctas (0 = one CTA per SM).  The grid is launched cooperatively, so the
 * runtime guarantees that all of this rank's CTAs are resident at once (CUDA error
 * "cooperative launch too large" otherwise) -- with one rank per GPU that is sufficient for
 * progress.  Ranks sharing one GPU under MPS must also fit together (num_ctas <= SMs / world);
 * without MPS their kernels time-slice and still make progress.  A rank that never arrives (a
 * crashed peer) makes the kernel trap after ~30 s instead of hanging the GPU.
 * world <= 16.  Errors: as q8_optim8bit_step, plus INVALID for bad world/rank/n_pad/epoch/num_ctas. */
q8_status q8_optim8bit_step_zero_fused(q8_kind kind, q8_dtype g_dtype, int32_t world, int32_t rank,
                                       const void* const* g_peers_host, float* const* p_peers_host,
                                       uint32_t* const* sig_peers_host, float* p_multicast, uint8_t* s1, uint8_t* s2,
                                       float* absmax1,
                                       float* absmax2, int64_t n_pad, int32_t blocksize, const q8_hparams* hp,
                                       int64_t step, uint32_t epoch, int32_t num_ctas, void* stream);

/* Bytes of one rank's signal pad for q8_optim8bit_step_zero_fused: 2 * world * num_ctas * 4
 * (num_ctas 0 = the current device's SM count).  -1 on bad input. */
int64_t q8_zero_signal_bytes(int32_t world, int32_t num_ctas);

/* Count the non-finite gradient elements (NaN or +-inf) of g: *count_dev = #{i : g_i not finite}
 * (failure detection: non-finite gradients are out of the step's contract, G13, so a
 * mixed-precision caller skips the step when the count is non-zero, as AMP's GradScaler does).
 *   g_dev      [n] gradients of g_dtype, 16-B aligned (read)
 *   count_dev  one uint64 on the device, 8-B aligned (written: zeroed then accumulated on stream)
 * Errors: INVALID for n < 0, NULL, misalignment or a bad dtype. */
q8_status q8_count_nonfinite(const void* g_dev, q8_dtype g_dtype, int64_t n, uint64_t* count_dev, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Prepared multi-tensor steps ("plans"): the paper's drop-in optimizer ("changing two lines of
 * code") steps the same parameter list every iteration, so the descriptor arrays of
 * q8_optim8bit_step_multi are built and validated once, kept by the library, and each step costs
 * one host call (plus, when backward re-allocates gradients, one q8_plan_set_grads).  A plan may mix
 * 8-bit-state tensors with 32-bit-state tensors (the Stable Embedding layer, "the only layer that
 * uses 32-bit optimizer states", S3.3 P:124-125): both are stepped by the SAME kernel launch.
 * ------------------------------------------------------------------------------------------- */
typedef struct q8_plan q8_plan;

/* Build a plan for kind (Q8_ADAM, Q8_ADAMW or Q8_MOMENTUM) over t8[n8] (8-bit states, as
 * q8_optim8bit_step_multi) and t32[n32] (32-bit states, as q8_optim32bit_step_multi); tensor k of
 * the plan is t8[k] for k < n8 and t32[k - n8] after that.  All buffers live on the current
 * device, which the plan remembers; the library copies the descriptors (caller keeps ownership
 * of every buffer and must keep them alive while the plan is used).  *out receives the plan.
 * Errors: as q8_optim8bit_step_multi / q8_optim32bit_step_multi; CUDA if the plan's device
 * counter cannot be allocated. */
q8_status q8_plan_create(q8_kind kind, q8_dtype g_dtype, const q8_tensor* t8, int32_t n8, const q8_tensor32* t32,
                         int32_t n32, int32_t blocksize, q8_plan** out);

/* Re-point the gradients: g_host[k] (a HOST array of n8 + n32 device pointers, 16-B aligned,
 * g_dtype) becomes tensor k's gradient; a NULL entry keeps the previous pointer.  Host-only (no
 * CUDA call), so it may run while earlier steps are in flight; takes effect at the next step call.
 * Errors: INVALID for count != n8 + n32 or a misaligned pointer. */
q8_status q8_plan_set_grads(q8_plan* plan, const void* const* g_host, int32_t count);

/* One step of every tensor of the plan with the host step counter `step` (>= 1, as
 * q8_optim8bit_step): one kernel launch per 384 tensors on `stream`.  Must be called with the
 * plan's device current (INVALID otherwise); hyper-parameters validated as q8_optim8bit_step. */
q8_status q8_plan_step(q8_plan* plan, const q8_hparams* hp, int64_t step, void* stream);

/* The same step with the step counter on the DEVICE (CUDA-graph capturable: no host value changes
 * between replays): the launch reads t - 1 from *step_dev (int64, device memory, 0 before the first
 * step), computes the scalars of G8-G10 for t on the device (in binary64, the same expressions as
 * the host path; see DESIGN.md 6.8 for the pow() caveat) and stores t back into *step_dev when it
 * completes.  Hyper-parameters are captured by value at the call. */
q8_status q8_plan_step_device(q8_plan* plan, const q8_hparams* hp, int64_t* step_dev, void* stream);

/* Free the plan (host descriptors and its device counter).  NULL is a no-op. */
void q8_plan_destroy(q8_plan* plan);

/* Diagnostics: the fp32 scalars one update at `step` uses (G8-G10, LAMB L1), computed on the
 * host -- out_host[10] = lr, beta1, beta2, 1-beta1, 1-beta2, step_size, eps_hat, wd, decay,
 * fast-path flag (as a float) -- and the same ten for each steps_dev[i] computed on the DEVICE
 * (out_dev[10 * n], device memory) by the code the capturable plan step runs. */
q8_status q8_step_scalars(q8_kind kind, const q8_hparams* hp, int64_t step, float* out_host);
q8_status q8_step_scalars_device(q8_kind kind, const q8_hparams* hp, const int64_t* steps_dev, int64_t n,
                                 float* out_dev, void* stream);

/* Thread-local description of the last error ("" after success). */
const char* q8_last_error(void);

/* Library version string, e.g. "q8 0.1 sm_100a". */
const char* q8_version(void);

#ifdef __cplusplus
}
#endif

#endif /* Q8_H */
