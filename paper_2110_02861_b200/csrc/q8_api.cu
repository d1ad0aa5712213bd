// q8_api.cu -- the C ABI declared in include/q8.h: validation, host scalars, per-device
// table cache and kernel launches.  No compute happens on the host except the once-per-
// process codebook/threshold construction (a1) and the per-call fp32 scalars (G8-G10).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/q8.h"
#include "q8_kernels.cuh"
#include "q8_codec.cuh"
#include "q8_launch.h"
#include "q8_step_kernel.cuh"
#include "q8_step32_kernel.cuh"
#include "q8_quantiles.cuh"
#include "q8_quant_kernel.cuh"

namespace q8 {
void build_dynamic_codebook(bool is_signed, float out[256]);
void build_eytzinger_thresholds(const float Q[256], float out[256]);
void build_sorted_thresholds(const float Q[256], float out[256]);
bool build_bucket_lut(const float T[256], bool is_signed, int shift, int key_min, int entries, uint8_t* lut);
}  // namespace q8

namespace {

thread_local std::string g_last_error;

q8_status fail(q8_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

q8_status ok() {
    g_last_error.clear();
    return Q8_OK;
}

q8_status cuda_fail(cudaError_t e, const char* what) {
    return fail(Q8_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// ---------------------------------------------------------------- per-device state
constexpr int kMaxDevices = 64;
struct DeviceState {
    float* tabs = nullptr;  // kTabFloats device floats
    int sms = 0;
};
std::mutex g_mu;
DeviceState g_dev[kMaxDevices];

q8_status device_state(DeviceState** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) return fail(Q8_ERR_UNSUPPORTED, "device ordinal %d out of range", dev);
    std::lock_guard<std::mutex> lock(g_mu);
    DeviceState& d = g_dev[dev];
    if (d.tabs == nullptr) {
        static float host[q8::kTabFloats];
        q8::build_dynamic_codebook(true, host + q8::kTabQs);
        q8::build_eytzinger_thresholds(host + q8::kTabQs, host + q8::kTabTs);
        q8::build_sorted_thresholds(host + q8::kTabQs, host + q8::kTabSs);
        q8::build_dynamic_codebook(false, host + q8::kTabQu);
        q8::build_eytzinger_thresholds(host + q8::kTabQu, host + q8::kTabTu);
        q8::build_sorted_thresholds(host + q8::kTabQu, host + q8::kTabSu);
        uint8_t* lut = reinterpret_cast<uint8_t*>(host + q8::kTabLut);
        if (!q8::build_bucket_lut(host + q8::kTabSs, true, q8::kShiftS, 0, q8::kLutSBytes, lut) ||
            !q8::build_bucket_lut(host + q8::kTabSu, false, q8::kShiftU, q8::kLutUKeyMin, q8::kLutUBytes,
                                  lut + q8::kLutSBytes))
            return fail(Q8_ERR_CUDA, "internal: bucket table spans more than two codes");
        float* ptr = nullptr;
        e = cudaMalloc(&ptr, sizeof host);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tables)");
        e = cudaMemcpy(ptr, host, sizeof host, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(ptr);
            return cuda_fail(e, "cudaMemcpy(tables)");
        }
        int sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) {
            cudaFree(ptr);
            return cuda_fail(e, "cudaDeviceGetAttribute");
        }
        d.sms = sms;
        d.tabs = ptr;
    }
    *out = &d;
    return Q8_OK;
}

// Resident CTAs per SM for a kernel (cached per function pointer by the caller).
int ctas_per_sm(const void* fn) {
    const char* env = std::getenv("Q8_CTAS_PER_SM");
    if (env && std::atoi(env) > 0) return std::atoi(env);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, q8::kThreads, 0) != cudaSuccess || occ < 1) occ = 1;
    return occ;
}

int64_t grid_for(const DeviceState* d, int occ, int64_t nblocks) {
    int64_t g = static_cast<int64_t>(d->sms) * occ;
    return nblocks < g ? nblocks : g;
}

// ---------------------------------------------------------------- hparams
q8_status validate_hparams(q8_kind kind, const q8_hparams* hp, int64_t step) {
    if (!hp) return fail(Q8_ERR_INVALID, "hparams is NULL");
    if (kind != Q8_ADAM && kind != Q8_ADAMW && kind != Q8_MOMENTUM && kind != Q8_LAMB && kind != Q8_LARS)
        return fail(Q8_ERR_INVALID, "bad kind %d", kind);
    if (!(hp->lr >= 0.0) || !std::isfinite(hp->lr)) return fail(Q8_ERR_INVALID, "lr must be finite and >= 0");
    if (!(hp->beta1 >= 0.0 && hp->beta1 < 1.0)) return fail(Q8_ERR_INVALID, "beta1 must be in [0, 1)");
    if (!(hp->weight_decay >= 0.0) || !std::isfinite(hp->weight_decay))
        return fail(Q8_ERR_INVALID, "weight_decay must be finite and >= 0");
    if (q8::two_states(kind)) {
        if (!(hp->beta2 >= 0.0 && hp->beta2 < 1.0)) return fail(Q8_ERR_INVALID, "beta2 must be in [0, 1)");
        if (!(hp->eps > 0.0) || !std::isfinite(hp->eps)) return fail(Q8_ERR_INVALID, "eps must be finite and > 0");
    }
    if (step < 1) return fail(Q8_ERR_INVALID, "step must be >= 1 (got %lld)", static_cast<long long>(step));
    return Q8_OK;
}

// Element-wise entry points take the Adam family and Momentum only.
q8_status reject_layerwise(q8_kind kind) {
    if (kind == Q8_LAMB || kind == Q8_LARS)
        return fail(Q8_ERR_INVALID, "kind %d is layer-wise: use q8_optim8bit_step_layerwise", kind);
    return Q8_OK;
}

// fp32 scalars of the update, computed in double and rounded once (G8-G10; LAMB L1).
q8::StepScalars make_scalars(const q8_hparams* hp, int64_t step, q8_kind kind = Q8_ADAM) {
    return q8::compute_scalars(kind, hp->lr, hp->beta1, hp->beta2, hp->eps, hp->weight_decay, hp->bias_correction, step);
}

q8_status validate_tensor(q8_kind kind, q8_dtype gdt, const q8_tensor& t, int idx) {
    if (t.n < 0) return fail(Q8_ERR_INVALID, "tensor %d: n < 0", idx);
    if (t.n == 0) return Q8_OK;
    const bool two = q8::two_states(kind);
    if (!t.p || !t.g || !t.s1 || !t.absmax1 || (two && (!t.s2 || !t.absmax2)))
        return fail(Q8_ERR_INVALID, "tensor %d: NULL buffer with n > 0", idx);
    if (!aligned(t.p, 16)) return fail(Q8_ERR_INVALID, "tensor %d: p not 16-byte aligned", idx);
    // 16 B: the step kernel moves each full block with TMA bulk copies (16-byte granules)
    if (!aligned(t.g, 16)) return fail(Q8_ERR_INVALID, "tensor %d: g not 16-byte aligned", idx);
    if (!aligned(t.s1, 16) || (two && !aligned(t.s2, 16)))
        return fail(Q8_ERR_INVALID, "tensor %d: codes not 16-byte aligned", idx);
    if (!aligned(t.absmax1, 4) || (two && !aligned(t.absmax2, 4)))
        return fail(Q8_ERR_INVALID, "tensor %d: absmax not 4-byte aligned", idx);
    return Q8_OK;
}

// ---------------------------------------------------------------- launch dispatch
int search_variant() {
    static const int v = [] {
        const char* env = std::getenv("Q8_SEARCH");
        return (env && std::strcmp(env, "eytzinger") == 0) ? q8::SEARCH_EYTZINGER : q8::SEARCH_BUCKET;
    }();
    return v;
}

// Sub-blocks (256-thread groups, one 2048-element block each) per persistent CTA: 4 for 16-bit
// gradients, 3 for fp32 (shared-memory bound); Q8_NSUB=2|3|4 overrides (tuning).
int nsub_variant(q8_dtype gdt) {
    static const int env = [] {
        const char* e = std::getenv("Q8_NSUB");
        const int n = e ? std::atoi(e) : 0;
        return (n >= 2 && n <= 4) ? n : 0;
    }();
    const int mx = gdt == Q8_F32 ? 3 : 4;
    return env ? std::min(env, mx) : mx;
}

// Kernels already opted into their dynamic shared memory, per device (the attribute is set
// per device: a process stepping tensors on two GPUs needs it on both).
std::mutex g_smem_mu;
struct SmemDone {
    int dev;
    const void* fn;
};
SmemDone g_smem_done[1024];
int g_smem_count = 0;

template <int MAXT>
q8_status dispatch_step(q8_kind kind, q8_dtype gdt, const q8::StepParams<MAXT>& P, const DeviceState* d,
                        cudaStream_t st, int plan = 0) {
    static const int subt = [] {
        const char* e = std::getenv("Q8_SUBT");
        const int v = e ? std::atoi(e) : 0;
        return (v == 128 || v == 256) ? v : 0;
    }();
    const q8::LaunchCtx ctx{d->tabs, d->sms, st, search_variant(), nsub_variant(gdt), subt, plan};
    const q8::StepParams<1>* single = nullptr;
    const q8::StepParams<q8::kMultiMaxT>* multi = nullptr;
    if constexpr (MAXT == 1) single = &P; else multi = &P;
    cudaError_t e = cudaErrorInvalidValue;
    switch (gdt) {
        case Q8_F32: e = q8::launch_step_g0(kind, single, multi, ctx); break;
        case Q8_F16: e = q8::launch_step_g1(kind, single, multi, ctx); break;
        case Q8_BF16: e = q8::launch_step_g2(kind, single, multi, ctx); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "optim8bit_step_kernel launch");
    return Q8_OK;
}

// Plans of <= kSmallMaxT non-empty tensors: one launch with the 192-entry descriptor table.
q8_status dispatch_plan_small(q8_kind kind, q8_dtype gdt, const q8::StepParams<q8::kSmallMaxT>& P,
                              const DeviceState* d, cudaStream_t st) {
    const q8::LaunchCtx ctx{d->tabs, d->sms, st, q8::SEARCH_BUCKET, 0, 0, 1};
    cudaError_t e = cudaErrorInvalidValue;
    switch (gdt) {
        case Q8_F32: e = q8::launch_plan_small_g0(kind, P, ctx); break;
        case Q8_F16: e = q8::launch_plan_small_g1(kind, P, ctx); break;
        case Q8_BF16: e = q8::launch_plan_small_g2(kind, P, ctx); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "optim8bit_step_kernel launch");
    return Q8_OK;
}

q8_status check_common(q8_dtype gdt, int32_t blocksize) {
    if (gdt != Q8_F32 && gdt != Q8_F16 && gdt != Q8_BF16) return fail(Q8_ERR_INVALID, "bad g_dtype %d", gdt);
    if (blocksize != q8::kBlock)
        return fail(Q8_ERR_UNSUPPORTED, "blocksize %d unsupported on the GPU (only 2048)", blocksize);
    return Q8_OK;
}

}  // namespace

namespace {
// Launch the TMA-pipelined quantizer (q8_quant_kernel.cuh): one persistent CTA per SM at most.
template <int QTAB, bool kSigned, bool TW>
q8_status launch_quant(const DeviceState* d, const float* code, const float* x, float* absmax, uint8_t* codes,
                       int64_t n, cudaStream_t st) {
    const auto fn = q8::quantize_tma_kernel<QTAB, kSigned, TW>;
    cudaError_t e = q8::ensure_smem(reinterpret_cast<const void*>(fn), q8::kQtSmemBytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(quantizer)");
    const int64_t nb = (n + q8::kBlock - 1) / q8::kBlock;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((nb + q8::kQNSub - 1) / q8::kQNSub, d->sms));
    fn<<<grid, q8::kQNSub * q8::kQSubT, q8::kQtSmemBytes, st>>>(d->tabs, code, x, absmax, codes, n, nb);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "quantize_tma_kernel launch");
    return Q8_OK;
}
}  // namespace

cudaError_t q8::ensure_smem(const void* fn, int smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_smem_mu);
    for (int i = 0; i < g_smem_count; ++i)
        if (g_smem_done[i].fn == fn && g_smem_done[i].dev == dev) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (g_smem_count < static_cast<int>(sizeof g_smem_done / sizeof g_smem_done[0]))
        g_smem_done[g_smem_count++] = SmemDone{dev, fn};
    return cudaSuccess;
}

extern "C" {

const char* q8_last_error(void) { return g_last_error.c_str(); }

const char* q8_version(void) { return "q8 0.1 sm_100a"; }

q8_status q8_create_linear_codebook(int32_t is_signed, float* out_host) {
    if (!out_host) return fail(Q8_ERR_INVALID, "out_host is NULL");
    for (int i = 0; i < 256; ++i) {
        // linear quantization (T3 caption P:214), reading L0: signed (i - 127)/128 -- even spacing
        // 1/128, exact 0 at index 127 and +1 at 255 (the dynamic type's layout of its specials);
        // unsigned i/255.  Computed in double and rounded once (both are exact in binary32).
        const double v = is_signed ? static_cast<double>(i - 127) / 128.0 : static_cast<double>(i) / 255.0;
        out_host[i] = static_cast<float>(v);
    }
    return ok();
}

// ---------------------------------------------------------------- SRAM-Quantiles (App G)
namespace {
// Resident CTAs per SM are cached process-wide: the library runs only on sm_100a devices, whose
// SMs have identical register files and shared memory, so the occupancy of a kernel is the same on
// every device; the shared-memory opt-in itself is per device (ensure_smem).
int quantile_rows(const DeviceState* d, int64_t nchunks) {
    if (q8::ensure_smem(reinterpret_cast<const void*>(q8::sram_quantiles_kernel), q8::kQSmemBytes) != cudaSuccess)
        return 1;
    static int occ = [] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, q8::sram_quantiles_kernel, q8::kQThreads,
                                                          q8::kQSmemBytes) != cudaSuccess || o < 1)
            o = 1;
        const char* env = std::getenv("Q8_QUANTILE_CTAS_PER_SM");
        if (env && std::atoi(env) > 0) o = std::atoi(env);
        return o;
    }();
    return static_cast<int>(grid_for(d, occ, nchunks));
}
}  // namespace

int64_t q8_quantiles_workspace_bytes(int64_t n) {
    if (n < 1) return -1;
    DeviceState* d = nullptr;
    if (device_state(&d) != Q8_OK) return -1;
    const int64_t nchunks = (n + q8::kQChunk - 1) / q8::kQChunk;
    return static_cast<int64_t>(quantile_rows(d, nchunks)) * q8::kQuantiles * static_cast<int64_t>(sizeof(double));
}

q8_status q8_estimate_quantiles(const float* x_dev, int64_t n, float* quantiles_dev, float* code_dev,
                                void* workspace_dev, int64_t workspace_bytes, void* stream) {
    if (n < 1) return fail(Q8_ERR_INVALID, "n must be >= 1 (quantiles of an empty tensor are undefined)");
    if (!x_dev || !quantiles_dev || !workspace_dev) return fail(Q8_ERR_INVALID, "NULL buffer");
    if (!aligned(x_dev, 16) || !aligned(workspace_dev, 16) || !aligned(quantiles_dev, 4) ||
        (code_dev && !aligned(code_dev, 4)))
        return fail(Q8_ERR_INVALID, "misaligned buffer (x and workspace 16 B)");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    const int64_t nchunks = (n + q8::kQChunk - 1) / q8::kQChunk;
    const int rows = quantile_rows(d, nchunks);
    const int64_t need = static_cast<int64_t>(rows) * q8::kQuantiles * static_cast<int64_t>(sizeof(double));
    if (workspace_bytes < need)
        return fail(Q8_ERR_INVALID, "workspace too small: %lld < %lld bytes", static_cast<long long>(workspace_bytes),
                    static_cast<long long>(need));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* partial = static_cast<double*>(workspace_dev);
    q8::sram_quantiles_kernel<<<rows, q8::kQThreads, q8::kQSmemBytes, st>>>(x_dev, n, nchunks, partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "sram_quantiles_kernel launch");
    q8::quantiles_finalize_kernel<<<1, 288, 0, st>>>(partial, rows, nchunks, quantiles_dev, code_dev);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "quantiles_finalize_kernel launch");
    return ok();
}

q8_status q8_create_quantile_codebook(const float* quantiles_host, float* out_host) {
    if (!quantiles_host || !out_host) return fail(Q8_ERR_INVALID, "NULL buffer");
    // Eq.5: midpoints of consecutive quantiles, in double; normalized into [-1, 1] by the
    // largest magnitude (Fig. 6 caption), rounded once (reading Q5)
    double mid[256], M = 0.0;
    for (int i = 0; i < 256; ++i) {
        mid[i] = (static_cast<double>(quantiles_host[i]) + static_cast<double>(quantiles_host[i + 1])) * 0.5;
        M = std::max(M, std::fabs(mid[i]));
    }
    if (!(M > 0.0) || !std::isfinite(M)) return fail(Q8_ERR_INVALID, "every Eq.5 midpoint is zero (or non-finite)");
    for (int i = 0; i < 256; ++i) out_host[i] = static_cast<float>(mid[i] / M);
    return ok();
}

q8_status q8_count_nonfinite(const void* g_dev, q8_dtype g_dtype, int64_t n, uint64_t* count_dev, void* stream) {
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (!count_dev) return fail(Q8_ERR_INVALID, "count_dev is NULL");
    if (g_dtype != Q8_F32 && g_dtype != Q8_F16 && g_dtype != Q8_BF16) return fail(Q8_ERR_INVALID, "bad g_dtype %d", g_dtype);
    if (n > 0 && !g_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (n > 0 && !aligned(g_dev, 16)) return fail(Q8_ERR_INVALID, "g not 16-byte aligned");
    if (!aligned(count_dev, 8)) return fail(Q8_ERR_INVALID, "count_dev not 8-byte aligned");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(count_dev, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(count)");
    if (n == 0) return ok();
    const int per = g_dtype == Q8_F32 ? 4 : 8;
    const int64_t nv = (n / per + q8::kThreads - 1) / q8::kThreads;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(nv, 4 * d->sms)));
    auto* out = reinterpret_cast<unsigned long long*>(count_dev);
    switch (g_dtype) {
        case Q8_F32: q8::count_nonfinite_kernel<q8::G_F32><<<grid, q8::kThreads, 0, st>>>(g_dev, n, out); break;
        case Q8_F16: q8::count_nonfinite_kernel<q8::G_F16><<<grid, q8::kThreads, 0, st>>>(g_dev, n, out); break;
        case Q8_BF16: q8::count_nonfinite_kernel<q8::G_BF16><<<grid, q8::kThreads, 0, st>>>(g_dev, n, out); break;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "count_nonfinite_kernel launch");
    return ok();
}

q8_status q8_quantize_tensorwise(const float* code_dev, const float* x_dev, float* absmax_dev, uint8_t* codes_dev,
                                 int64_t n, void* stream) {
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (n == 0) return ok();
    if (!code_dev || !x_dev || !absmax_dev || !codes_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (!aligned(x_dev, 16) || !aligned(codes_dev, 4) || !aligned(absmax_dev, 4) || !aligned(code_dev, 4))
        return fail(Q8_ERR_INVALID, "misaligned buffer (x 16 B, codes 4 B)");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(absmax_dev, 0, sizeof(float), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(absmax)");
    const int64_t n4 = (n / 4 + q8::kThreads - 1) / q8::kThreads;
    const unsigned grid_r = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(n4, 4 * d->sms)));
    q8::tensor_absmax_kernel<<<grid_r, q8::kThreads, 0, st>>>(x_dev, n, reinterpret_cast<unsigned int*>(absmax_dev));
    if (q8_status s = launch_quant<q8::QTAB_GENERIC, true, true>(d, code_dev, x_dev, absmax_dev, codes_dev, n, st);
        s != Q8_OK)
        return s;
    return ok();
}

q8_status q8_dequantize_tensorwise(const float* code_dev, const uint8_t* codes_dev, const float* absmax_dev,
                                   float* out_dev, int64_t n, void* stream) {
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (n == 0) return ok();
    if (!code_dev || !codes_dev || !absmax_dev || !out_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (!aligned(out_dev, 16) || !aligned(codes_dev, 4) || !aligned(absmax_dev, 4) || !aligned(code_dev, 4))
        return fail(Q8_ERR_INVALID, "misaligned buffer (out 16 B, codes 4 B)");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    const int64_t nb = (n + q8::kBlock - 1) / q8::kBlock;
    static int occ = ctas_per_sm(reinterpret_cast<const void*>(q8::dequantize_blockwise_kernel<true>));
    q8::dequantize_blockwise_kernel<true><<<static_cast<unsigned>(grid_for(d, occ, nb)), q8::kThreads, 0,
                                            static_cast<cudaStream_t>(stream)>>>(code_dev, codes_dev, absmax_dev,
                                                                                 out_dev, n, nb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "dequantize_tensorwise launch");
    return ok();
}

q8_status q8_create_dynamic_codebook(int32_t is_signed, float* out_host) {
    if (!out_host) return fail(Q8_ERR_INVALID, "out_host is NULL");
    q8::build_dynamic_codebook(is_signed != 0, out_host);
    return ok();
}

q8_status q8_quantize_blockwise(const float* code_dev, const float* x_dev, float* absmax_dev, uint8_t* codes_dev,
                                int64_t n, int32_t blocksize, void* stream) {
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (blocksize != q8::kBlock) return fail(Q8_ERR_UNSUPPORTED, "blocksize %d unsupported (only 2048)", blocksize);
    if (n == 0) return ok();
    if (!code_dev || !x_dev || !absmax_dev || !codes_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (!aligned(x_dev, 16) || !aligned(codes_dev, 4) || !aligned(absmax_dev, 4) || !aligned(code_dev, 4))
        return fail(Q8_ERR_INVALID, "misaligned buffer (x 16 B, codes 4 B)");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    if (q8_status s = launch_quant<q8::QTAB_GENERIC, true, false>(d, code_dev, x_dev, absmax_dev, codes_dev, n,
                                                                   static_cast<cudaStream_t>(stream));
        s != Q8_OK)
        return s;
    return ok();
}

q8_status q8_quantize_blockwise_dynamic(int32_t is_signed, const float* x_dev, float* absmax_dev, uint8_t* codes_dev,
                                        int64_t n, int32_t blocksize, void* stream) {
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (blocksize != q8::kBlock) return fail(Q8_ERR_UNSUPPORTED, "blocksize %d unsupported (only 2048)", blocksize);
    if (n == 0) return ok();
    if (!x_dev || !absmax_dev || !codes_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (!aligned(x_dev, 16) || !aligned(codes_dev, 4) || !aligned(absmax_dev, 4))
        return fail(Q8_ERR_INVALID, "misaligned buffer (x 16 B, codes 4 B)");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const q8_status s = is_signed
                            ? launch_quant<q8::QTAB_BUILTIN, true, false>(d, nullptr, x_dev, absmax_dev, codes_dev, n, st)
                            : launch_quant<q8::QTAB_BUILTIN, false, false>(d, nullptr, x_dev, absmax_dev, codes_dev, n, st);
    if (s != Q8_OK) return s;
    return ok();
}

q8_status q8_dequantize_blockwise(const float* code_dev, const uint8_t* codes_dev, const float* absmax_dev,
                                  float* out_dev, int64_t n, int32_t blocksize, void* stream) {
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (blocksize != q8::kBlock) return fail(Q8_ERR_UNSUPPORTED, "blocksize %d unsupported (only 2048)", blocksize);
    if (n == 0) return ok();
    if (!code_dev || !codes_dev || !absmax_dev || !out_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (!aligned(out_dev, 16) || !aligned(codes_dev, 4) || !aligned(absmax_dev, 4) || !aligned(code_dev, 4))
        return fail(Q8_ERR_INVALID, "misaligned buffer (out 16 B, codes 4 B)");
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    const int64_t nb = (n + q8::kBlock - 1) / q8::kBlock;
    static int occ = ctas_per_sm(reinterpret_cast<const void*>(q8::dequantize_blockwise_kernel<false>));
    q8::dequantize_blockwise_kernel<false><<<static_cast<unsigned>(grid_for(d, occ, nb)), q8::kThreads, 0,
                                      static_cast<cudaStream_t>(stream)>>>(code_dev, codes_dev, absmax_dev, out_dev, n,
                                                                            nb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "dequantize_blockwise_kernel launch");
    return ok();
}

q8_status q8_optim8bit_step(q8_kind kind, float* p, const void* g, q8_dtype g_dtype, uint8_t* s1, uint8_t* s2,
                            float* absmax1, float* absmax2, int64_t n, int32_t blocksize, const q8_hparams* hp,
                            int64_t step, void* stream) {
    if (q8_status s = reject_layerwise(kind); s != Q8_OK) return s;
    if (q8_status s = check_common(g_dtype, blocksize); s != Q8_OK) return s;
    if (q8_status s = validate_hparams(kind, hp, step); s != Q8_OK) return s;
    q8_tensor t{p, g, s1, s2, absmax1, absmax2, n};
    if (q8_status s = validate_tensor(kind, g_dtype, t, 0); s != Q8_OK) return s;
    if (n == 0) return ok();
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    q8::StepParams<1> P;
    P.s = make_scalars(hp, step);
    P.scale = nullptr;
    P.num_tensors = 1;
    P.block_start[0] = 0;
    P.total_blocks = P.block_start[1] = (n + q8::kBlock - 1) / q8::kBlock;
    P.t[0] = q8::TensorDesc{p, g, s1, s2, absmax1, absmax2, n};
    if (q8_status s = dispatch_step<1>(kind, g_dtype, P, d, static_cast<cudaStream_t>(stream)); s != Q8_OK) return s;
    return ok();
}

q8_status q8_optim8bit_step_multi(q8_kind kind, q8_dtype g_dtype, const q8_tensor* tensors_host, int32_t num_tensors,
                                  int32_t blocksize, const q8_hparams* hp, int64_t step, void* stream) {
    if (q8_status s = reject_layerwise(kind); s != Q8_OK) return s;
    if (q8_status s = check_common(g_dtype, blocksize); s != Q8_OK) return s;
    if (q8_status s = validate_hparams(kind, hp, step); s != Q8_OK) return s;
    if (num_tensors < 0) return fail(Q8_ERR_INVALID, "num_tensors < 0");
    if (num_tensors > 0 && !tensors_host) return fail(Q8_ERR_INVALID, "tensors_host is NULL");
    for (int i = 0; i < num_tensors; ++i)
        if (q8_status s = validate_tensor(kind, g_dtype, tensors_host[i], i); s != Q8_OK) return s;
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    constexpr int MAXT = Q8_MAX_TENSORS_PER_LAUNCH;
    static thread_local q8::StepParams<MAXT> P;  // ~24 KB; kernel parameter (copied at launch)
    P.s = make_scalars(hp, step);
    P.scale = nullptr;
    int i = 0;
    while (i < num_tensors) {
        int k = 0;
        int64_t blocks = 0;
        for (; i < num_tensors && k < MAXT; ++i) {
            const q8_tensor& t = tensors_host[i];
            if (t.n == 0) continue;
            P.t[k] = q8::TensorDesc{t.p, t.g, t.s1, t.s2, t.absmax1, t.absmax2, t.n};
            P.block_start[k] = blocks;
            blocks += (t.n + q8::kBlock - 1) / q8::kBlock;
            ++k;
        }
        if (k == 0) break;
        P.num_tensors = k;
        P.block_start[k] = blocks;
        P.total_blocks = blocks;
        if (q8_status s = dispatch_step<MAXT>(kind, g_dtype, P, d, static_cast<cudaStream_t>(stream)); s != Q8_OK)
            return s;
    }
    return ok();
}

}  // extern "C"

// ---------------------------------------------------------------- 32-bit-state step

namespace {

q8_status validate_tensor32(q8_kind kind, const q8_tensor32& t, int idx) {
    if (t.n < 0) return fail(Q8_ERR_INVALID, "tensor %d: n < 0", idx);
    if (t.n == 0) return Q8_OK;
    if (!t.p || !t.g || !t.m || (kind != Q8_MOMENTUM && !t.r))
        return fail(Q8_ERR_INVALID, "tensor %d: NULL buffer with n > 0", idx);
    if (!aligned(t.p, 16) || !aligned(t.g, 16) || !aligned(t.m, 16) || (kind != Q8_MOMENTUM && !aligned(t.r, 16)))
        return fail(Q8_ERR_INVALID, "tensor %d: buffers must be 16-byte aligned", idx);
    return Q8_OK;
}

template <int MAXT>
q8_status launch_step32(q8_kind kind, q8_dtype gdt, const q8::StepParams<MAXT>& P, const DeviceState* d,
                        cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(P.total_blocks, 8LL * d->sms));
#define Q8_CASE32(K, G)                                                                     \
    if (kind == K && gdt == G) {                                                            \
        q8::optim32bit_step_kernel<K, G, MAXT><<<grid, q8::kThreads, 0, st>>>(P);             \
        cudaError_t e = cudaGetLastError();                                                 \
        return e == cudaSuccess ? Q8_OK : cuda_fail(e, "optim32bit_step_kernel launch");     \
    }
    Q8_CASE32(Q8_ADAM, Q8_F32) Q8_CASE32(Q8_ADAM, Q8_F16) Q8_CASE32(Q8_ADAM, Q8_BF16)
    Q8_CASE32(Q8_ADAMW, Q8_F32) Q8_CASE32(Q8_ADAMW, Q8_F16) Q8_CASE32(Q8_ADAMW, Q8_BF16)
    Q8_CASE32(Q8_MOMENTUM, Q8_F32) Q8_CASE32(Q8_MOMENTUM, Q8_F16) Q8_CASE32(Q8_MOMENTUM, Q8_BF16)
#undef Q8_CASE32
    return fail(Q8_ERR_INVALID, "bad kind/dtype");
}

}  // namespace

extern "C" {

q8_status q8_optim32bit_step_multi(q8_kind kind, q8_dtype g_dtype, const q8_tensor32* tensors_host,
                                   int32_t num_tensors, const q8_hparams* hp, int64_t step, void* stream) {
    if (q8_status s = reject_layerwise(kind); s != Q8_OK) return s;
    if (q8_status s = check_common(g_dtype, q8::kBlock); s != Q8_OK) return s;
    if (q8_status s = validate_hparams(kind, hp, step); s != Q8_OK) return s;
    if (num_tensors < 0) return fail(Q8_ERR_INVALID, "num_tensors < 0");
    if (num_tensors > 0 && !tensors_host) return fail(Q8_ERR_INVALID, "tensors_host is NULL");
    for (int i = 0; i < num_tensors; ++i)
        if (q8_status s = validate_tensor32(kind, tensors_host[i], i); s != Q8_OK) return s;
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    constexpr int MAXT = Q8_MAX_TENSORS_PER_LAUNCH;
    static thread_local q8::StepParams<MAXT> P;
    P.s = make_scalars(hp, step);
    P.scale = nullptr;
    int i = 0;
    while (i < num_tensors) {
        int k = 0;
        int64_t blocks = 0;
        for (; i < num_tensors && k < MAXT; ++i) {
            const q8_tensor32& t = tensors_host[i];
            if (t.n == 0) continue;
            P.t[k] = q8::TensorDesc{t.p, t.g, reinterpret_cast<uint8_t*>(t.m), reinterpret_cast<uint8_t*>(t.r),
                                    nullptr, nullptr, t.n};
            P.block_start[k] = blocks;
            blocks += (t.n + q8::kBlock - 1) / q8::kBlock;
            ++k;
        }
        if (k == 0) break;
        P.num_tensors = k;
        P.block_start[k] = blocks;
        P.total_blocks = blocks;
        if (q8_status s = launch_step32<MAXT>(kind, g_dtype, P, d, static_cast<cudaStream_t>(stream)); s != Q8_OK)
            return s;
    }
    return ok();
}

}  // extern "C"

// ---------------------------------------------------------------- layer-wise step (LAMB / LARS)

namespace {

constexpr int kLwChunk = Q8_MAX_TENSORS_PER_LAUNCH;

// Workspace layout: float scale[num_tensors] (rounded up to 16 B), then double2 partial[] sized
// for the largest chunk of kLwChunk consecutive tensors.
// Workspace layout (q8.h): [0, kLwCountBytes) the per-tensor block counters of the LARS norms pass (zero
// between calls: the pass resets them) -- at a FIXED offset, so a workspace reused for other tensor lists
// still finds them zero; then the 16-B grid barrier of the one-launch LARS step; then the scales
// (Q8_LAYERWISE_SCALE_OFFSET); then the binary64 partials.
constexpr int64_t kLwCountBytes = 4 * kLwChunk;
static_assert(kLwCountBytes + 16 == Q8_LAYERWISE_SCALE_OFFSET, "q8.h scale offset");
int64_t lw_scale_bytes(int32_t num_tensors) { return (static_cast<int64_t>(num_tensors) * 4 + 15) / 16 * 16; }

int64_t lw_partial_blocks(const q8_tensor* t, int32_t num_tensors) {
    int64_t best = 0;
    for (int32_t c = 0; c < num_tensors; c += kLwChunk) {
        int64_t blocks = 0;
        for (int32_t i = c; i < std::min(num_tensors, c + kLwChunk); ++i) blocks += (t[i].n + q8::kBlock - 1) / q8::kBlock;
        best = std::max(best, blocks);
    }
    return best;
}

// The layer-wise launches, chunk by chunk of <= MAXT tensors, with descriptor table P (MAXT = kLwChunk, or
// kSmallMaxT for short lists).
template <int MAXT>
q8_status layerwise_chunks(q8::StepParams<MAXT>& P, q8_kind kind, q8_dtype g_dtype, const q8_tensor* tensors_host,
                           int32_t num_tensors, const q8_hparams* hp, double trust_coefficient, int64_t step,
                           uint8_t* ws, const q8::LaunchCtx& ctx) {
    unsigned int* count = reinterpret_cast<unsigned int*>(ws);
    float* scale = reinterpret_cast<float*>(ws + Q8_LAYERWISE_SCALE_OFFSET);
    double2* partial = reinterpret_cast<double2*>(ws + Q8_LAYERWISE_SCALE_OFFSET + lw_scale_bytes(num_tensors));
    P.s = make_scalars(hp, step, kind);
    P.lw.lr = hp->lr;
    P.lw.eta = trust_coefficient;
    P.lw.wd = hp->weight_decay;
    P.lw.gbar = reinterpret_cast<unsigned int*>(ws + kLwCountBytes);
    for (int32_t c = 0; c < num_tensors; c += MAXT) {
        // every tensor of the chunk keeps its slot (empty ones have no blocks) so that
        // scale[i] belongs to tensors_host[i]
        const int k = std::min(num_tensors - c, MAXT);
        int64_t blocks = 0;
        for (int j = 0; j < k; ++j) {
            const q8_tensor& t = tensors_host[c + j];
            P.t[j] = q8::TensorDesc{t.p, t.g, t.s1, t.s2, t.absmax1, t.absmax2, t.n};
            P.block_start[j] = blocks;
            blocks += (t.n + q8::kBlock - 1) / q8::kBlock;
        }
        P.num_tensors = k;
        P.block_start[k] = blocks;
        P.total_blocks = blocks;
        P.scale = scale + c;
        P.partial = partial;
        cudaError_t e = cudaErrorInvalidValue;
        switch (g_dtype) {
            case Q8_F32: e = q8::launch_layerwise_g0(kind, P, ctx, partial, scale + c, count, hp->lr, trust_coefficient,
                                                     hp->weight_decay); break;
            case Q8_F16: e = q8::launch_layerwise_g1(kind, P, ctx, partial, scale + c, count, hp->lr, trust_coefficient,
                                                     hp->weight_decay); break;
            case Q8_BF16: e = q8::launch_layerwise_g2(kind, P, ctx, partial, scale + c, count, hp->lr, trust_coefficient,
                                                      hp->weight_decay); break;
        }
        if (e != cudaSuccess) return cuda_fail(e, "layer-wise step launch");
    }
    return ok();
}

}  // namespace

extern "C" {

int64_t q8_layerwise_workspace_bytes(const q8_tensor* tensors_host, int32_t num_tensors) {
    if (num_tensors < 0 || (num_tensors > 0 && !tensors_host)) return -1;
    for (int32_t i = 0; i < num_tensors; ++i)
        if (tensors_host[i].n < 0) return -1;
    // + the per-tensor block counters of the LARS norms pass (one launch chunk), + 16 B: the grid barrier
    // of the one-launch LARS step
    return lw_scale_bytes(num_tensors) + 16 * q8::kNormSlots * lw_partial_blocks(tensors_host, num_tensors) +
           kLwCountBytes + 16;
}

q8_status q8_optim8bit_step_layerwise(q8_kind kind, q8_dtype g_dtype, const q8_tensor* tensors_host,
                                      int32_t num_tensors, int32_t blocksize, const q8_hparams* hp,
                                      double trust_coefficient, int64_t step, void* workspace_dev,
                                      int64_t workspace_bytes, void* stream) {
    if (kind != Q8_LAMB && kind != Q8_LARS) return fail(Q8_ERR_INVALID, "kind %d is not layer-wise (LAMB/LARS)", kind);
    if (q8_status s = check_common(g_dtype, blocksize); s != Q8_OK) return s;
    if (q8_status s = validate_hparams(kind, hp, step); s != Q8_OK) return s;
    if (kind == Q8_LARS && !(trust_coefficient > 0.0 && std::isfinite(trust_coefficient)))
        return fail(Q8_ERR_INVALID, "trust_coefficient must be finite and > 0");
    if (num_tensors < 0) return fail(Q8_ERR_INVALID, "num_tensors < 0");
    if (num_tensors > 0 && !tensors_host) return fail(Q8_ERR_INVALID, "tensors_host is NULL");
    for (int i = 0; i < num_tensors; ++i)
        if (q8_status s = validate_tensor(kind, g_dtype, tensors_host[i], i); s != Q8_OK) return s;
    if (num_tensors == 0) return ok();
    const int64_t need = q8_layerwise_workspace_bytes(tensors_host, num_tensors);
    if (!workspace_dev || !aligned(workspace_dev, 16))
        return fail(Q8_ERR_INVALID, "workspace must be a non-NULL 16-byte aligned device buffer");
    if (workspace_bytes < need)
        return fail(Q8_ERR_INVALID, "workspace too small: %lld < %lld bytes", static_cast<long long>(workspace_bytes),
                    static_cast<long long>(need));
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    uint8_t* const ws = static_cast<uint8_t*>(workspace_dev);
    const q8::LaunchCtx ctx{d->tabs, d->sms, static_cast<cudaStream_t>(stream), q8::SEARCH_BUCKET, 0, 0};
    // lists of <= kSmallMaxT tensors: the half-size descriptor table (fewer parameter bytes per launch)
    if (num_tensors <= q8::kSmallMaxT) {
        static thread_local q8::StepParams<q8::kSmallMaxT> Ps;
        return layerwise_chunks(Ps, kind, g_dtype, tensors_host, num_tensors, hp, trust_coefficient, step, ws, ctx);
    }
    static thread_local q8::StepParams<kLwChunk> P;
    return layerwise_chunks(P, kind, g_dtype, tensors_host, num_tensors, hp, trust_coefficient, step, ws, ctx);
}

}  // extern "C"

// ---------------------------------------------------------------- fused ZeRO-1 step + peer memory

extern "C" {

int64_t q8_zero_signal_bytes(int32_t world, int32_t num_ctas) {
    if (world < 1 || world > q8::kMaxWorld || num_ctas < 0) return -1;
    int ctas = num_ctas;
    if (ctas == 0) {
        DeviceState* d = nullptr;
        if (device_state(&d) != Q8_OK) return -1;
        ctas = d->sms;
    }
    return static_cast<int64_t>(2) * world * ctas * 4;
}

q8_status q8_optim8bit_step_zero_fused(q8_kind kind, q8_dtype g_dtype, int32_t world, int32_t rank,
                                       const void* const* g_peers_host, float* const* p_peers_host,
                                       uint32_t* const* sig_peers_host, float* p_multicast, uint8_t* s1, uint8_t* s2,
                                       float* absmax1,
                                       float* absmax2, int64_t n_pad, int32_t blocksize, const q8_hparams* hp,
                                       int64_t step, uint32_t epoch, int32_t num_ctas, void* stream) {
    if (q8_status s = reject_layerwise(kind); s != Q8_OK) return s;
    if (q8_status s = check_common(g_dtype, blocksize); s != Q8_OK) return s;
    if (q8_status s = validate_hparams(kind, hp, step); s != Q8_OK) return s;
    if (world < 1 || world > q8::kMaxWorld) return fail(Q8_ERR_INVALID, "world must be in [1, %d]", q8::kMaxWorld);
    if (rank < 0 || rank >= world) return fail(Q8_ERR_INVALID, "rank %d out of [0, %d)", rank, world);
    if (n_pad < 0 || n_pad % (static_cast<int64_t>(world) * q8::kBlock) != 0)
        return fail(Q8_ERR_INVALID, "n_pad must be a multiple of world * 2048 (ZeRO padding)");
    if (epoch == 0) return fail(Q8_ERR_INVALID, "epoch must be >= 1 (signal pads start zeroed)");
    if (n_pad == 0) return ok();
    if (!g_peers_host || !p_peers_host || !sig_peers_host) return fail(Q8_ERR_INVALID, "peer arrays are NULL");
    for (int r = 0; r < world; ++r) {
        if (!g_peers_host[r] || !p_peers_host[r] || !sig_peers_host[r])
            return fail(Q8_ERR_INVALID, "rank %d: NULL peer pointer", r);
        if (!aligned(g_peers_host[r], 16) || !aligned(p_peers_host[r], 16) || !aligned(sig_peers_host[r], 4))
            return fail(Q8_ERR_INVALID, "rank %d: peer buffers must be 16-byte aligned", r);
    }
    const int64_t shard = n_pad / world;
    q8_tensor t{p_peers_host[rank] + static_cast<int64_t>(rank) * shard, g_peers_host[rank], s1, s2, absmax1, absmax2,
                shard};
    if (q8_status s = validate_tensor(kind, g_dtype, t, 0); s != Q8_OK) return s;
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    const int grid = num_ctas == 0 ? d->sms : num_ctas;
    if (grid < 1 || grid > d->sms)
        return fail(Q8_ERR_INVALID, "num_ctas must be in [1, %d] (all CTAs of all ranks must be co-resident)", d->sms);
    q8::StepParams<1> P;
    P.s = make_scalars(hp, step);
    P.scale = nullptr;
    P.partial = nullptr;
    P.num_tensors = 1;
    P.block_start[0] = 0;
    P.total_blocks = P.block_start[1] = shard / q8::kBlock;
    // this rank's own gradient shard is read through the TMA stages like the plain step's
    const int64_t gsz = g_dtype == Q8_F32 ? 4 : 2;
    P.t[0] = q8::TensorDesc{t.p, static_cast<const uint8_t*>(g_peers_host[rank]) + static_cast<int64_t>(rank) * shard * gsz,
                            s1, s2, absmax1, absmax2, shard};
    std::memset(&P.z, 0, sizeof P.z);
    for (int r = 0; r < world; ++r) {
        P.z.g[r] = g_peers_host[r];
        P.z.p[r] = p_peers_host[r];
        P.z.sig[r] = sig_peers_host[r];
    }
    if (p_multicast && !aligned(p_multicast, 16)) return fail(Q8_ERR_INVALID, "p_multicast not 16-byte aligned");
    P.z.p_mc = p_multicast;
    P.z.off = static_cast<int64_t>(rank) * shard;
    P.z.world = world;
    P.z.rank = rank;
    P.z.epoch = epoch;
    P.z.pow2 = (world & (world - 1)) == 0;
    P.z.invw = static_cast<float>(1.0 / world);
    const q8::LaunchCtx ctx{d->tabs, d->sms, static_cast<cudaStream_t>(stream), q8::SEARCH_BUCKET, 0, 0};
    cudaError_t e = cudaErrorInvalidValue;
    switch (g_dtype) {
        case Q8_F32: e = q8::launch_zero_g0(kind, P, ctx, grid); break;
        case Q8_F16: e = q8::launch_zero_g1(kind, P, ctx, grid); break;
        case Q8_BF16: e = q8::launch_zero_g2(kind, P, ctx, grid); break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "fused ZeRO step launch");
    return ok();
}

}  // extern "C"

// ---------------------------------------------------------------- plans (prepared multi-tensor steps)

struct q8_plan {
    int dev = 0;
    q8_kind kind = Q8_ADAM;
    q8_dtype gdt = Q8_F32;
    int32_t count = 0;
    std::vector<std::unique_ptr<q8::StepParams<q8::kMultiMaxT>>> chunks;
    // plans of <= kSmallMaxT non-empty tensors: their one launch with the 192-entry table (chunks empty)
    std::unique_ptr<q8::StepParams<q8::kSmallMaxT>> small;
    std::vector<int32_t> chunk_of, slot_of;  // per plan tensor; -1 for empty tensors
    unsigned int* done = nullptr;             // CTA completion counter of capturable launches
};

namespace {

__global__ void step_scalars_kernel(int kind, double lr, double beta1, double beta2, double eps, double wd, int bc,
                                    const int64_t* steps, int64_t n, float* out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const q8::StepScalars s = q8::compute_scalars(kind, lr, beta1, beta2, eps, wd, bc, steps[i]);
        float* o = out + 10 * i;
        o[0] = s.lr; o[1] = s.beta1; o[2] = s.beta2; o[3] = s.omb1; o[4] = s.omb2;
        o[5] = s.step_size; o[6] = s.eps_hat; o[7] = s.wd; o[8] = s.decay; o[9] = static_cast<float>(s.fast_div);
    }
}

q8_status plan_device_check(const q8_plan* plan) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev != plan->dev)
        return fail(Q8_ERR_INVALID, "plan was built on device %d but device %d is current", plan->dev, dev);
    return Q8_OK;
}

}  // namespace

extern "C" {

q8_status q8_plan_create(q8_kind kind, q8_dtype g_dtype, const q8_tensor* t8, int32_t n8, const q8_tensor32* t32,
                         int32_t n32, int32_t blocksize, q8_plan** out) {
    if (!out) return fail(Q8_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (q8_status s = reject_layerwise(kind); s != Q8_OK) return s;
    if (kind != Q8_ADAM && kind != Q8_ADAMW && kind != Q8_MOMENTUM) return fail(Q8_ERR_INVALID, "bad kind %d", kind);
    if (q8_status s = check_common(g_dtype, blocksize); s != Q8_OK) return s;
    if (n8 < 0 || n32 < 0) return fail(Q8_ERR_INVALID, "tensor counts must be >= 0");
    if ((n8 > 0 && !t8) || (n32 > 0 && !t32)) return fail(Q8_ERR_INVALID, "tensor array is NULL");
    for (int i = 0; i < n8; ++i)
        if (q8_status s = validate_tensor(kind, g_dtype, t8[i], i); s != Q8_OK) return s;
    for (int i = 0; i < n32; ++i)
        if (q8_status s = validate_tensor32(kind, t32[i], n8 + i); s != Q8_OK) return s;
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    auto plan = std::make_unique<q8_plan>();
    cudaError_t e = cudaGetDevice(&plan->dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    plan->kind = kind;
    plan->gdt = g_dtype;
    plan->count = n8 + n32;
    plan->chunk_of.assign(plan->count, -1);
    plan->slot_of.assign(plan->count, -1);
    constexpr int MAXT = q8::kMultiMaxT;
    q8::StepParams<MAXT>* P = nullptr;
    int64_t blocks = 0;
    for (int k = 0; k < plan->count; ++k) {
        q8::TensorDesc T;
        if (k < n8) {
            const q8_tensor& t = t8[k];
            T = q8::TensorDesc{t.p, t.g, t.s1, t.s2, t.absmax1, t.absmax2, t.n};
        } else {  // 32-bit states: a1 == NULL marks the tensor, s1/s2 carry m/r (TensorDesc)
            const q8_tensor32& t = t32[k - n8];
            T = q8::TensorDesc{t.p, t.g, reinterpret_cast<uint8_t*>(t.m), reinterpret_cast<uint8_t*>(t.r), nullptr,
                               nullptr, t.n};
        }
        if (T.n == 0) continue;
        if (!P || P->num_tensors == MAXT) {
            plan->chunks.push_back(std::make_unique<q8::StepParams<MAXT>>());
            P = plan->chunks.back().get();
            P->scale = nullptr;
            P->partial = nullptr;
            P->num_tensors = 0;
            blocks = 0;
        }
        const int slot = P->num_tensors++;
        P->t[slot] = T;
        P->block_start[slot] = blocks;
        blocks += (T.n + q8::kBlock - 1) / q8::kBlock;
        P->block_start[slot + 1] = blocks;
        P->total_blocks = blocks;
        plan->chunk_of[k] = static_cast<int32_t>(plan->chunks.size() - 1);
        plan->slot_of[k] = slot;
    }
    if (plan->chunks.size() == 1 && plan->chunks[0]->num_tensors <= q8::kSmallMaxT) {
        const q8::StepParams<MAXT>& B = *plan->chunks[0];
        plan->small = std::make_unique<q8::StepParams<q8::kSmallMaxT>>();
        q8::StepParams<q8::kSmallMaxT>& S = *plan->small;
        S.scale = B.scale;
        S.partial = B.partial;
        S.num_tensors = B.num_tensors;
        S.total_blocks = B.total_blocks;
        for (int j = 0; j <= B.num_tensors; ++j) S.block_start[j] = B.block_start[j];
        for (int j = 0; j < B.num_tensors; ++j) S.t[j] = B.t[j];
        plan->chunks.clear();  // chunk_of stays 0: the slot indices are the small table's
    }
    e = cudaMalloc(&plan->done, sizeof(unsigned int));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(plan counter)");
    e = cudaMemset(plan->done, 0, sizeof(unsigned int));
    if (e != cudaSuccess) {
        cudaFree(plan->done);
        return cuda_fail(e, "cudaMemset(plan counter)");
    }
    *out = plan.release();
    return ok();
}

q8_status q8_plan_set_grads(q8_plan* plan, const void* const* g_host, int32_t count) {
    if (!plan || !g_host) return fail(Q8_ERR_INVALID, "NULL argument");
    if (count != plan->count) return fail(Q8_ERR_INVALID, "count %d != the plan's %d tensors", count, plan->count);
    for (int k = 0; k < count; ++k) {
        const void* g = g_host[k];
        if (!g || plan->chunk_of[k] < 0) continue;
        if (!aligned(g, 16)) return fail(Q8_ERR_INVALID, "tensor %d: g not 16-byte aligned", k);
        if (plan->small)
            plan->small->t[plan->slot_of[k]].g = g;
        else
            plan->chunks[plan->chunk_of[k]]->t[plan->slot_of[k]].g = g;
    }
    return ok();
}

q8_status q8_plan_step(q8_plan* plan, const q8_hparams* hp, int64_t step, void* stream) {
    if (!plan) return fail(Q8_ERR_INVALID, "plan is NULL");
    if (q8_status s = validate_hparams(plan->kind, hp, step); s != Q8_OK) return s;
    if (q8_status s = plan_device_check(plan); s != Q8_OK) return s;
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    const q8::StepScalars sc = make_scalars(hp, step);
    if (plan->small) {
        plan->small->s = sc;
        plan->small->ds.step = nullptr;
        const q8_status s = dispatch_plan_small(plan->kind, plan->gdt, *plan->small, d, static_cast<cudaStream_t>(stream));
        return s == Q8_OK ? ok() : s;
    }
    for (auto& P : plan->chunks) {
        P->s = sc;
        P->ds.step = nullptr;
        if (q8_status s =
                dispatch_step<q8::kMultiMaxT>(plan->kind, plan->gdt, *P, d, static_cast<cudaStream_t>(stream), 1);
            s != Q8_OK)
            return s;
    }
    return ok();
}

q8_status q8_plan_step_device(q8_plan* plan, const q8_hparams* hp, int64_t* step_dev, void* stream) {
    if (!plan || !step_dev) return fail(Q8_ERR_INVALID, "NULL argument");
    if (q8_status s = validate_hparams(plan->kind, hp, 1); s != Q8_OK) return s;
    if (!aligned(step_dev, 8)) return fail(Q8_ERR_INVALID, "step_dev not 8-byte aligned");
    if (q8_status s = plan_device_check(plan); s != Q8_OK) return s;
    DeviceState* d = nullptr;
    if (q8_status s = device_state(&d); s != Q8_OK) return s;
    auto arm = [&](auto& P, bool last) {
        P.s = make_scalars(hp, 1);  // placeholder; the kernel uses ds (its wd decides the L2 variant)
        P.ds.step = step_dev;
        P.ds.done = plan->done;
        P.ds.advance = last ? 1 : 0;
        P.ds.kind = plan->kind;
        P.ds.lr = hp->lr;
        P.ds.beta1 = hp->beta1;
        P.ds.beta2 = hp->beta2;
        P.ds.eps = hp->eps;
        P.ds.wd = hp->weight_decay;
        P.ds.bias_correction = hp->bias_correction;
    };
    if (plan->small) {
        arm(*plan->small, true);
        q8_status s = dispatch_plan_small(plan->kind, plan->gdt, *plan->small, d, static_cast<cudaStream_t>(stream));
        plan->small->ds.step = nullptr;
        return s == Q8_OK ? ok() : s;
    }
    const size_t nc = plan->chunks.size();
    for (size_t c = 0; c < nc; ++c) {
        auto& P = plan->chunks[c];
        arm(*P, c + 1 == nc);
        q8_status s =
            dispatch_step<q8::kMultiMaxT>(plan->kind, plan->gdt, *P, d, static_cast<cudaStream_t>(stream), 1);
        P->ds.step = nullptr;
        if (s != Q8_OK) return s;
    }
    return ok();
}

void q8_plan_destroy(q8_plan* plan) {
    if (!plan) return;
    if (plan->done) cudaFree(plan->done);
    delete plan;
}

q8_status q8_step_scalars(q8_kind kind, const q8_hparams* hp, int64_t step, float* out_host) {
    if (!out_host) return fail(Q8_ERR_INVALID, "out_host is NULL");
    if (q8_status s = validate_hparams(kind, hp, step); s != Q8_OK) return s;
    const q8::StepScalars s = make_scalars(hp, step, kind);
    const float v[10] = {s.lr, s.beta1, s.beta2, s.omb1, s.omb2, s.step_size, s.eps_hat, s.wd, s.decay,
                         static_cast<float>(s.fast_div)};
    std::memcpy(out_host, v, sizeof v);
    return ok();
}

q8_status q8_step_scalars_device(q8_kind kind, const q8_hparams* hp, const int64_t* steps_dev, int64_t n,
                                 float* out_dev, void* stream) {
    if (q8_status s = validate_hparams(kind, hp, 1); s != Q8_OK) return s;
    if (n < 0) return fail(Q8_ERR_INVALID, "n < 0");
    if (n == 0) return ok();
    if (!steps_dev || !out_dev) return fail(Q8_ERR_INVALID, "NULL buffer with n > 0");
    if (!aligned(steps_dev, 8) || !aligned(out_dev, 4)) return fail(Q8_ERR_INVALID, "misaligned buffer");
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024));
    step_scalars_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        kind, hp->lr, hp->beta1, hp->beta2, hp->eps, hp->weight_decay, hp->bias_correction, steps_dev, n, out_dev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "step_scalars_kernel launch");
    return ok();
}

}  // extern "C"
