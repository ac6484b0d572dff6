// Pointwise (1x1, pad 0, any stride) binary convolution on the POPC pipe: ResNet-18's
// downsample shortcuts (C = 64 / 128 -> 2C filters, stride 2, BatchNorm, f32 NCHW output).
//
// Replaces the same reference path as the tcgen05 engines -- QConv2d.forward(INFER_PACKED)
// (layers.py:225-245) = im2col (tensor.py:60-78) -> pack_matrix_b (bitpack.py:152-169) ->
// xnor_gemm (gemm.py:128-139) -- bit-identically, for K = C <= 128.
//
// Why not the tensor cores: with K <= 128 a pixel is 1-2 u64 words and an output costs
// CW (xor + 2 popc) integer instructions, while every output is 4 bytes of f32 written to HBM.
// The layer is bound by its OUTPUT stream (layer 2's downsample: 103 MB written, 1.6 MB read),
// which a tensor-core tile pipeline (operand expansion, TMEM round trip, epilogue warps) only
// slows down: 35 us on bnn_sconv.cu against 27.5 us here (HBM write floor 16 us).  This is the
// LOP3 / POPC arm of the north-star contest winning on its own ground.
//
// One thread = one output pixel x a group of 64 filters: the pixel's words stay in registers,
// filter words and the per-filter epilogue parameters are broadcast from SMEM, and for every
// filter a warp writes 32 consecutive pixels of the NCHW plane (one 128-byte line).
#include "bnn_common.cuh"

namespace bnn {
namespace pw {

constexpr int kThreads = 256;    // pixels per CTA
constexpr int kFgDefault = 64;   // filters per CTA (blockIdx.y)

struct Geom {
    const uint64_t *x;  // packed NHWC [B, H, W, CW]
    const uint64_t *w;  // [F, CW]
    float *y;           // f32 NCHW [B, F, OH, OW]
    const float *res;   // optional residual, same layout
    int H, W, OH, OW, sh, sw, F, K;
    long long NP;       // B * OH * OW
};

template <int CW, int kFg, int kMagic>
__global__ void __launch_bounds__(kThreads) xnor_pw_kernel(const Geom g, const Epilogue ep) {
    __shared__ uint64_t s_w[kFg * CW];
    __shared__ float4 s_bn[kFg];   // mean, inv_std, gamma, beta
    __shared__ float2 s_aff[kFg];  // scale, shift
    // let the next kernel start its prologue; weights and parameters are constants of the
    // layer, so they are staged before waiting for the producer of x
    asm volatile("griddepcontrol.launch_dependents;\n");
    const int f0 = blockIdx.y * kFg;
    const int nf = g.F - f0 < kFg ? g.F - f0 : kFg;
    const bool has_bn = ep.bn_mean != nullptr;
    for (int i = threadIdx.x; i < nf * CW; i += kThreads) s_w[i] = __ldg(g.w + (int64_t)f0 * CW + i);
    for (int i = threadIdx.x; i < nf; i += kThreads) {
        if (has_bn)
            s_bn[i] = make_float4(__ldg(ep.bn_mean + f0 + i), __ldg(ep.bn_inv + f0 + i),
                                  __ldg(ep.bn_gamma + f0 + i), __ldg(ep.bn_beta + f0 + i));
        s_aff[i] = make_float2(ep.scale ? __ldg(ep.scale + f0 + i) : 1.0f,
                               ep.shift ? __ldg(ep.shift + f0 + i) : 0.0f);
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    __syncthreads();
    const int64_t m = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (m >= g.NP) return;
    const int ohw = g.OH * g.OW;
    const int64_t b = m / ohw;
    const int p = (int)(m - b * ohw);
    const int oy = p / g.OW, ox = p - oy * g.OW;
    const uint64_t *xin = g.x + ((b * g.H + (int64_t)oy * g.sh) * g.W + (int64_t)ox * g.sw) * CW;
    uint64_t xw[CW];
    if constexpr (CW % 2 == 0) {
#pragma unroll
        for (int i = 0; i < CW; i += 2) {
            const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(xin + i));
            xw[i] = v.x, xw[i + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < CW; ++i) xw[i] = __ldg(xin + i);
    }
    const int64_t obase = (b * g.F + f0) * ohw + p;
    float *out = g.y + obase;
    const float *res = g.res ? g.res + obase : nullptr;
    const bool dot = ep.domain == BNN_DOT;
    const bool scale = ep.scale != nullptr, shift = ep.shift != nullptr;
    const float keff = (float)ep.k_eff, klog = (float)ep.k_logical;
#pragma unroll 8
    for (int f = 0; f < nf; ++f) {
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < CW; ++i) cnt += __popcll(xw[i] ^ s_w[f * CW + i]);
        // Epilogue::apply in the reference op order (tails are 0 in both operands)
        float v;
        if constexpr (kMagic) {
            // counts -> f32 without I2F: for 0 <= n < 2^23, as_float(0x4B000000 | n) = 2^23 + n;
            // P = k_eff - X and 2P - K are small integers, exact in f32 in any order
            const float pc = __fsub_rn(keff, __fsub_rn(__int_as_float(0x4B000000 | cnt), 8388608.0f));
            v = dot ? __fmaf_rn(2.0f, pc, -klog) : pc;
        } else {
            const int pc = ep.k_eff - cnt;
            v = (float)(dot ? 2 * pc - ep.k_logical : pc);
        }
        const float2 a = s_aff[f];
        if (scale) v = __fmul_rn(v, a.x);
        if (shift) v = __fadd_rn(v, a.y);
        if (has_bn) {
            const float4 q = s_bn[f];  // layers.py:598-602
            v = __fadd_rn(__fmul_rn(q.z, __fmul_rn(__fsub_rn(v, q.x), q.y)), q.w);
        }
        if (res) v = __fadd_rn(v, __ldg(res + (int64_t)f * ohw));
        out[(int64_t)f * ohw] = v;
    }
}

// OH * OW % 4 == 0: one thread = 4 consecutive pixels of a plane x kFg filters, so every output
// instruction is a 16-byte store (a warp writes 512 contiguous bytes per filter, as a fill kernel
// does) and a filter's words / parameters are read from SMEM once per 4 outputs
template <int CW, int kFg>
__global__ void __launch_bounds__(kThreads) xnor_pw4_kernel(const Geom g, const Epilogue ep) {
    __shared__ uint64_t s_w[kFg * CW];
    __shared__ float4 s_bn[kFg];
    __shared__ float2 s_aff[kFg];
    asm volatile("griddepcontrol.launch_dependents;\n");
    const int f0 = blockIdx.y * kFg;
    const int nf = g.F - f0 < kFg ? g.F - f0 : kFg;
    const bool has_bn = ep.bn_mean != nullptr;
    for (int i = threadIdx.x; i < nf * CW; i += kThreads) s_w[i] = __ldg(g.w + (int64_t)f0 * CW + i);
    for (int i = threadIdx.x; i < nf; i += kThreads) {
        if (has_bn)
            s_bn[i] = make_float4(__ldg(ep.bn_mean + f0 + i), __ldg(ep.bn_inv + f0 + i),
                                  __ldg(ep.bn_gamma + f0 + i), __ldg(ep.bn_beta + f0 + i));
        s_aff[i] = make_float2(ep.scale ? __ldg(ep.scale + f0 + i) : 1.0f,
                               ep.shift ? __ldg(ep.shift + f0 + i) : 0.0f);
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    __syncthreads();
    const int64_t m = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * 4;  // first of 4 pixels
    if (m >= g.NP) return;
    const int ohw = g.OH * g.OW;
    const int64_t b = m / ohw;       // (ohw % 4 == 0: the 4 pixels share the image)
    const int p = (int)(m - b * ohw);
    uint64_t xw[4][CW];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int pu = p + u;
        const int oy = pu / g.OW, ox = pu - oy * g.OW;
        const uint64_t *xin = g.x + ((b * g.H + (int64_t)oy * g.sh) * g.W + (int64_t)ox * g.sw) * CW;
        if constexpr (CW % 2 == 0) {
#pragma unroll
            for (int i = 0; i < CW; i += 2) {
                const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(xin + i));
                xw[u][i] = v.x, xw[u][i + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < CW; ++i) xw[u][i] = __ldg(xin + i);
        }
    }
    const int64_t obase = (b * g.F + f0) * ohw + p;
    float *out = g.y + obase;
    const float *res = g.res ? g.res + obase : nullptr;
    const bool dot = ep.domain == BNN_DOT;
    const bool scale = ep.scale != nullptr, shift = ep.shift != nullptr;
    const float keff = (float)ep.k_eff, klog = (float)ep.k_logical;
#pragma unroll 4
    for (int f = 0; f < nf; ++f) {
        uint64_t wv[CW];
#pragma unroll
        for (int i = 0; i < CW; ++i) wv[i] = s_w[f * CW + i];
        const float2 a = s_aff[f];
        const float4 q = s_bn[f];
        float4 r4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (res) r4 = __ldg(reinterpret_cast<const float4 *>(res + (int64_t)f * ohw));
        const float rr[4] = {r4.x, r4.y, r4.z, r4.w};
        float o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int cnt = 0;
#pragma unroll
            for (int i = 0; i < CW; ++i) cnt += __popcll(xw[u][i] ^ wv[i]);
            const float pc = __fsub_rn(keff, __fsub_rn(__int_as_float(0x4B000000 | cnt), 8388608.0f));
            float v = dot ? __fmaf_rn(2.0f, pc, -klog) : pc;
            if (scale) v = __fmul_rn(v, a.x);
            if (shift) v = __fadd_rn(v, a.y);
            if (has_bn) v = __fadd_rn(__fmul_rn(q.z, __fmul_rn(__fsub_rn(v, q.x), q.y)), q.w);
            if (res) v = __fadd_rn(v, rr[u]);
            o[u] = v;
        }
        *reinterpret_cast<float4 *>(out + (int64_t)f * ohw) = make_float4(o[0], o[1], o[2], o[3]);
    }
}

}  // namespace pw

// Eligible: 1x1 kernel, no padding, C <= 128 in whole or partial words (tails 0; at C = 256 the
// eight POPCs per output lose to the pre-expanded tensor-core engine, 25.6 vs 16.3 us), f32 output,
// no sign-pack output.  Returns BNN_EUNSUP otherwise (the caller falls through).
int launch_pwconv(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W, const uint64_t *w,
                  int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw_,
                  int64_t oh, int64_t ow, float *y, const Epilogue &ep, cudaStream_t s,
                  const float *res) {
    using namespace pw;
    const int64_t CW = ceil_div(C, 64);
    if (kh != 1 || kw != 1 || ph != 0 || pw_ != 0 || (CW != 1 && CW != 2) || y == nullptr ||
        ep.pack_out != nullptr)
        return BNN_EUNSUP;
    if (CW >= 2 && (reinterpret_cast<uintptr_t>(x) & 15) != 0) return BNN_EUNSUP;
    const int64_t NP = B * oh * ow;
    if (NP <= 0 || F <= 0) return BNN_OK;
    if (oh * ow >= (1ll << 24) || ceil_div(F, kFgDefault) > 65535) return BNN_EUNSUP;
    Geom g{};
    g.x = x, g.w = w, g.y = y, g.res = res;
    g.H = (int)H, g.W = (int)W, g.OH = (int)oh, g.OW = (int)ow, g.sh = (int)sh, g.sw = (int)sw;
    g.F = (int)F, g.K = (int)C, g.NP = NP;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // 64 filters per CTA and the I2F-free count conversion: measured best of {32, 64, 128} x
    // {I2F, magic} at batch 256 (27.5 / 19.8 us for ResNet-18's layer-2 / layer-3 downsample
    // against 35.4 / 26.2 us on the tensor-core engines) and at batch 32 (6.6 vs 10.6 us)
    // one-word pixels on large batches: the 4-pixel kernel (16-byte stores), 16 filters per CTA
    // to keep the grid large (ResNet-18 layer-2 downsample at batch 256: 22.9 vs 27.5 us; at
    // batch 32 and for two-word pixels, which sit on the POPC pipe's rate, the scalar kernel is
    // as fast or faster)
    const bool vec4 = CW == 1 && NP >= 131072 && (oh * ow) % 4 == 0 &&
                      (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                      (res == nullptr || (reinterpret_cast<uintptr_t>(res) & 15) == 0);
    if (vec4) {
        cfg.gridDim = dim3((unsigned)ceil_div(NP, kThreads * 4), (unsigned)ceil_div(F, 16));
        cudaLaunchKernelEx(&cfg, xnor_pw4_kernel<1, 16>, g, ep);
        return check_launch("xnor_pw4_kernel");
    }
    cfg.gridDim = dim3((unsigned)ceil_div(NP, kThreads), (unsigned)ceil_div(F, kFgDefault));
    if (CW == 1) cudaLaunchKernelEx(&cfg, xnor_pw_kernel<1, kFgDefault, 1>, g, ep);
    else cudaLaunchKernelEx(&cfg, xnor_pw_kernel<2, kFgDefault, 1>, g, ep);
    return check_launch("xnor_pw_kernel");
}

}  // namespace bnn
