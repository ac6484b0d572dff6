// Internal helpers shared by the sm_100a kernels of libbnn_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bnn_b200.h"

namespace bnn {

// thread-local last error (bnn_last_error); set_error returns the status
int set_error(int status, const char *fmt, ...);
int check_launch(const char *what);

inline cudaStream_t as_stream(bnn_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Debug knobs (bnn_debug_set, include/bnn_b200.h): process-wide, not thread-safe,
// all 0 by default; the product path never sets them (tools/ experiments only).
struct DebugKnobs {
    int64_t umma_bits = 0;      // BNN_DEBUG_UMMA_BITS: tcgen05 engine debug bit flags
    int64_t fp4_bn = 0;         // BNN_DEBUG_FP4_BN: force the kind::mxf4 tile N
    int64_t pair_kw32 = 0;      // BNN_DEBUG_PAIR_KW32: 2-CTA pairs from this K (u32 words)
    int64_t stem_bits = 0;      // BNN_DEBUG_STEM_BITS: stem kernel debug bit flags
    int64_t pack_pix = 0;       // BNN_DEBUG_PACK_PIX: pack kernel variant (0 = default)
    int64_t pack_ch = 0;        // BNN_DEBUG_PACK_CH: channels per lane (0 = default 8)
    int64_t stempost_simple = 0;  // BNN_DEBUG_STEMPOST_SIMPLE: unbanded stem post-op
    int64_t grid_cap = 0;       // BNN_DEBUG_GRID_CAP: persistent tcgen05 kernels use <= this many
                                // CTAs (tests: many tiles per CTA, every ring wraps)
    uint64_t *trace_buf = nullptr;  // bnn_umma_trace
};
extern DebugKnobs g_debug;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Epilogue parameters common to the GEMM and conv kernels.
//   X  = sum over all stored words of popc(a ^ b)
//   P  = k_eff - X     (k_eff absorbs the tail correction, see capi)
//   v  = domain == DOT ? 2P - K : P ;  out = v * scale[m] + shift[m]
struct Epilogue {
    int32_t k_eff;
    int32_t k_logical;
    int32_t domain;
    const float *scale;
    const float *shift;
    // multi-bit (bit-plane) operands: value = (alpha * code + beta) / gamma per
    // operand; out = (aA aB S + aA bB sumA[m] + bA aB sumB[n] + K bA bB) / (gA gB)
    int32_t a_alpha = 1, a_beta = 0, b_alpha = 1, b_beta = 0;
    float inv_gamma = 1.0f;
    // optional fused inference BatchNorm in the reference's op order
    // (layers.py:598-602): gamma * ((x - mean) * inv_std) + beta, each op rounded
    const float *bn_mean = nullptr, *bn_inv = nullptr, *bn_gamma = nullptr, *bn_beta = nullptr;
    // optional sign-pack of the final value (next layer's QActivation + pack):
    // u32 word (n * pack_ld32 + m / 32), bit m % 32 = out[m, n] >= 0
    uint32_t *pack_out = nullptr;
    int64_t pack_ld32 = 0;
    int32_t *pack_flags = nullptr;
    // host-side dispatch: tcgen05 engine variant of this call (BNN_ALGO_UMMA_V0 + v;
    // AUTO / UMMA = 2), read by the launcher only
    int32_t variant = 2;
    __device__ __forceinline__ float bn(float f, int m) const {
        if (!bn_mean) return f;
        const float xh = __fmul_rn(__fsub_rn(f, __ldg(bn_mean + m)), __ldg(bn_inv + m));
        return __fadd_rn(__fmul_rn(__ldg(bn_gamma + m), xh), __ldg(bn_beta + m));
    }
    __device__ __forceinline__ float apply(int32_t x, int m) const {
        int32_t p = k_eff - x;
        int32_t v = domain == BNN_DOT ? 2 * p - k_logical : p;
        float f = (float)v;
        if (scale) f = __fmul_rn(f, __ldg(scale + m));
        if (shift) f = __fadd_rn(f, __ldg(shift + m));
        return bn(f, m);
    }
};

}  // namespace bnn
