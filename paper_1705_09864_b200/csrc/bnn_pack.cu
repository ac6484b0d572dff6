// Sign-binarise + bit-pack kernels (HBM-bound) and word re-layout helpers.
//
// Reference functions replaced (paths under /root/reference/pkg/src/bitnn):
//   binarize            bitpack.py:30-42    x >= 0 -> +1 (so -0.0 -> +1)
//   pack_matrix_a       bitpack.py:144-149  rows along K, LSB-first, tail fill
//   pack_matrix_b       bitpack.py:152-169  columns along K -> [W, N]
//   _validate_signs     bitpack.py:69-75    (STRICT mode flag)
//   audit_padding       bitpack.py:197-215
//   im2col + pack_matrix_b activation side of QConv2d (layers.py:230-236),
//                       here as a NCHW -> packed NHWC transpose-pack.
#include <cstdio>

#include "bnn_common.cuh"

namespace bnn {

__device__ __forceinline__ uint32_t sign_bit(float v) { return v >= 0.0f ? 1u : 0u; }

__device__ __forceinline__ uint32_t smem_u32_pack(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// streaming 16-byte load that does not allocate in L1 (the input is read once)
__device__ __forceinline__ float4 ld_stream(const float *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// Per-element checks: bit0 = non-finite, bit1 = not exactly +-1 (strict mode).
__device__ __forceinline__ int elem_flags(float v, int mode) {
    int f = isfinite(v) ? 0 : BNN_FLAG_NONFINITE;
    if (mode == BNN_PACK_STRICT && v != 1.0f && v != -1.0f) f |= BNN_FLAG_NOTSIGN;
    return f;
}

__device__ __forceinline__ void flush_flags(int f, int32_t *flags) {
    // one atomic per warp at most
    int any = __reduce_or_sync(0xffffffffu, f);
    if (any && flags && (threadIdx.x & 31) == 0) atomicOr(flags, any);
}

// ---------------------------------------------------------------- binarize
__global__ void binarize_kernel(const float *__restrict__ x, int64_t n, float *__restrict__ out,
                                int32_t *flags) {
    int f = 0;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        float v = x[i];
        f |= elem_flags(v, BNN_PACK_SIGN);
        out[i] = v >= 0.0f ? 1.0f : -1.0f;
    }
    flush_flags(f, flags);
}

// ---------------------------------------------------------------- pack rows
// One warp per row; each iteration covers 128 consecutive elements (4 per
// lane, float4 when aligned) and emits 2 u64 words.  Lane l owns elements
// 4l..4l+3, i.e. nibble l%8 of u32 word l/8; an OR-butterfly over the 8
// lanes of a group assembles each u32 word.
template <bool kVec4>
__global__ void pack_rows_kernel(const float *__restrict__ x, int64_t R, int64_t K, int64_t ldx,
                                 uint64_t *__restrict__ out, int64_t ldo, int pad_bit, int mode,
                                 int32_t *__restrict__ row_popc, int32_t *flags) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= R) return;  // warp-uniform
    const float *xr = x + row * ldx;
    const int64_t W = ceil_div(K, 64);
    int f = 0;
    int popc = 0;
    for (int64_t base = 0; base < W * 64; base += 128) {
        const int64_t e = base + 4 * lane;
        float v[4];
        if (kVec4 && e + 3 < K) {
            float4 q = __ldg(reinterpret_cast<const float4 *>(xr + e));
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = e + i < K ? __ldg(xr + e + i) : 0.0f;
        }
        uint32_t nib = 0, valid = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            bool in = e + i < K;
            uint32_t b = in ? sign_bit(v[i]) : (uint32_t)pad_bit;
            nib |= b << i;
            valid |= (in ? 1u : 0u) << i;
            if (in) f |= elem_flags(v[i], mode);
        }
        popc += __popc(nib & valid);
        uint32_t w = nib << (4 * (lane & 7));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        uint32_t hi = __shfl_down_sync(0xffffffffu, w, 8);
        const int64_t wi = base / 64 + (lane >> 4);
        if ((lane & 15) == 0 && wi < W) out[row * ldo + wi] = (uint64_t)w | ((uint64_t)hi << 32);
    }
    flush_flags(f, flags);
    if (row_popc) {
        popc = __reduce_add_sync(0xffffffffu, popc);
        if (lane == 0) row_popc[row] = popc;
    }
}

// ---------------------------------------------------------------- pack cols
// layout 'b': thread per (word w, column n); 64 coalesced loads along K.
__global__ void pack_cols_kernel(const float *__restrict__ x, int64_t K, int64_t N, int64_t ldx,
                                 uint64_t *__restrict__ out, int64_t ldo, int pad_bit, int mode,
                                 int32_t *flags) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t w = blockIdx.y;
    int f = 0;
    if (n < N) {
        uint64_t word = 0;
#pragma unroll 16
        for (int b = 0; b < 64; ++b) {
            int64_t k = w * 64 + b;
            uint64_t bit;
            if (k < K) {
                float v = __ldg(x + k * ldx + n);
                f |= elem_flags(v, mode);
                bit = sign_bit(v);
            } else {
                bit = (uint64_t)pad_bit;
            }
            word |= bit << b;
        }
        out[w * ldo + n] = word;
    }
    flush_flags(f, flags);
}

// ---------------------------------------------------------------- pack NCHW
// x [B, C, H, W] -> out [B*H*W, Cw] u64 (NHWC words, channel tail 0).
// CTA = (128 pixels, one 64-channel word, image b), 256 threads.
//  1. fully coalesced loads: each warp instruction reads 512 contiguous bytes
//     (one channel, 128 pixels); 8 x 16 B per thread in flight, no L1 alloc;
//     staged in a 64 x 128 f32 SMEM tile whose 16-byte units are XOR-swizzled
//     by (channel & 7), so both the row writes and the column reads below are
//     bank-conflict free.
//  2. transpose by ballot: lane l reads 4 pixels of channel 32h + l
//     (ld.shared.v4) and one __ballot_sync per pixel yields that pixel's u32
//     channel word -- 32 elements per VOTE instruction.
// Finiteness: per float4, an overflow-free FFMA sum of |x|/4 propagates NaN/Inf.
constexpr int kPackPix = 128;
template <bool kVec4, bool kStrict>
__global__ void __launch_bounds__(256) pack_nchw_kernel(const float *__restrict__ x, int64_t B,
                                                        int64_t C, int64_t HW, int64_t Cw,
                                                        uint32_t *__restrict__ out32,
                                                        int32_t *flags) {
    __shared__ __align__(16) float tile[64 * kPackPix];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * kPackPix;
    const int64_t cw = blockIdx.y, b = blockIdx.z;
    const int nc = (int)(C - cw * 64 < 64 ? C - cw * 64 : 64);
    const float *src = x + (b * C + cw * 64) * HW + p0;
    int f = 0;
    const bool full = kVec4 && nc == 64 && p0 + kPackPix <= HW;
    float4 q[8];
    if (full) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + 256 * i;  // 2048 float4 = 64 channels x 32 quads
            const float *pp = src + (e >> 5) * HW + 4 * (e & 31);
            asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(q[i].x), "=f"(q[i].y), "=f"(q[i].z), "=f"(q[i].w)
                         : "l"(pp));
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + 256 * i;
            const int c = e >> 5, p = 4 * (e & 31);
            float t[4] = {-1.f, -1.f, -1.f, -1.f};  // absent channels / pixels: bit 0
            if (c < nc)
                for (int j = 0; j < 4; ++j)
                    if (p0 + p + j < HW) t[j] = __ldg(src + c * HW + p + j);
            q[i] = make_float4(t[0], t[1], t[2], t[3]);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = tid + 256 * i;
        const int c = e >> 5, unit = e & 31;
        const float sum = fmaf(fabsf(q[i].x), 0.25f, fmaf(fabsf(q[i].y), 0.25f,
                          fmaf(fabsf(q[i].z), 0.25f, fabsf(q[i].w) * 0.25f)));
        if (!(sum <= 3.402823466e38f)) f |= BNN_FLAG_NONFINITE;
        if (kStrict && c < nc) {
            const float tv[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (p0 + 4 * unit + j < HW && tv[j] != 1.0f && tv[j] != -1.0f)
                    f |= BNN_FLAG_NOTSIGN;
        }
        *reinterpret_cast<float4 *>(&tile[c * kPackPix + 4 * (unit ^ (c & 7))]) = q[i];
    }
    __syncthreads();
    // 64 items = (2 channel halves) x (32 pixel quads); 8 per warp
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        const int item = warp * 8 + it;
        const int h = item & 1, quad = item >> 1;
        const int c = 32 * h + lane;
        const float4 t = *reinterpret_cast<const float4 *>(&tile[c * kPackPix + 4 * (quad ^ (c & 7))]);
        const bool ok = c < nc;
        const uint32_t w0 = __ballot_sync(0xffffffffu, ok && t.x >= 0.0f);  // sign(-0) = +1
        const uint32_t w1 = __ballot_sync(0xffffffffu, ok && t.y >= 0.0f);
        const uint32_t w2 = __ballot_sync(0xffffffffu, ok && t.z >= 0.0f);
        const uint32_t w3 = __ballot_sync(0xffffffffu, ok && t.w >= 0.0f);
        if (lane < 4) {
            const int64_t p = p0 + 4 * quad + lane;
            const uint32_t w = lane == 0 ? w0 : lane == 1 ? w1 : lane == 2 ? w2 : w3;
            if (p < HW) out32[(b * HW + p) * (2 * Cw) + 2 * cw + h] = w;
        }
    }
    flush_flags(f, flags);
}

// ---------------------------------------------------------------- transpose
__global__ void words_transpose_kernel(const uint64_t *__restrict__ in, int64_t rows,
                                       int64_t cols, int64_t ldi, uint64_t *__restrict__ out,
                                       int64_t ldo) {
    __shared__ uint64_t tile[32][33];
    const int64_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * ldi + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * ldo + r] = tile[threadIdx.x][i];
    }
}

// ---------------------------------------------------------------- audit
__global__ void audit_padding_kernel(const uint64_t *__restrict__ words, int64_t vectors,
                                     int64_t last_off, int64_t ld_vec, uint64_t mask,
                                     uint64_t expect, int32_t *bad) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int f = 0;
    if (v < vectors) f = ((words[v * ld_vec + last_off] & mask) != expect) ? 1 : 0;
    if (__any_sync(0xffffffffu, f) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// ---------------------------------------------------------------- conv weights
// w_ref: [F, ceil(C*kh*kw/64)] with bit (c*kh + i)*kw + j  (layers.py:221)
// w_dev: [F, kh*kw, Cw] with bit c%64 of word (i*kw + j)*Cw + c/64
__global__ void conv_weights_reorder_kernel(const uint64_t *__restrict__ w_ref, int64_t F,
                                            int64_t C, int64_t kh, int64_t kw, int64_t Cw,
                                            uint64_t *__restrict__ w_dev) {
    const int64_t per_f = kh * kw * Cw;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= F * per_f) return;
    const int64_t f = idx / per_f, r = idx % per_f;
    const int64_t tap = r / Cw, cw = r % Cw;
    const int64_t i = tap / kw, j = tap % kw;
    const int64_t wref = ceil_div(C * kh * kw, 64);
    const uint64_t *src = w_ref + f * wref;
    uint64_t word = 0;
    for (int b = 0; b < 64; ++b) {
        int64_t c = cw * 64 + b;
        if (c >= C) break;
        int64_t bit = (c * kh + i) * kw + j;
        word |= ((src[bit >> 6] >> (bit & 63)) & 1ull) << b;
    }
    w_dev[idx] = word;
}

// ---------------------------------------------------------------- pack NCHW (TMA)
// Streaming variant for HW % 4 == 0: CTA = (image b, 32-channel group g,
// pixel chunk).  One elected thread issues 32 cp.async.bulk copies (one
// contiguous channel segment each, TMA engine, mbarrier complete_tx) into a
// SMEM tile whose row pitch is chosen so lane l's 16-byte column reads fall in
// distinct bank quads; then each warp transposes 4 pixels per ld.shared.v4
// with four __ballot_sync (32 channels -> one u32 word per pixel).
constexpr int kTmaPixMax = 1024;  // pixels per CTA chunk (<= 132 KB of SMEM)
__device__ __forceinline__ int tma_pitch(int npix) { return ((npix + 31) & ~31) + 4; }

template <bool kStrict>
__global__ void __launch_bounds__(256) pack_nchw_tma_kernel(const float *__restrict__ x,
                                                            int64_t C, int64_t HW, int64_t Cw,
                                                            uint32_t *__restrict__ out32,
                                                            int32_t *flags) {
    extern __shared__ __align__(128) float tile_t[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t g = blockIdx.y, b = blockIdx.z;
    const int64_t p0 = (int64_t)blockIdx.x * kTmaPixMax;
    const int npix = (int)(HW - p0 < kTmaPixMax ? HW - p0 : kTmaPixMax);
    const int pitch = tma_pitch(npix);
    const int nc = (int)(C - g * 32 < 32 ? C - g * 32 : 32);
    const uint32_t sbar = smem_u32_pack(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t bytes = (uint32_t)npix * 4u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sbar),
                     "r"(bytes * (uint32_t)nc)
                     : "memory");
        for (int c = 0; c < nc; ++c) {
            const float *src = x + (b * C + g * 32 + c) * HW + p0;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                "[%3];\n" ::"r"(smem_u32_pack(tile_t + c * pitch)),
                "l"(src), "r"(bytes), "r"(sbar)
                : "memory");
        }
    }
    // wait for the tile (phase 0)
    {
        uint32_t done = 0;
        do {
            asm volatile(
                "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                "selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(sbar)
                : "memory");
        } while (!done);
    }
    int f = 0;
    const bool cok = lane < nc;
    const int nquads = (npix + 3) >> 2;
    for (int qd = warp; qd < nquads; qd += 8) {
        float4 t = make_float4(-1.f, -1.f, -1.f, -1.f);
        if (cok) t = *reinterpret_cast<const float4 *>(tile_t + lane * pitch + 4 * qd);
        const float tv[4] = {t.x, t.y, t.z, t.w};
        const int left = npix - 4 * qd;  // valid pixels in this quad (>= 1)
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float a = (j < left && cok) ? tv[j] : 0.f;
            sum = fmaf(fabsf(a), 0.25f, sum);
            if (kStrict && j < left && cok && a != 1.0f && a != -1.0f) f |= BNN_FLAG_NOTSIGN;
        }
        if (!(sum <= 3.402823466e38f)) f |= BNN_FLAG_NONFINITE;
        const uint32_t w0 = __ballot_sync(0xffffffffu, cok && t.x >= 0.0f);  // sign(-0) = +1
        const uint32_t w1 = __ballot_sync(0xffffffffu, cok && t.y >= 0.0f);
        const uint32_t w2 = __ballot_sync(0xffffffffu, cok && t.z >= 0.0f);
        const uint32_t w3 = __ballot_sync(0xffffffffu, cok && t.w >= 0.0f);
        if (lane < 4 && lane < left) {
            const int64_t p = p0 + 4 * qd + lane;
            const uint32_t w = lane == 0 ? w0 : lane == 1 ? w1 : lane == 2 ? w2 : w3;
            out32[(b * HW + p) * (2 * Cw) + g] = w;
        }
    }
    flush_flags(f, flags);
}

// ================================================================ launchers
int launch_binarize(const float *x, int64_t n, float *out, int32_t *flags, cudaStream_t s) {
    if (n == 0) return BNN_OK;
    int blocks = (int)(ceil_div(n, 256) < 148 * 16 ? ceil_div(n, 256) : 148 * 16);
    binarize_kernel<<<blocks, 256, 0, s>>>(x, n, out, flags);
    return check_launch("binarize_kernel");
}

int launch_pack_rows(const float *x, int64_t R, int64_t K, int64_t ldx, uint64_t *out,
                     int64_t ldo, int pad_bit, int mode, int32_t *row_popc, int32_t *flags,
                     cudaStream_t s) {
    if (R == 0 || K == 0) return BNN_OK;
    const int64_t blocks = ceil_div(R * 32, 256);
    const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    if (vec)
        pack_rows_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(x, R, K, ldx, out, ldo, pad_bit,
                                                               mode, row_popc, flags);
    else
        pack_rows_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(x, R, K, ldx, out, ldo, pad_bit,
                                                                mode, row_popc, flags);
    return check_launch("pack_rows_kernel");
}

int launch_pack_cols(const float *x, int64_t K, int64_t N, int64_t ldx, uint64_t *out,
                     int64_t ldo, int pad_bit, int mode, int32_t *flags, cudaStream_t s) {
    if (K == 0 || N == 0) return BNN_OK;
    dim3 grid((unsigned)ceil_div(N, 256), (unsigned)ceil_div(K, 64));
    pack_cols_kernel<<<grid, 256, 0, s>>>(x, K, N, ldx, out, ldo, pad_bit, mode, flags);
    return check_launch("pack_cols_kernel");
}

int launch_pack_nchw(const float *x, int64_t B, int64_t C, int64_t H, int64_t W, uint64_t *out,
                     int mode, int32_t *flags, cudaStream_t s) {
    const int64_t HW = H * W, Cw = ceil_div(C, 64);
    if (B == 0 || HW == 0 || C == 0) return BNN_OK;
    uint32_t *o32 = reinterpret_cast<uint32_t *>(out);
    const bool strict = mode == BNN_PACK_STRICT;
    const bool aligned = (HW % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    if (aligned) {
        // TMA streaming path: 32-channel groups, contiguous bulk copies
        const int chunk = (int)(HW < kTmaPixMax ? HW : kTmaPixMax);
        const int pitch = ((chunk + 31) & ~31) + 4;
        const int smem = 32 * pitch * 4;
        dim3 grid((unsigned)ceil_div(HW, kTmaPixMax), (unsigned)ceil_div(C, 32), (unsigned)B);
        if (strict) {
            static bool cfg = false;
            if (!cfg) cudaFuncSetAttribute(pack_nchw_tma_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * (kTmaPixMax + 4) * 4), cfg = true;
            pack_nchw_tma_kernel<true><<<grid, 256, smem, s>>>(x, C, HW, Cw, o32, flags);
        } else {
            static bool cfg = false;
            if (!cfg) cudaFuncSetAttribute(pack_nchw_tma_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * (kTmaPixMax + 4) * 4), cfg = true;
            pack_nchw_tma_kernel<false><<<grid, 256, smem, s>>>(x, C, HW, Cw, o32, flags);
        }
        // channel-tail words of odd 32-groups (C % 64 in (0, 32]) must read 0
        if (ceil_div(C, 32) % 2 == 1) {
            cudaMemset2DAsync(o32 + 2 * Cw - 1, 2 * Cw * 4, 0, 4, (size_t)(B * HW), s);
        }
        return check_launch("pack_nchw_tma_kernel");
    }
    dim3 grid((unsigned)ceil_div(HW, kPackPix), (unsigned)Cw, (unsigned)B);
    if (strict)
        pack_nchw_kernel<false, true><<<grid, 256, 0, s>>>(x, B, C, HW, Cw, o32, flags);
    else
        pack_nchw_kernel<false, false><<<grid, 256, 0, s>>>(x, B, C, HW, Cw, o32, flags);
    return check_launch("pack_nchw_kernel");
}

int launch_words_transpose(const uint64_t *in, int64_t rows, int64_t cols, int64_t ldi,
                           uint64_t *out, int64_t ldo, cudaStream_t s) {
    if (rows == 0 || cols == 0) return BNN_OK;
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
    words_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, rows, cols, ldi, out, ldo);
    return check_launch("words_transpose_kernel");
}

int launch_audit_padding(const uint64_t *words, int64_t vectors, int64_t n_bits, int64_t ld_vec,
                         int64_t ld_word, int pad_fill, int32_t *bad, cudaStream_t s) {
    const int rem = (int)(n_bits % 64);
    if (rem == 0 || vectors == 0) return BNN_OK;
    const uint64_t mask = ~((1ull << rem) - 1ull);
    const uint64_t expect = pad_fill ? mask : 0ull;
    const int64_t last_off = (ceil_div(n_bits, 64) - 1) * ld_word;
    audit_padding_kernel<<<(unsigned)ceil_div(vectors, 256), 256, 0, s>>>(
        words, vectors, last_off, ld_vec, mask, expect, bad);
    return check_launch("audit_padding_kernel");
}

int launch_conv_weights_reorder(const uint64_t *w_ref, int64_t F, int64_t C, int64_t kh,
                                int64_t kw, uint64_t *w_dev, cudaStream_t s) {
    const int64_t Cw = ceil_div(C, 64);
    const int64_t total = F * kh * kw * Cw;
    if (total == 0) return BNN_OK;
    conv_weights_reorder_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, s>>>(w_ref, F, C, kh,
                                                                              kw, Cw, w_dev);
    return check_launch("conv_weights_reorder_kernel");
}

}  // namespace bnn
