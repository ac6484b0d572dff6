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
#include <cstdlib>

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
template <bool kVec4, int kIters>
__global__ void pack_rows_kernel(const float *__restrict__ x, int64_t R, int64_t K, int64_t ldx,
                                 uint64_t *__restrict__ out, int64_t ldo, int pad_bit, int mode,
                                 int32_t *flags, int64_t nseg) {
    // warp per (row, segment of kIters x 128 elements); every load of the segment is
    // issued before the first is consumed, so a warp keeps kIters x 512 B in flight
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t row = gw / nseg, seg = gw - row * nseg;
    if (row >= R) return;  // warp-uniform
    const float *xr = x + row * ldx;
    const int64_t W = ceil_div(K, 64);
    const int64_t base0 = seg * (128 * kIters);
    float v[kIters][4];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const int64_t e = base0 + 128 * it + 4 * lane;
        if (kVec4 && e + 3 < K) {
            const float4 q = __ldg(reinterpret_cast<const float4 *>(xr + e));
            v[it][0] = q.x; v[it][1] = q.y; v[it][2] = q.z; v[it][3] = q.w;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[it][i] = e + i < K ? __ldg(xr + e + i) : 0.0f;
        }
    }
    int f = 0;
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
        const int64_t base = base0 + 128 * it;
        if (base >= W * 64) break;  // warp-uniform
        const int64_t e = base + 4 * lane;
        uint32_t nib = 0, valid = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            bool in = e + i < K;
            uint32_t b = in ? sign_bit(v[it][i]) : (uint32_t)pad_bit;
            nib |= b << i;
            valid |= (in ? 1u : 0u) << i;
            if (in) f |= elem_flags(v[it][i], mode);
        }
        uint32_t w = nib << (4 * (lane & 7));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        uint32_t hi = __shfl_down_sync(0xffffffffu, w, 8);
        const int64_t wi = base / 64 + (lane >> 4);
        if ((lane & 15) == 0 && wi < W) out[row * ldo + wi] = (uint64_t)w | ((uint64_t)hi << 32);
    }
    flush_flags(f, flags);
}

// popcount of each packed row's K valid bits (tail bits past K masked off)
__global__ void row_popc_kernel(const uint64_t *__restrict__ words, int64_t R, int64_t W,
                                int64_t ldo, int64_t K, int32_t *__restrict__ row_popc) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= R) return;
    int popc = 0;
    for (int64_t w = lane; w < W; w += 32) {
        uint64_t v = words[row * ldo + w];
        const int64_t left = K - 64 * w;
        if (left < 64) v &= (1ull << left) - 1ull;
        popc += __popcll(v);
    }
    popc = __reduce_add_sync(0xffffffffu, popc);
    if (lane == 0) row_popc[row] = popc;
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
// CTA = (64 pixels of image b, all channels in chunks of 256), 256 threads.
//  1. cp.async 16-byte pieces (a warp covers two 256-byte channel rows per
//     instruction) into a 256 x 64 f32 SMEM tile whose 16-byte units are
//     XOR-swizzled by (channel & 7) -- conflict-free column reads below;
//  2. transpose by ballot: lane l reads 4 pixels of channel 32g + l
//     (ld.shared.v4) and one __ballot_sync per pixel yields that pixel's
//     32-channel u32 word (32 elements per VOTE);
//  3. the words are collected in SMEM and written as one contiguous
//     64 x (Cw u64) block with 16-byte stores (scattered 4-byte stores of the
//     words themselves made the previous versions L2-transaction bound).
// Finiteness: per float4, an overflow-free FFMA sum of |x|/4 propagates NaN/Inf.
template <int kPackPix, bool kVec4, bool kStrict>
__global__ void __launch_bounds__(256) pack_nchw_kernel(const float *__restrict__ x, int64_t B,
                                                        int64_t C, int64_t HW, int64_t Cw,
                                                        uint32_t *__restrict__ out32,
                                                        int32_t *flags) {
    constexpr int kPackChunkC = 16384 / kPackPix;  // 64 KB of f32 per pass
    constexpr int kUnits = kPackPix / 4;           // 16-byte units per channel row
    extern __shared__ __align__(128) uint8_t pk_smem[];
    float *tile = reinterpret_cast<float *>(pk_smem);                       // [chunkC][pix]
    uint32_t *words = reinterpret_cast<uint32_t *>(pk_smem + kPackChunkC * kPackPix * 4);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t p0 = (int64_t)blockIdx.x * kPackPix;
    const int64_t b = blockIdx.y;
    const int npix = (int)(HW - p0 < kPackPix ? HW - p0 : kPackPix);
    const int nw32 = (int)(2 * Cw);  // u32 words per pixel
    int f = 0;
    for (int64_t c0 = 0; c0 < C; c0 += kPackChunkC) {
        const int nc = (int)(C - c0 < kPackChunkC ? C - c0 : kPackChunkC);
        const float *src = x + (b * C + c0) * HW + p0;
        // kPackChunkC channels x kUnits units of 16 B = 4096 pieces, 16 per thread
#pragma unroll 4
        for (int i = 0; i < 16; ++i) {
            const int e = tid + 256 * i;
            const int c = e / kUnits, u = e % kUnits;
            const uint32_t dst = smem_u32_pack(tile + c * kPackPix + 4 * (u ^ (c & 7)));
            if (kVec4) {
                const int valid = (c < nc) ? (npix - 4 * u) : 0;
                const int bytes = valid >= 4 ? 16 : (valid > 0 ? 4 * valid : 0);
                const float *sp = bytes ? src + c * HW + 4 * u : x;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst),
                             "l"(sp), "r"(bytes));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool ok = c < nc && 4 * u + j < npix;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst + 4 * j),
                                 "l"(ok ? src + c * HW + 4 * u + j : x), "r"(ok ? 4 : 0));
                }
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        // transpose: items = kUnits pixel quads x (nc / 32) channel groups, 8 warps
        const int ngroups = (nc + 31) >> 5;
        const uint32_t tile_s = smem_u32_pack(tile), words_s = smem_u32_pack(words);
        const int gbase = (int)(c0 >> 5);
        for (int item = warp; item < kUnits * ngroups; item += 8) {
            const int q4 = item % kUnits, g = item / kUnits;
            const int c = 32 * g + lane;
            const bool cok = c < nc;
            float4 t;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                         : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                         : "r"(tile_s + (uint32_t)(c * kPackPix + 4 * (q4 ^ (c & 7))) * 4u));
            // zero-filled tails are finite, so no per-element validity test is needed
            const float sum = fmaf(fabsf(t.x), 0.25f, fmaf(fabsf(t.y), 0.25f,
                              fmaf(fabsf(t.z), 0.25f, fabsf(t.w) * 0.25f)));
            f |= (cok && !(sum <= 3.402823466e38f)) ? BNN_FLAG_NONFINITE : 0;
            if (kStrict && cok) {
                const int left = npix - 4 * q4;
                const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < left && tv[j] != 1.0f && tv[j] != -1.0f) f |= BNN_FLAG_NOTSIGN;
            }
            const uint32_t w0 = __ballot_sync(0xffffffffu, cok && t.x >= 0.0f);  // sign(-0) = +1
            const uint32_t w1 = __ballot_sync(0xffffffffu, cok && t.y >= 0.0f);
            const uint32_t w2 = __ballot_sync(0xffffffffu, cok && t.z >= 0.0f);
            const uint32_t w3 = __ballot_sync(0xffffffffu, cok && t.w >= 0.0f);
            const uint32_t w = (lane & 2) ? ((lane & 1) ? w3 : w2) : ((lane & 1) ? w1 : w0);
            if (lane < 4)
                asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(
                                 words_s + (uint32_t)((4 * q4 + lane) * nw32 + gbase + g) * 4u),
                             "r"(w));
        }
        __syncthreads();  // tile reuse by the next channel chunk
    }
    // channel-tail u32 words past ceil(C/32) (odd group count) are zero
    for (int i = tid; i < kPackPix; i += 256)
        for (int g = (int)((C + 31) >> 5); g < nw32; ++g) words[i * nw32 + g] = 0;  // tail halves
    __syncthreads();
    // contiguous write-out: npix pixels x nw32 u32 words
    uint32_t *dst = out32 + (b * HW + p0) * nw32;
    const int total = npix * nw32;
    if (((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && (total & 3) == 0) {
        for (int i = tid; i < total / 4; i += 256)
            reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(words)[i];
    } else {
        for (int i = tid; i < total; i += 256) dst[i] = words[i];
    }
    flush_flags(f, flags);
}

// Direct NCHW -> packed NHWC: thread per (pixel, 64-channel word).  The 64
// channel loads of a thread are independent and unrolled, and the 32 lanes of a
// warp are 32 consecutive pixels, so every load instruction is one coalesced
// 128-byte row segment and a warp keeps 64 x 128 B in flight -- the HBM-bound
// shape of this pass (4 B read per 1/8 B written) with no shared memory and no
// block barrier.  Channel tails (C % 64) are 0 bits, like the tiled kernel.
template <bool kStrict>
__global__ void __launch_bounds__(256) pack_nchw_direct_kernel(const float *__restrict__ x,
                                                                 int64_t B, int64_t C, int64_t HW,
                                                                 int64_t Cw,
                                                                 uint64_t *__restrict__ out,
                                                                 int32_t *flags) {
    const int64_t gp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // global pixel
    const int64_t cw = blockIdx.y;                                      // 64-channel word
    int f = 0;
    if (gp < B * HW) {
        const int64_t b = gp / HW, p = gp - b * HW;
        const int64_t c0 = cw * 64;
        const int nc = (int)(C - c0 < 64 ? C - c0 : 64);
        const float *src = x + (b * C + c0) * HW + p;
        uint32_t half[2] = {0u, 0u};
        float nf = 0.0f;  // + v * 0 for every element: NaN iff some element is not finite
        if (nc == 64) {
            float v[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] = __ldg(src + (int64_t)j * HW);
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                // bit = v >= 0 (sign(-0) = +1): the u32 image is > 0x80000000 only for
                // negative values other than -0 (and negative NaNs, flagged below)
                if (!(__float_as_uint(v[j]) > 0x80000000u)) half[j >> 5] |= 1u << (j & 31);
                nf = __fmaf_rn(v[j], 0.0f, nf);
                if (kStrict && v[j] != 1.0f && v[j] != -1.0f) f |= BNN_FLAG_NOTSIGN;
            }
        } else {
            for (int j = 0; j < nc; ++j) {  // channel tail word: bits past C stay 0
                const float v = __ldg(src + (int64_t)j * HW);
                if (!(__float_as_uint(v) > 0x80000000u)) half[j >> 5] |= 1u << (j & 31);
                nf = __fmaf_rn(v, 0.0f, nf);
                if (kStrict && v != 1.0f && v != -1.0f) f |= BNN_FLAG_NOTSIGN;
            }
        }
        if (nf != 0.0f) f |= BNN_FLAG_NONFINITE;
        out[gp * Cw + cw] = (uint64_t)half[0] | ((uint64_t)half[1] << 32);
    }
    flush_flags(f, flags);
}

// NCHW -> packed NHWC for H*W % 4 == 0: a group of G = 32 / kCh adjacent lanes
// owns one (4-pixel quad, 32-channel u32 word); each lane loads kCh channel rows
// of the quad (16-byte loads, all issued before any is consumed) and the group
// ORs its partial words with shuffles.  Many small independent loads per SM keep
// HBM busy (the pass is 4 B read per 1/8 B written), at ~3 ALU ops per element.
template <bool kStrict, int kCh>
__global__ void __launch_bounds__(256) pack_nchw_quad_kernel(const float *__restrict__ x,
                                                               int64_t B, int64_t C, int64_t HW,
                                                               int64_t cs32,
                                                               uint32_t *__restrict__ out32,
                                                               int32_t *flags) {
    constexpr int G = 32 / kCh;
    // let a programmatic-dependent consumer (the conv kernel) launch and run its setup
    // while this pass finishes; it waits for our results in griddepcontrol.wait
    asm volatile("griddepcontrol.launch_dependents;\n");
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int sub = (int)(t % G);
    const int64_t gq = t / G;          // pixel quad
    const int64_t wi = blockIdx.y;     // u32 word in pixel
    int f = 0;
    uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
    const bool ok = gq * 4 < B * HW;
    const int64_t gp = gq * 4;
    if (ok) {
        const int64_t b = gp / HW, p = gp - b * HW;
        const int64_t c0 = wi * 32 + sub * kCh;
        const int nc = (int)(C - c0 < kCh ? (C - c0 > 0 ? C - c0 : 0) : kCh);
        const float *src = x + (b * C + c0) * HW + p;
        float nf = 0.0f;  // + v * 0 over every element: NaN iff one is not finite
        float4 v[kCh];
#pragma unroll
        for (int j = 0; j < kCh; ++j)
            v[j] = j < nc ? __ldg(reinterpret_cast<const float4 *>(src + (int64_t)j * HW))
                          : make_float4(-1.0f, -1.0f, -1.0f, -1.0f);
#pragma unroll
        for (int j = 0; j < kCh; ++j) {
            // bit = v >= 0 (sign(-0) = +1): u32 image > 0x80000000 only for values < 0;
            // channels past C were loaded as -1 -> 0 bits
            const int sh = sub * kCh + j;
            w0 |= (__float_as_uint(v[j].x) > 0x80000000u ? 0u : 1u) << sh;
            w1 |= (__float_as_uint(v[j].y) > 0x80000000u ? 0u : 1u) << sh;
            w2 |= (__float_as_uint(v[j].z) > 0x80000000u ? 0u : 1u) << sh;
            w3 |= (__float_as_uint(v[j].w) > 0x80000000u ? 0u : 1u) << sh;
            nf = __fmaf_rn(v[j].x, 0.0f, __fmaf_rn(v[j].y, 0.0f, nf));
            nf = __fmaf_rn(v[j].z, 0.0f, __fmaf_rn(v[j].w, 0.0f, nf));
            if (kStrict && j < nc) {
                const float tv[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (tv[i] != 1.0f && tv[i] != -1.0f) f |= BNN_FLAG_NOTSIGN;
            }
        }
        if (nf != 0.0f) f |= BNN_FLAG_NONFINITE;
    }
#pragma unroll
    for (int m = 1; m < G; m <<= 1) {  // OR the group's channel sub-blocks
        w0 |= __shfl_xor_sync(0xffffffffu, w0, m);
        w1 |= __shfl_xor_sync(0xffffffffu, w1, m);
        w2 |= __shfl_xor_sync(0xffffffffu, w2, m);
        w3 |= __shfl_xor_sync(0xffffffffu, w3, m);
    }
    if (ok && sub == 0) {
        uint32_t *o = out32 + gp * cs32 + wi;
        o[0] = w0;
        o[cs32] = w1;
        o[2 * cs32] = w2;
        o[3 * cs32] = w3;
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

// ---------------------------------------------------------------- pack planes
// k-bit quantize + bit-plane pack (multi-bit act_bit / weight_bit):
// x [R, K] f32 -> planes[p][R][ldo] u64, plane p holding bit p of each code.
// Codes follow the reference's float32 op order exactly (qmath.py:44-84, no
// FMA contraction): unsigned grid  code = floor(x * L + 0.5), x in [0, 1];
// signed grid  code = floor((0.5 * clip(x, -1, 1) + 0.5) * L + 0.5).
template <int kBits>
__global__ void pack_planes_kernel(const float *__restrict__ x, int64_t R, int64_t K, int64_t ldx,
                                   int grid_signed, uint64_t *__restrict__ out, int64_t ldo,
                                   int64_t plane_stride, int32_t *flags) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= R) return;  // warp-uniform
    const float L = (float)((1 << kBits) - 1);
    const float *xr = x + row * ldx;
    const int64_t W = ceil_div(K, 64);
    int f = 0;
    for (int64_t base = 0; base < W * 64; base += 128) {
        const int64_t e = base + 4 * lane;
        uint32_t nib[kBits];
#pragma unroll
        for (int p = 0; p < kBits; ++p) nib[p] = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (e + i < K) {
                const float v = __ldg(xr + e + i);
                if (!isfinite(v)) f |= BNN_FLAG_NONFINITE;
                float y;
                if (grid_signed) {
                    const float c = fminf(fmaxf(v, -1.0f), 1.0f);
                    y = __fadd_rn(__fmul_rn(0.5f, c), 0.5f);
                } else {
                    if (v < 0.0f || v > 1.0f) f |= BNN_FLAG_RANGE;
                    y = v;
                }
                const uint32_t code = (uint32_t)floorf(__fadd_rn(__fmul_rn(y, L), 0.5f));
#pragma unroll
                for (int p = 0; p < kBits; ++p) nib[p] |= ((code >> p) & 1u) << i;
            }
        }
        const int64_t wi = base / 64 + (lane >> 4);
#pragma unroll
        for (int p = 0; p < kBits; ++p) {
            uint32_t w = nib[p] << (4 * (lane & 7));
            w |= __shfl_xor_sync(0xffffffffu, w, 1);
            w |= __shfl_xor_sync(0xffffffffu, w, 2);
            w |= __shfl_xor_sync(0xffffffffu, w, 4);
            const uint32_t hi = __shfl_down_sync(0xffffffffu, w, 8);
            if ((lane & 15) == 0 && wi < W)
                out[p * plane_stride + row * ldo + wi] = (uint64_t)w | ((uint64_t)hi << 32);
        }
    }
    flush_flags(f, flags);
}

// ---------------------------------------------------------------- BN + ReLU + maxpool
// Fused float post-op of a full-precision stem (ResNet-18 configs[3]):
// y = maxpool_kxk/s/p(relu(gamma * ((x - mean) * inv_std) + beta)), NCHW f32.
// Every op is the reference's float32 op (layers.py:598-602, each rounded, no
// FMA), so the result is bit-identical to the unfused torch / NumPy sequence.
// One thread per output element; the k*k window reads hit L1/L2.
__global__ void bn_relu_maxpool_kernel(const float *__restrict__ x, int64_t B, int64_t C,
                                       int64_t H, int64_t W, const float *__restrict__ mean,
                                       const float *__restrict__ inv, const float *__restrict__ gamma,
                                       const float *__restrict__ beta, int relu, int k, int st,
                                       int pd, int64_t OH, int64_t OW, float *__restrict__ y,
                                       int bpp) {
    // bpp blocks per (image, channel) plane; 32-bit index math inside the plane
    const int64_t plane = blockIdx.x / bpp;
    const int c = (int)(plane % C);
    const int p = (int)(blockIdx.x - plane * bpp) * blockDim.x + threadIdx.x;
    const int oh = (int)OH, ow = (int)OW, h = (int)H, w = (int)W;
    if (p >= oh * ow) return;
    const int oy = p / ow, ox = p - (p / ow) * ow;
    const float m = __ldg(mean + c), iv = __ldg(inv + c), g = __ldg(gamma + c), bt = __ldg(beta + c);
    const float *src = x + plane * H * W;
    float best = -INFINITY;
    for (int i = 0; i < k; ++i) {
        const int iy = oy * st - pd + i;
        if (iy < 0 || iy >= h) continue;
        for (int j = 0; j < k; ++j) {
            const int ix = ox * st - pd + j;
            if (ix < 0 || ix >= w) continue;
            float v = __ldg(src + iy * w + ix);
            v = __fadd_rn(__fmul_rn(g, __fmul_rn(__fsub_rn(v, m), iv)), bt);
            if (relu) v = fmaxf(v, 0.0f);
            best = fmaxf(best, v);
        }
    }
    y[plane * OH * OW + p] = best;
}

// Banded variant of the same post-op (the product path for the ResNet stem):
// one CTA per (plane, band of R output rows) stages the band's input rows in
// SMEM with coalesced loads, pools first and applies BatchNorm + ReLU once per
// output.  Exact: f(v) = relu?(bt + g * ((v - m) * iv)) with every op rounded is
// monotone non-decreasing in v for g >= 0 and non-increasing for g < 0 (iv > 0),
// so max over the window of f(v) = f(max v) (g >= 0) or f(min v) (g < 0) --
// bit-identical to applying f to every element first.  Out-of-image window
// positions are skipped (-inf padding of maxpool).
__global__ void bn_relu_maxpool_band_kernel(const float *__restrict__ x, int C, int H, int W,
                                            const float *__restrict__ mean,
                                            const float *__restrict__ inv,
                                            const float *__restrict__ gamma,
                                            const float *__restrict__ beta, int relu, int k,
                                            int st, int pd, int OH, int OW, int R, int nbands,
                                            float *__restrict__ y) {
    extern __shared__ float band[];
    const int64_t plane = blockIdx.x / nbands;
    const int c = (int)(plane % C);
    const int r0 = (int)(blockIdx.x - plane * nbands) * R;
    const int rows = min(R, OH - r0);
    const int iy0 = r0 * st - pd;
    const int nrows = (rows - 1) * st + k;
    const float *src = x + plane * H * W;
    // stage input rows iy0 .. iy0 + nrows - 1 (rows outside the image are skipped later)
    const bool vec = (W % 4 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    if (vec) {
        const int w4 = W / 4;
        for (int i = threadIdx.x; i < nrows * w4; i += blockDim.x) {
            const int r = i / w4, j = i - r * w4, iy = iy0 + r;
            if (iy >= 0 && iy < H)
                reinterpret_cast<float4 *>(band)[i] =
                    __ldcs(reinterpret_cast<const float4 *>(src + (int64_t)iy * W) + j);
        }
    } else {
        for (int i = threadIdx.x; i < nrows * W; i += blockDim.x) {
            const int r = i / W, j = i - r * W, iy = iy0 + r;
            if (iy >= 0 && iy < H) band[i] = __ldcs(src + (int64_t)iy * W + j);
        }
    }
    __syncthreads();
    const float m = __ldg(mean + c), iv = __ldg(inv + c), g = __ldg(gamma + c), bt = __ldg(beta + c);
    const bool up = !(g < 0.0f);
    float *dst = y + plane * OH * OW + (int64_t)r0 * OW;
    for (int o = threadIdx.x; o < rows * OW; o += blockDim.x) {
        const int oy = o / OW, ox = o - oy * OW;
        float hi = -INFINITY, lo = INFINITY;
        for (int i = 0; i < k; ++i) {
            const int iy = (r0 + oy) * st - pd + i;
            if (iy < 0 || iy >= H) continue;
            const float *row = band + (oy * st + i) * W;
            for (int j = 0; j < k; ++j) {
                const int ix = ox * st - pd + j;
                if (ix < 0 || ix >= W) continue;
                const float v = row[ix];
                hi = fmaxf(hi, v);
                lo = fminf(lo, v);
            }
        }
        float v = up ? hi : lo;
        v = __fadd_rn(__fmul_rn(g, __fmul_rn(__fsub_rn(v, m), iv)), bt);
        if (relu) v = fmaxf(v, 0.0f);
        dst[o] = v;
    }
}

// Max pooling of sign-packed NHWC words (no padding): out = OR of the window's
// words.  sign(max(v)) = OR(sign(v_i)) for the predicate v >= 0, so this equals
// packing the max-pooled f32 tensor.  One thread per output word.
__global__ void maxpool_packed_kernel(const uint64_t *__restrict__ in, int64_t H, int64_t W,
                                      int64_t Cw, int k, int st, int64_t OH, int64_t OW,
                                      int64_t total, uint64_t *__restrict__ out,
                                      int64_t out_bstride) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int64_t cw = i % Cw, p = i / Cw;
    const int64_t ox = p % OW, oy = (p / OW) % OH, b = p / (OW * OH);
    const uint64_t *src = in + ((b * H + oy * st) * W + ox * st) * Cw + cw;
    uint64_t v = 0;
    for (int r = 0; r < k; ++r)
        for (int c = 0; c < k; ++c) v |= __ldg(src + ((int64_t)r * W + c) * Cw);
    // (out_bstride: words between images; a consumer GEMM wants 16-byte aligned rows)
    out[b * out_bstride + (i - b * OH * OW * Cw)] = v;
}

// Shortcut add + sign-pack: y = a + r (f32, the block output, same rounding as
// torch) and the packed NHWC sign words of y for the next block's convs.  One
// thread per (pixel, 32-channel word); the warp's threads are consecutive pixels,
// so every channel plane is read and written in 128-byte runs.
// (a and y may alias: the networks add in place; every element is read before the
// same thread writes it, so no __restrict__ on them)
__global__ void add_pack_nchw_kernel(const float *a, const float *__restrict__ r,
                                     int64_t B, int64_t C, int64_t HW, int64_t cs32,
                                     float *y, uint32_t *__restrict__ out32,
                                     int32_t *flags) {
    const int64_t gp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pixel over B * HW
    const int64_t wi = blockIdx.y;                                        // u32 word in pixel
    int f = 0;
    if (gp < B * HW) {
        const int64_t b = gp / HW, p = gp - b * HW, c0 = wi * 32;
        const int nc = (int)(C - c0 < 32 ? (C - c0 > 0 ? C - c0 : 0) : 32);
        const int64_t base = (b * C + c0) * HW + p;
        float va[32], vr[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            va[j] = j < nc ? __ldcs(a + base + (int64_t)j * HW) : -1.0f;
            vr[j] = j < nc ? __ldcs(r + base + (int64_t)j * HW) : 0.0f;
        }
        uint32_t w = 0;
        float nf = 0.0f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float v = __fadd_rn(va[j], vr[j]);
            if (j < nc) y[base + (int64_t)j * HW] = v;
            w |= (v >= 0.0f ? 1u : 0u) << j;  // sign(-0) = +1; channels past C: -1 -> 0
            nf = __fmaf_rn(v, 0.0f, nf);
        }
        if (nf != 0.0f) f |= BNN_FLAG_NONFINITE;
        out32[gp * cs32 + wi] = w;
    }
    flush_flags(f, flags);
}

// popcount64 (bitpack.py:49-52, hardware POPC) and popcount64_soft (:55-66, the
// shift/mask SWAR sequence with the same constants), one u64 word per thread
template <bool kSoft>
__global__ void popcount64_kernel(const uint64_t *__restrict__ w, int64_t n,
                                  uint8_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x = __ldg(w + i);
        if (kSoft) {
            x -= (x >> 1) & 0x5555555555555555ull;
            x = (x & 0x3333333333333333ull) + ((x >> 2) & 0x3333333333333333ull);
            x = (x + (x >> 4)) & 0x0F0F0F0F0F0F0F0Full;
            out[i] = (uint8_t)((x * 0x0101010101010101ull) >> 56);
        } else {
            out[i] = (uint8_t)__popcll(x);
        }
    }
}

// The classifier head of a network: y[b, o] = sum_c mean_hw(x[b, c]) * w[o, c] + bias[o]
// (GlobalAvgPool -> Dense, layers.py:266-317).  Every output is computed in one fixed
// order that depends only on its own image -- channel means summed over hw in order,
// then lane-strided partial dot products and a fixed shuffle tree -- so an image's
// logits are bit-identical whatever batch (or batch shard) it is computed in.
// Pass 1: one thread per (image, channel) mean.  Pass 2: a CTA per (8 images, 64
// outputs), pooled rows in SMEM, one warp per output row (W rows read coalesced).
__global__ void avgpool_kernel(const float *__restrict__ x, int64_t BC, int HW,
                               float *__restrict__ pooled) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= BC) return;
    const float *p = x + i * HW;
    float s = 0.0f;
    for (int t = 0; t < HW; ++t) s = __fadd_rn(s, __ldg(p + t));
    pooled[i] = __fdiv_rn(s, (float)HW);
}

// Pass 2: a CTA per (16 images, 64 outputs) tile; four groups of 64 threads each take a
// quarter of K (k tiles of 32 staged in SMEM row-major with a 33-float pitch: coalesced
// fills, conflict-free column reads), each thread a 4 x 4 register tile with a sequential
// FMA chain over its quarter; the four partial sums are added in the fixed order
// ((q0 + q1) + q2) + q3 -- the same order for every image, any batch.  (One group walking
// all of K took 35 us for 512 -> 1000 at batch 256: eight serial load-latency rounds.)
constexpr int kFcImg = 16, kFcOut = 64, kFcK = 32, kFcPitch = kFcK + 1, kFcGroups = 4;
__global__ void __launch_bounds__(64 * kFcGroups) fc_rows_kernel(const float *__restrict__ pooled, int B,
                                                                 int C, const float *__restrict__ w,
                                                                 const float *__restrict__ bias, int O,
                                                                 float *__restrict__ y) {
    __shared__ float sp_all[kFcGroups][kFcImg * kFcPitch];
    __shared__ float sw_all[kFcGroups][kFcOut * kFcPitch];
    const int b0 = blockIdx.x * kFcImg, o0 = blockIdx.y * kFcOut;
    const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
    const int og = t & 15, ig = t >> 4;  // outputs 4 og .. +3, images 4 ig .. +3
    float *sp = sp_all[grp], *sw = sw_all[grp];
    const int kq = (C + kFcGroups - 1) / kFcGroups;  // this group's K range [kb, ke)
    const int kb = grp * kq, ke = kb + kq < C ? kb + kq : C;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    // programmatic dependent launch: the first weight tile (a constant of the layer) is loaded
    // while the pooling kernel finishes; `pooled` is read after griddepcontrol.wait
    constexpr int kP = kFcImg * kFcK / 64, kW = kFcOut * kFcK / 64;
    float vw[kW];
    {
        const int kn = ke - kb < kFcK ? (ke - kb > 0 ? ke - kb : 0) : kFcK;
#pragma unroll
        for (int u = 0; u < kW; ++u) {
            const int i = t + 64 * u, r = i / kFcK, k = i - r * kFcK;
            vw[u] = (o0 + r < O && k < kn) ? __ldg(w + (int64_t)(o0 + r) * C + kb + k) : 0.0f;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;\n");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    for (int k0 = kb; k0 < kb + kq; k0 += kFcK) {  // (every group runs the same trip count: the barriers)
        const int kn = ke - k0 < kFcK ? (ke - k0 > 0 ? ke - k0 : 0) : kFcK;
        {   // all of a thread's tile loads in flight before its SMEM stores
            float vp[kP];
#pragma unroll
            for (int u = 0; u < kP; ++u) {
                const int i = t + 64 * u, r = i / kFcK, k = i - r * kFcK;
                vp[u] = (b0 + r < B && k < kn) ? __ldg(pooled + (int64_t)(b0 + r) * C + k0 + k) : 0.0f;
            }
            if (k0 != kb) {
#pragma unroll
                for (int u = 0; u < kW; ++u) {
                    const int i = t + 64 * u, r = i / kFcK, k = i - r * kFcK;
                    vw[u] = (o0 + r < O && k < kn) ? __ldg(w + (int64_t)(o0 + r) * C + k0 + k) : 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < kP; ++u) {
                const int i = t + 64 * u, r = i / kFcK, k = i - r * kFcK;
                sp[r * kFcPitch + k] = vp[u];
            }
#pragma unroll
            for (int u = 0; u < kW; ++u) {
                const int i = t + 64 * u, r = i / kFcK, k = i - r * kFcK;
                sw[r * kFcPitch + k] = vw[u];
            }
        }
        __syncthreads();
        for (int k = 0; k < kn; ++k) {
            float p4[4], w4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p4[i] = sp[(4 * ig + i) * kFcPitch + k];
#pragma unroll
            for (int j = 0; j < 4; ++j) w4[j] = sw[(4 * og + j) * kFcPitch + k];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(p4[i], w4[j], acc[i][j]);
        }
        __syncthreads();
    }
    // partial sums of groups 1..3 -> SMEM (the weight tiles are consumed), group 0 adds them in order
    float *red = &sw_all[0][0];  // [3][64 threads][16]
    if (grp > 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) red[((grp - 1) * 64 + t) * 16 + 4 * i + j] = acc[i][j];
    }
    __syncthreads();
    if (grp == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int bi = b0 + 4 * ig + i, o = o0 + 4 * og + j;
                float v = acc[i][j];
#pragma unroll
                for (int q = 0; q < kFcGroups - 1; ++q) v = __fadd_rn(v, red[(q * 64 + t) * 16 + 4 * i + j]);
                if (bi < B && o < O) {
                    if (bias) v = __fadd_rn(v, __ldg(bias + o));
                    y[(int64_t)bi * O + o] = v;
                }
            }
    }
}

// Pass 1: a CTA per 64 consecutive (image, channel) rows, staged in SMEM by coalesced
// 16-byte loads; each thread sums its row in order t = 0 .. HW-1, then / HW
__global__ void __launch_bounds__(128) avgpool_rows_kernel(const float *__restrict__ x, int64_t BC,
                                                           int HW, float *__restrict__ pooled) {
    extern __shared__ float rows[];  // [64][HW]
    // programmatic dependent launch: the classifier GEMM may start its weight loads now; x is
    // the previous kernel's output
    asm volatile("griddepcontrol.launch_dependents;\n");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const int64_t r0 = (int64_t)blockIdx.x * 64;
    const int nr = BC - r0 < 64 ? (int)(BC - r0) : 64;
    const float *src = x + r0 * HW;
    const int n = nr * HW;
    if (((reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int n4 = n >> 2;
        for (int i = threadIdx.x; i < n4; i += blockDim.x)
            reinterpret_cast<float4 *>(rows)[i] = __ldg(reinterpret_cast<const float4 *>(src) + i);
        for (int i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) rows[i] = __ldg(src + i);
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) rows[i] = __ldg(src + i);
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        const float *p = rows + threadIdx.x * HW;
        float s = 0.0f;
        for (int t = 0; t < HW; ++t) s = __fadd_rn(s, p[t]);
        pooled[r0 + threadIdx.x] = __fdiv_rn(s, (float)HW);
    }
}

// ================================================================ launchers
int launch_avgpool_fc(const float *x, int64_t B, int64_t C, int64_t HW, const float *w,
                      const float *bias, int64_t O, float *y, float *pooled, cudaStream_t s) {
    if (B == 0) return BNN_OK;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    if (HW <= 256) {  // (64 rows of HW floats staged in SMEM)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)ceil_div(B * C, 64));
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = (size_t)64 * HW * 4;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, avgpool_rows_kernel, x, B * C, (int)HW, pooled);
    } else {
        avgpool_kernel<<<(unsigned)ceil_div(B * C, 256), 256, 0, s>>>(x, B * C, (int)HW, pooled);
    }
    int rc = check_launch("avgpool_kernel");
    if (rc) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ceil_div(B, kFcImg), (unsigned)ceil_div(O, kFcOut));
    cfg.blockDim = dim3(64 * kFcGroups);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fc_rows_kernel, (const float *)pooled, (int)B, (int)C, w, bias, (int)O, y);
    return check_launch("fc_rows_kernel");
}
int launch_popcount64(const uint64_t *w, int64_t n, uint8_t *out, int soft, cudaStream_t s) {
    if (n == 0) return BNN_OK;
    const int64_t blocks = ceil_div(n, 256) < 4096 ? ceil_div(n, 256) : 4096;
    if (soft) popcount64_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(w, n, out);
    else popcount64_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(w, n, out);
    return check_launch("popcount64_kernel");
}
int launch_add_pack_nchw(const float *a, const float *r, int64_t B, int64_t C, int64_t H,
                         int64_t W, float *y, uint64_t *out, int32_t *flags, cudaStream_t s) {
    const int64_t HW = H * W, Cw = ceil_div(C, 64);
    if (B == 0 || HW == 0) return BNN_OK;
    dim3 g((unsigned)ceil_div(B * HW, 128), (unsigned)(2 * Cw));
    add_pack_nchw_kernel<<<g, 128, 0, s>>>(a, r, B, C, HW, 2 * Cw, y,
                                           reinterpret_cast<uint32_t *>(out), flags);
    return check_launch("add_pack_nchw_kernel");
}
int launch_maxpool_packed(const uint64_t *in, int64_t B, int64_t H, int64_t W, int64_t Cw, int k,
                          int st, uint64_t *out, int64_t out_bstride, cudaStream_t s) {
    const int64_t OH = (H - k) / st + 1, OW = (W - k) / st + 1;
    const int64_t total = B * OH * OW * Cw;
    if (total == 0) return BNN_OK;
    maxpool_packed_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, s>>>(
        in, H, W, Cw, k, st, OH, OW, total, out, out_bstride > 0 ? out_bstride : OH * OW * Cw);
    return check_launch("maxpool_packed_kernel");
}
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
    constexpr int kIters = 4;
    const int64_t W = ceil_div(K, 64);
    const int64_t nseg = ceil_div(W, 2 * kIters);  // warps per row
    const bool vec = (ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    const unsigned blocks = (unsigned)ceil_div(R * nseg * 32, 256);
    if (vec)
        pack_rows_kernel<true, kIters><<<blocks, 256, 0, s>>>(x, R, K, ldx, out, ldo, pad_bit, mode,
                                                              flags, nseg);
    else
        pack_rows_kernel<false, kIters><<<blocks, 256, 0, s>>>(x, R, K, ldx, out, ldo, pad_bit,
                                                               mode, flags, nseg);
    int rc = check_launch("pack_rows_kernel");
    if (rc == BNN_OK && row_popc) {
        row_popc_kernel<<<(unsigned)ceil_div(R * 32, 256), 256, 0, s>>>(out, R, W, ldo, K, row_popc);
        rc = check_launch("row_popc_kernel");
    }
    return rc;
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
    const bool vec4 = (HW % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    int pix = (int)g_debug.pack_pix;  // debug knob; 0 (default): direct kernel
    if (pix != 0 && pix != 64 && pix != 128 && pix != 256) pix = 0;
    if (pix == 0 && vec4) {
        int ch = (int)g_debug.pack_ch;  // debug knob: channels per lane 8 (default), 16, 32
        if (ch != 8 && ch != 16 && ch != 32) ch = 8;
        const int64_t threads = ceil_div(B * HW, 4) * (32 / ch);
        dim3 g((unsigned)ceil_div(threads, 256), (unsigned)(2 * Cw));
#define BNN_QUAD(K)                                                                            \
    if (ch == K) {                                                                             \
        if (strict) pack_nchw_quad_kernel<true, K><<<g, 256, 0, s>>>(x, B, C, HW, 2 * Cw, o32, flags); \
        else pack_nchw_quad_kernel<false, K><<<g, 256, 0, s>>>(x, B, C, HW, 2 * Cw, o32, flags);      \
    }
        BNN_QUAD(8)
        BNN_QUAD(16)
        BNN_QUAD(32)
#undef BNN_QUAD
        return check_launch("pack_nchw_quad_kernel");
    }
    if (pix == 0) {
        dim3 g((unsigned)ceil_div(B * HW, 256), (unsigned)Cw);
        if (strict) pack_nchw_direct_kernel<true><<<g, 256, 0, s>>>(x, B, C, HW, Cw, out, flags);
        else pack_nchw_direct_kernel<false><<<g, 256, 0, s>>>(x, B, C, HW, Cw, out, flags);
        return check_launch("pack_nchw_direct_kernel");
    }
    const int smem = 16384 * 4 + pix * (int)(2 * Cw) * 4;
    if (smem > 200 * 1024) return set_error(BNN_EUNSUP, "too many channels for the pack kernel");
    dim3 grid((unsigned)ceil_div(HW, pix), (unsigned)B);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<grid, 256, smem, s>>>(x, B, C, HW, Cw, o32, flags);
    };
#define BNN_PACK_SEL(P)                                                  \
    if (pix == P) {                                                      \
        if (vec4 && !strict) launch(pack_nchw_kernel<P, true, false>);   \
        else if (vec4) launch(pack_nchw_kernel<P, true, true>);          \
        else if (!strict) launch(pack_nchw_kernel<P, false, false>);     \
        else launch(pack_nchw_kernel<P, false, true>);                   \
    }
    BNN_PACK_SEL(64)
    BNN_PACK_SEL(128)
    BNN_PACK_SEL(256)
#undef BNN_PACK_SEL
    return check_launch("pack_nchw_kernel");
}

int launch_pack_planes(const float *x, int64_t R, int64_t K, int64_t ldx, int bits, int grid,
                       uint64_t *out, int64_t ldo, int64_t plane_stride, int32_t *flags,
                       cudaStream_t s) {
    if (R == 0 || K == 0) return BNN_OK;
    const int64_t blocks = ceil_div(R * 32, 256);
    if (bits == 2)
        pack_planes_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(x, R, K, ldx, grid, out, ldo,
                                                               plane_stride, flags);
    else
        return set_error(BNN_EUNSUP, "bit-plane packing supports bits == 2");
    return check_launch("pack_planes_kernel");
}

int launch_bn_relu_maxpool(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                           const float *mean, const float *inv, const float *gamma,
                           const float *beta, int relu, int k, int st, int pd, float *y,
                           cudaStream_t s) {
    const int64_t OH = (H + 2 * pd - k) / st + 1, OW = (W + 2 * pd - k) / st + 1;
    const int64_t total = B * C * OH * OW;
    if (total == 0) return BNN_OK;
    // banded SMEM kernel: R output rows per CTA (~8 KB+ of input rows per band)
    int64_t R = (8192 / 4) / (W * st > 0 ? W * st : 1);
    R = R < 1 ? 1 : (R > OH ? OH : R);
    const int64_t band_bytes = (((R - 1) * st + k) * W) * 4;
    const int64_t nbands = ceil_div(OH, R);
    if (band_bytes <= 48 * 1024 && OH * OW < (1ll << 31) && H * W < (1ll << 31) &&
        B * C * nbands <= 0x7fffffffll && !g_debug.stempost_simple) {
        bn_relu_maxpool_band_kernel<<<(unsigned)(B * C * nbands), 256, (size_t)band_bytes, s>>>(
            x, (int)C, (int)H, (int)W, mean, inv, gamma, beta, relu, k, st, pd, (int)OH, (int)OW,
            (int)R, (int)nbands, y);
        return check_launch("bn_relu_maxpool_band_kernel");
    }
    const int64_t bpp = ceil_div(OH * OW, 256);
    if (OH * OW > (1ll << 30) || H * W > (1ll << 30) || B * C * bpp > 0x7fffffffll)
        return set_error(BNN_EUNSUP, "bn_relu_maxpool: tensor too large");
    bn_relu_maxpool_kernel<<<(unsigned)(B * C * bpp), 256, 0, s>>>(
        x, B, C, H, W, mean, inv, gamma, beta, relu, k, st, pd, OH, OW, y, (int)bpp);
    return check_launch("bn_relu_maxpool_kernel");
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


// ---------------------------------------------------------------------------
// split-K combine: out = alpha * sum_s partials[s] + beta.  The partials are
// popcount-domain counts of disjoint, word-aligned K ranges (integers < 2^24),
// so every f32 add is exact and the result is bit-identical to one unsplit
// launch: P = sum_s P_s (popcount domain) or 2P - K (dot domain, qmath.py:102-109).
// Streaming, HBM-bound: splits x 4 B read + 4 B written per output.
__global__ void sum_partials_kernel(const float *__restrict__ p, int splits, int64_t count,
                                    int64_t stride, float alpha, float beta,
                                    float *__restrict__ out, bool vec) {
    const int64_t n4 = vec ? count >> 2 : 0;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += step) {
        float4 acc = __ldcs(reinterpret_cast<const float4 *>(p) + i);
        for (int s = 1; s < splits; ++s) {
            const float4 v = __ldcs(reinterpret_cast<const float4 *>(p + s * stride) + i);
            acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
        }
        acc.x = fmaf(alpha, acc.x, beta), acc.y = fmaf(alpha, acc.y, beta);
        acc.z = fmaf(alpha, acc.z, beta), acc.w = fmaf(alpha, acc.w, beta);
        reinterpret_cast<float4 *>(out)[i] = acc;
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += step) {
        float acc = p[i];
        for (int s = 1; s < splits; ++s) acc += p[s * stride + i];
        out[i] = fmaf(alpha, acc, beta);
    }
}

int launch_sum_partials(const float *p, int splits, int64_t count, int64_t stride, float alpha,
                        float beta, float *out, cudaStream_t s) {
    if (count == 0) return BNN_OK;
    const int64_t blocks = ceil_div(ceil_div(count, 4), 256);
    const int64_t cap = 8LL * 148;
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(out)) & 15) == 0 &&
                     (stride & 3) == 0;
    sum_partials_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, s>>>(
        p, splits, count, stride, alpha, beta, out, vec);
    return check_launch("sum_partials_kernel");
}

}  // namespace bnn
