// Operand loaders and output stores shared by the xnor engines.
//
// A loader maps (row, u32 word index) of a K-contiguous packed operand to a
// shared-memory write: DenseRows for plain [rows, ld] word matrices,
// ConvRows for the implicit-im2col view of packed NHWC activations.  A
// store maps (m, n) of the GEMM view to the output tensor.
#pragma once

#include <cuda.h>

#include "bnn_common.cuh"

namespace bnn {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kBytes>
__device__ __forceinline__ void cp_async(uint32_t dst, const void *src, int src_bytes) {
    if constexpr (kBytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                     "r"(src_bytes));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(dst), "l"(src),
                     "n"(kBytes), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// byte offset of piece p (of kVec words) of row r inside a [rows][32-word] tile
template <int kVec>
__device__ __forceinline__ uint32_t tile_off(int r, int p) {
    const int byte = p * kVec * 4;  // logical byte within the 128-B row
    const int c16 = byte >> 4;
    return (uint32_t)(r * 128 + ((c16 ^ (r & 7)) << 4) + (byte & 15));
}

// ------------------------------------------------------------------ loaders
// Dense operand: row r of a [rows, ld32] u32 matrix, kw32 valid words.
struct DenseRows {
    const uint32_t *base;
    int64_t ld32;
    int64_t rows;
    int64_t kw32;
    int64_t plane32 = 0;  // u32 stride between bit planes (multi-bit operands)
    struct Cursor { const uint32_t *p; bool ok; };
    __device__ Cursor row(int64_t r) const { return {base + r * ld32, r < rows}; }
    // load kVec words at word w of this row into smem address dst
    template <int kVec>
    __device__ void load(Cursor &c, int w, uint32_t dst, int plane = 0) const {
        const int left = (int)kw32 - w;  // K < 2^24 -> word counts fit in 32 bits
        int bytes = (!c.ok || left <= 0) ? 0 : (left >= kVec ? kVec * 4 : left * 4);
        const uint32_t *src = bytes ? c.p + plane * plane32 + w : base;
        cp_async<kVec * 4>(dst, src, bytes);
    }
};

// Implicit im2col rows: row n = output pixel (b, oy, ox); word w = tap-major
// (i, j, channel word).  Out-of-image taps read the constant "+1" word
// (valid channel bits set, channel tail 0), the reference's zero-pad-then-
// binarize composition (tensor.py:73-74 + bitpack.py:39).
struct ConvRows {
    const uint32_t *x;  // NHWC words, pixel stride cs32
    int64_t npix;       // B * oh * ow
    int H, W, cs32, C, kw, sh, sw, ph, pw, oh, ow;
    int64_t kw32;       // kh * kw * cs32
    // (tap_w0, i, j) track the current kernel tap incrementally: callers walk
    // w upwards within a row, so no division is needed per load
    struct Cursor { const uint32_t *img; int iy0, ix0; bool ok; int64_t tap_w0; int i, j; };
    __device__ Cursor row(int64_t n) const {
        Cursor c;
        c.ok = n < npix;
        int64_t nn = c.ok ? n : 0;
        int64_t ohw = (int64_t)oh * ow;
        int64_t b = nn / ohw;
        int pix = (int)(nn - b * ohw);
        int oy = pix / ow, ox = pix - (pix / ow) * ow;
        c.img = x + b * (int64_t)H * W * cs32;
        c.iy0 = oy * sh - ph;
        c.ix0 = ox * sw - pw;
        c.tap_w0 = 0;
        c.i = c.j = 0;
        return c;
    }
    template <int kVec>
    __device__ void load(Cursor &c, int w, uint32_t dst, int plane = 0) const {
        if (!c.ok || w >= kw32) {
            cp_async<kVec * 4>(dst, x, 0);
            return;
        }
        if (w < c.tap_w0) c.tap_w0 = 0, c.i = 0, c.j = 0;  // new pass over the row
        while (w >= c.tap_w0 + cs32) {
            c.tap_w0 += cs32;
            if (++c.j == kw) c.j = 0, ++c.i;
        }
        const int cw = (int)(w - c.tap_w0);  // (tap_w0 is int64 for ld math)
        int iy = c.iy0 + c.i, ix = c.ix0 + c.j;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) {
            cp_async<kVec * 4>(dst, c.img + ((int64_t)iy * W + ix) * cs32 + cw, kVec * 4);
        } else {
            uint32_t v[kVec];
#pragma unroll
            for (int q = 0; q < kVec; ++q) {
                int valid = C - 32 * (cw + q);
                v[q] = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
            }
            if constexpr (kVec == 4)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(dst), "r"(v[0]),
                             "r"(v[1]), "r"(v[2]), "r"(v[3]));
            else
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(dst), "r"(v[0]),
                             "r"(v[1]));
        }
    }
};

// ------------------------------------------------------------------ stores
// Stores optionally add a residual tensor of the output's own layout (fused
// "+ shortcut" of a residual block; f32 add, the same rounding as x + r).
struct GemmStore {
    static constexpr bool kConv = false;
    static constexpr bool kPack = false;  // fused sign-pack epilogue instantiations
    static constexpr bool kSwap = false;  // rows = output pixels, columns = filters
    float *C;
    int64_t ldc_m, ldc_n, M, N;
    const float *res = nullptr;
    // optional TMA store map over C ([M, N] f32, 32 x 32 boxes, SWIZZLE_128B);
    // the tcgen05 epilogue uses it when has_map (row-major, no residual)
    int has_map = 0;
    CUtensorMap omap;
    __device__ bool ok(int64_t m, int64_t n) const { return m < M && n < N; }
    __device__ void put(int64_t m, int64_t n, float v) const {
        const int64_t i = m * ldc_m + n * ldc_n;
        C[i] = res ? __fadd_rn(v, __ldg(res + i)) : v;
    }
    __device__ void put_raw(int64_t m, int64_t n, float v) const { C[m * ldc_m + n * ldc_n] = v; }
    __device__ float res_at(int64_t m, int64_t n) const { return __ldg(res + m * ldc_m + n * ldc_n); }
    // element (m, n) lives at out_ptr()[col_off(n) + m * m_stride()]
    __device__ int64_t col_off(int64_t n) const { return n * ldc_n; }
    __device__ float *out_ptr() const { return C; }
    __device__ const float *res_of(const float *p) const { return res + (p - C); }
    __device__ bool has_out() const { return C != nullptr; }
    // g[j] += res[m, n + j] for the first w columns (j < w, n + j < N)
    __device__ void add_res_row(int64_t m, int64_t n, int w, float *g) const {
        const float *r = res + m * ldc_m + n * ldc_n;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < w && n + j < N) g[j] = __fadd_rn(g[j], __ldg(r + j * ldc_n));
    }
    // column view for the staged epilogue: &C[m, n] = col_base(n) + m * m_stride()
    __device__ bool n_contiguous() const { return ldc_n == 1; }
    __device__ float *col_base(int64_t n) const { return C + n * ldc_n; }
    __device__ int64_t m_stride() const { return ldc_m; }
    __device__ int64_t rows() const { return M; }
    __device__ int64_t cols() const { return N; }
    // contiguous output run starting at (m, n), at most maxlen columns (n_contiguous only)
    __device__ int run(int64_t m, int64_t n, int maxlen, float *&p) const {
        p = C + m * ldc_m + n;
        return (int)(N - n < maxlen ? N - n : maxlen);
    }
    // column group n..n+3: base pointer (row 0) and whether a float4 store is legal
    // for every row (n_contiguous only)
    __device__ bool col4(int64_t n, float *&col) const {
        col = C + n;
        return n + 3 < N && ((reinterpret_cast<uintptr_t>(col) | (uintptr_t)(ldc_m * 4)) & 15) == 0;
    }
    // four consecutive n of one row m (m < M checked by the caller)
    __device__ void put4(int64_t m, int64_t n, const float *v) const {
        float *p = C + m * ldc_m + n * ldc_n;
        if (ldc_n == 1 && n + 3 < N && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
            *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (n + i < N) p[i * ldc_n] = v[i];
        }
    }
};

struct ConvStore {  // y NCHW [B, F, oh*ow]; m = filter, n = b*ohw + pixel
    static constexpr bool kConv = true;
    static constexpr bool kPack = false;
    static constexpr bool kSwap = false;
    float *y;
    int64_t F, ohw, npix;
    const float *res = nullptr;
    // optional TMA store map over y ({ohw, F, B} f32, 32 x 32 x 1 boxes, SWIZZLE_128B)
    int has_map = 0;
    CUtensorMap omap;
    __device__ bool ok(int64_t m, int64_t n) const { return m < F && n < npix; }
    __device__ void put(int64_t m, int64_t n, float v) const {
        int64_t b = n / ohw, p = n - b * ohw;
        const int64_t i = (b * F + m) * ohw + p;
        y[i] = res ? __fadd_rn(v, __ldg(res + i)) : v;
    }
    __device__ void put_raw(int64_t m, int64_t n, float v) const {
        int64_t b = n / ohw, p = n - b * ohw;
        y[(b * F + m) * ohw + p] = v;
    }
    __device__ float res_at(int64_t m, int64_t n) const {
        int64_t b = n / ohw, p = n - b * ohw;
        return __ldg(res + (b * F + m) * ohw + p);
    }
    // element (m, n) lives at out_ptr()[col_off(n) + m * m_stride()]
    __device__ int64_t col_off(int64_t n) const {
        const int64_t b = n / ohw;
        return b * F * ohw + (n - b * ohw);
    }
    __device__ float *out_ptr() const { return y; }
    __device__ const float *res_of(const float *p) const { return res + (p - y); }
    __device__ bool has_out() const { return y != nullptr; }
    // g[j] += res[m, n + j] for the first w columns (j < w, n + j < npix); the
    // run of 32 pixels may straddle images
    __device__ void add_res_row(int64_t m, int64_t n, int w, float *g) const {
        int64_t b = n / ohw, p = n - b * ohw;
        const float *r = res + (b * F + m) * ohw + p;
        if (w == 32 && p + 32 <= ohw && n + 32 <= npix && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 t = __ldg(reinterpret_cast<const float4 *>(r) + j);
                g[4 * j] = __fadd_rn(g[4 * j], t.x);
                g[4 * j + 1] = __fadd_rn(g[4 * j + 1], t.y);
                g[4 * j + 2] = __fadd_rn(g[4 * j + 2], t.z);
                g[4 * j + 3] = __fadd_rn(g[4 * j + 3], t.w);
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j < w && n + j < npix) g[j] = __fadd_rn(g[j], __ldg(r));
            ++r;
            if (++p == ohw) {  // next image: same channel m
                p = 0;
                r += (F - 1) * ohw;
            }
        }
    }
    __device__ bool n_contiguous() const { return true; }  // within an image
    __device__ float *col_base(int64_t n) const {
        int64_t b = n / ohw, p = n - b * ohw;
        return y + b * F * ohw + p;
    }
    __device__ int64_t m_stride() const { return ohw; }
    __device__ int64_t rows() const { return F; }
    __device__ int64_t cols() const { return npix; }
    __device__ bool col4(int64_t n, float *&col) const {
        const int64_t b = n / ohw, pp = n - b * ohw;
        col = y + b * F * ohw + pp;
        return pp + 3 < ohw && n + 3 < npix &&
               ((reinterpret_cast<uintptr_t>(col) | (uintptr_t)(ohw * 4)) & 15) == 0;
    }
    __device__ int run(int64_t m, int64_t n, int maxlen, float *&p) const {
        const int64_t b = n / ohw, pp = n - b * ohw;
        p = y + (b * F + m) * ohw + pp;
        int64_t len = ohw - pp;
        if (npix - n < len) len = npix - n;
        return (int)(len < maxlen ? len : maxlen);
    }
    __device__ void put4(int64_t m, int64_t n, const float *v) const {
        int64_t b = n / ohw, p = n - b * ohw;
        float *dst = y + (b * F + m) * ohw + p;
        if (p + 3 < ohw && n + 3 < npix && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (n + i < npix) put(m, n + i, v[i]);
        }
    }
};

// Swapped conv orientation (filters <= 64): GEMM rows m = output pixels
// (b * ohw + p, implicit im2col rows, one TMEM lane each), columns n = filters.
// Element (m, n) of y NCHW [B, F, ohw] sits at row_off(m) + n * ohw, so for a
// fixed filter the 32 lanes of a warp store 32 consecutive pixels.  The
// per-filter epilogue parameters (BN) are per column; the sign-pack word of a
// pixel is built in its own lane.
struct ConvStoreT {
    static constexpr bool kConv = true;
    static constexpr bool kPack = false;
    static constexpr bool kSwap = true;
    float *y;
    int64_t F, ohw, npix;
    const float *res = nullptr;
    int has_map = 0;
    CUtensorMap omap;
    __device__ int64_t rows() const { return npix; }
    __device__ int64_t cols() const { return F; }
    __device__ int64_t m_stride() const { return 1; }
    __device__ bool n_contiguous() const { return false; }
    __device__ bool has_out() const { return y != nullptr; }
    __device__ int64_t row_off(int64_t m) const {
        const int64_t b = m / ohw;
        return b * F * ohw + (m - b * ohw);
    }
};
struct ConvStoreTPk : ConvStoreT {
    static constexpr bool kPack = true;
};

// the same stores, instantiating the tcgen05 epilogue's sign-pack output
struct GemmStorePk : GemmStore {
    static constexpr bool kPack = true;
};
struct ConvStorePk : ConvStore {
    static constexpr bool kPack = true;
};

}  // namespace bnn
