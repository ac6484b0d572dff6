// extern "C" boundary of libbnn_b200.so: argument validation (mirroring the
// reference's ValueError cases), thread-local error reporting, and engine
// dispatch.  See include/bnn_b200.h for the contract of each entry point.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "bnn_common.cuh"

namespace bnn {

static thread_local char g_err[512] = "";
DebugKnobs g_debug;

int set_error(int status, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return status;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(BNN_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return BNN_OK;
}

// engines (defined in the kernel translation units)
int launch_binarize(const float *, int64_t, float *, int32_t *, cudaStream_t);
int launch_popcount64(const uint64_t *, int64_t, uint8_t *, int, cudaStream_t);
int launch_avgpool_fc(const float *, int64_t, int64_t, int64_t, const float *, const float *,
                      int64_t, float *, float *, cudaStream_t);
int launch_pack_rows(const float *, int64_t, int64_t, int64_t, uint64_t *, int64_t, int, int,
                     int32_t *, int32_t *, cudaStream_t);
int launch_pack_cols(const float *, int64_t, int64_t, int64_t, uint64_t *, int64_t, int, int,
                     int32_t *, cudaStream_t);
int launch_pack_nchw(const float *, int64_t, int64_t, int64_t, int64_t, uint64_t *, int,
                     int32_t *, cudaStream_t);
int launch_words_transpose(const uint64_t *, int64_t, int64_t, int64_t, uint64_t *, int64_t,
                           cudaStream_t);
int launch_audit_padding(const uint64_t *, int64_t, int64_t, int64_t, int64_t, int, int32_t *,
                         cudaStream_t);
int launch_conv_weights_reorder(const uint64_t *, int64_t, int64_t, int64_t, int64_t,
                                uint64_t *, cudaStream_t);
int launch_xnor_gemm_popc(const uint64_t *, int64_t, const uint64_t *, int64_t, int64_t,
                          int64_t, int64_t, float *, int64_t, int64_t, const Epilogue &,
                          cudaStream_t, const float *);
int launch_xnor_gemm_xp(const uint64_t *, int64_t, const uint64_t *, int64_t, int64_t, int64_t, int64_t,
                        float *, int64_t, int64_t, const Epilogue &, cudaStream_t, const float *, void *,
                        int64_t);
int64_t xnor_gemm_xp_workspace(int64_t M, int64_t N, int64_t K);
int launch_bconv2d_xp(const uint64_t *, int64_t, int64_t, int64_t, int64_t, const uint64_t *, int64_t,
                      int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, float *,
                      const Epilogue &, cudaStream_t, const float *, void *, int64_t);
int64_t bconv2d_xp_workspace(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                             int64_t);
int launch_bitplane_gemm_xp(const uint64_t *, int64_t, int64_t, const uint64_t *, int64_t, int64_t, int64_t,
                            int64_t, int64_t, float *, int64_t, int64_t, const Epilogue &, cudaStream_t,
                            void *, int64_t);
// AUTO: shapes from which the pre-expanded engine wins (measured, profiles/r02)
static bool xp_auto(int64_t M, int64_t N, int64_t K) {
    return M >= 1024 && N >= 1024 && K >= 2048 && (double)M * (double)N * (double)K >= 3.0e10;
}
int launch_xnor_gemm_umma(const uint64_t *, int64_t, const uint64_t *, int64_t, int64_t,
                          int64_t, int64_t, float *, int64_t, int64_t, const Epilogue &,
                          cudaStream_t, const float *);
int launch_bconv2d_umma(const uint64_t *, int64_t, int64_t, int64_t, int64_t, const uint64_t *,
                        int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                        int64_t, float *, const Epilogue &, cudaStream_t, const float *);
int launch_pwconv(const uint64_t *, int64_t, int64_t, int64_t, int64_t, const uint64_t *, int64_t,
                  int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, float *,
                  const Epilogue &, cudaStream_t, const float *);
int launch_xnor_gemm_bmma(const uint64_t *, int64_t, const uint64_t *, int64_t, int64_t,
                          int64_t, int64_t, float *, int64_t, int64_t, const Epilogue &,
                          cudaStream_t, const float *);
int launch_bconv2d_bmma(const uint64_t *, int64_t, int64_t, int64_t, int64_t, const uint64_t *,
                        int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                        int64_t, float *, const Epilogue &, cudaStream_t, const float *);
int launch_sum_partials(const float *, int, int64_t, int64_t, float, float, float *, cudaStream_t);
int launch_pack_planes(const float *, int64_t, int64_t, int64_t, int, int, uint64_t *, int64_t,
                       int64_t, int32_t *, cudaStream_t);
int launch_bitplane_gemm_umma(const uint64_t *, int64_t, int64_t, const uint64_t *, int64_t,
                              int64_t, int64_t, int64_t, int64_t, float *, int64_t, int64_t,
                              const Epilogue &, cudaStream_t);
int launch_bn_relu_maxpool(const float *, int64_t, int64_t, int64_t, int64_t, const float *,
                           const float *, const float *, const float *, int, int, int, int,
                           float *, cudaStream_t);
int launch_conv2d_f32_tc(const float *, int64_t, int64_t, int64_t, int64_t, const float *,
                         const float *, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                         int64_t, int64_t, int64_t, float *, cudaStream_t);
int launch_conv_bn_relu_maxpool_tc(const float *, int64_t, int64_t, int64_t, int64_t,
                                   const float *, int64_t, int64_t, int64_t, int64_t, int64_t,
                                   int64_t, int64_t, const float *, const float *, const float *,
                                   const float *, int, float *, cudaStream_t, int, uint64_t *,
                                   int32_t *, int);
int launch_maxpool_packed(const uint64_t *, int64_t, int64_t, int64_t, int64_t, int, int,
                          uint64_t *, int64_t, cudaStream_t);
int launch_add_pack_nchw(const float *, const float *, int64_t, int64_t, int64_t, int64_t, float *,
                         uint64_t *, int32_t *, cudaStream_t);
int launch_bconv2d_popc(const uint64_t *, int64_t, int64_t, int64_t, int64_t, const uint64_t *,
                        int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                        int64_t, float *, const Epilogue &, cudaStream_t, const float *);

}  // namespace bnn

using namespace bnn;

#define BNN_REQUIRE(cond, status, ...) \
    do {                               \
        if (!(cond)) return set_error(status, __VA_ARGS__); \
    } while (0)

static const int64_t kMaxKExact = 1 << 24;  // gemm.py:43-44

extern "C" {

int bnn_abi_version(void) { return 2; }

int bnn_debug_set(int knob, int64_t value) {
    switch (knob) {
        case BNN_DEBUG_UMMA_BITS: g_debug.umma_bits = value; return BNN_OK;
        case BNN_DEBUG_FP4_BN: g_debug.fp4_bn = value; return BNN_OK;
        case BNN_DEBUG_PAIR_KW32: g_debug.pair_kw32 = value; return BNN_OK;
        case BNN_DEBUG_STEM_BITS: g_debug.stem_bits = value; return BNN_OK;
        case BNN_DEBUG_PACK_PIX: g_debug.pack_pix = value; return BNN_OK;
        case BNN_DEBUG_PACK_CH: g_debug.pack_ch = value; return BNN_OK;
        case BNN_DEBUG_STEMPOST_SIMPLE: g_debug.stempost_simple = value; return BNN_OK;
        case BNN_DEBUG_GRID_CAP: g_debug.grid_cap = value; return BNN_OK;
        default: return set_error(BNN_EINVAL, "unknown debug knob %d", knob);
    }
}

const char *bnn_last_error(void) { return g_err; }

const char *bnn_status_string(int status) {
    switch (status) {
        case BNN_OK: return "ok";
        case BNN_EINVAL: return "invalid argument";
        case BNN_EDIMS: return "GEMM dims must be positive";
        case BNN_EKEXACT: return "K exceeds the float32-exact range";
        case BNN_EPAD: return "pad fill must be 0 or 1";
        case BNN_EALIGN: return "leading dimension too small";
        case BNN_EGEOM: return "invalid convolution geometry";
        case BNN_EUNSUP: return "unsupported configuration";
        case BNN_ECUDA: return "CUDA error";
        default: return "unknown status";
    }
}

int bnn_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

int bnn_binarize_f32(const float *x, int64_t n, float *out, int32_t *flags, bnn_stream_t stream) {
    BNN_REQUIRE(n >= 0, BNN_EINVAL, "n must be non-negative");
    BNN_REQUIRE(n == 0 || (x && out), BNN_EINVAL, "null pointer");
    return launch_binarize(x, n, out, flags, as_stream(stream));
}

int bnn_popcount64(const uint64_t *words, int64_t n, uint8_t *out, int soft,
                   bnn_stream_t stream) {
    BNN_REQUIRE(n >= 0, BNN_EINVAL, "n must be non-negative");
    BNN_REQUIRE(n == 0 || (words && out), BNN_EINVAL, "null pointer");
    return launch_popcount64(words, n, out, soft, as_stream(stream));
}

int bnn_pack_rows_f32(const float *x, int64_t R, int64_t K, int64_t ldx, uint64_t *out,
                      int64_t ldo, int pad_bit, int mode, int32_t *row_popc, int32_t *flags,
                      bnn_stream_t stream) {
    BNN_REQUIRE(R >= 0 && K >= 0, BNN_EINVAL, "negative size");
    BNN_REQUIRE(pad_bit == 0 || pad_bit == 1, BNN_EPAD, "pad_fill must be 0 or 1, got %d", pad_bit);
    BNN_REQUIRE(mode == BNN_PACK_SIGN || mode == BNN_PACK_STRICT, BNN_EINVAL, "bad mode");
    BNN_REQUIRE(ldx >= K && ldo >= ceil_div(K, 64), BNN_EALIGN, "leading dimension too small");
    BNN_REQUIRE(R * K == 0 || (x && out), BNN_EINVAL, "null pointer");
    return launch_pack_rows(x, R, K, ldx, out, ldo, pad_bit, mode, row_popc, flags,
                            as_stream(stream));
}

int bnn_pack_cols_f32(const float *x, int64_t K, int64_t N, int64_t ldx, uint64_t *out,
                      int64_t ldo, int pad_bit, int mode, int32_t *flags, bnn_stream_t stream) {
    BNN_REQUIRE(K >= 0 && N >= 0, BNN_EINVAL, "negative size");
    BNN_REQUIRE(pad_bit == 0 || pad_bit == 1, BNN_EPAD, "pad_fill must be 0 or 1, got %d", pad_bit);
    BNN_REQUIRE(mode == BNN_PACK_SIGN || mode == BNN_PACK_STRICT, BNN_EINVAL, "bad mode");
    BNN_REQUIRE(ldx >= N && ldo >= N, BNN_EALIGN, "leading dimension too small");
    BNN_REQUIRE(K * N == 0 || (x && out), BNN_EINVAL, "null pointer");
    return launch_pack_cols(x, K, N, ldx, out, ldo, pad_bit, mode, flags, as_stream(stream));
}

int bnn_pack_nchw_f32(const float *x, int64_t B, int64_t C, int64_t H, int64_t W, uint64_t *out,
                      int mode, int32_t *flags, bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 0 && H >= 0 && W >= 0, BNN_EINVAL, "negative size");
    BNN_REQUIRE(mode == BNN_PACK_SIGN || mode == BNN_PACK_STRICT, BNN_EINVAL, "bad mode");
    BNN_REQUIRE(B * C * H * W == 0 || (x && out), BNN_EINVAL, "null pointer");
    BNN_REQUIRE(ceil_div(C, 64) <= 65535 && B <= 65535, BNN_EUNSUP, "C or B too large");
    return launch_pack_nchw(x, B, C, H, W, out, mode, flags, as_stream(stream));
}

int bnn_words_transpose(const uint64_t *in, int64_t rows, int64_t cols, int64_t ldi,
                        uint64_t *out, int64_t ldo, bnn_stream_t stream) {
    BNN_REQUIRE(rows >= 0 && cols >= 0, BNN_EINVAL, "negative size");
    BNN_REQUIRE(ldi >= cols && ldo >= rows, BNN_EALIGN, "leading dimension too small");
    BNN_REQUIRE(rows * cols == 0 || (in && out), BNN_EINVAL, "null pointer");
    return launch_words_transpose(in, rows, cols, ldi, out, ldo, as_stream(stream));
}

int bnn_audit_padding(const uint64_t *words, int64_t vectors, int64_t n_bits, int64_t ld_vec,
                      int64_t ld_word, int pad_fill, int32_t *bad, bnn_stream_t stream) {
    BNN_REQUIRE(vectors >= 0 && n_bits >= 0, BNN_EINVAL, "negative size");
    BNN_REQUIRE(pad_fill == 0 || pad_fill == 1, BNN_EPAD, "pad_fill must be 0 or 1");
    BNN_REQUIRE(bad != nullptr, BNN_EINVAL, "null flag pointer");
    return launch_audit_padding(words, vectors, n_bits, ld_vec, ld_word, pad_fill, bad,
                                as_stream(stream));
}

static int check_gemm_dims(int64_t M, int64_t N, int64_t K) {
    // GemmDims.__post_init__ (gemm.py:170-177)
    BNN_REQUIRE(M >= 1 && N >= 1 && K >= 1, BNN_EDIMS,
                "GEMM dims must be positive, got M=%lld N=%lld K=%lld", (long long)M,
                (long long)N, (long long)K);
    BNN_REQUIRE(K < kMaxKExact, BNN_EKEXACT,
                "K=%lld exceeds %lld; popcounts would lose exactness in float32 outputs",
                (long long)K, (long long)(kMaxKExact - 1));
    return BNN_OK;
}

// engine of an algo code: POPC / BMMA / UMMA (AUTO and the tcgen05 variants map to
// UMMA, the variant recorded in ep.variant), or -1 for an unknown code
static int engine_of(int algo, Epilogue &ep) {
    if (algo >= BNN_ALGO_UMMA_V0 && algo <= BNN_ALGO_UMMA_V4) {
        ep.variant = algo - BNN_ALGO_UMMA_V0;
        return BNN_ALGO_UMMA;
    }
    ep.variant = 2;
    if (algo == BNN_ALGO_AUTO || algo == BNN_ALGO_UMMA || algo == BNN_ALGO_UMMA_XP) return BNN_ALGO_UMMA;
    if (algo == BNN_ALGO_POPC || algo == BNN_ALGO_BMMA) return algo;
    return -1;
}
static bool is_umma(int algo) {
    return algo == BNN_ALGO_AUTO || algo == BNN_ALGO_UMMA || algo == BNN_ALGO_UMMA_XP ||
           (algo >= BNN_ALGO_UMMA_V0 && algo <= BNN_ALGO_UMMA_V4);
}

static void fill_epilogue(Epilogue &ep, const bnn_epilogue *e) {
    ep.scale = e->scale;
    ep.shift = e->shift;
    ep.bn_mean = e->bn_mean;
    ep.bn_inv = e->bn_inv_std;
    ep.bn_gamma = e->bn_gamma;
    ep.bn_beta = e->bn_beta;
    ep.pack_out = reinterpret_cast<uint32_t *>(e->pack_out);
    ep.pack_ld32 = 2 * e->pack_ld;
    ep.pack_flags = e->pack_flags;
}

// the fused sign-pack output (tcgen05 engine only) and the optional f32 output
static int check_pack_out(const bnn_epilogue *e, int64_t M, int algo, const float *out) {
    if (!e->pack_out) {
        BNN_REQUIRE(out, BNN_EINVAL, "null pointer");
        return BNN_OK;
    }
    BNN_REQUIRE(is_umma(algo), BNN_EUNSUP,
                "the fused sign-pack epilogue runs on the tcgen05 engine only");
    BNN_REQUIRE(e->pack_ld >= ceil_div(M, 64), BNN_EALIGN, "pack_ld=%lld smaller than ceil(M/64)=%lld",
                (long long)e->pack_ld, (long long)ceil_div(M, 64));
    return BNN_OK;
}

static int xnor_gemm_impl(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                          int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                          int64_t ldc_n, const bnn_epilogue *e, int algo, bnn_stream_t stream,
                          void *ws, int64_t ws_bytes) {
    int rc = check_gemm_dims(M, N, K);
    if (rc) return rc;
    BNN_REQUIRE(e != nullptr, BNN_EINVAL, "null epilogue");
    BNN_REQUIRE((a_pad == 0 || a_pad == 1) && (b_pad == 0 || b_pad == 1), BNN_EPAD,
                "pad fills must be 0 or 1");
    const int64_t W = ceil_div(K, 64);
    BNN_REQUIRE(lda >= W && ldb >= W, BNN_EALIGN, "lda/ldb smaller than ceil(K/64)=%lld",
                (long long)W);
    BNN_REQUIRE(A && B, BNN_EINVAL, "null pointer");
    rc = check_pack_out(e, M, algo, C);
    if (rc) return rc;
    const int domain = e->domain;
    BNN_REQUIRE(domain == BNN_POPCOUNT || domain == BNN_DOT, BNN_EINVAL, "bad domain %d", domain);
    BNN_REQUIRE(!e->bn_mean || (e->bn_inv_std && e->bn_gamma && e->bn_beta), BNN_EINVAL,
                "BatchNorm epilogue needs mean, inv_std, gamma and beta");
    // Tail correction (bitpack.py:12-15): positions K..64W-1 contribute
    // popc(a_pad ^ b_pad) each to X, so P = K - (X - tail) = k_eff - X.
    const int64_t tail = (64 * W - K) * (int64_t)(a_pad ^ b_pad);
    Epilogue ep{(int32_t)(K + tail), (int32_t)K, domain, nullptr, nullptr};
    fill_epilogue(ep, e);
    switch (engine_of(algo, ep)) {
        case BNN_ALGO_POPC:
            return launch_xnor_gemm_popc(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep,
                                         as_stream(stream), e->residual);
        case BNN_ALGO_BMMA:
            return launch_xnor_gemm_bmma(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep,
                                         as_stream(stream), e->residual);
        case BNN_ALGO_UMMA:
            // large GEMMs with a workspace: operands expanded once in HBM, 2-CTA TMA-fed
            // kind::mxf4 GEMM (bnn_gemm_xp.cu); AUTO takes it from xp_auto_min_ops on
            if (algo == BNN_ALGO_UMMA_XP || (algo == BNN_ALGO_AUTO && ws && xp_auto(M, N, K))) {
                rc = launch_xnor_gemm_xp(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep,
                                         as_stream(stream), e->residual, ws, ws_bytes);
                if (rc != BNN_EUNSUP) return rc;
                if (algo == BNN_ALGO_UMMA_XP)
                    return set_error(BNN_EUNSUP, "pre-expanded engine: plain epilogue and a 128-byte aligned "
                                     "workspace of bnn_xnor_gemm_ws_bytes() needed");
            }
            return launch_xnor_gemm_umma(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep,
                                         as_stream(stream), e->residual);
        default:
            return set_error(BNN_EUNSUP, "algorithm %d not available", algo);
    }
}

int bnn_xnor_gemm_ex(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                     int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                     int64_t ldc_n, const bnn_epilogue *e, int algo, bnn_stream_t stream) {
    return xnor_gemm_impl(A, lda, B, ldb, M, N, K, a_pad, b_pad, C, ldc_m, ldc_n, e, algo, stream,
                          nullptr, 0);
}

int64_t bnn_xnor_gemm_ws_bytes(int64_t M, int64_t N, int64_t K) {
    if (M < 1 || N < 1 || K < 1) return 0;
    return xnor_gemm_xp_workspace(M, N, K);
}

int bnn_xnor_gemm_ws(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                     int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                     int64_t ldc_n, int domain, int algo, void *ws, int64_t ws_bytes,
                     bnn_stream_t stream) {
    bnn_epilogue e{domain, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    BNN_REQUIRE(ws_bytes >= 0 && (ws || ws_bytes == 0), BNN_EINVAL, "bad workspace");
    return xnor_gemm_impl(A, lda, B, ldb, M, N, K, a_pad, b_pad, C, ldc_m, ldc_n, &e, algo, stream, ws,
                          ws_bytes);
}

int bnn_xnor_gemm(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                  int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                  int64_t ldc_n, int domain, const float *scale, const float *shift, int algo,
                  bnn_stream_t stream) {
    bnn_epilogue e{domain, scale, shift, nullptr, nullptr, nullptr, nullptr, nullptr};
    return bnn_xnor_gemm_ex(A, lda, B, ldb, M, N, K, a_pad, b_pad, C, ldc_m, ldc_n, &e, algo,
                            stream);
}

int bnn_pack_planes_f32(const float *x, int64_t R, int64_t K, int64_t ldx, int bits, int grid,
                        uint64_t *out, int64_t ldo, int64_t plane_stride, int32_t *flags,
                        bnn_stream_t stream) {
    BNN_REQUIRE(R >= 0 && K >= 0, BNN_EINVAL, "negative size");
    BNN_REQUIRE(bits == 2, BNN_EUNSUP, "bit-plane path supports bits == 2, got %d", bits);
    BNN_REQUIRE(grid == BNN_GRID_UNSIGNED || grid == BNN_GRID_SIGNED, BNN_EINVAL, "bad grid");
    BNN_REQUIRE(ldx >= K && ldo >= ceil_div(K, 64) && plane_stride >= R * ldo, BNN_EALIGN,
                "leading dimension / plane stride too small");
    BNN_REQUIRE(R * K == 0 || (x && out), BNN_EINVAL, "null pointer");
    return launch_pack_planes(x, R, K, ldx, bits, grid, out, ldo, plane_stride, flags,
                              as_stream(stream));
}

int bnn_bitplane_gemm(const uint64_t *A, int64_t lda, int64_t a_plane_stride, int a_grid,
                      const uint64_t *B, int64_t ldb, int64_t b_plane_stride, int b_grid,
                      int bits, int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                      int64_t ldc_n, bnn_stream_t stream) {
    return bnn_bitplane_gemm_ws(A, lda, a_plane_stride, a_grid, B, ldb, b_plane_stride, b_grid, bits, M,
                                N, K, C, ldc_m, ldc_n, 0, nullptr, 0, stream);
}

int bnn_bitplane_gemm_ws(const uint64_t *A, int64_t lda, int64_t a_plane_stride, int a_grid,
                         const uint64_t *B, int64_t ldb, int64_t b_plane_stride, int b_grid,
                         int bits, int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                         int64_t ldc_n, int algo, void *ws, int64_t ws_bytes, bnn_stream_t stream) {
    int rc = check_gemm_dims(M, N, K);
    if (rc) return rc;
    BNN_REQUIRE(bits == 2, BNN_EUNSUP, "bit-plane path supports bits == 2, got %d", bits);
    BNN_REQUIRE((a_grid == BNN_GRID_UNSIGNED || a_grid == BNN_GRID_SIGNED) &&
                    (b_grid == BNN_GRID_UNSIGNED || b_grid == BNN_GRID_SIGNED),
                BNN_EINVAL, "bad grid");
    const int64_t W = ceil_div(K, 64);
    BNN_REQUIRE(lda >= W && ldb >= W && a_plane_stride >= M * lda && b_plane_stride >= N * ldb,
                BNN_EALIGN, "leading dimension / plane stride too small");
    BNN_REQUIRE(A && B && C, BNN_EINVAL, "null pointer");
    const int L = (1 << bits) - 1;
    Epilogue ep{(int32_t)K, (int32_t)K, BNN_POPCOUNT, nullptr, nullptr};
    ep.a_alpha = a_grid == BNN_GRID_SIGNED ? 2 : 1;
    ep.a_beta = a_grid == BNN_GRID_SIGNED ? -L : 0;
    ep.b_alpha = b_grid == BNN_GRID_SIGNED ? 2 : 1;
    ep.b_beta = b_grid == BNN_GRID_SIGNED ? -L : 0;
    ep.inv_gamma = 1.0f / (float)(L * L);
    BNN_REQUIRE(algo == BNN_ALGO_AUTO || algo == BNN_ALGO_UMMA || algo == BNN_ALGO_UMMA_XP, BNN_EUNSUP,
                "bit-plane GEMM: algo must be AUTO, UMMA or UMMA_XP");
    BNN_REQUIRE(ws_bytes >= 0 && (ws || ws_bytes == 0), BNN_EINVAL, "bad workspace");
    // codes as e2m1 grid values in a workspace + the 2-CTA kind::mxf4 GEMM (bnn_gemm_xp.cu)
    if (algo == BNN_ALGO_UMMA_XP || (algo == BNN_ALGO_AUTO && ws && xp_auto(M, N, K))) {
        rc = launch_bitplane_gemm_xp(A, lda, a_plane_stride, B, ldb, b_plane_stride, M, N, K, C, ldc_m,
                                     ldc_n, ep, as_stream(stream), ws, ws_bytes);
        if (rc != BNN_EUNSUP) return rc;
        if (algo == BNN_ALGO_UMMA_XP)
            return set_error(BNN_EUNSUP, "pre-expanded engine: 9 K < 2^24 and a 128-byte aligned "
                             "workspace of bnn_xnor_gemm_ws_bytes() needed");
    }
    return launch_bitplane_gemm_umma(A, lda, a_plane_stride, B, ldb, b_plane_stride, M, N, K, C,
                                     ldc_m, ldc_n, ep, as_stream(stream));
}

int bnn_bn_relu_maxpool_f32(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                            const float *mean, const float *inv_std, const float *gamma,
                            const float *beta, int relu, int k, int stride, int pad, float *y,
                            bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 0 && H >= 1 && W >= 1 && k >= 1 && stride >= 1 && pad >= 0 &&
                    pad < k && H + 2 * pad >= k && W + 2 * pad >= k,
                BNN_EGEOM, "invalid pooling geometry");
    BNN_REQUIRE(x && y && mean && inv_std && gamma && beta, BNN_EINVAL, "null pointer");
    return launch_bn_relu_maxpool(x, B, C, H, W, mean, inv_std, gamma, beta, relu, k, stride, pad,
                                  y, as_stream(stream));
}

int bnn_conv2d_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                      const float *w, const float *bias, int64_t F, int64_t kh, int64_t kw,
                      int64_t sh, int64_t sw, int64_t ph, int64_t pw, float *y,
                      bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && F >= 1 && kh >= 1 && kw >= 1 &&
                    sh >= 1 && sw >= 1 && ph >= 0 && pw >= 0 && H + 2 * ph >= kh &&
                    W + 2 * pw >= kw,
                BNN_EGEOM, "invalid convolution geometry");
    BNN_REQUIRE(x && w && y, BNN_EINVAL, "null pointer");
    const int64_t oh = (H + 2 * ph - kh) / sh + 1, ow = (W + 2 * pw - kw) / sw + 1;
    return launch_conv2d_f32_tc(x, B, C, H, W, w, bias, F, kh, kw, sh, sw, ph, pw, oh, ow, y,
                                as_stream(stream));
}

int bnn_conv_bn_relu_maxpool_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                    const float *w, int64_t F, int64_t kh, int64_t kw,
                                    int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                    const float *mean, const float *inv_std, const float *gamma,
                                    const float *beta, int relu, float *y, bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && F >= 1 && kh >= 1 && kw >= 1 &&
                    sh >= 1 && sw >= 1 && ph >= 0 && pw >= 0 && H + 2 * ph >= kh &&
                    W + 2 * pw >= kw,
                BNN_EGEOM, "invalid convolution geometry");
    BNN_REQUIRE(x && w && y && mean && inv_std && gamma && beta, BNN_EINVAL, "null pointer");
    return launch_conv_bn_relu_maxpool_tc(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, mean,
                                          inv_std, gamma, beta, relu, y, as_stream(stream), 0,
                                          nullptr, nullptr, 0);
}

int bnn_conv_bn_relu_maxpool_pack_f32_tc(const float *x, int64_t B, int64_t C, int64_t H,
                                         int64_t W, const float *w, int64_t F, int64_t kh,
                                         int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                         const float *mean, const float *inv_std,
                                         const float *gamma, const float *beta, int relu,
                                         float *y, uint64_t *out_words, int32_t *flags,
                                         bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && F >= 1 && kh >= 1 && kw >= 1 &&
                    sh >= 1 && sw >= 1 && ph >= 0 && pw >= 0 && H + 2 * ph >= kh &&
                    W + 2 * pw >= kw,
                BNN_EGEOM, "invalid convolution geometry");
    BNN_REQUIRE(x && w && y && mean && inv_std && gamma && beta && out_words, BNN_EINVAL,
                "null pointer");
    return launch_conv_bn_relu_maxpool_tc(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, mean,
                                          inv_std, gamma, beta, relu, y, as_stream(stream), 0,
                                          out_words, flags, 0);
}

int bnn_conv_tanh_maxpool2_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                  const float *w, const float *bias, int64_t F, int64_t kh,
                                  int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                  int pool_first, float *y, bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && F >= 1 && kh >= 1 && kw >= 1 &&
                    sh >= 1 && sw >= 1 && ph >= 0 && pw >= 0 && H + 2 * ph >= kh &&
                    W + 2 * pw >= kw,
                BNN_EGEOM, "invalid convolution geometry");
    BNN_REQUIRE(x && w && y, BNN_EINVAL, "null pointer");
    return launch_conv_bn_relu_maxpool_tc(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, bias,
                                          nullptr, nullptr, nullptr, 0, y, as_stream(stream), 1,
                                          nullptr, nullptr, pool_first);
}

int bnn_conv_tanh_maxpool2_pack_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                       const float *w, const float *bias, int64_t F, int64_t kh,
                                       int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                       int pool_first, float *y, uint64_t *out_words,
                                       int32_t *flags, bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && F >= 1 && kh >= 1 && kw >= 1 &&
                    sh >= 1 && sw >= 1 && ph >= 0 && pw >= 0 && H + 2 * ph >= kh &&
                    W + 2 * pw >= kw,
                BNN_EGEOM, "invalid convolution geometry");
    BNN_REQUIRE(x && w && out_words, BNN_EINVAL, "null pointer");
    return launch_conv_bn_relu_maxpool_tc(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, bias,
                                          nullptr, nullptr, nullptr, 0, y, as_stream(stream), 1,
                                          out_words, flags, pool_first);
}

int bnn_maxpool_packed(const uint64_t *in, int64_t B, int64_t H, int64_t W, int64_t Cw, int k,
                       int stride, uint64_t *out, bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && H >= 1 && W >= 1 && Cw >= 1 && k >= 1 && stride >= 1 && H >= k &&
                    W >= k,
                BNN_EGEOM, "invalid pooling geometry");
    BNN_REQUIRE(B == 0 || (in && out), BNN_EINVAL, "null pointer");
    BNN_REQUIRE(ceil_div(B * H * W * Cw, 256) < (1ll << 31), BNN_EUNSUP, "tensor too large");
    return launch_maxpool_packed(in, B, H, W, Cw, k, stride, out, 0, as_stream(stream));
}

int bnn_maxpool_packed_ld(const uint64_t *in, int64_t B, int64_t H, int64_t W, int64_t Cw, int k,
                          int stride, uint64_t *out, int64_t out_batch_stride, bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && H >= 1 && W >= 1 && Cw >= 1 && k >= 1 && stride >= 1 && H >= k &&
                    W >= k,
                BNN_EGEOM, "invalid pooling geometry");
    BNN_REQUIRE(B == 0 || (in && out), BNN_EINVAL, "null pointer");
    BNN_REQUIRE(ceil_div(B * H * W * Cw, 256) < (1ll << 31), BNN_EUNSUP, "tensor too large");
    const int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    BNN_REQUIRE(out_batch_stride >= OH * OW * Cw, BNN_EALIGN, "batch stride smaller than an image");
    return launch_maxpool_packed(in, B, H, W, Cw, k, stride, out, out_batch_stride, as_stream(stream));
}

int bnn_sum_partials_f32(const float *partials, int splits, int64_t count, int64_t stride,
                         int domain, int64_t K, float *out, bnn_stream_t stream) {
    BNN_REQUIRE(splits >= 1 && count >= 0, BNN_EINVAL, "invalid size");
    BNN_REQUIRE(splits == 1 || stride >= count, BNN_EALIGN, "stride smaller than count");
    BNN_REQUIRE(domain == BNN_POPCOUNT || domain == BNN_DOT, BNN_EINVAL, "bad domain %d", domain);
    int rc = check_gemm_dims(1, 1, K);
    if (rc) return rc;
    BNN_REQUIRE(count == 0 || (partials && out), BNN_EINVAL, "null pointer");
    const float alpha = domain == BNN_DOT ? 2.0f : 1.0f;
    const float beta = domain == BNN_DOT ? -(float)K : 0.0f;
    return launch_sum_partials(partials, splits, count, stride, alpha, beta, out, as_stream(stream));
}

int bnn_add_pack_nchw_f32(const float *a, const float *residual, int64_t B, int64_t C, int64_t H,
                          int64_t W, float *y, uint64_t *out_words, int32_t *flags,
                          bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1, BNN_EGEOM, "invalid shape");
    BNN_REQUIRE(B == 0 || (a && residual && y && out_words), BNN_EINVAL, "null pointer");
    return launch_add_pack_nchw(a, residual, B, C, H, W, y, out_words, flags, as_stream(stream));
}

int bnn_avgpool_fc_f32(const float *x, int64_t B, int64_t C, int64_t HW, const float *w,
                       const float *bias, int64_t O, float *y, float *pooled,
                       bnn_stream_t stream) {
    BNN_REQUIRE(B >= 0 && C >= 1 && HW >= 1 && O >= 1, BNN_EINVAL, "invalid size");
    BNN_REQUIRE(B < (1ll << 31) && C * HW < (1ll << 31) && O < (1ll << 31), BNN_EUNSUP,
                "tensor too large");
    BNN_REQUIRE(B == 0 || (x && w && y && pooled), BNN_EINVAL, "null pointer");
    return launch_avgpool_fc(x, B, C, HW, w, bias, O, y, pooled, as_stream(stream));
}

int64_t bnn_conv_channel_words(int64_t C) { return C > 0 ? ceil_div(C, 64) : 0; }

int bnn_conv_weights_reorder(const uint64_t *w_ref, int64_t F, int64_t C, int64_t kh,
                             int64_t kw, uint64_t *w_dev, bnn_stream_t stream) {
    BNN_REQUIRE(F >= 1 && C >= 1 && kh >= 1 && kw >= 1, BNN_EGEOM, "invalid conv weight shape");
    BNN_REQUIRE(w_ref && w_dev, BNN_EINVAL, "null pointer");
    return launch_conv_weights_reorder(w_ref, F, C, kh, kw, w_dev, as_stream(stream));
}

static int bconv2d_impl(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                        const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                        int64_t sw, int64_t ph, int64_t pw, float *y, const bnn_epilogue *e, int algo,
                        bnn_stream_t stream, void *ws, int64_t ws_bytes) {
    // tensor.conv_output_hw (tensor.py:15-27)
    BNN_REQUIRE(B >= 1 && C >= 1 && H >= 1 && W >= 1 && F >= 1 && kh >= 1 && kw >= 1 &&
                    sh >= 1 && sw >= 1 && ph >= 0 && pw >= 0,
                BNN_EGEOM, "invalid convolution geometry");
    const int64_t oh = (H + 2 * ph - kh) / sh + 1, ow = (W + 2 * pw - kw) / sw + 1;
    BNN_REQUIRE(H + 2 * ph >= kh && W + 2 * pw >= kw && oh >= 1 && ow >= 1, BNN_EGEOM,
                "kernel %lldx%lld does not fit input %lldx%lld with pad %lld,%lld",
                (long long)kh, (long long)kw, (long long)H, (long long)W, (long long)ph,
                (long long)pw);
    const int64_t K = C * kh * kw;
    int rc = check_gemm_dims(F, B * oh * ow, K);
    if (rc) return rc;
    BNN_REQUIRE(e != nullptr, BNN_EINVAL, "null epilogue");
    BNN_REQUIRE(x_words && w_dev, BNN_EINVAL, "null pointer");
    rc = check_pack_out(e, F, algo, y);
    if (rc) return rc;
    const int domain = e->domain;
    BNN_REQUIRE(domain == BNN_POPCOUNT || domain == BNN_DOT, BNN_EINVAL, "bad domain %d", domain);
    BNN_REQUIRE(!e->bn_mean || (e->bn_inv_std && e->bn_gamma && e->bn_beta), BNN_EINVAL,
                "BatchNorm epilogue needs mean, inv_std, gamma and beta");
    BNN_REQUIRE(H * W * bnn_conv_channel_words(C) < (1ll << 31), BNN_EUNSUP, "image too large");
    Epilogue ep{(int32_t)K, (int32_t)K, domain, nullptr, nullptr};  // all tails are 0
    fill_epilogue(ep, e);
    switch (engine_of(algo, ep)) {
        case BNN_ALGO_POPC:
            return launch_bconv2d_popc(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, oh,
                                       ow, y, ep, as_stream(stream), e->residual);
        case BNN_ALGO_BMMA:
            return launch_bconv2d_bmma(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, oh,
                                       ow, y, ep, as_stream(stream), e->residual);
        case BNN_ALGO_UMMA:
            // AUTO, 1x1 / pad 0 / C <= 128 with an f32 output (ResNet downsample shortcuts): the
            // layer is bound by its output stream, and the POPC-pipe pointwise kernel writes it at
            // HBM speed (bnn_pwconv.cu); debug bit 1 << 29 keeps the tensor-core engines
            if (algo == BNN_ALGO_AUTO && !(g_debug.umma_bits & (1 << 29))) {
                rc = launch_pwconv(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, oh, ow, y, ep,
                                   as_stream(stream), e->residual);
                if (rc != BNN_EUNSUP) return rc;
            }
            // C % 256 == 0 with a workspace: activations (+1 halo) and weights expanded once to
            // e2m1 codes, im2col-TMA-fed 2-CTA kind::mxf4 GEMM with the full fused epilogue
            // (AUTO: every C % 256 == 0 conv -- ResNet-18 layer 4: 22 vs 45 us per conv; at C = 256,
            // expansion pass included, level on plain outputs (C2 17.7 vs 17.7 us) and ahead with a fused
            // shortcut: ResNet-18 213k -> 220k images/s, C2 step 963 -> 1002 TOPS)
            if (algo == BNN_ALGO_UMMA_XP || (algo == BNN_ALGO_AUTO && ws && C >= 256)) {
                rc = launch_bconv2d_xp(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, oh, ow, y,
                                       ep, as_stream(stream), e->residual, ws, ws_bytes);
                if (rc != BNN_EUNSUP) return rc;
                if (algo == BNN_ALGO_UMMA_XP)
                    return set_error(BNN_EUNSUP, "pre-expanded conv engine: C %% 256 == 0, F %% 64 == 0 "
                                     "and a workspace of bnn_bconv2d_ws_bytes() needed");
            }
            return launch_bconv2d_umma(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, oh,
                                       ow, y, ep, as_stream(stream), e->residual);
        default:
            return set_error(BNN_EUNSUP, "algorithm %d not available", algo);
    }
}

int bnn_bconv2d_ex(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                   const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                   int64_t sw, int64_t ph, int64_t pw, float *y, const bnn_epilogue *e, int algo,
                   bnn_stream_t stream) {
    return bconv2d_impl(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, y, e, algo, stream,
                        nullptr, 0);
}

int64_t bnn_bconv2d_ws_bytes(int64_t B, int64_t C, int64_t H, int64_t W, int64_t F, int64_t kh,
                             int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw) {
    if (B < 1 || C < 1 || H < 1 || W < 1 || F < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 ||
        pw < 0 || C % 256 != 0 || F % 64 != 0 || F > 1024 || sh > 8 || sw > 8 || kh > 128 || kw > 128)
        return 0;
    return bconv2d_xp_workspace(B, C, H, W, F, kh, kw, ph, pw);
}

int bnn_bconv2d_ws(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                   const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                   int64_t ph, int64_t pw, float *y, const bnn_epilogue *e, int algo, void *ws,
                   int64_t ws_bytes, bnn_stream_t stream) {
    BNN_REQUIRE(ws_bytes >= 0 && (ws || ws_bytes == 0), BNN_EINVAL, "bad workspace");
    return bconv2d_impl(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, y, e, algo, stream, ws,
                        ws_bytes);
}

int bnn_bconv2d(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                int64_t ph, int64_t pw, float *y, int domain, const float *scale,
                const float *shift, int algo, bnn_stream_t stream) {
    bnn_epilogue e{domain, scale, shift, nullptr, nullptr, nullptr, nullptr, nullptr};
    return bnn_bconv2d_ex(x_words, B, C, H, W, w_dev, F, kh, kw, sh, sw, ph, pw, y, &e, algo,
                          stream);
}

}  // extern "C"
