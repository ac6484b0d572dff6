/*
 * bnn_b200.h -- C ABI of the B200-native binarise -> bit-pack -> xnor-popcount
 * path (BMXNet, arXiv 1705.09864).
 *
 * Every entry point takes plain device pointers allocated by the caller
 * (PyTorch in the Python host layer), sizes as int64_t, and an explicit CUDA
 * stream.  Nothing allocates device memory internally, every option is a
 * per-call argument (engine and tcgen05 variant in `algo`, epilogue in
 * bnn_epilogue), and every call is asynchronous on `stream`.  The only global
 * mutable state is the thread-local error message and the DEBUG knobs at the
 * end of this file (process-wide, not thread-safe, off by default, never set
 * by the product path).  Return value: 0 on success, a negative BNN_E*
 * code for an invalid argument (the reference raises ValueError for these),
 * or BNN_ECUDA (> 0) when a CUDA launch failed.  bnn_last_error() returns a
 * thread-local message for the last failing call.
 *
 * ABI version 2 (bnn_abi_version).
 *
 * Word format (reference bitpack.py:1-16): bit k of a packed vector is bit
 * k % 64 of u64 word k / 64 (LSB-first); bit 1 <=> sign +1, bit 0 <=> -1.
 * A layout-'a' matrix is [rows, ceil(K/64)] words, row-major.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/bitnn):
 *   bnn_binarize_f32        bitpack.binarize              bitpack.py:30-42
 *   bnn_popcount64          bitpack.popcount64 / popcount64_soft
 *                                                         bitpack.py:49-66
 *   bnn_pack_rows_f32       bitpack.pack_matrix_a(binarize(x)) / pack_row
 *                                                         bitpack.py:144-149,172-182
 *   bnn_pack_cols_f32       bitpack.pack_matrix_b         bitpack.py:152-169
 *   bnn_pack_nchw_f32       tensor.im2col + binarize + pack_matrix_b, the
 *                           activation side of QConv2d.forward
 *                                                         layers.py:230-236
 *   bnn_words_transpose     BitMatrix layout 'b' <-> 'a'  bitpack.py:90-141
 *   bnn_audit_padding       bitpack.audit_padding         bitpack.py:197-215
 *   bnn_xnor_gemm           gemm.xnor_gemm_{base,blocked,unrolled,parallel}
 *                                                         gemm.py:226-291
 *   bnn_conv_weights_reorder QConv2d.pack (load-time re-layout only)
 *                                                         layers.py:215-223
 *   bnn_bconv2d             QConv2d.forward(INFER_PACKED) layers.py:225-245
 */
#ifndef BNN_B200_H
#define BNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t-compatible opaque handle (0 = legacy default stream). */
typedef struct CUstream_st *bnn_stream_t;

enum bnn_status {
    BNN_OK = 0,
    BNN_EINVAL = -1,   /* bad pointer / negative size / bad enum           */
    BNN_EDIMS = -2,    /* GemmDims: M, N, K must be >= 1 (gemm.py:170-172)  */
    BNN_EKEXACT = -3,  /* K >= 2^24 loses f32 exactness (gemm.py:173-177)   */
    BNN_EPAD = -4,     /* pad fill must be 0 or 1 (bitpack.py:109-111)      */
    BNN_EALIGN = -5,   /* leading dimension smaller than the row            */
    BNN_EGEOM = -6,    /* conv geometry (tensor.py:15-27)                   */
    BNN_EUNSUP = -7,   /* algorithm not available for this shape           */
    BNN_ECUDA = 1      /* CUDA launch / runtime error                      */
};

/* Output domain of the GEMM epilogue (qmath.py:87-109). */
enum bnn_domain {
    BNN_POPCOUNT = 0,  /* P = popcount(xnor(a, b)) in [0, K] (gemm.py:3-8) */
    BNN_DOT = 1        /* 2P - K, the signed dot product                    */
};

/* Inner-product engine.  AUTO picks the measured winner for the shape (the
 * tcgen05 engine, variant 2).  The explicit tcgen05 variants exist for the
 * engine contest and as independent parity checks; all results are identical. */
enum bnn_algo {
    BNN_ALGO_AUTO = 0,
    BNN_ALGO_POPC = 1, /* CUDA cores: LOP3 xor + POPC                        */
    BNN_ALGO_BMMA = 2, /* warp mma.sync m16n8k256 b1 .and.popc (emulated     */
                       /* on sm_100a: IMMA.U8 subroutine calls)              */
    BNN_ALGO_UMMA = 3, /* tcgen05.mma on bits expanded in SMEM = variant 2   */
    /* AUTO / UMMA route by shape (all bit-identical): stride-1 convs with C <= 128 ->
     * the shifted-window kernel (bnn_wconv.cu), other small-channel convs ->
     * bnn_sconv.cu, GEMMs with N <= 256 and K <= 4096 -> the 8-CTA-cluster split-K
     * kernel (bnn_gemm_splitk.cu), everything else -> the general engine below.
     * AUTO only: 1x1 / pad 0 convs with C <= 128 and an f32 output (no sign-pack output) run
     * the POPC-pipe pointwise kernel (bnn_pwconv.cu): they are bound by their output stream. */
    /* tcgen05 engine variants (BNN_ALGO_UMMA_V0 + v):
     *   V0: kind::i8, 128 x 256 tiles, A and B through SMEM
     *   V1: kind::i8, expanded weights in TMEM, tile N from {128..192}
     *   V2: kind::mxf4 (e2m1 expansion, 2x the i8 MMA rate) for TMA-fed operands,
     *       kind::i8 V0/V1 for cp.async-fed shapes (the default)
     *   V3: kind::mxf4 with the expanded A operand in TMEM (N tiles <= 192)
     *   V4: V2, and convs with <= 64 filters in the swapped orientation
     *       (rows = output pixels, 128 x 64 tiles) */
    BNN_ALGO_UMMA_V0 = 16,
    BNN_ALGO_UMMA_V1 = 17,
    BNN_ALGO_UMMA_V2 = 18,
    BNN_ALGO_UMMA_V3 = 19,
    BNN_ALGO_UMMA_V4 = 20,
    /* bnn_xnor_gemm_ws only: force the pre-expanded engine (bnn_gemm_xp.cu): both operands
     * expanded once in HBM to e2m1 +-1 codes, then a 2-CTA (cta_group::2) TMA-fed kind::mxf4
     * GEMM whose accumulator is the signed dot product itself.  AUTO takes it for large
     * shapes when a workspace is given; BNN_EUNSUP without one. */
    BNN_ALGO_UMMA_XP = 24
};

/* Flags written (OR-ed) by the pack kernels into a caller int32. */
enum bnn_flags {
    BNN_FLAG_NONFINITE = 1, /* NaN/Inf seen: binarize raises ValueError    */
    BNN_FLAG_NOTSIGN = 2,   /* strict mode: an entry was not exactly +-1     */
    BNN_FLAG_RANGE = 4      /* unsigned grid: an input outside [0, 1]        */
};

/* Quantization grids of the multi-bit path (qmath.py:50-84), levels L = 2^bits - 1. */
enum bnn_grid {
    BNN_GRID_UNSIGNED = 0, /* quantize:        v = code / L,        x in [0, 1] */
    BNN_GRID_SIGNED = 1    /* quantize_signed: v = (2 code - L) / L, clip(x, -1, 1) */
};

/* Pack-kernel input modes. */
enum bnn_pack_mode {
    BNN_PACK_SIGN = 0,  /* binarize on the fly: x >= 0 -> 1 (sign(-0) = +1) */
    BNN_PACK_STRICT = 1 /* input must already be +-1 (_validate_signs)      */
};

int bnn_abi_version(void);
const char *bnn_last_error(void);
const char *bnn_status_string(int status);
/* number of SMs of the current device (0 if none) */
int bnn_device_sm_count(void);

/* bitpack.binarize: out[i] = x[i] >= 0 ? +1 : -1 (f32).  Sets
 * BNN_FLAG_NONFINITE in *flags (if non-null) when an input is not finite. */
int bnn_binarize_f32(const float *x, int64_t n, float *out, int32_t *flags,
                     bnn_stream_t stream);

/* bitpack.popcount64 (soft = 0, hardware POPC) / popcount64_soft (soft = 1, the
 * shift/mask sequence): out[i] = popcount(words[i]) as u8, i < n. */
int bnn_popcount64(const uint64_t *words, int64_t n, uint8_t *out, int soft,
                   bnn_stream_t stream);

/* pack_matrix_a(binarize(x)): x [R, K] f32, row stride ldx elements ->
 * out [R, ldo] u64 words (ldo >= ceil(K/64)); tail bits of the last word =
 * pad_bit.  Optional row_popc[R] receives popcount of each row's valid bits. */
int bnn_pack_rows_f32(const float *x, int64_t R, int64_t K, int64_t ldx, uint64_t *out,
                      int64_t ldo, int pad_bit, int mode, int32_t *row_popc, int32_t *flags,
                      bnn_stream_t stream);

/* pack_matrix_b: x [K, N] f32 (row stride ldx) -> out [ceil(K/64), ldo] u64
 * words (layout 'b', column n packed along K), tail bits = pad_bit. */
int bnn_pack_cols_f32(const float *x, int64_t K, int64_t N, int64_t ldx, uint64_t *out,
                      int64_t ldo, int pad_bit, int mode, int32_t *flags, bnn_stream_t stream);

/* Activation side of the binary conv: x NCHW [B, C, H, W] f32 -> packed
 * NHWC words out [B*H*W, ceil(C/64)] (channel c at bit c%64 of word c/64,
 * channel tail bits 0). */
int bnn_pack_nchw_f32(const float *x, int64_t B, int64_t C, int64_t H, int64_t W, uint64_t *out,
                      int mode, int32_t *flags, bnn_stream_t stream);

/* out[c, r] = in[r, c] for a [rows, cols] u64 word matrix (layout 'b' <-> K-contiguous). */
int bnn_words_transpose(const uint64_t *in, int64_t rows, int64_t cols, int64_t ldi,
                        uint64_t *out, int64_t ldo, bnn_stream_t stream);

/* audit_padding over `vectors` packed vectors of n_bits each: vector v's
 * last word is words[v * ld_vec + (W-1) * ld_word].  Sets *bad (device
 * int32, caller-zeroed) to 1 when a tail bit differs from pad_fill. */
int bnn_audit_padding(const uint64_t *words, int64_t vectors, int64_t n_bits, int64_t ld_vec,
                      int64_t ld_word, int pad_fill, int32_t *bad, bnn_stream_t stream);

/* xnor-popcount GEMM, both operands K-contiguous:
 *   A [M, lda] u64 (weights, layout 'a'), tail fill a_pad
 *   B [N, ldb] u64 (activations, one packed vector per row), tail fill b_pad
 *   P[m, n] = #{k < K : bit_k(A[m]) == bit_k(B[n])}
 *   C[m * ldc_m + n * ldc_n] = (domain == DOT ? 2P - K : P) * scale[m] + shift[m]
 * scale/shift are optional (null = 1 / 0).  K < 2^24. */
int bnn_xnor_gemm(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                  int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                  int64_t ldc_n, int domain, const float *scale, const float *shift, int algo,
                  bnn_stream_t stream);

/* bnn_xnor_gemm with a device workspace (same reference functions, gemm.py:226-291; plain
 * DOT / POPCOUNT output, no affine).  With ws_bytes >= bnn_xnor_gemm_ws_bytes(M, N, K)
 * (128-byte aligned; (M + N) * ceil(K / 64) * 32 bytes) large GEMMs run the pre-expanded
 * engine (BNN_ALGO_UMMA_XP above); every other case, and ws == NULL, is exactly
 * bnn_xnor_gemm.  Results are bit-identical either way.  The workspace is scratch: it is
 * overwritten by every call and must not be shared by calls on different streams. */
int64_t bnn_xnor_gemm_ws_bytes(int64_t M, int64_t N, int64_t K);
int bnn_xnor_gemm_ws(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                     int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                     int64_t ldc_n, int domain, int algo, void *ws, int64_t ws_bytes,
                     bnn_stream_t stream);

/* Multi-bit path (act_bit = weight_bit = bits):
 * k-bit quantize + bit-plane pack, x [R, K] f32 -> out[p * plane_stride + r * ldo + w]
 * (plane p = bit p of every code).  bits == 2. */
int bnn_pack_planes_f32(const float *x, int64_t R, int64_t K, int64_t ldx, int bits, int grid,
                        uint64_t *out, int64_t ldo, int64_t plane_stride, int32_t *flags,
                        bnn_stream_t stream);

/* Bit-plane GEMM: out[m, n] = sum_k v_a(m, k) * v_b(n, k) where v = grid value
 * of the code assembled from `bits` planes (A weights [bits][M][lda], B
 * activations [bits][N][ldb]).  Exact integer numerator, one f32 rounding of
 * the final division by L^2.  Engine: tcgen05 (codes expanded to u8 in SMEM /
 * TMEM; the MMA accumulates sum(code_a * code_b)). */
int bnn_bitplane_gemm(const uint64_t *A, int64_t lda, int64_t a_plane_stride, int a_grid,
                      const uint64_t *B, int64_t ldb, int64_t b_plane_stride, int b_grid,
                      int bits, int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                      int64_t ldc_n, bnn_stream_t stream);

/* bnn_bitplane_gemm with a device workspace of bnn_xnor_gemm_ws_bytes(M, N, K) bytes: large
 * shapes (and algo == BNN_ALGO_UMMA_XP) write each 2-bit code's grid value as an e2m1 number
 * (0..3 or -3, -1, +1, +3: exact) into the workspace and run the pre-expanded 2-CTA
 * kind::mxf4 GEMM, whose f32 accumulator is the integer numerator itself (9 K < 2^24); same
 * single f32 rounding, bit-identical outputs.  algo: AUTO, UMMA (planes engine) or UMMA_XP. */
int bnn_bitplane_gemm_ws(const uint64_t *A, int64_t lda, int64_t a_plane_stride, int a_grid,
                         const uint64_t *B, int64_t ldb, int64_t b_plane_stride, int b_grid,
                         int bits, int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                         int64_t ldc_n, int algo, void *ws, int64_t ws_bytes, bnn_stream_t stream);

/* Fused epilogue of the GEMM / conv (all fields optional except domain):
 *   v  = domain == BNN_DOT ? 2P - K : P
 *   v  = v * scale[m] + shift[m]                                  (affine)
 *   v  = gamma[m] * ((v - mean[m]) * inv_std[m]) + beta[m]         (inference
 *        BatchNorm in the reference's op order, layers.py:598-602, each op
 *        rounded as NumPy float32 does -- bit-identical to an unfused BN)
 *   out = v + residual[same index as out]                          (shortcut)
 *   sign-pack (tcgen05 engine only; the next layer's QActivation + pack,
 *   layers.py:409-413 -> bitpack.py:30-42,78-87, fused):
 *        bit m % 64 of pack_out[n * pack_ld + m / 64] = (out[m, n] >= 0)
 *        (-0.0 -> 1 like binarize), bits m >= M are 0, words past ceil(M/64)
 *        are not written; n is the output column:
 *        the NHWC pixel b*oh*ow + y*ow + x of a conv (packed NHWC input of the
 *        next bnn_bconv2d), the batch row of a GEMM (K-contiguous rows of the
 *        next layer).  pack_flags[0] is set to 1 when an out value is NaN/Inf
 *        (binarize's ValueError, bitpack.py:37-38).  The f32 output pointer may
 *        be null when only the packed words are wanted.
 */
typedef struct bnn_epilogue {
    int domain;
    const float *scale, *shift;
    const float *bn_mean, *bn_inv_std, *bn_gamma, *bn_beta;
    const float *residual;
    uint64_t *pack_out;   /* optional sign-packed copy of out, [cols][pack_ld] u64 */
    int64_t pack_ld;      /* >= ceil(M / 64) */
    int32_t *pack_flags;  /* optional non-finite flag word */
} bnn_epilogue;

/* bnn_xnor_gemm / bnn_bconv2d with the full fused epilogue. */
int bnn_xnor_gemm_ex(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                     int64_t N, int64_t K, int a_pad, int b_pad, float *C, int64_t ldc_m,
                     int64_t ldc_n, const bnn_epilogue *ep, int algo, bnn_stream_t stream);

/* bnn_bconv2d_ex with a device workspace (QConv2d.forward INFER_PACKED, layers.py:225-245, same
 * fused epilogue and results).  For C % 256 == 0, F % 64 == 0 and F <= 1024 (any stride <= 8)
 * and ws_bytes >= bnn_bconv2d_ws_bytes(...) (128-byte aligned), AUTO and BNN_ALGO_UMMA_XP run the
 * pre-expanded engine: activations (with a physical halo of +1 codes) and weights expanded once
 * to e2m1 codes in the workspace, im2col-mode TMA loads, 2-CTA kind::mxf4 GEMM with rows =
 * output pixels.  bnn_bconv2d_ws_bytes returns 0 for geometries the engine does not take;
 * every other case, and ws == NULL, is exactly bnn_bconv2d_ex.  The workspace is scratch. */
int64_t bnn_bconv2d_ws_bytes(int64_t B, int64_t C, int64_t H, int64_t W, int64_t F, int64_t kh,
                             int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw);
int bnn_bconv2d_ws(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                   const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                   int64_t ph, int64_t pw, float *y, const bnn_epilogue *e, int algo, void *ws,
                   int64_t ws_bytes, bnn_stream_t stream);

/* Float post-op of a full-precision stem conv (ResNet-18, configs[3]):
 * y = maxpool_k/stride/pad(relu?(BN(x))) with BN in the reference's op order,
 * bit-identical to the unfused sequence.  NCHW f32. */
int bnn_bn_relu_maxpool_f32(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                            const float *mean, const float *inv_std, const float *gamma,
                            const float *beta, int relu, int k, int stride, int pad, float *y,
                            bnn_stream_t stream);

/* Full-precision convolution of a network's float stem layer (reference
 * Conv2d, layers.py:81-141; ResNet-18 conv7x7/2 3->64, LeNet conv5x5 1->64):
 * y[B, F, oh, ow] = conv(x[B, C, H, W], w[F, C, kh, kw]) (+ bias[F]), zero
 * padding, NCHW f32.  tcgen05 kind::tf32 with a hi/lo operand split (three
 * terms x_hi w_hi + x_hi w_lo + x_lo w_hi; the ResNet-18 geometry -- C = 3, 7x7,
 * stride 2, pad 3, W = 224 -- runs the gather-free kernel bnn_stem_s2.cu, which
 * accumulates all four terms), f32 accumulate: f32 accuracy, rounding differs
 * from a CUDA-core f32 conv only in summation order.  F == 64 and
 * C*kh*kw <= 320 (BNN_EUNSUP otherwise). */
int bnn_conv2d_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                      const float *w, const float *bias, int64_t F, int64_t kh, int64_t kw,
                      int64_t sh, int64_t sw, int64_t ph, int64_t pw, float *y,
                      bnn_stream_t stream);

/* The ResNet-18 stem as one kernel: y = maxpool_3x3/2/1(relu?(BN(conv(x, w))))
 * (bnn_conv2d_f32_tc's conv, bnn_bn_relu_maxpool_f32's post-op; no bias).  The
 * pool runs on sign-adjusted conv outputs before the BatchNorm -- exact, since
 * the rounded BN + ReLU is monotone per channel -- so only the pooled tensor
 * is written.  BNN_EUNSUP outside F == 64, C*kh*kw <= 320, conv width <= 128,
 * W % 4 == 0 (run the two calls instead). */
int bnn_conv_bn_relu_maxpool_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                    const float *w, int64_t F, int64_t kh, int64_t kw,
                                    int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                    const float *mean, const float *inv_std, const float *gamma,
                                    const float *beta, int relu, float *y, bnn_stream_t stream);

/* The same, also writing the sign-packed NHWC words of y (the first binary
 * block's input; flags as the pack kernels), so no pack pass follows the stem. */
int bnn_conv_bn_relu_maxpool_pack_f32_tc(const float *x, int64_t B, int64_t C, int64_t H,
                                         int64_t W, const float *w, int64_t F, int64_t kh,
                                         int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                         const float *mean, const float *inv_std,
                                         const float *gamma, const float *beta, int relu,
                                         float *y, uint64_t *out_words, int32_t *flags,
                                         bnn_stream_t stream);

/* LeNet's float stem as one kernel: y = maxpool_2x2/2(tanh(conv(x, w) + bias))
 * (reference Conv2d -> Tanh -> MaxPool2d, layers.py:81-141, 480-540), the same
 * per-element f32 ops as the unfused sequence; bias may be null.  pool_first = 1
 * pools before the tanh (exact iff bnn_probe_tanh_monotone reported 0 violations
 * on this device; measured no faster, so callers pass 0).  BNN_EUNSUP outside
 * F == 64, C*kh*kw <= 320, conv width <= 128, W % 4 == 0. */
int bnn_conv_tanh_maxpool2_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                  const float *w, const float *bias, int64_t F, int64_t kh,
                                  int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                  int pool_first, float *y, bnn_stream_t stream);

/* The same kernel also writing the sign-packed NHWC words of y (u64 [B, PH, PW, F / 64]: the
 * next QConvolution's QActivation(act_bit = 1) + pack, bitpack.py:30-42 / 152-169, fused) and
 * OR-ing BNN_FLAG_NONFINITE into *flags (may be null).  y may be null: a binary consumer reads
 * only the words, and the f32 tensor is then never written. */
int bnn_conv_tanh_maxpool2_pack_f32_tc(const float *x, int64_t B, int64_t C, int64_t H, int64_t W,
                                       const float *w, const float *bias, int64_t F, int64_t kh,
                                       int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw,
                                       int pool_first, float *y, uint64_t *out_words,
                                       int32_t *flags, bnn_stream_t stream);

/* Adds to *violations_dev (device u64) the number of adjacent finite floats
 * a < b with tanhf(a) > tanhf(b) (exhaustive, ~4e9 evaluations).  0 means the
 * f32 tanh is monotone, which makes pooling before the tanh exact. */
int bnn_probe_tanh_monotone(unsigned long long *violations_dev, bnn_stream_t stream);

/* Max pooling of sign-packed NHWC words: out bit = OR over the k x k / stride
 * window (no padding) = sign(maxpool(x)) (x >= 0 is monotone: the max is >= 0
 * iff some element is) -- the pool between a binary layer's packed output and
 * the next binary layer. in [B, H, W, Cw] u64 -> out [B, OH, OW, Cw]. */
int bnn_maxpool_packed(const uint64_t *in, int64_t B, int64_t H, int64_t W, int64_t Cw, int k,
                       int stride, uint64_t *out, bnn_stream_t stream);
/* The same with out_batch_stride u64 words between the images of out (>= OH * OW * Cw): a
 * following QFullyConnected reads each image as one packed row, and an even stride keeps those
 * rows 16-byte aligned for the TMA-fed engine (LeNet: 49 words per image -> stride 50). */
int bnn_maxpool_packed_ld(const uint64_t *in, int64_t B, int64_t H, int64_t W, int64_t Cw, int k,
                          int stride, uint64_t *out, int64_t out_batch_stride, bnn_stream_t stream);

/* A residual block's output y = a + residual (NCHW f32, f32 add as torch) and its
 * sign-packed NHWC words (the next block's conv input); flags as the pack kernels.
 * (Used after 64-filter convs, where the conv epilogue without the shortcut add is
 * faster than the fused one.) */
int bnn_add_pack_nchw_f32(const float *a, const float *residual, int64_t B, int64_t C, int64_t H,
                          int64_t W, float *y, uint64_t *out_words, int32_t *flags,
                          bnn_stream_t stream);

/* Split-K combine (small GEMMs such as config 1: too few output tiles to fill
 * the SMs, so the caller runs word-aligned K ranges as concurrent popcount-
 * domain GEMMs into `splits` partial buffers, partial s at partials + s*stride,
 * and sums them here):  out[i] = sum_s partials[s*stride + i], or 2*sum - K
 * when domain == BNN_DOT.  The partials are integer counts < 2^24, so the
 * result is bit-identical to one unsplit bnn_xnor_gemm (the reference's
 * int32 accumulation, gemm.py:128-139, then .astype(float32)). */
int bnn_sum_partials_f32(const float *partials, int splits, int64_t count, int64_t stride,
                         int domain, int64_t K, float *out, bnn_stream_t stream);

/* A network's classifier head, GlobalAvgPool -> Dense (layers.py:266-317):
 * y[b, o] = sum_c (sum_t x[b, c, t] / HW) * w[o, c] + bias[o] (bias may be null),
 * x [B, C, HW] f32, w [O, C] f32, y [B, O] f32, pooled: caller scratch of B * C
 * f32 (receives the channel means).  Each output is summed in a fixed order that
 * depends only on its own image, so logits are bit-identical for any batch size or
 * batch shard (multi-GPU batch sharding).  Two launches (pool, classifier). */
int bnn_avgpool_fc_f32(const float *x, int64_t B, int64_t C, int64_t HW, const float *w,
                       const float *bias, int64_t O, float *y, float *pooled,
                       bnn_stream_t stream);

/* Words per pixel of the packed NHWC activation layout: ceil(C / 64). */
int64_t bnn_conv_channel_words(int64_t C);

/* Load-time re-layout of QConv2d.pack() words (layout 'a' of
 * W.reshape(F, C*kh*kw), bit order (c, i, j), layers.py:221) into the device
 * tap-major order [F, kh*kw, ceil(C/64)] (bit order (i, j, c), channel tail
 * 0).  Popcount is permutation-invariant, so outputs are unchanged. */
int bnn_conv_weights_reorder(const uint64_t *w_ref, int64_t F, int64_t C, int64_t kh,
                             int64_t kw, uint64_t *w_dev, bnn_stream_t stream);

/* Implicit-im2col binary convolution (QConv2d.forward INFER_PACKED):
 *   x_words  packed NHWC [B, H, W, ceil(C/64)] (bnn_pack_nchw_f32)
 *   w_dev    [F, kh*kw*ceil(C/64)] (bnn_conv_weights_reorder)
 *   y        f32 NCHW [B, F, oh, ow]
 * Spatial padding follows the reference composition im2col(zero pad) ->
 * binarize: a pad position is sign(0) = +1. */
int bnn_bconv2d(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                int64_t ph, int64_t pw, float *y, int domain, const float *scale,
                const float *shift, int algo, bnn_stream_t stream);


/* Roofline probe (synchronous): measured issue rate of a pipe on the
 * current device.  pipe 0 = POPC (32-bit population counts per second);
 * pipe 1 = dense tcgen05.mma kind::i8 and pipe 2 = kind::mxf4 (MACs per
 * second, one CTA per SM issuing 128x256 MMAs back to back); pipes 3 / 4 / 5 =
 * kind::mxf4 128x64 with A in TMEM / 128x64 from SMEM / 128x256 with A in TMEM.
 * `sink` is a caller-allocated device u32 the kernel may write. */
int bnn_probe_pipe_peak(int pipe, int64_t iters, uint32_t *sink, double *ops_per_sec,
                        bnn_stream_t stream);

int bnn_bconv2d_ex(const uint64_t *x_words, int64_t B, int64_t C, int64_t H, int64_t W,
                   const uint64_t *w_dev, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                   int64_t sw, int64_t ph, int64_t pw, float *y, const bnn_epilogue *ep, int algo,
                   bnn_stream_t stream);

/* ------------------------------------------------------------------------
 * DEBUG knobs.  Process-wide, NOT thread-safe, all off by default; the product
 * path never sets them (they serve the experiment scripts under tools/).  Some
 * produce wrong results on purpose (timing ablations).
 * ------------------------------------------------------------------------ */
enum bnn_debug_knob {
    BNN_DEBUG_UMMA_BITS = 1,       /* tcgen05 engine debug bit flags: 16 timelines into the
                                    * bnn_umma_trace buffer, 1 << 15 no cluster split-K,
                                    * 1 << 17 shifted-window conv also for C >= 256,
                                    * 1 << 19 no shifted-window conv, 1 << 14 two
                                    * superstages per TMA load, 1 << 29 no POPC pointwise
                                    * (1x1) conv route, 1 << 18 no small-channel
                                    * kernels, bits 21-24 role ablations (wrong results) */
    BNN_DEBUG_FP4_BN = 2,          /* force the kind::mxf4 tile N (0 = by shape)     */
    BNN_DEBUG_PAIR_KW32 = 3,       /* 2-CTA pairs from this K in u32 words (0 = off) */
    BNN_DEBUG_STEM_BITS = 4,       /* float-stem kernels: 1 / 2 / 4 ablations (wrong results),
                                    * 8 timeline, 16 the im2col-gather kernel for every shape */
    BNN_DEBUG_PACK_PIX = 5,        /* NCHW pack kernel variant (0 = default)         */
    BNN_DEBUG_PACK_CH = 6,         /* NCHW pack channels per lane (0 = default 8)    */
    BNN_DEBUG_STEMPOST_SIMPLE = 7, /* unbanded BN/ReLU/maxpool kernel                */
    BNN_DEBUG_GRID_CAP = 8         /* tcgen05 kernels: at most this many CTAs (0 = #SMs) */
};
int bnn_debug_set(int knob, int64_t value);

/* Debug timeline of the tcgen05 engine: buf is a device array of
 * (#SMs x 16) u64 %globaltimer stamps written by later launches
 * (slot 0 start, 1 setup done, 2 first stage consumed, 3/6/9 tile MMA done,
 * 4/7/10 epilogue start, 5/8/11 epilogue end, 12 exit); null disables. */
int bnn_umma_trace(uint64_t *buf);

/* Debug: arm the tcgen05 engine's wait watchdog (the plain-epilogue kernels) with
 * a device log of BNN_WATCHDOG_WORDS u64 (word 0 count, 1..64 records of a wait
 * that did not complete in ~2 s -- block / warp / barrier / parity --, then the
 * progress marks and raw barrier words; the kernel traps), or null. */
#define BNN_WATCHDOG_WORDS 225
int bnn_umma_watchdog(uint64_t *log);

/* Debug: *dst = %globaltimer (ns) when a one-thread kernel on `stream` runs. */
int bnn_debug_stamp(uint64_t *dst, bnn_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* BNN_B200_H */
