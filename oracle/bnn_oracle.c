/*
 * bnn_oracle.c -- CPU restatement of the reference's binarise/pack/xnor path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path lives in
 * paper_1705_09864_b200/csrc and fails loudly without its CUDA library.
 *
 * Each function restates one reference function (bitnn, /root/reference/pkg/
 * src/bitnn/...) in plain C.  Parity of this restatement is pinned by
 * tests/test_oracle_golden.py against vectors produced by the reference
 * itself (tests/golden/gen_golden_vectors.py).
 *
 * Word format (bitpack.py:1-16): bit k of a packed vector lives in u64 word
 * k/64 at bit k%64 (LSB-first); bit value 1 <=> sign +1.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ENONFINITE (-1)
#define ORC_ENOTSIGN (-2)
#define ORC_EINVAL (-3)

/* host ISA is unknown at build time (the .so is built here and shipped to
 * the GPU box): let the loader pick AVX-512 VPOPCNTQ / AVX2 / generic. */
#define ORC_CLONES __attribute__((target_clones("arch=icelake-server", "arch=haswell", "default")))

static inline int64_t words_per_bits(int64_t n) { return (n + 63) / 64; }

/* ------------------------------------------------------------------ */
/* simple static row partition over pthreads: same contract as
 * xnor_gemm_parallel, gemm.py:254-284 (contiguous disjoint spans,
 * result independent of the worker count).                             */
typedef void (*span_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { span_fn fn; void *ctx; int64_t lo, hi; } span_job;

static void *span_entry(void *p) {
    span_job *j = (span_job *)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static void run_spans(span_fn fn, void *ctx, int64_t total, int threads) {
    if (threads < 1) threads = 1;
    if (threads > total) threads = (int)(total > 0 ? total : 1);
    if (threads == 1) { fn(ctx, 0, total); return; }
    int64_t step = (total + threads - 1) / threads;
    pthread_t tid[256];
    span_job job[256];
    if (threads > 256) threads = 256;
    int n = 0;
    for (int64_t lo = 0; lo < total && n < threads; lo += step, ++n) {
        job[n].fn = fn; job[n].ctx = ctx; job[n].lo = lo;
        job[n].hi = lo + step < total ? lo + step : total;
        pthread_create(&tid[n], NULL, span_entry, &job[n]);
    }
    for (int i = 0; i < n; ++i) pthread_join(tid[i], NULL);
}

/* ------------------------------------------------------------------ */
/* bitpack.binarize (bitpack.py:30-42): sign(x) with x >= 0 -> +1 (so
 * -0.0 and 0.0 map to +1); any non-finite input raises ValueError
 * (:37-38) -> ORC_ENONFINITE here.                                      */
int orc_binarize_f32(const float *x, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return ORC_ENONFINITE;
    for (int64_t i = 0; i < n; ++i) out[i] = x[i] >= 0.0f ? 1.0f : -1.0f;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* pack_matrix_a (bitpack.py:144-149) via _pack_last_axis (:78-87):
 * +-1 rows [R, K] -> u64 words [R, ceil(K/64)], tail bits = pad_fill.
 * _validate_signs (:69-75): every entry must be exactly +-1.          */
typedef struct { const float *x; int64_t K; uint64_t *out; int pad; int bad; } pack_rows_ctx;

static void pack_rows_span(void *p, int64_t lo, int64_t hi) {
    pack_rows_ctx *c = (pack_rows_ctx *)p;
    int64_t W = words_per_bits(c->K);
    for (int64_t r = lo; r < hi; ++r) {
        const float *row = c->x + r * c->K;
        for (int64_t w = 0; w < W; ++w) {
            uint64_t word = 0;
            for (int b = 0; b < 64; ++b) {
                int64_t k = w * 64 + b;
                int bit;
                if (k < c->K) {
                    float v = row[k];
                    if (v == 1.0f) bit = 1;
                    else if (v == -1.0f) bit = 0;
                    else { c->bad = 1; bit = 0; }
                } else {
                    bit = c->pad;
                }
                word |= (uint64_t)bit << b;
            }
            c->out[r * W + w] = word;
        }
    }
}

int orc_pack_rows(const float *signs, int64_t R, int64_t K, uint64_t *out, int pad_fill,
                  int threads) {
    if (R < 0 || K < 0 || (pad_fill != 0 && pad_fill != 1)) return ORC_EINVAL;
    pack_rows_ctx c = {signs, K, out, pad_fill, 0};
    run_spans(pack_rows_span, &c, R, threads);
    return c.bad ? ORC_ENOTSIGN : ORC_OK;
}

/* pack_matrix_b (bitpack.py:152-169): +-1 columns of [K, N] -> words
 * [ceil(K/64), N] (K-major), tail bits = pad_fill (the reference uses 1). */
typedef struct { const float *x; int64_t K, N; uint64_t *out; int pad; int bad; } pack_cols_ctx;

ORC_CLONES static void pack_cols_span(void *p, int64_t lo, int64_t hi) {
    pack_cols_ctx *c = (pack_cols_ctx *)p;
    int64_t W = words_per_bits(c->K);
    /* lo/hi index words of K; inner loop over contiguous N like the
     * reference's byte interleave (:165-168) */
    for (int64_t w = lo; w < hi; ++w) {
        uint64_t *dst = c->out + w * c->N;
        for (int64_t n = 0; n < c->N; ++n) dst[n] = 0;
        for (int b = 0; b < 64; ++b) {
            int64_t k = w * 64 + b;
            if (k < c->K) {
                const float *src = c->x + k * c->N;
                for (int64_t n = 0; n < c->N; ++n) {
                    float v = src[n];
                    uint64_t bit;
                    if (v == 1.0f) bit = 1;
                    else if (v == -1.0f) bit = 0;
                    else { c->bad = 1; bit = 0; }
                    dst[n] |= bit << b;
                }
            } else if (c->pad) {
                for (int64_t n = 0; n < c->N; ++n) dst[n] |= (uint64_t)1 << b;
            }
        }
    }
    (void)W;
}

int orc_pack_cols(const float *signs, int64_t K, int64_t N, uint64_t *out, int pad_fill,
                  int threads) {
    if (K < 0 || N < 0 || (pad_fill != 0 && pad_fill != 1)) return ORC_EINVAL;
    pack_cols_ctx c = {signs, K, N, out, pad_fill, 0};
    run_spans(pack_cols_span, &c, words_per_bits(K), threads);
    return c.bad ? ORC_ENOTSIGN : ORC_OK;
}

/* Fused binarize + pack of raw f32 rows, as the reference composes
 * pack_matrix_a(binarize(x)) (layers.py:221, gemm.py:406-408).  Returns
 * ORC_ENONFINITE if any element is NaN/Inf (bitpack.py:37-38).          */
typedef struct { const float *x; int64_t K; uint64_t *out; int pad; int bad; } bpack_ctx;

ORC_CLONES static void bpack_rows_span(void *p, int64_t lo, int64_t hi) {
    bpack_ctx *c = (bpack_ctx *)p;
    int64_t W = words_per_bits(c->K);
    for (int64_t r = lo; r < hi; ++r) {
        const float *row = c->x + r * c->K;
        for (int64_t w = 0; w < W; ++w) {
            uint64_t word = 0;
            for (int b = 0; b < 64; ++b) {
                int64_t k = w * 64 + b;
                uint64_t bit;
                if (k < c->K) {
                    float v = row[k];
                    if (!isfinite(v)) c->bad = 1;
                    bit = v >= 0.0f;
                } else {
                    bit = (uint64_t)c->pad;
                }
                word |= bit << b;
            }
            c->out[r * W + w] = word;
        }
    }
}

int orc_binarize_pack_rows(const float *x, int64_t R, int64_t K, uint64_t *out, int pad_fill,
                           int threads) {
    if (R < 0 || K < 0 || (pad_fill != 0 && pad_fill != 1)) return ORC_EINVAL;
    bpack_ctx c = {x, K, out, pad_fill, 0};
    run_spans(bpack_rows_span, &c, R, threads);
    return c.bad ? ORC_ENONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------ */
/* xnor kernel family (gemm.py:80-159), restated on the parallel
 * variant's traversal (gemm.py:117-139 hot loop, :254-284 partition):
 * C[m, n] = sum_w popcount(~(A[m, w] ^ B[w, n])), int32 accumulate.
 * A: layout 'a' [M, W]; B: layout 'b' [W, N].  Tails must be
 * complementary (a: 0, b: 1) so whole-word counts are exact
 * (bitpack.py:12-15).                                                  */
typedef struct {
    const uint64_t *a, *b; int64_t N, W; int32_t *c; int64_t block_rows, block_words;
} xnor_ctx;

ORC_CLONES static void xnor_span(void *p, int64_t m0, int64_t m1) {
    xnor_ctx *x = (xnor_ctx *)p;
    const int64_t N = x->N, W = x->W;
    for (int64_t mb = m0; mb < m1; mb += x->block_rows) {
        int64_t m_hi = mb + x->block_rows < m1 ? mb + x->block_rows : m1;
        for (int64_t wb = 0; wb < W; wb += x->block_words) {
            int64_t w_hi = wb + x->block_words < W ? wb + x->block_words : W;
            for (int64_t m = mb; m < m_hi; ++m) {
                int32_t *crow = x->c + m * N;
                int64_t w = wb;
                for (; w + 2 <= w_hi; w += 2) {
                    uint64_t a0 = x->a[m * W + w], a1 = x->a[m * W + w + 1];
                    const uint64_t *b0 = x->b + w * N, *b1 = x->b + (w + 1) * N;
                    for (int64_t j = 0; j < N; ++j)
                        crow[j] += (int32_t)__builtin_popcountll(~(a0 ^ b0[j])) +
                                   (int32_t)__builtin_popcountll(~(a1 ^ b1[j]));
                }
                if (w < w_hi) {
                    uint64_t a0 = x->a[m * W + w];
                    const uint64_t *b0 = x->b + w * N;
                    for (int64_t j = 0; j < N; ++j)
                        crow[j] += (int32_t)__builtin_popcountll(~(a0 ^ b0[j]));
                }
            }
        }
    }
}

/* C must be zeroed by the caller (gemm.py:453 allocates zeros). */
void orc_xnor_gemm(const uint64_t *a, const uint64_t *b, int64_t M, int64_t N, int64_t W,
                   int32_t *c, int threads) {
    xnor_ctx x = {a, b, N, W, c, 32, 512}; /* DEFAULT_BLOCK_ROWS/WORDS gemm.py:46-47 */
    run_spans(xnor_span, &x, M, threads);
}

/* Row-major B variant: both operands K-contiguous ([M, W] and [N, W]).
 * Identity: P = K_eff - sum popc(a ^ b).  Used by the
 * CPU baseline on the same operand layout the GPU consumes.            */
typedef struct { const uint64_t *a, *b; int64_t N, W; int32_t *c; } xnor_rr_ctx;

ORC_CLONES static void xnor_rr_span(void *p, int64_t m0, int64_t m1) {
    xnor_rr_ctx *x = (xnor_rr_ctx *)p;
    const int64_t N = x->N, W = x->W;
    for (int64_t m = m0; m < m1; ++m) {
        const uint64_t *ar = x->a + m * W;
        for (int64_t n = 0; n < N; ++n) {
            const uint64_t *br = x->b + n * W;
            int32_t s = 0;
            for (int64_t w = 0; w < W; ++w) s += (int32_t)__builtin_popcountll(ar[w] ^ br[w]);
            x->c[m * N + n] = s;
        }
    }
}

void orc_xor_popc_gemm_rowrow(const uint64_t *a, const uint64_t *b, int64_t M, int64_t N,
                              int64_t W, int32_t *c, int threads) {
    xnor_rr_ctx x = {a, b, N, W, c};
    run_spans(xnor_rr_span, &x, M, threads);
}

/* ------------------------------------------------------------------ */
/* tensor.im2col (tensor.py:60-78 / _im2col_fill :30-42): [B,C,H,W] ->
 * [C*kh*kw, B*oh*ow]; rows (c,i,j), columns (b,oy,ox); zero padding
 * (np.pad, :73-74).                                                    */
typedef struct {
    const float *x; int B, C, H, W, kh, kw, sh, sw, ph, pw, oh, ow; float *cols;
} im2col_ctx;

static void im2col_span(void *p, int64_t lo, int64_t hi) {
    im2col_ctx *c = (im2col_ctx *)p;
    int64_t ncol = (int64_t)c->B * c->oh * c->ow;
    for (int64_t row = lo; row < hi; ++row) {
        int ci = (int)(row / (c->kh * c->kw));
        int i = (int)((row / c->kw) % c->kh);
        int j = (int)(row % c->kw);
        float *dst = c->cols + row * ncol;
        for (int bi = 0; bi < c->B; ++bi)
            for (int oy = 0; oy < c->oh; ++oy) {
                int iy = oy * c->sh + i - c->ph;
                for (int ox = 0; ox < c->ow; ++ox) {
                    int ix = ox * c->sw + j - c->pw;
                    float v = 0.0f;
                    if (iy >= 0 && iy < c->H && ix >= 0 && ix < c->W)
                        v = c->x[(((int64_t)bi * c->C + ci) * c->H + iy) * c->W + ix];
                    dst[((int64_t)bi * c->oh + oy) * c->ow + ox] = v;
                }
            }
    }
}

int orc_im2col_f32(const float *x, int B, int C, int H, int W, int kh, int kw, int sh, int sw,
                   int ph, int pw, float *cols, int threads) {
    /* tensor.conv_output_hw (tensor.py:15-27) */
    if (B < 1 || C < 1 || H < 1 || W < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 ||
        pw < 0)
        return ORC_EINVAL;
    int oh = (H + 2 * ph - kh) / sh + 1, ow = (W + 2 * pw - kw) / sw + 1;
    if (oh < 1 || ow < 1) return ORC_EINVAL;
    im2col_ctx c = {x, B, C, H, W, kh, kw, sh, sw, ph, pw, oh, ow, cols};
    run_spans(im2col_span, &c, (int64_t)C * kh * kw, threads);
    return ORC_OK;
}

int orc_version(void) { return 1; }
