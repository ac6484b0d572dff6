// BNN_ALGO_UMMA entry points (tcgen05 engine; kernel in bnn_umma_impl.cuh).
// Outputs with the fused sign-pack epilogue dispatch to bnn_gemm_umma_pk.cu.
#include "bnn_umma_impl.cuh"

namespace bnn {


int launch_xnor_gemm_umma_pk(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                             int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                             int64_t ldc_n, const Epilogue &ep, cudaStream_t s, const float *res);
int launch_bconv2d_umma_pk(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                           const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                           int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y,
                           const Epilogue &ep, cudaStream_t s, const float *res);

int launch_xnor_gemm_splitk(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb, int64_t M,
                            int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                            const Epilogue &ep, cudaStream_t s, const float *res);

int launch_xnor_gemm_umma(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                          int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                          const Epilogue &ep, cudaStream_t s, const float *res) {
    if (ep.pack_out)
        return launch_xnor_gemm_umma_pk(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep, s, res);
    if (ep.variant == 2) {  // small GEMMs: one cluster per row tile, in-kernel split-K
        const int rc = launch_xnor_gemm_splitk(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep, s, res);
        if (rc != BNN_EUNSUP) return rc;
    }
    return launch_xnor_gemm_umma_t<GemmStore>(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep, s, res);
}

int launch_bitplane_gemm_umma(const uint64_t *A, int64_t lda, int64_t a_plane,
                              const uint64_t *B, int64_t ldb, int64_t b_plane, int64_t M,
                              int64_t N, int64_t K, float *C, int64_t ldc_m, int64_t ldc_n,
                              const Epilogue &ep, cudaStream_t s) {
    const int64_t kw32 = 2 * ceil_div(K, 64);
    DenseRows a{reinterpret_cast<const uint32_t *>(A), 2 * lda, M, kw32, 2 * a_plane};
    DenseRows b{reinterpret_cast<const uint32_t *>(B), 2 * ldb, N, kw32, 2 * b_plane};
    GemmStore st{C, ldc_m, ldc_n, M, N};
    const bool vec4 = (lda % 2 == 0) && (ldb % 2 == 0) && (a_plane % 2 == 0) &&
                      (b_plane % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
    switch (choose_bn(M, N)) {
        case 128:
            return vec4 ? launch_umma_cfg<128, true, 4, DenseRows, DenseRows, GemmStore, 2>(a, b, st, ep, M, N, kw32, s)
                        : launch_umma_cfg<128, true, 2, DenseRows, DenseRows, GemmStore, 2>(a, b, st, ep, M, N, kw32, s);
        default:
            return vec4 ? launch_umma_cfg<192, true, 4, DenseRows, DenseRows, GemmStore, 2>(a, b, st, ep, M, N, kw32, s)
                        : launch_umma_cfg<192, true, 2, DenseRows, DenseRows, GemmStore, 2>(a, b, st, ep, M, N, kw32, s);
    }
}

int launch_bconv2d_umma(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                        const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                        int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y,
                        const Epilogue &ep, cudaStream_t s, const float *res) {
    if (ep.pack_out)
        return launch_bconv2d_umma_pk(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, oh, ow, y, ep,
                                      s, res);
    return launch_bconv2d_umma_t<ConvStore>(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, oh, ow, y,
                                            ep, s, res);
}

}  // namespace bnn

// debug: arm the wait watchdog of this translation unit's kernels (the plain-epilogue
// instantiations; buf = device u64[BNN_WATCHDOG_WORDS]: count, records, marks), or null
extern "C" int bnn_umma_watchdog(uint64_t *buf) {
    cudaMemcpyToSymbol(bnn::umma::g_wait_log, &buf, sizeof(buf));
    return bnn::check_launch("bnn_umma_watchdog");
}

extern "C" int bnn_umma_trace(uint64_t *buf) {
    // debug: buf = device array of (#SMs x 16) u64 timestamps, or null to disable
    bnn::g_debug.trace_buf = buf;
    return BNN_OK;
}
