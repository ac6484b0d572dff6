// BNN_ALGO_UMMA entry points with the fused sign-pack epilogue:
// the next layer's QActivation + pack (layers.py:409-413, bitpack.py:30-42,78-87)
// run in the epilogue.  Separate instantiations (Store::kPack) so the plain
// epilogue keeps its register budget; this translation unit compiles in
// parallel with bnn_gemm_umma.cu.
#include "bnn_umma_impl.cuh"

namespace bnn {

int launch_xnor_gemm_umma_pk(const uint64_t *A, int64_t lda, const uint64_t *B, int64_t ldb,
                             int64_t M, int64_t N, int64_t K, float *C, int64_t ldc_m,
                             int64_t ldc_n, const Epilogue &ep, cudaStream_t s, const float *res) {
    return launch_xnor_gemm_umma_t<GemmStorePk>(A, lda, B, ldb, M, N, K, C, ldc_m, ldc_n, ep, s,
                                                res);
}

int launch_bconv2d_umma_pk(const uint64_t *x, int64_t B, int64_t C, int64_t H, int64_t W,
                           const uint64_t *w, int64_t F, int64_t kh, int64_t kw, int64_t sh,
                           int64_t sw, int64_t ph, int64_t pw, int64_t oh, int64_t ow, float *y,
                           const Epilogue &ep, cudaStream_t s, const float *res) {
    return launch_bconv2d_umma_t<ConvStorePk>(x, B, C, H, W, w, F, kh, kw, sh, sw, ph, pw, oh, ow,
                                              y, ep, s, res);
}

}  // namespace bnn
