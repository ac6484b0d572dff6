// Pipe-peak probes: measure the roofline denominators the bench reports
// against (the POPC pipe has no vendor figure for sm_100a; SURVEY 0 asks
// for a microbenchmark before the 16/clk/SM figure is used).
#include "bnn_common.cuh"

namespace bnn {

// 8 independent LOP3+POPC chains per thread: one ALU op per POPC, so the
// loop is POPC-bound unless POPC runs at the full ALU rate.
__global__ void probe_popc_kernel(uint32_t seed, int64_t iters, uint32_t *sink) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    const uint32_t k0 = seed ^ 0x5bd1e995u, k1 = seed ^ 0x1b873593u;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __popc(v[i] ^ ((i & 1) ? k1 : k0));
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc ^= v[i];
    if (acc == 0x12345678u) sink[0] = acc;  // keep the loop alive
}

}  // namespace bnn

using namespace bnn;

extern "C" int bnn_probe_pipe_peak(int pipe, int64_t iters, uint32_t *sink,
                                   double *ops_per_sec, bnn_stream_t stream) {
    if (pipe != 0 || iters < 1 || !ops_per_sec || !sink)
        return set_error(BNN_EINVAL, "probe: pipe must be 0 (POPC), iters >= 1, sink non-null");
    int sms = bnn_device_sm_count();
    if (sms <= 0) return set_error(BNN_ECUDA, "probe: no CUDA device");
    cudaStream_t s = as_stream(stream);
    const int threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe_popc_kernel<<<blocks, threads, 0, s>>>(1u, iters / 8 + 1, sink);  // warm-up
    cudaEventRecord(e0, s);
    probe_popc_kernel<<<blocks, threads, 0, s>>>(7u, iters, sink);
    cudaEventRecord(e1, s);
    int rc = check_launch("probe_popc_kernel");
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    *ops_per_sec = (double)blocks * threads * (double)iters * 8.0 / (ms * 1e-3);
    return BNN_OK;
}

// debug: dst[0] = %globaltimer when this one-thread kernel runs (timeline probes)
static __global__ void stamp_kernel(uint64_t *dst) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *dst = t;
}

extern "C" int bnn_debug_stamp(uint64_t *dst, bnn_stream_t stream) {
    stamp_kernel<<<1, 1, 0, as_stream(stream)>>>(dst);
    return check_launch("stamp_kernel");
}
