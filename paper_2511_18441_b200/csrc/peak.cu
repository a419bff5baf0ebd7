// FP32 FMA throughput probe: the roofline denominator for the rasteriser, which
// is FP32-issue bound (no tensor cores, little HBM traffic).  Every SM runs
// 8 independent FFMA chains per thread; the result is FLOP/s (2 per FFMA) over
// CUDA events on the given stream.
#include "common.cuh"

namespace rcgs {

__global__ void __launch_bounds__(256) fma_peak_kernel(int iters, float seed, float* __restrict__ sink) {
    float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
    float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
    const float m = 0.9999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fmaf(a0, m, c);
            a1 = fmaf(a1, m, c);
            a2 = fmaf(a2, m, c);
            a3 = fmaf(a3, m, c);
            a4 = fmaf(a4, m, c);
            a5 = fmaf(a5, m, c);
            a6 = fmaf(a6, m, c);
            a7 = fmaf(a7, m, c);
        }
    }
    const float r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 1234.5f) sink[threadIdx.x] = r;  // keep the chains alive
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_fp32_peak(int32_t iters, double* h_flops, void* stream) {
    RCGS_CHECK_ARG(h_flops != nullptr && iters > 0, "bad argument");
    cudaStream_t s = as_stream(stream);
    int dev = 0, sms = 0, per_sm = 0;
    RCGS_CUDA(cudaGetDevice(&dev));
    RCGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RCGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fma_peak_kernel, 256, 0));
    const int blocks = sms * (per_sm > 0 ? per_sm : 1);
    float* sink = nullptr;
    RCGS_TRY(dalloc(&sink, 256, s));
    cudaEvent_t e0, e1;
    RCGS_CUDA(cudaEventCreate(&e0));
    RCGS_CUDA(cudaEventCreate(&e1));
    fma_peak_kernel<<<blocks, 256, 0, s>>>(iters / 4 + 1, 1.f, sink);  // warm-up
    RCGS_CUDA(cudaEventRecord(e0, s));
    fma_peak_kernel<<<blocks, 256, 0, s>>>(iters, 1.f, sink);
    RCGS_CUDA(cudaEventRecord(e1, s));
    RCGS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RCGS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dfree(sink, s);
    *h_flops = (double)blocks * 256.0 * (double)iters * 16.0 * 8.0 * 2.0 / (ms * 1e-3);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}
