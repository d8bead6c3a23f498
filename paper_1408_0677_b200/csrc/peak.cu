// peak.cu -- FP32 / FP64 FMA-pipe peak kernels for the roofline denominators
// (MEASURED_PEAKS.json carries only HBM and bf16; SURVEY.md §7 hard part 6).
// Each thread runs 8 independent FMA chains; the caller times the launch with
// CUDA events and divides 2 * 8 * iters * blocks * 256 by the duration.
#include "common.cuh"

namespace mdc {
template <typename T>
__global__ void __launch_bounds__(256) peak_fma(T *sink, int iters) {
    T a[8];
    T x = (T)threadIdx.x * (T)1e-7, y = (T)0.999999;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = x + (T)k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], y, x);
        }
    }
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == (T)-1.2345) sink[0] = s;  // never true; keeps the chains alive
}
}  // namespace mdc

extern "C" int mdc_peak_ffma(float *sink, int32_t blocks, int32_t iters, void *stream) {
    mdc::peak_fma<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
extern "C" int mdc_peak_dfma(double *sink, int32_t blocks, int32_t iters, void *stream) {
    mdc::peak_fma<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
