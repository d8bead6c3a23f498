// capi.cu -- error reporting and device queries shared by the C-ABI.
#include <string>

#include "common.cuh"

namespace mdc {
static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
int num_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return sms;
}
}  // namespace mdc

extern "C" const char *mdc_last_error(void) { return mdc::g_err.c_str(); }
extern "C" int mdc_version(void) { return 1; }
extern "C" int mdc_num_sms(void) { return mdc::num_sms(); }

extern "C" int mdc_copy_2d_async(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width_bytes,
                                 size_t height, void *stream) {
    MDC_REQUIRE(dst && src, "null pointer");
    MDC_CHECK_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, height, cudaMemcpyDefault,
                                     (cudaStream_t)stream));
    return MDC_OK;
}
