// common.cuh -- shared helpers for libmdc (B200 / sm_100a).
#pragma once
#include <mutex>
#include <set>
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/mdc.h"

namespace mdc {

void set_error(const std::string &msg);

#define MDC_CHECK_CUDA(expr)                                                                \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess) {                                                            \
            ::mdc::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));           \
            return MDC_ECUDA;                                                               \
        }                                                                                   \
    } while (0)

#define MDC_CHECK_LAUNCH()                                                                  \
    do {                                                                                    \
        cudaError_t _e = cudaGetLastError();                                                \
        if (_e != cudaSuccess) {                                                            \
            ::mdc::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e) +      \
                             " at " + __FILE__ + ":" + std::to_string(__LINE__));           \
            return MDC_ECUDA;                                                               \
        }                                                                                   \
    } while (0)

#define MDC_REQUIRE(cond, msg)                                                              \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            ::mdc::set_error(msg);                                                          \
            return MDC_EINVAL;                                                              \
        }                                                                                   \
    } while (0)

int num_sms();

// fp64 arithmetic with the reference's exact rounding sequence (no FMA
// contraction): numpy evaluates each binary op with one IEEE rounding.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }


// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device),
// thread-safe (the service launches from several Python threads and one
// process may drive more than one device).
inline cudaError_t ensure_dynamic_smem(const void *kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

}  // namespace mdc
