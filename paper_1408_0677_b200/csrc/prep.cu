// prep.cu -- device-side MLS input staging (field.py:596-613 `compute_field`
// set-up): column means pm / qm, centred controls pc = p - pm, and the padded
// target block q (qc, or dq = qc - pc[:, axis] for the mean variant,
// _kernels.py:52-67) in the kernel's compute dtype.  Replaces ~40 ms of host
// numpy per 100k x 32 frame with a few microseconds of device work after one
// H2D of the raw (pinned) inputs.
//
// The means use a fixed chunking and a fixed reduction order, so they are
// deterministic and identical on every rank (row-band sharding stays
// bit-identical to one GPU); they can differ from numpy's pairwise mean in
// the last bit, which the fp64 (1e-10) and fp32 (1e-4) contracts absorb.
#include "common.cuh"

namespace mdc {

constexpr int PREP_CH = 128;  // fixed row chunks for the column sums
constexpr int PREP_RL = 8;    // row lanes per block

// part[ch][c] = sum of column c over row chunk ch; columns 0,1 = positions,
// 2.. = targets.  block (32 columns, PREP_RL row lanes), fixed lane order.
__global__ void prep_partial_kernel(int64_t n, int d, const double *pos, const double *tv, double *part) {
    __shared__ double red[PREP_RL][32];
    const int ch = blockIdx.x;
    const int c = blockIdx.y * 32 + threadIdx.x;
    const int ncol = d + 2;
    const int64_t r0 = n * ch / PREP_CH, r1 = n * (ch + 1) / PREP_CH;
    double s = 0.0;
    if (c < ncol) {
        for (int64_t i = r0 + threadIdx.y; i < r1; i += PREP_RL)
            s += c < 2 ? pos[2 * i + c] : tv[i * d + (c - 2)];
    }
    red[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && c < ncol) {
        double t = 0.0;
        for (int l = 0; l < PREP_RL; ++l) t += red[l][threadIdx.x];
        part[(int64_t)ch * ncol + c] = t;
    }
}

__global__ void prep_mean_kernel(int64_t n, int d, const double *part, double *pm, double *qm) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int ncol = d + 2;
    if (c >= ncol) return;
    double s = 0.0;
    for (int ch = 0; ch < PREP_CH; ++ch) s += part[(int64_t)ch * ncol + c];
    const double m = s / (double)n;
    if (c < 2)
        pm[c] = m;
    else
        qm[c - 2] = m;
}

template <typename T>
__global__ void prep_center_kernel(int64_t n, int d, int ldq, int mean_variant, const double *pos, const double *tv,
                                   const int32_t *axis, const double *pm, const double *qm, double *pc, T *q) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * ldq) return;
    const int64_t i = e / ldq;
    const int c = (int)(e - i * ldq);
    if (c < 2) pc[2 * i + c] = pos[2 * i + c] - pm[c];
    T v = T(0);
    if (c < d) {
        double x = tv[i * d + c] - qm[c];
        if (mean_variant) {
            const int a = axis[c];
            x = x - (pos[2 * i + a] - pm[a]);
        }
        v = (T)x;
    }
    q[e] = v;
}

}  // namespace mdc

extern "C" size_t mdc_mls_prepare_workspace_bytes(int32_t d) {
    return sizeof(double) * (size_t)mdc::PREP_CH * (size_t)(d + 2) + 256;
}

extern "C" int mdc_mls_prepare(int64_t n, int32_t d, const double *positions, const double *tvals, int32_t variant,
                               int32_t dtype, const int32_t *axis, int32_t ldq, double *pc, void *q, double *pm,
                               double *qm, void *workspace, size_t workspace_bytes, void *stream) {
    using namespace mdc;
    MDC_REQUIRE(n >= 1 && d >= 1 && ldq >= d, "bad sizes");
    MDC_REQUIRE(positions && tvals && pc && q && pm && qm && workspace, "null pointer");
    MDC_REQUIRE(dtype == MDC_F32 || dtype == MDC_F64, "dtype must be MDC_F32 or MDC_F64");
    MDC_REQUIRE(variant != MDC_MEAN || axis, "mean variant needs the axis map");
    MDC_REQUIRE(workspace_bytes >= mdc_mls_prepare_workspace_bytes(d), "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    double *part = reinterpret_cast<double *>(workspace);
    const int ncol = d + 2;
    prep_partial_kernel<<<dim3(PREP_CH, (ncol + 31) / 32), dim3(32, PREP_RL), 0, s>>>(n, d, positions, tvals, part);
    prep_mean_kernel<<<(ncol + 127) / 128, 128, 0, s>>>(n, d, part, pm, qm);
    const int64_t total = n * (int64_t)ldq;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    const int mv = variant == MDC_MEAN ? 1 : 0;
    if (dtype == MDC_F32)
        prep_center_kernel<float><<<blocks, 256, 0, s>>>(n, d, ldq, mv, positions, tvals, axis, pm, qm, pc,
                                                         reinterpret_cast<float *>(q));
    else
        prep_center_kernel<double><<<blocks, 256, 0, s>>>(n, d, ldq, mv, positions, tvals, axis, pm, qm, pc,
                                                          reinterpret_cast<double *>(q));
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
