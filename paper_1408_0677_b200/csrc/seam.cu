// seam.cu -- one-to-one replacements of the reference's numba kernels.
//
// Same argument meaning and out-parameter convention as
// /root/reference/pkg/src/mdcontour/_kernels.py (mean_field :52-67,
// affine_field :70-124, rigid_field :127-175, bh_forces :178-230), with every
// array a DEVICE pointer.  A maintainer binds these from _kernels.py with
// ctypes and nothing else in the reference changes.  They
// evaluate the reference's own one-pass fp64 formulas (global-frame moments),
// so their outputs track the numba kernels to a few ulps; the fused,
// throughput path is mdc_mls_field (mls.cu).
#include <math.h>

#include "common.cuh"

namespace mdc {

constexpr int SEAM_T = 256;

__device__ __forceinline__ double seam_weight(double d2, double alpha) {
    // _kernels.py:37-49
    if (d2 < 1e-300) d2 = 1e-300;
    if (alpha == 1.0) return 1.0 / d2;
    if (alpha == 1.5) return 1.0 / (d2 * sqrt(d2));
    if (alpha == 0.5) return 1.0 / sqrt(d2);
    if (alpha == 2.0) return 1.0 / (d2 * d2);
    return pow(d2, -alpha);
}

template <int VAR>
__global__ void __launch_bounds__(SEAM_T) seam_mls_kernel(int64_t npix, const double *vx, const double *vy,
                                                         int64_t n, const double *px, const double *py,
                                                         const double *qx, const double *qy, double alpha,
                                                         double reg_eps, double *out, double *norm_out) {
    __shared__ double4 sc[SEAM_T];
    int64_t i = (int64_t)blockIdx.x * SEAM_T + threadIdx.x;
    bool ok = i < npix;
    double x = ok ? vx[i] : 0.0, y = ok ? vy[i] : 0.0;
    double sw = 0, mpx = 0, mpy = 0, mqx = 0, mqy = 0, mpxpx = 0, mpxpy = 0, mpypy = 0;
    double mpxqx = 0, mpxqy = 0, mpyqx = 0, mpyqy = 0;
    for (int64_t base = 0; base < n; base += SEAM_T) {
        int64_t j = base + threadIdx.x;
        __syncthreads();
        if (j < n) sc[threadIdx.x] = make_double4(px[j], py[j], qx[j], qy[j]);
        __syncthreads();
        int cnt = (int)min((int64_t)SEAM_T, n - base);
        for (int jj = 0; jj < cnt; ++jj) {
            double4 c = sc[jj];
            double dx = __dsub_rn(c.x, x), dy = __dsub_rn(c.y, y);
            double w = seam_weight(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), alpha);
            sw = __dadd_rn(sw, w);
            if (VAR == MDC_MEAN) {
                mqx = __dadd_rn(mqx, __dmul_rn(w, c.z));
                mqy = __dadd_rn(mqy, __dmul_rn(w, c.w));
                continue;
            }
            mpx = __dadd_rn(mpx, __dmul_rn(w, c.x));
            mpy = __dadd_rn(mpy, __dmul_rn(w, c.y));
            mqx = __dadd_rn(mqx, __dmul_rn(w, c.z));
            mqy = __dadd_rn(mqy, __dmul_rn(w, c.w));
            if (VAR == MDC_AFFINE) {
                mpxpx = __dadd_rn(mpxpx, __dmul_rn(__dmul_rn(w, c.x), c.x));
                mpxpy = __dadd_rn(mpxpy, __dmul_rn(__dmul_rn(w, c.x), c.y));
                mpypy = __dadd_rn(mpypy, __dmul_rn(__dmul_rn(w, c.y), c.y));
            }
            mpxqx = __dadd_rn(mpxqx, __dmul_rn(__dmul_rn(w, c.x), c.z));
            mpxqy = __dadd_rn(mpxqy, __dmul_rn(__dmul_rn(w, c.x), c.w));
            mpyqx = __dadd_rn(mpyqx, __dmul_rn(__dmul_rn(w, c.y), c.z));
            mpyqy = __dadd_rn(mpyqy, __dmul_rn(__dmul_rn(w, c.y), c.w));
        }
    }
    if (!ok) return;
    if (VAR == MDC_MEAN) {  // _kernels.py:66-67 (q passed as dq)
        out[2 * i] = x + mqx / sw;
        out[2 * i + 1] = y + mqy / sw;
        return;
    }
    double psx = mpx / sw, psy = mpy / sw, qsx = mqx / sw, qsy = mqy / sw;
    double b00 = mpxqx - qsx * mpx, b01 = mpxqy - qsy * mpx;
    double b10 = mpyqx - qsx * mpy, b11 = mpyqy - qsy * mpy;
    double dx = x - psx, dy = y - psy;
    if (VAR == MDC_AFFINE) {  // _kernels.py:102-124
        double a00 = mpxpx - psx * mpx, a01 = mpxpy - psx * mpy, a11 = mpypy - psy * mpy;
        double reg = reg_eps * (a00 + a11);
        a00 += reg;
        a11 += reg;
        double det = a00 * a11 - a01 * a01;
        double m00 = (a11 * b00 - a01 * b10) / det, m01 = (a11 * b01 - a01 * b11) / det;
        double m10 = (a00 * b10 - a01 * b00) / det, m11 = (a00 * b11 - a01 * b01) / det;
        out[2 * i] = dx * m00 + dy * m10 + qsx;
        out[2 * i + 1] = dx * m01 + dy * m11 + qsy;
        return;
    }
    // rigid, _kernels.py:153-175
    double s = b00 + b11, d = b10 - b01;
    double fx = dx * s + dy * d, fy = dy * s - dx * d;
    double norm = hypot(fx, fy);
    if (norm_out) norm_out[i] = norm;  // field.py:263-265: the scalar evaluator raises on it
    if (norm < 1e-12) {
        out[2 * i] = x + (mqx - mpx) / sw;
        out[2 * i + 1] = y + (mqy - mpy) / sw;
    } else {
        double r = hypot(dx, dy) / norm;
        out[2 * i] = fx * r + qsx;
        out[2 * i + 1] = fy * r + qsy;
    }
}

// _kernels.py:178-230, one thread per point over the caller's flat tree.
__global__ void seam_bh_kernel(int64_t n, const double *pts, const int64_t *perm, const int64_t *lo,
                               const int64_t *hi, const int64_t *left, const int64_t *right,
                               const double *com, const double *mass, const double *size,
                               const double *bmin, const double *bmax, double c, double eta, double theta,
                               double *out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double xi = pts[2 * i], yi = pts[2 * i + 1], fx = 0.0, fy = 0.0;
    int64_t stack[128];
    int sp = 1;
    stack[0] = 0;
    while (sp > 0) {
        int64_t node = stack[--sp];
        if (left[node] < 0) {
            for (int64_t k = lo[node]; k < hi[node]; ++k) {
                int64_t j = perm[k];
                if (j == i) continue;
                double dx = xi - pts[2 * j], dy = yi - pts[2 * j + 1];
                double r2 = dx * dx + dy * dy;
                double w = c / (r2 * sqrt(r2) + eta);
                fx += w * dx;
                fy += w * dy;
            }
            continue;
        }
        double gx = bmin[2 * node] - xi;
        if (gx < 0.0) gx = xi - bmax[2 * node];
        if (gx < 0.0) gx = 0.0;
        double gy = bmin[2 * node + 1] - yi;
        if (gy < 0.0) gy = yi - bmax[2 * node + 1];
        if (gy < 0.0) gy = 0.0;
        double box_dist = sqrt(gx * gx + gy * gy);
        if (size[node] < theta * box_dist) {
            double dx = xi - com[2 * node], dy = yi - com[2 * node + 1];
            double r = sqrt(dx * dx + dy * dy);
            double coef = c * mass[node] / (r * r * r + eta);
            fx += coef * dx;
            fy += coef * dy;
        } else {
            stack[sp++] = left[node];
            stack[sp++] = right[node];
        }
    }
    out[2 * i] = fx;
    out[2 * i + 1] = fy;
}

template <int VAR>
static int launch_seam(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                       const double *py, const double *qx, const double *qy, double alpha, double reg_eps,
                       double *out, void *stream, double *norm_out = nullptr) {
    MDC_REQUIRE(npix >= 0 && n >= 1, "need at least one control");
    MDC_REQUIRE(vx && vy && px && py && qx && qy && out, "null device pointer");
    if (npix == 0) return MDC_OK;
    seam_mls_kernel<VAR><<<(unsigned)((npix + SEAM_T - 1) / SEAM_T), SEAM_T, 0, (cudaStream_t)stream>>>(
        npix, vx, vy, n, px, py, qx, qy, alpha, reg_eps, out, norm_out);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

}  // namespace mdc

extern "C" int mdc_mean_field(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                              const double *py, const double *dqx, const double *dqy, double alpha,
                              double *out, void *stream) {
    return mdc::launch_seam<MDC_MEAN>(npix, vx, vy, n, px, py, dqx, dqy, alpha, 0.0, out, stream);
}

extern "C" int mdc_affine_field(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                                const double *py, const double *qx, const double *qy, double alpha,
                                double reg_eps, double *out, void *stream) {
    return mdc::launch_seam<MDC_AFFINE>(npix, vx, vy, n, px, py, qx, qy, alpha, reg_eps, out, stream);
}

extern "C" int mdc_rigid_field(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                               const double *py, const double *qx, const double *qy, double alpha, double *out,
                               void *stream) {
    return mdc::launch_seam<MDC_RIGID>(npix, vx, vy, n, px, py, qx, qy, alpha, 0.0, out, stream);
}

extern "C" int mdc_rigid_field_norm(int64_t npix, const double *vx, const double *vy, int64_t n,
                                    const double *px, const double *py, const double *qx, const double *qy,
                                    double alpha, double *out, double *norm_out, void *stream) {
    MDC_REQUIRE(norm_out != nullptr, "null norm_out");
    return mdc::launch_seam<MDC_RIGID>(npix, vx, vy, n, px, py, qx, qy, alpha, 0.0, out, stream, norm_out);
}

extern "C" int mdc_bh_forces(int64_t n, const double *points, const int64_t *perm, const int64_t *lo,
                             const int64_t *hi, const int64_t *left, const int64_t *right, const double *com,
                             const double *mass, const double *size, const double *bmin, const double *bmax,
                             double c, double eta, double theta, double *out, void *stream) {
    MDC_REQUIRE(n >= 0, "n must be >= 0");
    MDC_REQUIRE(points && perm && lo && hi && left && right && com && mass && size && bmin && bmax && out,
                "null device pointer");
    if (n == 0) return MDC_OK;
    mdc::seam_bh_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        n, points, perm, lo, hi, left, right, com, mass, size, bmin, bmax, c, eta, theta, out);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
