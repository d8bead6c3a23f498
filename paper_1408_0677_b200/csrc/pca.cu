// pca.cu -- PCA projection numerics (projection.py:50-79) on B200, fp64.
//
//   mean      : column means, fixed 64-chunk partials summed in chunk order
//   cov       : centred X^T X / (n-1) as 32x32 tiles over 64 fixed row chunks,
//               partial tiles reduced in chunk order (deterministic)
//   eigh      : one-CTA parallel cyclic Jacobi (round-robin pairing, d/2
//               disjoint rotations per round), matrices in global memory
//   axes      : top-2 eigenpairs, descending, sign rule projection.py:71-74
//   positions : (x - mean) @ axes^T
#include <math.h>

#include "common.cuh"

namespace mdc {

constexpr int PCA_CH = 64;  // fixed row chunks -> run-to-run deterministic sums
constexpr int CT = 32;      // covariance tile

__global__ void col_partial_kernel(int64_t n, int d, const double *x, double *part) {
    int ch = blockIdx.x;
    int64_t r0 = n * ch / PCA_CH, r1 = n * (ch + 1) / PCA_CH;
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        double s = 0.0;
        for (int64_t i = r0; i < r1; ++i) s += x[i * d + j];
        part[(int64_t)ch * d + j] = s;
    }
}

__global__ void col_mean_kernel(int64_t n, int d, const double *part, double *mean) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d) return;
    double s = 0.0;
    for (int ch = 0; ch < PCA_CH; ++ch) s += part[(int64_t)ch * d + j];
    mean[j] = s / (double)n;
}

__global__ void __launch_bounds__(CT *CT) cov_partial_kernel(int64_t n, int d, const double *x,
                                                            const double *mean, double *part) {
    __shared__ double sa[CT][CT + 1], sb[CT][CT + 1];
    int ta = blockIdx.x * CT, tb = blockIdx.y * CT, ch = blockIdx.z;
    int tx = threadIdx.x % CT, ty = threadIdx.x / CT;
    int64_t r0 = n * ch / PCA_CH, r1 = n * (ch + 1) / PCA_CH;
    double acc = 0.0;
    for (int64_t base = r0; base < r1; base += CT) {
        int64_t i = base + ty;
        int ca = ta + tx, cb = tb + tx;
        sa[ty][tx] = (i < r1 && ca < d) ? x[i * d + ca] - mean[ca] : 0.0;
        sb[ty][tx] = (i < r1 && cb < d) ? x[i * d + cb] - mean[cb] : 0.0;
        __syncthreads();
#pragma unroll 8
        for (int r = 0; r < CT; ++r) acc += sa[r][ty] * sb[r][tx];
        __syncthreads();
    }
    int a = ta + ty, b = tb + tx;
    if (a < d && b < d) part[((int64_t)ch * d + a) * d + b] = acc;
}

__global__ void cov_reduce_kernel(int64_t n, int d, const double *part, double *cov, double *A) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)d * d) return;
    double s = 0.0;
    for (int ch = 0; ch < PCA_CH; ++ch) s += part[(int64_t)ch * d * d + e];
    s /= (double)(n - 1);
    cov[e] = s;
    A[e] = s;
}

// Parallel cyclic Jacobi, one CTA.  A (d x d) destroyed; V receives the
// eigenvectors as columns.  Round-robin "circle" pairing over m2 = d rounded
// up to even; the phantom index d (odd d) never rotates.
__global__ void __launch_bounds__(1024) jacobi_kernel(int d, double *A, double *V, double *evals,
                                                      double *axes, double *eig2) {
    extern __shared__ double sh[];
    double *cs = sh, *sn = sh + 512;
    int *pp = reinterpret_cast<int *>(sh + 1024), *qq = pp + 512;
    __shared__ double red[32];
    __shared__ int stop;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int e = tid; e < d * d; e += nt) V[e] = (e / d == e % d) ? 1.0 : 0.0;
    const int m2 = (d + 1) & ~1, np = m2 / 2;
    __syncthreads();
    for (int sweep = 0; sweep < 60; ++sweep) {
        // convergence test: off-diagonal vs total Frobenius mass
        double off = 0.0, tot = 0.0;
        for (int e = tid; e < d * d; e += nt) {
            double v = A[e] * A[e];
            tot += v;
            if (e / d != e % d) off += v;
        }
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            tot += __shfl_xor_sync(0xffffffffu, tot, o);
        }
        if ((tid & 31) == 0) red[tid >> 5] = off;
        __syncthreads();
        if (tid == 0) {
            double so = 0.0;
            for (int w = 0; w < (nt + 31) / 32; ++w) so += red[w];
            red[0] = so;
        }
        __syncthreads();
        double so = red[0];
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = tot;
        __syncthreads();
        if (tid == 0) {
            double st = 0.0;
            for (int w = 0; w < (nt + 31) / 32; ++w) st += red[w];
            stop = (so == 0.0 || so <= 1e-32 * st) ? 1 : 0;
        }
        __syncthreads();
        if (stop) break;
        for (int r = 0; r < m2 - 1; ++r) {
            for (int j = tid; j < np; j += nt) {
                int p, q;
                if (j == 0) {
                    p = 0;
                    q = 1 + r % (m2 - 1);
                } else {
                    p = 1 + (r + j) % (m2 - 1);
                    q = 1 + (r - j + (m2 - 1)) % (m2 - 1);
                }
                if (p > q) {
                    int t = p;
                    p = q;
                    q = t;
                }
                double c = 1.0, s = 0.0;
                if (q < d) {
                    double apq = A[p * d + q];
                    if (apq != 0.0) {
                        double app = A[p * d + p], aqq = A[q * d + q];
                        double th = (aqq - app) / (2.0 * apq);
                        double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                cs[j] = c;
                sn[j] = s;
                pp[j] = p;
                qq[j] = q < d ? q : -1;
            }
            __syncthreads();
            // rows: A <- J^T A
            for (int e = tid; e < np * d; e += nt) {
                int j = e / d, k = e % d;
                int p = pp[j], q = qq[j];
                if (q < 0 || sn[j] == 0.0) continue;
                double c = cs[j], s = sn[j];
                double apk = A[p * d + k], aqk = A[q * d + k];
                A[p * d + k] = c * apk - s * aqk;
                A[q * d + k] = s * apk + c * aqk;
            }
            __syncthreads();
            // columns: A <- A J, V <- V J
            for (int e = tid; e < np * d; e += nt) {
                int j = e / d, k = e % d;
                int p = pp[j], q = qq[j];
                if (q < 0 || sn[j] == 0.0) continue;
                double c = cs[j], s = sn[j];
                double akp = A[k * d + p], akq = A[k * d + q];
                A[k * d + p] = c * akp - s * akq;
                A[k * d + q] = s * akp + c * akq;
                double vkp = V[k * d + p], vkq = V[k * d + q];
                V[k * d + p] = c * vkp - s * vkq;
                V[k * d + q] = s * vkp + c * vkq;
            }
            __syncthreads();
        }
    }
    for (int k = tid; k < d; k += nt) evals[k] = A[k * d + k];
    __syncthreads();
    if (tid == 0) {
        // top-2 by descending eigenvalue (projection.py:61-63)
        int i0 = 0;
        for (int k = 1; k < d; ++k)
            if (evals[k] > evals[i0]) i0 = k;
        int i1 = i0 == 0 ? 1 : 0;
        for (int k = 0; k < d; ++k)
            if (k != i0 && evals[k] > evals[i1]) i1 = k;
        int idx[2] = {i0, i1};
        for (int a = 0; a < 2; ++a) {
            eig2[a] = fmax(evals[idx[a]], 0.0);
            int jm = 0;
            double best = -1.0;
            for (int k = 0; k < d; ++k) {
                double v = fabs(V[k * d + idx[a]]);
                if (v > best) {
                    best = v;
                    jm = k;
                }
            }
            double sgn = V[jm * d + idx[a]] < 0 ? -1.0 : 1.0;
            for (int k = 0; k < d; ++k) axes[a * d + k] = sgn * V[k * d + idx[a]];
        }
    }
}

__global__ void project_kernel(int64_t n, int d, const double *x, const double *mean,
                               const double *axes, double *pos) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s0 = 0.0, s1 = 0.0;
    for (int j = 0; j < d; ++j) {
        double c = x[i * d + j] - mean[j];
        s0 += c * axes[j];
        s1 += c * axes[d + j];
    }
    pos[2 * i] = s0;
    pos[2 * i + 1] = s1;
}

}  // namespace mdc

extern "C" size_t mdc_pca_workspace_bytes(int64_t n, int32_t d) {
    (void)n;
    size_t dd = (size_t)d * d;
    return sizeof(double) * ((size_t)mdc::PCA_CH * d + (size_t)mdc::PCA_CH * dd + 2 * dd + d + 256);
}

extern "C" int mdc_pca(int64_t n, int32_t d, const double *x, double *mean, double *cov,
                       double *eigenvalues, double *axes, double *positions, void *workspace,
                       void *stream) {
    using namespace mdc;
    MDC_REQUIRE(n >= 2 && d >= 2 && d <= 1024, "pca needs n >= 2 and 2 <= d <= 1024");
    MDC_REQUIRE(x && mean && cov && eigenvalues && axes && positions && workspace, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    double *w = reinterpret_cast<double *>(workspace);
    double *pmean = w;
    double *pcov = pmean + (size_t)PCA_CH * d;
    double *A = pcov + (size_t)PCA_CH * d * d;
    double *V = A + (size_t)d * d;
    double *ev = V + (size_t)d * d;
    col_partial_kernel<<<PCA_CH, 256, 0, s>>>(n, d, x, pmean);
    col_mean_kernel<<<(d + 255) / 256, 256, 0, s>>>(n, d, pmean, mean);
    dim3 g((d + CT - 1) / CT, (d + CT - 1) / CT, PCA_CH);
    cov_partial_kernel<<<g, CT * CT, 0, s>>>(n, d, x, mean, pcov);
    int64_t dd = (int64_t)d * d;
    cov_reduce_kernel<<<(unsigned)((dd + 255) / 256), 256, 0, s>>>(n, d, pcov, cov, A);
    size_t shm = sizeof(double) * 1024 + sizeof(int) * 1024;
    jacobi_kernel<<<1, 1024, shm, s>>>(d, A, V, ev, axes, eigenvalues);
    project_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, d, x, mean, axes, positions);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
