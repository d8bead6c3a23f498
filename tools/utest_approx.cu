// Accuracy of rsqrt.approx.ftz.f64 / rcp.approx.ftz.f64 and of one/two
// Newton corrections against correctly rounded fp64 (experiments only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/utest_approx tools/utest_approx.cu
#include <stdio.h>
#include <math.h>
__global__ void k(int n, double *err) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = exp2(-40.0 + 80.0 * (double)i / n) * (1.0 + 0.37 * sin((double)i));
    double y, r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double ry = 1.0 / sqrt(x), rr = 1.0 / x;
    double e = fma(-x * y, y, 1.0);
    double y1 = fma(y, 0.5 * e, y);
    double y2 = fma(y * e, fma(0.375, e, 0.5), y);
    double f = fma(-x, r, 1.0);
    double r1 = fma(r, f, r);
    double r2 = fma(r, fma(f, f, f), r);
    atomicMax((unsigned long long *)&err[0], __double_as_longlong(fabs(y / ry - 1)));
    atomicMax((unsigned long long *)&err[1], __double_as_longlong(fabs(y1 / ry - 1)));
    atomicMax((unsigned long long *)&err[2], __double_as_longlong(fabs(y2 / ry - 1)));
    atomicMax((unsigned long long *)&err[3], __double_as_longlong(fabs(r / rr - 1)));
    atomicMax((unsigned long long *)&err[4], __double_as_longlong(fabs(r1 / rr - 1)));
    atomicMax((unsigned long long *)&err[5], __double_as_longlong(fabs(r2 / rr - 1)));
}
int main() {
    double *e;
    cudaMallocManaged(&e, 6 * sizeof(double));
    for (int i = 0; i < 6; ++i) e[i] = 0;
    int n = 1 << 24;
    k<<<n / 256, 256>>>(n, e);
    cudaDeviceSynchronize();
    const char *nm[6] = {"rsqrt.approx", "rsqrt+1 newton", "rsqrt+2nd order", "rcp.approx", "rcp+1 newton", "rcp+2nd order"};
    for (int i = 0; i < 6; ++i) printf("%-18s max rel err %.3e (2^%.1f)\n", nm[i], e[i], log2(e[i] > 0 ? e[i] : 1e-300));
    return 0;
}
