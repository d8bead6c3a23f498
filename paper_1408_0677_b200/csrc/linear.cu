// linear.cu -- the "linear" field variant on B200: barycentric interpolation
// over the mesh triangles, extended outside the hull by the nearest hull
// triangle's plane.
//
// Replaces _kernels.rasterize_linear (_kernels.py:233-269; serial, the FIRST
// covering triangle wins) and _kernels.extend_hull (_kernels.py:272-313), as
// driven by field._linear_field (field.py:497-515).  First-wins becomes an
// atomicMin on the triangle index (owner = the lowest covering triangle),
// which is exactly the serial loop's outcome.  Compiled with -fmad=false so
// every inside test and barycentric weight is the reference's IEEE sequence.
#include <math.h>

#include "common.cuh"

namespace mdc {

struct LinArgs {
    int width, height, row0, row1;
    double x0, y1, sx, sy;
    int64_t n, ntri;
    int nch, dtype;
    const double *pos, *tvals;
    const int32_t *tris;  // ntri x 3
    const int32_t *hull;  // nhull x 3: u, v, triangle (field._hull_edges order)
    int nhull;
    void *out;
    int64_t out_cs, out_rs, out_ps;
    int32_t *owner;  // band pixels, all INT32_MAX between calls
};

__device__ __forceinline__ double2 P(const LinArgs &a, int i) { return reinterpret_cast<const double2 *>(a.pos)[i]; }

// one warp per triangle; lanes stride over the triangle's pixel bounding box
__global__ void tri_owner_kernel(LinArgs a) {
    int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (t >= a.ntri) return;
    int ia = a.tris[3 * t], ib = a.tris[3 * t + 1], ic = a.tris[3 * t + 2];
    double2 A = P(a, ia), B = P(a, ib), C = P(a, ic);
    double det = (B.x - A.x) * (C.y - A.y) - (B.y - A.y) * (C.x - A.x);
    if (det == 0.0) return;
    double xlo = fmin(A.x, fmin(B.x, C.x)), xhi = fmax(A.x, fmax(B.x, C.x));
    double ylo = fmin(A.y, fmin(B.y, C.y)), yhi = fmax(A.y, fmax(B.y, C.y));
    long long c0 = (long long)floor((xlo - a.x0) / a.sx - 0.5), c1 = (long long)ceil((xhi - a.x0) / a.sx);
    long long r0 = (long long)floor((a.y1 - yhi) / a.sy - 0.5), r1 = (long long)ceil((a.y1 - ylo) / a.sy);
    if (c0 < 0) c0 = 0;
    if (c1 > a.width - 1) c1 = a.width - 1;
    if (r0 < a.row0) r0 = a.row0;
    if (r1 > a.row1 - 1) r1 = a.row1 - 1;
    if (c0 > c1 || r0 > r1) return;
    long long bw = c1 - c0 + 1, cnt = bw * (r1 - r0 + 1);
    for (long long e = lane; e < cnt; e += 32) {
        long long row = r0 + e / bw, col = c0 + e % bw;
        double gy = a.y1 - ((double)row + 0.5) * a.sy;
        double gx = a.x0 + ((double)col + 0.5) * a.sx;
        double l1 = ((B.x - gx) * (C.y - gy) - (B.y - gy) * (C.x - gx)) / det;
        double l2 = ((C.x - gx) * (A.y - gy) - (C.y - gy) * (A.x - gx)) / det;
        double l3 = 1.0 - l1 - l2;
        if (l1 >= -1e-12 && l2 >= -1e-12 && l3 >= -1e-12)
            atomicMin(&a.owner[(row - a.row0) * (int64_t)a.width + col], (int32_t)t);
    }
}

__global__ void linear_value_kernel(LinArgs a) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t npix = (int64_t)(a.row1 - a.row0) * a.width;
    if (e >= npix) return;
    int64_t lr = e / a.width, col = e - lr * a.width;
    int64_t row = a.row0 + lr;
    double gy = a.y1 - ((double)row + 0.5) * a.sy;
    double gx = a.x0 + ((double)col + 0.5) * a.sx;
    int t = a.owner[e];
    a.owner[e] = INT32_MAX;
    if (t == INT32_MAX) {
        // extend_hull: nearest hull segment, strict <, hull order
        double best = INFINITY;
        int best_t = 0;
        for (int k = 0; k < a.nhull; ++k) {
            double2 U = P(a, a.hull[3 * k]), V = P(a, a.hull[3 * k + 1]);
            double ex = V.x - U.x, ey = V.y - U.y;
            double ee = ex * ex + ey * ey, s = 0.0;
            if (ee > 0.0) {
                s = ((gx - U.x) * ex + (gy - U.y) * ey) / ee;
                if (s < 0.0)
                    s = 0.0;
                else if (s > 1.0)
                    s = 1.0;
            }
            double ddx = gx - (U.x + s * ex), ddy = gy - (U.y + s * ey);
            double d2 = ddx * ddx + ddy * ddy;
            if (d2 < best) {
                best = d2;
                best_t = a.hull[3 * k + 2];
            }
        }
        t = best_t;
    }
    int ia = a.tris[3 * t], ib = a.tris[3 * t + 1], ic = a.tris[3 * t + 2];
    double2 A = P(a, ia), B = P(a, ib), C = P(a, ic);
    double det = (B.x - A.x) * (C.y - A.y) - (B.y - A.y) * (C.x - A.x);
    double l1 = ((B.x - gx) * (C.y - gy) - (B.y - gy) * (C.x - gx)) / det;
    double l2 = ((C.x - gx) * (A.y - gy) - (C.y - gy) * (A.x - gx)) / det;
    double l3 = 1.0 - l1 - l2;
    for (int k = 0; k < a.nch; ++k) {
        double v = l1 * a.tvals[(int64_t)ia * a.nch + k] + l2 * a.tvals[(int64_t)ib * a.nch + k] +
                   l3 * a.tvals[(int64_t)ic * a.nch + k];
        int64_t off = k * a.out_cs + lr * a.out_rs + col * a.out_ps;
        if (a.dtype == MDC_F32)
            reinterpret_cast<float *>(a.out)[off] = (float)v;
        else
            reinterpret_cast<double *>(a.out)[off] = v;
    }
}

}  // namespace mdc

extern "C" size_t mdc_linear_workspace_bytes(int32_t width, int32_t rows) {
    return (size_t)width * (size_t)rows * sizeof(int32_t);
}

extern "C" int mdc_linear_field(const MdcLinearArgs *p, void *stream) {
    using namespace mdc;
    MDC_REQUIRE(p && p->pos && p->tvals && p->tris && p->out && p->workspace, "null pointer");
    MDC_REQUIRE(p->ntri >= 1, "linear interpolation needs at least one triangle");
    MDC_REQUIRE(p->nhull >= 1 && p->hull, "linear interpolation needs the hull edge list");
    MDC_REQUIRE(0 <= p->row0 && p->row0 <= p->row1 && p->row1 <= p->height, "bad row band");
    MDC_REQUIRE(p->nch >= 1, "need at least one channel");
    LinArgs a;
    a.width = p->width;
    a.height = p->height;
    a.row0 = p->row0;
    a.row1 = p->row1;
    a.x0 = p->x0;
    a.y1 = p->y1;
    a.sx = p->sx;
    a.sy = p->sy;
    a.n = p->n;
    a.ntri = p->ntri;
    a.nch = p->nch;
    a.dtype = p->dtype;
    a.pos = p->pos;
    a.tvals = p->tvals;
    a.tris = p->tris;
    a.hull = p->hull;
    a.nhull = p->nhull;
    a.out = p->out;
    a.out_cs = p->out_cs;
    a.out_rs = p->out_rs;
    a.out_ps = p->out_ps;
    a.owner = reinterpret_cast<int32_t *>(p->workspace);
    cudaStream_t s = (cudaStream_t)stream;
    int64_t npix = (int64_t)(p->row1 - p->row0) * p->width;
    if (npix == 0) return MDC_OK;
    tri_owner_kernel<<<(unsigned)((p->ntri * 32 + 255) / 256), 256, 0, s>>>(a);
    linear_value_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(a);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
