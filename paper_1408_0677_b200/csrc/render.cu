// render.cu -- band shading + anti-aliased isocontours from an MLS field.
//
// Replaces render.line_coverage (render.py:116-126), _gradient_magnitudes
// (render.py:110-113, CoordinateField.jacobian = np.gradient, field.py:154-161),
// _band_indices / render_discrete (render.py:135-148), render_contours
// (render.py:129-132) and the compositing helpers _over / _to_image
// (render.py:91-102).  All arithmetic is fp64 in the reference's order, so a
// field that matches the reference renders to the same RGBA bytes.
#include <math.h>

#include "common.cuh"

namespace mdc {

struct RArgs {
    int mode, dtype, width, height, nimg, channels;
    const void *values;
    int64_t img_stride, cs, rs, ps;
    const double *spacing;
    double line_width;
    double lc[4], bg[4];
    const double *cmap;  // ncolors x 4, already /255
    int ncolors;
    uint8_t *out;        // nimg x H x W x 4
    float *coverage;     // optional nimg x H x W
};

template <typename T>
__device__ __forceinline__ double val(const RArgs &a, int img, int c, int r, int x) {
    const T *v = reinterpret_cast<const T *>(a.values);
    return (double)v[img * a.img_stride + c * a.cs + (int64_t)r * a.rs + (int64_t)x * a.ps];
}

// np.gradient along one axis (unit spacing, edge_order=1)
template <typename T>
__device__ __forceinline__ double grad(const RArgs &a, int img, int c, int r, int x, bool along_x) {
    int lim = along_x ? a.width : a.height;
    int i = along_x ? x : r;
    if (lim < 2) return 0.0;
    auto at = [&](int k) { return along_x ? val<T>(a, img, c, r, k) : val<T>(a, img, c, k, x); };
    if (i == 0) return at(1) - at(0);
    if (i == lim - 1) return at(lim - 1) - at(lim - 2);
    return (at(i + 1) - at(i - 1)) / 2.0;
}

__device__ __forceinline__ void over(double *base, const double *src, double alpha) {
    // render.py:91-97
    double aa = fmin(fmax(alpha, 0.0), 1.0) * src[3];
    for (int k = 0; k < 3; ++k) base[k] = base[k] * (1.0 - aa) + src[k] * aa;
    base[3] = base[3] * (1.0 - aa) + aa;
}

template <typename T>
__global__ void render_kernel(RArgs a) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t npix = (int64_t)a.width * a.height;
    if (e >= npix * a.nimg) return;
    int img = (int)(e / npix);
    int64_t pix = e - (int64_t)img * npix;
    int r = (int)(pix / a.width), x = (int)(pix - (int64_t)r * a.width);
    const double s = a.spacing[img];
    double cov = 0.0;
    long long band = 0;
    for (int c = 0; c < a.channels; ++c) {
        double v = val<T>(a, img, c, r, x);
        band += (long long)floor(v / s);
        if (a.mode != 1) {
            double dist = fabs(v - s * rint(v / s));
            double g = hypot(grad<T>(a, img, c, r, x, true), grad<T>(a, img, c, r, x, false));
            double px = g > 1e-30 ? dist / g : INFINITY;
            cov = fmax(cov, fmin(fmax(0.5 * a.line_width + 0.5 - px, 0.0), 1.0));
        }
    }
    double rgba[4];
    if (a.mode == 0) {  // contour: background + lines
        for (int k = 0; k < 4; ++k) rgba[k] = a.bg[k];
        over(rgba, a.lc, cov);
    } else {  // discrete (+contour)
        long long m = band % a.ncolors;
        if (m < 0) m += a.ncolors;
        for (int k = 0; k < 4; ++k) rgba[k] = a.cmap[m * 4 + k];
        if (a.mode == 2) over(rgba, a.lc, cov);
    }
    uint8_t *o = a.out + e * 4;
    for (int k = 0; k < 4; ++k) o[k] = (uint8_t)fmin(fmax(rint(rgba[k] * 255.0), 0.0), 255.0);
    if (a.coverage) a.coverage[e] = (float)cov;
}

}  // namespace mdc

extern "C" int mdc_render(const MdcRenderArgs *p, void *stream) {
    using namespace mdc;
    MDC_REQUIRE(p && p->values && p->spacing && p->out, "null pointer");
    MDC_REQUIRE(p->mode >= 0 && p->mode <= 2, "mode must be MDC_RENDER_CONTOUR/DISCRETE/DISCRETE_CONTOUR");
    MDC_REQUIRE(p->channels == 1 || p->channels == 2, "channels must be 1 or 2");
    MDC_REQUIRE(p->width > 0 && p->height > 0 && p->nimg > 0, "bad raster");
    MDC_REQUIRE(p->mode == 0 || (p->colormap && p->ncolors > 0), "discrete modes need a colormap");
    RArgs a;
    a.mode = p->mode;
    a.dtype = p->dtype;
    a.width = p->width;
    a.height = p->height;
    a.nimg = p->nimg;
    a.channels = p->channels;
    a.values = p->values;
    a.img_stride = p->img_stride;
    a.cs = p->cs;
    a.rs = p->rs;
    a.ps = p->ps;
    a.spacing = p->spacing;
    a.line_width = p->line_width_px;
    for (int k = 0; k < 4; ++k) {
        a.lc[k] = p->line_color[k] / 255.0;
        a.bg[k] = p->background[k] / 255.0;
    }
    a.cmap = p->colormap;
    a.ncolors = p->ncolors;
    a.out = p->out;
    a.coverage = p->coverage;
    int64_t total = (int64_t)p->width * p->height * p->nimg;
    unsigned blocks = (unsigned)((total + 255) / 256);
    if (p->dtype == MDC_F32)
        render_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
    else
        render_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
