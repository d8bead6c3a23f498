// render.cu -- band shading + anti-aliased isocontours from an MLS field.
//
// Replaces render.line_coverage (render.py:116-126), _gradient_magnitudes
// (render.py:110-113, CoordinateField.jacobian = np.gradient, field.py:154-161),
// _band_indices / render_discrete (render.py:135-148), render_contours
// (render.py:129-132) and the compositing helpers _over / _to_image
// (render.py:91-102).  All arithmetic is fp64 in the reference's order, so a
// field that matches the reference renders to the same RGBA bytes.
#include <math.h>

#include <cub/cub.cuh>

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
    double corners[16];  // gradient corners /255
    double target_px;
    const uint8_t *tex;
    int tex_w, tex_h;
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

// np.mod(x, 1.0): fmod, then shifted into [0, 1) for negative remainders
__device__ __forceinline__ double mod1(double x) {
    double m = fmod(x, 1.0);
    if (m != 0.0 && m < 0.0) m += 1.0;
    return m;
}

// line_coverage at spacing s for one image (max over channels)
template <typename T>
__device__ __forceinline__ double coverage_at(const RArgs &a, int img, int r, int x, double s, const double *g) {
    double cov = 0.0;
    for (int c = 0; c < a.channels; ++c) {
        double v = val<T>(a, img, c, r, x);
        double dist = fabs(v - s * rint(v / s));
        double px = g[c] > 1e-30 ? dist / g[c] : INFINITY;
        cov = fmax(cov, fmin(fmax(0.5 * a.line_width + 0.5 - px, 0.0), 1.0));
    }
    return cov;
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
    double g[2] = {0.0, 0.0};
    for (int c = 0; c < a.channels; ++c)
        g[c] = hypot(grad<T>(a, img, c, r, x, true), grad<T>(a, img, c, r, x, false));
    double rgba[4];
    double cov = 0.0;
    if (a.mode == 0) {  // contour: background + lines (render.py:129-132)
        cov = coverage_at<T>(a, img, r, x, s, g);
        for (int k = 0; k < 4; ++k) rgba[k] = a.bg[k];
        over(rgba, a.lc, cov);
    } else if (a.mode == 1 || a.mode == 2) {  // discrete (+contour) (render.py:142-148)
        long long band = 0;
        for (int c = 0; c < a.channels; ++c) band += (long long)floor(val<T>(a, img, c, r, x) / s);
        long long m = band % a.ncolors;
        if (m < 0) m += a.ncolors;
        for (int k = 0; k < 4; ++k) rgba[k] = a.cmap[m * 4 + k];
        if (a.mode == 2) {
            cov = coverage_at<T>(a, img, r, x, s, g);
            over(rgba, a.lc, cov);
        }
    } else if (a.mode == 3) {  // adaptive (render.py:151-178): octaves 3..-3, coarse first
        const double lo = a.target_px / 4.0, hi = a.target_px;
        double remaining = 1.0;
        for (int k = 3; k >= -3; --k) {
            double sk = s * exp2((double)k);
            double pxb = g[0] > 1e-30 ? sk / g[0] : INFINITY;
            double t = fmin(fmax((pxb - lo) / (hi - lo), 0.0), 1.0);
            double op = t * t * (3.0 - 2.0 * t);
            double ck = coverage_at<T>(a, img, r, x, sk, g);
            remaining = remaining * (1.0 - ck * op);
        }
        cov = 1.0 - remaining;
        for (int k = 0; k < 4; ++k) rgba[k] = a.bg[k];
        over(rgba, a.lc, cov);
    } else if (a.mode == 4) {  // gradient (render.py:181-201)
        double fu = mod1(val<T>(a, img, 0, r, x) / s), fv = mod1(val<T>(a, img, 1, r, x) / s);
        double w00 = (1 - fu) * (1 - fv), w10 = fu * (1 - fv), w01 = (1 - fu) * fv, w11 = fu * fv;
        for (int k = 0; k < 4; ++k)
            rgba[k] = w00 * a.corners[k] + w10 * a.corners[4 + k] + w01 * a.corners[8 + k] + w11 * a.corners[12 + k];
        cov = coverage_at<T>(a, img, r, x, s, g);
        over(rgba, a.lc, cov);
    } else {  // texture (render.py:204-234), bilinear with wrap
        double fu = mod1(val<T>(a, img, 0, r, x) / s), fv = mod1(val<T>(a, img, 1, r, x) / s);
        double tx = fu * a.tex_w - 0.5, ty = fv * a.tex_h - 0.5;
        double fx0 = floor(tx), fy0 = floor(ty);
        double ax = tx - fx0, ay = ty - fy0;
        long long x0 = (long long)fx0, y0 = (long long)fy0;
        long long x1 = ((x0 + 1) % a.tex_w + a.tex_w) % a.tex_w, y1 = ((y0 + 1) % a.tex_h + a.tex_h) % a.tex_h;
        x0 = (x0 % a.tex_w + a.tex_w) % a.tex_w;
        y0 = (y0 % a.tex_h + a.tex_h) % a.tex_h;
        const uint8_t *t00 = a.tex + (y0 * a.tex_w + x0) * 4, *t01 = a.tex + (y0 * a.tex_w + x1) * 4;
        const uint8_t *t10 = a.tex + (y1 * a.tex_w + x0) * 4, *t11 = a.tex + (y1 * a.tex_w + x1) * 4;
        for (int k = 0; k < 4; ++k)
            rgba[k] = t00[k] / 255.0 * ((1 - ax) * (1 - ay)) + t01[k] / 255.0 * (ax * (1 - ay)) +
                      t10[k] / 255.0 * ((1 - ax) * ay) + t11[k] / 255.0 * (ax * ay);
    }
    uint8_t *o = a.out + e * 4;
    for (int k = 0; k < 4; ++k) o[k] = (uint8_t)fmin(fmax(rint(rgba[k] * 255.0), 0.0), 255.0);
    if (a.coverage) a.coverage[e] = (float)cov;
}

// ---------------------------------------------------------------------------
// Point overlay (render.py:237-257): every (pixel, point) pair of each disc's
// pixel box is keyed (pixel << 32 | point), radix-sorted, and each pixel then
// applies its discs in point order -- the reference's sequential _over.
__device__ __forceinline__ int ov_box(double r) { return (int)floor(2.0 * r + 5.0) + 1; }

__global__ void overlay_pairs_kernel(int64_t n, const double *pix, double r, int width, int height, int box,
                                     unsigned long long *keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long *k = keys + i * (int64_t)box * box;
    for (int e = 0; e < box * box; ++e) k[e] = ~0ULL;
    double px = pix[2 * i], py = pix[2 * i + 1];
    if (!(-r - 1 <= px && px <= width + r && -r - 1 <= py && py <= height + r)) return;
    long long c0 = max(0LL, (long long)floor(px - r - 1)), c1 = min((long long)width - 1, (long long)ceil(px + r + 1));
    long long r0 = max(0LL, (long long)floor(py - r - 1)), r1 = min((long long)height - 1, (long long)ceil(py + r + 1));
    if (c0 > c1 || r0 > r1) return;
    int e = 0;
    for (long long yy = r0; yy <= r1; ++yy)
        for (long long xx = c0; xx <= c1; ++xx)
            if (e < box * box) k[e++] = ((unsigned long long)(yy * width + xx) << 32) | (unsigned long long)i;
}

__global__ void overlay_apply_kernel(int64_t m, const unsigned long long *keys, const double *pix, double r,
                                     double c0, double c1, double c2, double c3, int width, uint8_t *img) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    unsigned long long k = keys[e];
    if (k == ~0ULL) return;
    unsigned p = (unsigned)(k >> 32);
    if (e > 0 && (unsigned)(keys[e - 1] >> 32) == p) return;  // first entry of the pixel's run
    int yy = (int)(p / (unsigned)width), xx = (int)(p % (unsigned)width);
    uint8_t *o = img + (size_t)p * 4;
    double base[4] = {o[0] / 255.0, o[1] / 255.0, o[2] / 255.0, o[3] / 255.0};
    const double src[4] = {c0, c1, c2, c3};
    for (int64_t q = e; q < m && (unsigned)(keys[q] >> 32) == p; ++q) {
        unsigned i = (unsigned)(keys[q] & 0xffffffffULL);
        double dist = hypot((double)xx - pix[2 * i], (double)yy - pix[2 * i + 1]);
        over(base, src, fmin(fmax(r + 0.5 - dist, 0.0), 1.0));
    }
    for (int k2 = 0; k2 < 4; ++k2) o[k2] = (uint8_t)fmin(fmax(rint(base[k2] * 255.0), 0.0), 255.0);
}

static size_t overlay_sort_bytes(int64_t m) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                   (int)m);
    return bytes;
}

}  // namespace mdc

extern "C" int mdc_render(const MdcRenderArgs *p, void *stream) {
    using namespace mdc;
    MDC_REQUIRE(p && p->values && p->spacing && p->out, "null pointer");
    MDC_REQUIRE(p->mode >= 0 && p->mode <= 5, "unknown render mode");
    MDC_REQUIRE(p->mode != 4 || p->channels == 2, "gradient mode requires a two-dimensional target");
    MDC_REQUIRE(p->mode != 5 || (p->channels == 2 && p->texture && p->tex_w > 0 && p->tex_h > 0),
                "texture mode requires a two-channel field and a texture");
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
    for (int k = 0; k < 16; ++k) a.corners[k] = p->gradient_corners[k] / 255.0;
    a.target_px = p->adaptive_target_px;
    a.tex = p->texture;
    a.tex_w = p->tex_w;
    a.tex_h = p->tex_h;
    int64_t total = (int64_t)p->width * p->height * p->nimg;
    unsigned blocks = (unsigned)((total + 255) / 256);
    if (p->dtype == MDC_F32)
        render_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
    else
        render_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

extern "C" size_t mdc_overlay_workspace_bytes(int64_t n, double radius) {
    int64_t box = (int64_t)floor(2.0 * radius + 5.0) + 1;
    int64_t m = n * box * box;
    return (size_t)(2 * m * sizeof(unsigned long long)) + mdc::overlay_sort_bytes(m) + 512;
}

extern "C" int mdc_overlay_points(uint8_t *img, int32_t width, int32_t height, int64_t n, const double *pix,
                                  double radius, const int32_t *color, void *workspace, size_t workspace_bytes,
                                  void *stream) {
    using namespace mdc;
    MDC_REQUIRE(img && pix && color && workspace, "null pointer");
    MDC_REQUIRE(width > 0 && height > 0 && n >= 0 && radius > 0, "bad overlay arguments");
    MDC_REQUIRE(workspace_bytes >= mdc_overlay_workspace_bytes(n, radius), "overlay workspace too small");
    MDC_REQUIRE((int64_t)width * height < (1LL << 32) && n < (1LL << 32), "overlay raster too large");
    if (n == 0) return MDC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int box = (int)floor(2.0 * radius + 5.0) + 1;
    int64_t m = n * (int64_t)box * box;
    char *w = reinterpret_cast<char *>(workspace);
    unsigned long long *k_in = reinterpret_cast<unsigned long long *>(w);
    unsigned long long *k_out = k_in + m;
    void *tmp = k_out + m;
    size_t tbytes = overlay_sort_bytes(m);
    overlay_pairs_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(n, pix, radius, width, height, box, k_in);
    MDC_CHECK_LAUNCH();
    MDC_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tbytes, k_in, k_out, (int)m, 0, 64, s));
    double c[4];
    for (int k = 0; k < 4; ++k) c[k] = color[k] / 255.0;
    overlay_apply_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(m, k_out, pix, radius, c[0], c[1], c[2], c[3],
                                                                    width, img);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
