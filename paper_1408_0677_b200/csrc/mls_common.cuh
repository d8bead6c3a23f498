// mls_common.cuh -- device helpers shared by the SIMT (mls.cu) and
// tensor-core (mls_tc.cu) MLS kernels.
#pragma once
#include <math.h>

#include "common.cuh"

namespace mdc {

enum AlphaMode { A_GENERIC = 0, A_ONE = 1, A_THREE_HALVES = 2, A_HALF = 3, A_TWO = 4 };

static inline int alpha_mode(double a) {
    if (a == 1.0) return A_ONE;
    if (a == 1.5) return A_THREE_HALVES;
    if (a == 0.5) return A_HALF;
    if (a == 2.0) return A_TWO;
    return A_GENERIC;
}

// ---- weights: w = d2^-alpha ------------------------------------------------
// fp64 reciprocal / reciprocal square root for the weights (MDC_F64_FASTW):
// the MUFU seed (2^-20) plus one second-order correction, ~1 ulp -- the
// library's correctly rounded sequences cost about twice the fp64 ops; the
// fp64 contract is 1e-10.  Inputs are >= 1e-300 (the weight floor), so the
// flush-to-zero seeds never see a subnormal.
#ifndef MDC_F64_FASTW
#define MDC_F64_FASTW 1
#endif
__device__ __forceinline__ double rsqrt64(double x) {
#if MDC_F64_FASTW
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
#else
    return rsqrt(x);
#endif
}
__device__ __forceinline__ double rcp64(double x) {
#if MDC_F64_FASTW
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
#else
    return 1.0 / x;
#endif
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int AM>
__device__ __forceinline__ float weight(float d2, float neg_alpha) {
    // fp32: no 1e-300 floor -- only pixels inside the snap radius can reach
    // d2 ~ 0 and those are overwritten by the snap pass (field.py:648).
    if (AM == A_THREE_HALVES) {
        float r = rsqrt_approx(d2);
        return r * r * r;
    } else if (AM == A_ONE) {
        return rcp_approx(d2);
    } else if (AM == A_HALF) {
        return rsqrt_approx(d2);
    } else if (AM == A_TWO) {
        float r = rcp_approx(d2);
        return r * r;
    } else {
        return ex2_approx(neg_alpha * lg2_approx(d2));
    }
}

// Packed form for two controls at once: the arithmetic runs as FFMA2/FMUL2
// (one issue slot for two lanes of fp32 work), the MUFU ops stay scalar.
// Lane-wise identical to weight<AM>(float).
template <int AM>
__device__ __forceinline__ float2 weight2(float2 d2, float neg_alpha) {
    if (AM == A_THREE_HALVES) {
        float2 r = make_float2(rsqrt_approx(d2.x), rsqrt_approx(d2.y));
        return __fmul2_rn(__fmul2_rn(r, r), r);
    } else if (AM == A_ONE) {
        return make_float2(rcp_approx(d2.x), rcp_approx(d2.y));
    } else if (AM == A_HALF) {
        return make_float2(rsqrt_approx(d2.x), rsqrt_approx(d2.y));
    } else if (AM == A_TWO) {
        float2 r = make_float2(rcp_approx(d2.x), rcp_approx(d2.y));
        return __fmul2_rn(r, r);
    } else {
        float2 l = __fmul2_rn(make_float2(lg2_approx(d2.x), lg2_approx(d2.y)), make_float2(neg_alpha, neg_alpha));
        return make_float2(ex2_approx(l.x), ex2_approx(l.y));
    }
}
template <int AM>
__device__ __forceinline__ double weight(double d2, double neg_alpha) {
    // fp64 mirrors _kernels.py:37-49 including the 1e-300 floor.
    if (d2 < 1e-300) d2 = 1e-300;
    if (AM == A_THREE_HALVES) {
        double r = rsqrt64(d2);
        return r * r * r;
    } else if (AM == A_ONE) {
        return rcp64(d2);
    } else if (AM == A_HALF) {
        return rsqrt64(d2);
    } else if (AM == A_TWO) {
        double r = rcp64(d2);
        return r * r;
    } else {
        return pow(d2, neg_alpha);
    }
}

// ---- tiling --------------------------------------------------------------
constexpr int NT = 256;  // threads per CTA == controls per shared-memory tile
#ifndef MDC_MLS_MINB
#define MDC_MLS_MINB 2  // CTAs per SM the register allocation must allow
#endif

template <typename T>
struct V2;
template <>
struct V2<float> {
    using type = float2;
};
template <>
struct V2<double> {
    using type = double2;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct KArgs {
    int width, row0, nrows;
    int64_t npix;             // nrows * width
    int64_t p_begin, p_end;   // band as global pixel indices [row0*W, row1*W)
    int64_t p_total;          // height * width
    int64_t tile0;            // first CTA tile (global, aligned to NT*R)
    double x0, y1, sx, sy, pmx, pmy;
    int64_t n;
    int d, ldq;
    double alpha, reg_eps;
    const double *pc;
    const void *q;
    const double *qm;
    const int32_t *axis;
    void *out;
    int64_t out_cs, out_rs, out_ps;
    int32_t *bands;
    int64_t band_cs, band_rs;
    const double *spacing;
    int32_t *nonfinite;
    uint32_t *rgba;
    const uint32_t *palette;
    int32_t palette_n;
    const double *pm_dev;  // non-null: pm is read here (device) instead of pmx / pmy
};

// Band epilogue (render.py:135-139) fused with the discrete shading
// (render.py:142-148): band = floor(f / s_k) and, when requested, the RGBA8
// colour palette[band mod n] (non-negative modulo, as np.mod).
template <typename A>
__device__ __forceinline__ void store_band(const A &a, int ch, int64_t lr, int64_t col, double f) {
    if (!a.bands && !a.rgba) return;
    const int32_t b = (int32_t)floor(f / a.spacing[ch]);
    const int64_t off = ch * a.band_cs + lr * a.band_rs + col;
    if (a.bands) a.bands[off] = b;
    if (a.rgba) {
        int m = b % a.palette_n;
        if (m < 0) m += a.palette_n;
        a.rgba[off] = a.palette[m];
    }
}

// Pixel centre (global linear pixel index p) in the globally-centred frame,
// bit-identical to `xs.ravel() - pm[0]` / `ys.ravel() - pm[1]` of
// field.py:611-613.
__device__ __forceinline__ void pixel_xy(const KArgs &a, int64_t p, double &vx, double &vy) {
    int64_t row = p / a.width;
    int col = (int)(p - row * a.width);
    double xs = dadd(a.x0, dmul((double)col + 0.5, a.sx));
    double ys = dsub(a.y1, dmul((double)row + 0.5, a.sy));
    const double pmx = a.pm_dev ? __ldg(a.pm_dev) : a.pmx, pmy = a.pm_dev ? __ldg(a.pm_dev + 1) : a.pmy;
    vx = dsub(xs, pmx);
    vy = dsub(ys, pmy);
}

// Stage tile `t` of the control positions (fp64, re-centred on o) into sxy,
// and issue the cp.async copies of its target block channels [c0, c0+DC).
template <typename T, int DC>
struct Stager {
    static constexpr int QV = (DC * (int)sizeof(T) + 15) / 16;  // 16 B vectors per control
    __device__ static void load_xy(const KArgs &a, int64_t t, double &rx, double &ry) {
        int64_t j = t * NT + threadIdx.x;
        if (j < a.n) {
            double2 v = reinterpret_cast<const double2 *>(a.pc)[j];
            rx = v.x;
            ry = v.y;
        } else {
            rx = 0.0;
            ry = 0.0;
        }
    }
    __device__ static void issue_q(const KArgs &a, int64_t t, int c0, T *sq) {
        // sq: NT controls x (QV*16/sizeof(T)) elements.  Requires ldq*sizeof(T)
        // and c0*sizeof(T) to be multiples of 16 (host pads ldq).
        const char *qb = reinterpret_cast<const char *>(a.q);
        for (int e = threadIdx.x; e < NT * QV; e += NT) {
            int jl = e / QV, v = e - jl * QV;
            int64_t j = t * NT + jl;
            if (j < a.n) {
                const char *src = qb + ((size_t)j * a.ldq + c0) * sizeof(T) + v * 16;
                cp_async16(reinterpret_cast<char *>(sq) + (size_t)e * 16, src);
            }
        }
        cp_async_commit();
    }
};

template <typename T>
__device__ __forceinline__ T to_t(double x) {
    return (T)x;
}

}  // namespace mdc
