/*
 * mdc_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity CHECKER, never the product: only tests/, the
 * `cpu_baseline` leg of bench.py, `bench.py --impl reference` and
 * __graft_entry__.smoke() may load it.  The shipped path is the CUDA library
 * paper_1408_0677_b200/libmdc.so, which never links or calls this code.
 *
 * Each function restates one routine of the upstream `mdcontour` package
 * (/root/reference/pkg/src/mdcontour) in plain C99 + OpenMP, fp64, with
 * floating-point contraction disabled (-ffp-contract=off) so that the
 * arithmetic is the same sequence of IEEE roundings as numba/numpy perform.
 * Parity of this restatement is pinned against golden vectors produced by
 * the reference itself (tests/golden/make_golden.py -> tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

EXPORT void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n < 1) n = 1;
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}

EXPORT int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* _kernels.py:37-49 `_weight` -- inverse power with fast paths. */
static inline double weight(double d2, double alpha) {
    if (d2 < 1e-300) d2 = 1e-300;
    if (alpha == 1.0) return 1.0 / d2;
    if (alpha == 1.5) return 1.0 / (d2 * sqrt(d2));
    if (alpha == 0.5) return 1.0 / sqrt(d2);
    if (alpha == 2.0) return 1.0 / (d2 * d2);
    return pow(d2, -alpha);
}

/* _kernels.py:52-67 `mean_field`. out is (npix, 2) row-major. */
EXPORT void orc_mean_field(int64_t npix, const double *vx, const double *vy, int64_t n,
                           const double *px, const double *py, const double *dqx,
                           const double *dqy, double alpha, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < npix; ++i) {
        double sw = 0.0, sx = 0.0, sy = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double dx = px[j] - vx[i];
            double dy = py[j] - vy[i];
            double w = weight(dx * dx + dy * dy, alpha);
            sw += w;
            sx += w * dqx[j];
            sy += w * dqy[j];
        }
        out[2 * i + 0] = vx[i] + sx / sw;
        out[2 * i + 1] = vy[i] + sy / sw;
    }
}

/* _kernels.py:70-124 `affine_field`: 12 global-frame moments, centred 2x2 solve. */
EXPORT void orc_affine_field(int64_t npix, const double *vx, const double *vy, int64_t n,
                             const double *px, const double *py, const double *qx,
                             const double *qy, double alpha, double reg_eps, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < npix; ++i) {
        double sw = 0, mpx = 0, mpy = 0, mqx = 0, mqy = 0, mpxpx = 0, mpxpy = 0, mpypy = 0;
        double mpxqx = 0, mpxqy = 0, mpyqx = 0, mpyqy = 0;
        for (int64_t j = 0; j < n; ++j) {
            double dx = px[j] - vx[i];
            double dy = py[j] - vy[i];
            double w = weight(dx * dx + dy * dy, alpha);
            sw += w;
            mpx += w * px[j];
            mpy += w * py[j];
            mqx += w * qx[j];
            mqy += w * qy[j];
            mpxpx += w * px[j] * px[j];
            mpxpy += w * px[j] * py[j];
            mpypy += w * py[j] * py[j];
            mpxqx += w * px[j] * qx[j];
            mpxqy += w * px[j] * qy[j];
            mpyqx += w * py[j] * qx[j];
            mpyqy += w * py[j] * qy[j];
        }
        double psx = mpx / sw, psy = mpy / sw, qsx = mqx / sw, qsy = mqy / sw;
        double a00 = mpxpx - psx * mpx;
        double a01 = mpxpy - psx * mpy;
        double a11 = mpypy - psy * mpy;
        double b00 = mpxqx - qsx * mpx;
        double b01 = mpxqy - qsy * mpx;
        double b10 = mpyqx - qsx * mpy;
        double b11 = mpyqy - qsy * mpy;
        double reg = reg_eps * (a00 + a11);
        a00 += reg;
        a11 += reg;
        double det = a00 * a11 - a01 * a01;
        double m00 = (a11 * b00 - a01 * b10) / det;
        double m01 = (a11 * b01 - a01 * b11) / det;
        double m10 = (a00 * b10 - a01 * b00) / det;
        double m11 = (a00 * b11 - a01 * b01) / det;
        double ddx = vx[i] - psx, ddy = vy[i] - psy;
        out[2 * i + 0] = ddx * m00 + ddy * m10 + qsx;
        out[2 * i + 1] = ddx * m01 + ddy * m11 + qsy;
    }
}

/* d-channel form of _kernels.py:70-124 `affine_field`: channel k equals
 * channel 0 of the reference's call with targets (q[:, k], 0) -- what the
 * reference CLI renders once per dimension (cli.py:143-165).  The moment sums
 * shared by all channels are accumulated once; every channel's own sums and
 * solve follow orc_affine_field's operation order, so each channel is
 * bit-identical to a separate 2-channel call.  q: (n, d) row-major,
 * out: (npix, d) row-major. */
/* -O3 lets gcc vectorise the per-channel loop; each channel's accumulator
 * still sees the same operations in the same order (no reassociation, no
 * contraction: -ffp-contract=off), so results are bit-identical. */
__attribute__((optimize("O3"))) EXPORT void orc_affine_field_d(int64_t npix, const double *vx, const double *vy, int64_t n,
                               const double *px, const double *py, int64_t d, const double *q,
                               double alpha, double reg_eps, double *out) {
#pragma omp parallel
    {
        double *mq = (double *)malloc(sizeof(double) * 3 * (size_t)d);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < npix; ++i) {
            double sw = 0, mpx = 0, mpy = 0, mpxpx = 0, mpxpy = 0, mpypy = 0;
            double *mqx = mq, *mpxqx = mq + d, *mpyqx = mq + 2 * d;
            for (int64_t k = 0; k < 3 * d; ++k) mq[k] = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                double dx = px[j] - vx[i];
                double dy = py[j] - vy[i];
                double w = weight(dx * dx + dy * dy, alpha);
                sw += w;
                mpx += w * px[j];
                mpy += w * py[j];
                mpxpx += w * px[j] * px[j];
                mpxpy += w * px[j] * py[j];
                mpypy += w * py[j] * py[j];
                const double *qj = q + j * d;
                for (int64_t k = 0; k < d; ++k) {
                    mqx[k] += w * qj[k];
                    mpxqx[k] += w * px[j] * qj[k];
                    mpyqx[k] += w * py[j] * qj[k];
                }
            }
            double psx = mpx / sw, psy = mpy / sw;
            double a00 = mpxpx - psx * mpx;
            double a01 = mpxpy - psx * mpy;
            double a11 = mpypy - psy * mpy;
            double reg = reg_eps * (a00 + a11);
            a00 += reg;
            a11 += reg;
            double det = a00 * a11 - a01 * a01;
            double ddx = vx[i] - psx, ddy = vy[i] - psy;
            for (int64_t k = 0; k < d; ++k) {
                double qsx = mqx[k] / sw;
                double b00 = mpxqx[k] - qsx * mpx;
                double b10 = mpyqx[k] - qsx * mpy;
                double m00 = (a11 * b00 - a01 * b10) / det;
                double m10 = (a00 * b10 - a01 * b00) / det;
                out[i * d + k] = ddx * m00 + ddy * m10 + qsx;
            }
        }
        free(mq);
    }
}

/* _kernels.py:127-175 `rigid_field`: similarity -> rotation, mean fallback. */
EXPORT void orc_rigid_field(int64_t npix, const double *vx, const double *vy, int64_t n,
                            const double *px, const double *py, const double *qx,
                            const double *qy, double alpha, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < npix; ++i) {
        double sw = 0, mpx = 0, mpy = 0, mqx = 0, mqy = 0, mpxqx = 0, mpxqy = 0, mpyqx = 0, mpyqy = 0;
        for (int64_t j = 0; j < n; ++j) {
            double dx = px[j] - vx[i];
            double dy = py[j] - vy[i];
            double w = weight(dx * dx + dy * dy, alpha);
            sw += w;
            mpx += w * px[j];
            mpy += w * py[j];
            mqx += w * qx[j];
            mqy += w * qy[j];
            mpxqx += w * px[j] * qx[j];
            mpxqy += w * px[j] * qy[j];
            mpyqx += w * py[j] * qx[j];
            mpyqy += w * py[j] * qy[j];
        }
        double psx = mpx / sw, psy = mpy / sw, qsx = mqx / sw, qsy = mqy / sw;
        double b00 = mpxqx - qsx * mpx;
        double b01 = mpxqy - qsy * mpx;
        double b10 = mpyqx - qsx * mpy;
        double b11 = mpyqy - qsy * mpy;
        double s = b00 + b11, d = b10 - b01;
        double ddx = vx[i] - psx, ddy = vy[i] - psy;
        double fx = ddx * s + ddy * d;
        double fy = ddy * s - ddx * d;
        double norm = hypot(fx, fy);
        if (norm < 1e-12) {
            out[2 * i + 0] = vx[i] + (mqx - mpx) / sw;
            out[2 * i + 1] = vy[i] + (mqy - mpy) / sw;
        } else {
            double r = hypot(ddx, ddy) / norm;
            out[2 * i + 0] = fx * r + qsx;
            out[2 * i + 1] = fy * r + qsy;
        }
    }
}

/* field.py:388-412 `_snap_control_pixels`: stamp exact targets within sqrt(eps),
 * nearest control wins (strict <, so the lower index wins exact ties).
 * coords is (h, w, nch) row-major; tvals is (n, nch). */
EXPORT void orc_snap(double *coords, int64_t h, int64_t w, int64_t nch, int64_t n,
                     const double *pos, const double *tvals, double x0, double y1, double sx,
                     double sy, double eps) {
    double *best = (double *)malloc(sizeof(double) * (size_t)(h * w));
    for (int64_t k = 0; k < h * w; ++k) best[k] = INFINITY;
    int64_t rx = (int64_t)ceil(sqrt(eps) / sx) + 1;
    int64_t ry = (int64_t)ceil(sqrt(eps) / sy) + 1;
    for (int64_t i = 0; i < n; ++i) {
        double pxf = (pos[2 * i] - x0) / sx - 0.5;
        double pyf = (y1 - pos[2 * i + 1]) / sy - 0.5;
        int64_t cx = (int64_t)rint(pxf), cy = (int64_t)rint(pyf);
        int64_t ylo = cy - ry > 0 ? cy - ry : 0, yhi = cy + ry + 1 < h ? cy + ry + 1 : h;
        int64_t xlo = cx - rx > 0 ? cx - rx : 0, xhi = cx + rx + 1 < w ? cx + rx + 1 : w;
        for (int64_t yy = ylo; yy < yhi; ++yy) {
            double ys = y1 - ((double)yy + 0.5) * sy;
            for (int64_t xx = xlo; xx < xhi; ++xx) {
                double xs = x0 + ((double)xx + 0.5) * sx;
                double ex = xs - pos[2 * i], ey = ys - pos[2 * i + 1];
                double d2 = ex * ex + ey * ey;
                if (d2 < eps && d2 < best[yy * w + xx]) {
                    best[yy * w + xx] = d2;
                    for (int64_t c = 0; c < nch; ++c) coords[(yy * w + xx) * nch + c] = tvals[i * nch + c];
                }
            }
        }
    }
    free(best);
}

/* ------------------------------------------------------------------------- */
/* bhtree.py:10-66 `KdTree`: median split, argmax-extent axis (ties -> x),
 * mid = count // 2, preorder numbering.  argpartition's membership is
 * restated as "the mid smallest under the total order (coord, index)". */

typedef struct {
    const double *pts;
    int axis;
} sort_ctx;

static __thread sort_ctx g_ctx;

static int cmp_idx(const void *a, const void *b) {
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    double u = g_ctx.pts[2 * i + g_ctx.axis], v = g_ctx.pts[2 * j + g_ctx.axis];
    if (u < v) return -1;
    if (u > v) return 1;
    return (i > j) - (i < j);
}

typedef struct {
    const double *pts;
    int64_t *perm, *lo, *hi, *left, *right;
    double *com, *mass, *size, *bmin, *bmax;
    int64_t count, leaf;
} kdtree;

static int64_t kd_new_node(kdtree *t, int64_t lo, int64_t hi) {
    int64_t i = t->count++;
    t->lo[i] = lo;
    t->hi[i] = hi;
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY, sx = 0, sy = 0;
    for (int64_t k = lo; k < hi; ++k) {
        const double *p = t->pts + 2 * t->perm[k];
        if (p[0] < mnx) mnx = p[0];
        if (p[0] > mxx) mxx = p[0];
        if (p[1] < mny) mny = p[1];
        if (p[1] > mxy) mxy = p[1];
        sx += p[0];
        sy += p[1];
    }
    t->bmin[2 * i] = mnx;
    t->bmin[2 * i + 1] = mny;
    t->bmax[2 * i] = mxx;
    t->bmax[2 * i + 1] = mxy;
    t->com[2 * i] = sx / (double)(hi - lo);
    t->com[2 * i + 1] = sy / (double)(hi - lo);
    t->mass[i] = (double)(hi - lo);
    t->size[i] = hypot(mxx - mnx, mxy - mny);
    t->left[i] = -1;
    t->right[i] = -1;
    return i;
}

static int64_t kd_build(kdtree *t, int64_t lo, int64_t hi) {
    int64_t node = kd_new_node(t, lo, hi);
    if (hi - lo <= t->leaf) return node;
    double ex = t->bmax[2 * node] - t->bmin[2 * node];
    double ey = t->bmax[2 * node + 1] - t->bmin[2 * node + 1];
    int axis = ey > ex ? 1 : 0;
    int64_t mid = (hi - lo) / 2;
    g_ctx.pts = t->pts;
    g_ctx.axis = axis;
    qsort(t->perm + lo, (size_t)(hi - lo), sizeof(int64_t), cmp_idx);
    if (mid == 0 || mid == hi - lo) return node;
    t->left[node] = kd_build(t, lo, lo + mid);
    t->right[node] = kd_build(t, lo + mid, hi);
    return node;
}

/* Returns the node count.  Arrays must hold cap = 4*(2n/leaf+2) entries
 * (bhtree.py:24), perm holds n. */
EXPORT int64_t orc_kdtree_build(int64_t n, const double *pts, int64_t leaf, int64_t *perm,
                                int64_t *lo, int64_t *hi, int64_t *left, int64_t *right,
                                double *com, double *mass, double *size, double *bmin,
                                double *bmax) {
    kdtree t = {pts, perm, lo, hi, left, right, com, mass, size, bmin, bmax, 0, leaf};
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    kd_build(&t, 0, n);
    return t.count;
}

/* _kernels.py:178-230 `bh_forces`: per-point explicit-stack DFS. */
EXPORT void orc_bh_forces(int64_t n, const double *pts, const int64_t *perm, const int64_t *lo,
                          const int64_t *hi, const int64_t *left, const int64_t *right,
                          const double *com, const double *mass, const double *size,
                          const double *bmin, const double *bmax, double c, double eta,
                          double theta, double *out) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
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
}

/* bhtree.py:69-95 `repulsive_forces` (tree + traversal). */
EXPORT void orc_repulsive_forces(int64_t n, const double *pts, double c, double eta, double theta,
                                 int64_t leaf, double *out) {
    if (n < 2) {
        memset(out, 0, sizeof(double) * 2 * (size_t)n);
        return;
    }
    int64_t cap = 4 * (2 * n / (leaf > 1 ? leaf : 1) + 2);
    int64_t *ib = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 4 * cap));
    double *db = (double *)malloc(sizeof(double) * (size_t)(8 * cap));
    int64_t *perm = ib, *lo = ib + n, *hi = lo + cap, *lf = hi + cap, *rt = lf + cap;
    double *com = db, *mass = db + 2 * cap, *size = mass + cap, *bmin = size + cap, *bmax = bmin + 2 * cap;
    orc_kdtree_build(n, pts, leaf, perm, lo, hi, lf, rt, com, mass, size, bmin, bmax);
    orc_bh_forces(n, pts, perm, lo, hi, lf, rt, com, mass, size, bmin, bmax, c, eta, theta, out);
    free(ib);
    free(db);
}

/* ------------------------------------------------------------------------- */
/* Layout: layout.py:216-286. */

/* layout.py:216-231 `_spring_forces`: CSR in source-major order, bincount sums
 * each node's edges sequentially in edge order. */
EXPORT void orc_spring_forces(int64_t n, const double *pos, const int64_t *off, const int64_t *tgt,
                              double spring, double eta, double dlen, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double fx = 0.0, fy = 0.0;
        for (int64_t e = off[i]; e < off[i + 1]; ++e) {
            int64_t j = tgt[e];
            double dx = pos[2 * i] - pos[2 * j], dy = pos[2 * i + 1] - pos[2 * j + 1];
            double r = hypot(dx, dy);
            double coef = -spring * log((r + eta) / dlen);
            fx += coef * dx;
            fy += coef * dy;
        }
        out[2 * i] = fx;
        out[2 * i + 1] = fy;
    }
}

/* layout.py:234-256 `_node_edge_forces`: per corner k, `forces -= bincount(...)`.
 * Restated per triangle in (k, t) order; the per-k partial sums are formed in
 * triangle order exactly like np.bincount, then subtracted k = 0, 1, 2. */
EXPORT void orc_node_edge_forces(int64_t n, const double *pos, int64_t ntri, const int64_t *tris,
                                 double c, double eta, double *out) {
    double *part = (double *)calloc((size_t)(2 * n), sizeof(double));
    for (int64_t i = 0; i < 2 * n; ++i) out[i] = 0.0;
    for (int k = 0; k < 3; ++k) {
        memset(part, 0, sizeof(double) * 2 * (size_t)n);
        for (int64_t t = 0; t < ntri; ++t) {
            int64_t v = tris[3 * t + k], a = tris[3 * t + (k + 1) % 3], b = tris[3 * t + (k + 2) % 3];
            double ex = pos[2 * b] - pos[2 * a], ey = pos[2 * b + 1] - pos[2 * a + 1];
            double ee = ex * ex + ey * ey;
            if (ee == 0.0) ee = 1.0;
            double tt = ((pos[2 * v] - pos[2 * a]) * ex + (pos[2 * v + 1] - pos[2 * a + 1]) * ey) / ee;
            double rx = pos[2 * a] + tt * ex - pos[2 * v];
            double ry = pos[2 * a + 1] + tt * ey - pos[2 * v + 1];
            double nr = hypot(rx, ry);
            double coef = nr >= 1e-12 ? c / (nr * nr + eta) / nr : 0.0;
            part[2 * v] += coef * rx;
            part[2 * v + 1] += coef * ry;
        }
        for (int64_t i = 0; i < 2 * n; ++i) out[i] -= part[i];
    }
    free(part);
}

/* layout.py:119-184 `_limit_constraints` + `clamp_factors`: nine rows per
 * triangle (3 midsegment lines x 3 vertices), per-node min, clip to [0, 1]. */
EXPORT void orc_clamp_factors(int64_t n, const double *pos, const double *disp, int64_t ntri,
                              const int64_t *tris, double eta, double *s) {
    for (int64_t i = 0; i < n; ++i) s[i] = INFINITY;
    for (int64_t t = 0; t < ntri; ++t) {
        const int64_t *tr = tris + 3 * t;
        double ax = pos[2 * tr[0]], ay = pos[2 * tr[0] + 1];
        double bx = pos[2 * tr[1]], by = pos[2 * tr[1] + 1];
        double cx = pos[2 * tr[2]], cy = pos[2 * tr[2] + 1];
        double mabx = 0.5 * (ax + bx), maby = 0.5 * (ay + by);
        double mbcx = 0.5 * (bx + cx), mbcy = 0.5 * (by + cy);
        double mcax = 0.5 * (cx + ax), mcay = 0.5 * (cy + ay);
        double ptx[3] = {mabx, mabx, mbcx}, pty[3] = {maby, maby, mbcy};
        double drx[3] = {mcax - mabx, mbcx - mabx, mcax - mbcx};
        double dry[3] = {mcay - maby, mbcy - maby, mcay - mbcy};
        for (int l = 0; l < 3; ++l) {
            double nx = -dry[l], ny = drx[l];
            double ln = hypot(nx, ny);
            if (ln == 0.0) ln = 1.0;
            nx /= ln;
            ny /= ln;
            for (int k = 0; k < 3; ++k) {
                int64_t v = tr[k];
                double relx = pos[2 * v] - ptx[l], rely = pos[2 * v + 1] - pty[l];
                double sgn = relx * nx + rely * ny;
                double side = sgn >= 0.0 ? 1.0 : -1.0;
                double dist = fabs(sgn);
                double allowed = dist - eta > 0.0 ? dist - eta : 0.0;
                double toward = -side * (disp[2 * v] * nx + disp[2 * v + 1] * ny);
                double f = toward > allowed ? allowed / toward : 1.0;
                if (f < s[v]) s[v] = f;
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        double v = s[i];
        if (v == INFINITY) v = 1.0;
        s[i] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
}

/* layout.py:266-286 `layout_step` on a frozen snapshot; writes pos_out. */
EXPORT void orc_layout_step(int64_t n, const double *pos, double *pos_out, const int64_t *off,
                            const int64_t *tgt, int64_t ntri, const int64_t *tris, double c,
                            double spring, double dlen, double eta, double theta, int64_t leaf,
                            double temperature) {
    double *f = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    double *g = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    double *s = (double *)malloc(sizeof(double) * (size_t)n);
    orc_repulsive_forces(n, pos, c, eta, theta, leaf, f);
    orc_spring_forces(n, pos, off, tgt, spring, eta, dlen, g);
    for (int64_t i = 0; i < 2 * n; ++i) f[i] += g[i];
    orc_node_edge_forces(n, pos, ntri, tris, c, eta, g);
    for (int64_t i = 0; i < 2 * n; ++i) f[i] += g[i];
    for (int64_t i = 0; i < n; ++i) {
        double mag = hypot(f[2 * i], f[2 * i + 1]);
        if (mag > temperature) {
            double k = temperature / mag;
            f[2 * i] *= k;
            f[2 * i + 1] *= k;
        }
    }
    orc_clamp_factors(n, pos, f, ntri, tris, eta, s);
    for (int64_t i = 0; i < n; ++i) {
        pos_out[2 * i] = pos[2 * i] + s[i] * f[2 * i];
        pos_out[2 * i + 1] = pos[2 * i + 1] + s[i] * f[2 * i + 1];
    }
    free(f);
    free(g);
    free(s);
}

/* ------------------------------------------------------------------------- */
/* projection.py:50-79 `pca_project` numerics: covariance (n-1) + a symmetric
 * eigensolver.  LAPACK `eigh` is restated as cyclic Jacobi (eigenpairs are
 * unique up to sign for distinct eigenvalues; the sign is fixed by the caller
 * with the reference's largest-|component|-positive rule). */
EXPORT void orc_covariance(int64_t n, int64_t d, const double *x, double *mean, double *cov) {
    for (int64_t j = 0; j < d; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += x[i * d + j];
        mean[j] = s / (double)n;
    }
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < d; ++a)
        for (int64_t b = 0; b < d; ++b) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s += (x[i * d + a] - mean[a]) * (x[i * d + b] - mean[b]);
            cov[a * d + b] = s / (double)(n - 1);
        }
}

/* Cyclic Jacobi on a symmetric d x d matrix (destroyed).  evals ascending is
 * NOT imposed here; evecs[:, k] pairs with evals[k]. */
EXPORT void orc_jacobi_eigh(int64_t d, double *a, double *evals, double *evecs) {
    for (int64_t i = 0; i < d * d; ++i) evecs[i] = 0.0;
    for (int64_t i = 0; i < d; ++i) evecs[i * d + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int64_t p = 0; p < d; ++p)
            for (int64_t q = 0; q < d; ++q) {
                tot += a[p * d + q] * a[p * d + q];
                if (p != q) off += a[p * d + q] * a[p * d + q];
            }
        if (off <= 1e-30 * tot || off == 0.0) break;
        for (int64_t p = 0; p < d - 1; ++p)
            for (int64_t q = p + 1; q < d; ++q) {
                double apq = a[p * d + q];
                if (apq == 0.0) continue;
                double app = a[p * d + p], aqq = a[q * d + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
                for (int64_t k = 0; k < d; ++k) {
                    double akp = a[k * d + p], akq = a[k * d + q];
                    a[k * d + p] = cs * akp - sn * akq;
                    a[k * d + q] = sn * akp + cs * akq;
                }
                for (int64_t k = 0; k < d; ++k) {
                    double apk = a[p * d + k], aqk = a[q * d + k];
                    a[p * d + k] = cs * apk - sn * aqk;
                    a[q * d + k] = sn * apk + cs * aqk;
                }
                for (int64_t k = 0; k < d; ++k) {
                    double vkp = evecs[k * d + p], vkq = evecs[k * d + q];
                    evecs[k * d + p] = cs * vkp - sn * vkq;
                    evecs[k * d + q] = sn * vkp + cs * vkq;
                }
            }
    }
    for (int64_t i = 0; i < d; ++i) evals[i] = a[i * d + i];
}

/* ------------------------------------------------------------------------- */
/* Linear variant: _kernels.py:233-313 `rasterize_linear` (serial, first
 * triangle wins) + `extend_hull` (nearest hull segment, strict <, hull order),
 * as driven by field._linear_field (field.py:497-515).  out (h, w, nch),
 * tvals (n, nch); hull arrays from field._hull_edges order. */
EXPORT void orc_linear_field(int64_t n, const double *pos, const double *tvals, int64_t nch, int64_t ntri,
                             const int64_t *tris, int64_t nh, const int64_t *hull_u, const int64_t *hull_v,
                             const int64_t *hull_t, double x0, double y1, double sx, double sy, int64_t w,
                             int64_t h, double *out) {
    unsigned char *assigned = (unsigned char *)calloc((size_t)(w * h), 1);
    for (int64_t t = 0; t < ntri; ++t) {
        int64_t ia = tris[3 * t], ib = tris[3 * t + 1], ic = tris[3 * t + 2];
        double ax = pos[2 * ia], ay = pos[2 * ia + 1], bx = pos[2 * ib], by = pos[2 * ib + 1];
        double cx = pos[2 * ic], cy = pos[2 * ic + 1];
        double det = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
        if (det == 0.0) continue;
        double xlo = fmin(ax, fmin(bx, cx)), xhi = fmax(ax, fmax(bx, cx));
        double ylo = fmin(ay, fmin(by, cy)), yhi = fmax(ay, fmax(by, cy));
        int64_t c0 = (int64_t)floor((xlo - x0) / sx - 0.5); if (c0 < 0) c0 = 0;
        int64_t c1 = (int64_t)ceil((xhi - x0) / sx); if (c1 > w - 1) c1 = w - 1;
        int64_t r0 = (int64_t)floor((y1 - yhi) / sy - 0.5); if (r0 < 0) r0 = 0;
        int64_t r1 = (int64_t)ceil((y1 - ylo) / sy); if (r1 > h - 1) r1 = h - 1;
        for (int64_t row = r0; row <= r1; ++row) {
            double gy = y1 - ((double)row + 0.5) * sy;
            for (int64_t col = c0; col <= c1; ++col) {
                if (assigned[row * w + col]) continue;
                double gx = x0 + ((double)col + 0.5) * sx;
                double l1 = ((bx - gx) * (cy - gy) - (by - gy) * (cx - gx)) / det;
                double l2 = ((cx - gx) * (ay - gy) - (cy - gy) * (ax - gx)) / det;
                double l3 = 1.0 - l1 - l2;
                if (l1 >= -1e-12 && l2 >= -1e-12 && l3 >= -1e-12) {
                    assigned[row * w + col] = 1;
                    for (int64_t k = 0; k < nch; ++k)
                        out[(row * w + col) * nch + k] =
                            l1 * tvals[ia * nch + k] + l2 * tvals[ib * nch + k] + l3 * tvals[ic * nch + k];
                }
            }
        }
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t row = 0; row < h; ++row) {
        double gy = y1 - ((double)row + 0.5) * sy;
        for (int64_t col = 0; col < w; ++col) {
            if (assigned[row * w + col]) continue;
            double gx = x0 + ((double)col + 0.5) * sx;
            double best = INFINITY;
            int64_t best_t = 0;
            for (int64_t k = 0; k < nh; ++k) {
                double axp = pos[2 * hull_u[k]], ayp = pos[2 * hull_u[k] + 1];
                double bxp = pos[2 * hull_v[k]], byp = pos[2 * hull_v[k] + 1];
                double ex = bxp - axp, ey = byp - ayp, ee = ex * ex + ey * ey, s = 0.0;
                if (ee > 0.0) {
                    s = ((gx - axp) * ex + (gy - ayp) * ey) / ee;
                    if (s < 0.0) s = 0.0;
                    else if (s > 1.0) s = 1.0;
                }
                double ddx = gx - (axp + s * ex), ddy = gy - (ayp + s * ey);
                double d2 = ddx * ddx + ddy * ddy;
                if (d2 < best) {
                    best = d2;
                    best_t = hull_t[k];
                }
            }
            int64_t ia = tris[3 * best_t], ib = tris[3 * best_t + 1], ic = tris[3 * best_t + 2];
            double ax = pos[2 * ia], ay = pos[2 * ia + 1], bx = pos[2 * ib], by = pos[2 * ib + 1];
            double cx = pos[2 * ic], cy = pos[2 * ic + 1];
            double det = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
            double l1 = ((bx - gx) * (cy - gy) - (by - gy) * (cx - gx)) / det;
            double l2 = ((cx - gx) * (ay - gy) - (cy - gy) * (ax - gx)) / det;
            double l3 = 1.0 - l1 - l2;
            for (int64_t k = 0; k < nch; ++k)
                out[(row * w + col) * nch + k] =
                    l1 * tvals[ia * nch + k] + l2 * tvals[ib * nch + k] + l3 * tvals[ic * nch + k];
        }
    }
    free(assigned);
}
