// mls.cu -- global-support moving-least-squares field on B200 (sm_100a).
//
// Replaces _kernels.mean_field / affine_field / rigid_field
// (/root/reference/pkg/src/mdcontour/_kernels.py:52-175) as dispatched by
// field.compute_field (field.py:582-659), fused with the band epilogue
// render._band_indices (render.py:135-139), and field._snap_control_pixels
// (field.py:388-412).
//
// Formulation (SURVEY.md §8a M6'): every pixel v works in a pixel-tile-local
// frame; with delta_j = p_j - v and phi_j = [1, dx_j, dy_j],
//     A = sum_j w_j phi_j phi_j^T   (3x3, 6 unique moments)
//     B = sum_j w_j phi_j q_j^T     (3 x d)
// and the affine MLS value is f_k = e0^T (A + diag(0,r,r))^{-1} B[:,k] with
// r = reg_eps * tr(Schur complement of A_00) -- algebraically identical to the
// reference's centred 2x2 solve (_kernels.py:102-124).  Because only row 0 of
// A^{-1} is needed, the kernel runs TWO passes over the controls:
//   pass 1:  the 6 moments -> c = A_reg^{-1} e0   (per pixel, solved in fp64)
//   pass 2:  f_k = sum_j w_j (c0 + c1 dx_j + c2 dy_j) q_jk
// which costs (13) + (9 + d) FMA-pipe ops per (pixel, control) pair instead
// of 14 + 3d for the one-pass RHS -- 2x fewer at d = 32.
// Controls stream through shared memory tile by tile (cp.async double
// buffering for the target block; positions are re-centred on the CTA's
// pixel tile in fp64 before being rounded to the compute dtype, which keeps
// fp32 cancellation relative to the tile size rather than the data extent).
#include <math.h>

#include "mls_common.cuh"

#ifndef MDC_SIMT_STATIC
#define MDC_SIMT_STATIC 1  // full control tiles run static-trip-count loops (same order)
#endif

namespace mdc {

// fp32 runs: partial sums cover one control tile (NT controls) and are then
// added into fp64 totals, bounding the rounding error by the tile length
// instead of N (a single fp32 accumulator over 100k controls misses the 1e-4
// fp32 contract; the affine pass-2 sum has heavy cancellation).  fp64
// kernels keep one accumulator (flush is a no-op).
template <typename T>
__device__ __forceinline__ void run_flush(T &part, double &tot) {
    if constexpr (sizeof(T) == 4) {
        tot += (double)part;
        part = T(0);
    }
}

// ------------------------------------------------------------------------------
// The fused kernel.  VAR: MDC_MEAN / MDC_AFFINE / MDC_RIGID; DC: channels per
// pass-2 chunk; R: pixels per thread.
// fp64 with 32-channel chunks: one pass 2 for d <= 32 (instead of two
// 16-channel passes, each re-evaluating the weights); 135 KB of staged
// controls, so one CTA per SM and the whole register file for it.
#ifndef MDC_F64_DC32
#define MDC_F64_DC32 2  // pixels per thread for the fp64 32-channel instantiation (0: off; A/B at config 3: 16-ch chunks 41.0, R = 1 49.2, R = 2 56.4 Mpixel*dim/s)
#endif
#ifndef MDC_SIMT_P1_UNROLL
#define MDC_SIMT_P1_UNROLL 8  // control-loop unroll of the scalar (fp64) passes (A/B, fp64 config 3 before the MUFU weights: 2 55.9, 4 56.5, 8 57.6)
#endif
#ifndef MDC_SIMT_P2_UNROLL
#define MDC_SIMT_P2_UNROLL 2
#endif
constexpr int SIMT_P1U = MDC_SIMT_P1_UNROLL, SIMT_P2U = MDC_SIMT_P2_UNROLL;
template <typename T, int DC>
constexpr int mls_minb() { return (sizeof(T) == 8 && DC == 32) ? 1 : MDC_MLS_MINB; }

template <typename T, int VAR, int AM, int DC, int R>
__global__ void __launch_bounds__(NT, mls_minb<T, DC>()) mls_kernel(KArgs a) {
    using T2 = typename V2<T>::type;
    constexpr int QE = Stager<T, DC>::QV * 16 / (int)sizeof(T);  // padded channels per control
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T2 *sxy = reinterpret_cast<T2 *>(smem_raw);
    T *sq0 = reinterpret_cast<T *>(smem_raw + NT * sizeof(T2));
    T *sq1 = sq0 + NT * QE;

    const int tid = threadIdx.x;
    // Tiles are aligned in GLOBAL pixel-index space, so a pixel's tile (and
    // hence its local frame and every rounding) does not depend on how the
    // frame is split into row bands: 1-GPU and N-GPU outputs are bit-identical.
    const int64_t tile_base = (a.tile0 + blockIdx.x) * (int64_t)(NT * R);
    const T neg_alpha = (T)(-a.alpha);

    // Tile-local frame origin: the centre pixel of this CTA's tile.
    double ox, oy;
    {
        int64_t mid = tile_base + (NT * R) / 2;
        if (mid >= a.p_total) mid = a.p_total - 1;
        pixel_xy(a, mid, ox, oy);
    }
    double vxg[R], vyg[R];  // global-centred pixel coordinates
    T vx[R], vy[R];         // tile-local
    bool active[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        int64_t p = tile_base + r * NT + tid;
        active[r] = p >= a.p_begin && p < a.p_end;
        if (!active[r]) p = p < a.p_begin ? a.p_begin : a.p_end - 1;
        pixel_xy(a, p, vxg[r], vyg[r]);
        vx[r] = to_t<T>(vxg[r] - ox);
        vy[r] = to_t<T>(vyg[r] - oy);
    }
    const int64_t ntiles = (a.n + NT - 1) / NT;
    // fp32 with two pixels per thread: the two pixels are the two lanes of
    // packed f32x2 arithmetic (FFMA2/FADD2/FMUL2, one issue slot for both);
    // control data is a broadcast operand.  Lane-wise identical to the scalar
    // code below except for the per-tile accumulation, which is also per lane.
    constexpr bool PK = sizeof(T) == 4 && R == 2;

    // Generic streaming loop over all control tiles; body(sxy, sq, count).
    auto stream_controls = [&](int c0, bool need_q, auto &&body) {
        double rx, ry;
        Stager<T, DC>::load_xy(a, 0, rx, ry);
        if (need_q) Stager<T, DC>::issue_q(a, 0, c0, sq0);
        for (int64_t t = 0; t < ntiles; ++t) {
            __syncthreads();  // previous tile fully consumed
            sxy[tid] = T2{to_t<T>(rx - ox), to_t<T>(ry - oy)};
            T *cur = (t & 1) ? sq1 : sq0;
            if (t + 1 < ntiles) {
                Stager<T, DC>::load_xy(a, t + 1, rx, ry);
                if (need_q) Stager<T, DC>::issue_q(a, t + 1, c0, (t & 1) ? sq0 : sq1);
            }
            if (need_q) {
                if (t + 1 < ntiles)
                    cp_async_wait<1>();
                else
                    cp_async_wait<0>();
            }
            __syncthreads();
            int cnt = (int)min((int64_t)NT, a.n - t * NT);
            body(cur, cnt);
        }
    };

    if constexpr (VAR == MDC_AFFINE) {
        // ---------------- pass 1: moments ----------------
        T sw[R], mx[R], my[R], sxx[R], sxy_[R], syy[R];
        double tsw[R], tmx[R], tmy[R], tsxx[R], tsxy[R], tsyy[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            sw[r] = mx[r] = my[r] = sxx[r] = sxy_[r] = syy[r] = T(0);
            tsw[r] = tmx[r] = tmy[r] = tsxx[r] = tsxy[r] = tsyy[r] = 0.0;
        }
        stream_controls(0, false, [&](const T *, int cnt) {
            if constexpr (PK) {
                const float2 nvx = make_float2(-vx[0], -vx[1]), nvy = make_float2(-vy[0], -vy[1]);
                float2 w2s = make_float2(0.f, 0.f), mx2 = w2s, my2 = w2s, xx2 = w2s, xy2 = w2s, yy2 = w2s;
                auto mom = [&](int j) {
                    const T2 p = sxy[j];
                    const float2 dx = __fadd2_rn(make_float2(p.x, p.x), nvx);
                    const float2 dy = __fadd2_rn(make_float2(p.y, p.y), nvy);
                    const float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                    const float2 wdx = __fmul2_rn(w, dx), wdy = __fmul2_rn(w, dy);
                    w2s = __fadd2_rn(w2s, w);
                    mx2 = __fadd2_rn(mx2, wdx);
                    my2 = __fadd2_rn(my2, wdy);
                    xx2 = __ffma2_rn(wdx, dx, xx2);
                    xy2 = __ffma2_rn(wdx, dy, xy2);
                    yy2 = __ffma2_rn(wdy, dy, yy2);
                };
#if MDC_SIMT_STATIC
                if (cnt == NT) {  // full tile: static trip count (same order)
#pragma unroll 16
                    for (int j = 0; j < NT; ++j) mom(j);
                } else
#endif
                {
#pragma unroll 4
                    for (int j = 0; j < cnt; ++j) mom(j);
                }
                tsw[0] += w2s.x; tsw[1] += w2s.y;
                tmx[0] += mx2.x; tmx[1] += mx2.y;
                tmy[0] += my2.x; tmy[1] += my2.y;
                tsxx[0] += xx2.x; tsxx[1] += xx2.y;
                tsxy[0] += xy2.x; tsxy[1] += xy2.y;
                tsyy[0] += yy2.x; tsyy[1] += yy2.y;
            } else {
#pragma unroll SIMT_P1U
                for (int j = 0; j < cnt; ++j) {
                    T2 p = sxy[j];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        T dx = p.x - vx[r], dy = p.y - vy[r];
                        T w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                        T wdx = w * dx, wdy = w * dy;
                        sw[r] += w;
                        mx[r] += wdx;
                        my[r] += wdy;
                        sxx[r] += wdx * dx;
                        sxy_[r] += wdx * dy;
                        syy[r] += wdy * dy;
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    run_flush(sw[r], tsw[r]);
                    run_flush(mx[r], tmx[r]);
                    run_flush(my[r], tmy[r]);
                    run_flush(sxx[r], tsxx[r]);
                    run_flush(sxy_[r], tsxy[r]);
                    run_flush(syy[r], tsyy[r]);
                }
            }
        });
        // per-pixel solve in fp64: c = (A + diag(0, reg, reg))^{-1} e0
        T c0[R], c1[R], c2[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double s = tsw[r] + (double)sw[r], m0 = tmx[r] + (double)mx[r], m1 = tmy[r] + (double)my[r];
            double a00 = (tsxx[r] + (double)sxx[r]) - m0 * m0 / s;
            double a01 = (tsxy[r] + (double)sxy_[r]) - m0 * m1 / s;
            double a11 = (tsyy[r] + (double)syy[r]) - m1 * m1 / s;
            double reg = a.reg_eps * (a00 + a11);
            a00 += reg;
            a11 += reg;
            double det = a00 * a11 - a01 * a01;
            double u0 = (a11 * m0 - a01 * m1) / det;
            double u1 = (a00 * m1 - a01 * m0) / det;
            c0[r] = to_t<T>(1.0 / s + (m0 * u0 + m1 * u1) / (s * s));
            c1[r] = to_t<T>(-u0 / s);
            c2[r] = to_t<T>(-u1 / s);
        }
        // ---------------- pass 2: weighted RHS, chunked over channels --------
        bool bad[R];
#pragma unroll
        for (int r = 0; r < R; ++r) bad[r] = false;
        for (int c0ch = 0; c0ch < a.d; c0ch += DC) {
            T acc[R][DC];
            double tacc[R][DC];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    acc[r][k] = T(0);
                    tacc[r][k] = 0.0;
                }
            stream_controls(c0ch, true, [&](const T *sq, int cnt) {
                if constexpr (PK) {
                    const float2 nvx = make_float2(-vx[0], -vx[1]), nvy = make_float2(-vy[0], -vy[1]);
                    const float2 c0v = make_float2(c0[0], c0[1]), c1v = make_float2(c1[0], c1[1]),
                                 c2v = make_float2(c2[0], c2[1]);
                    float2 acc2[DC];
#pragma unroll
                    for (int k = 0; k < DC; ++k) acc2[k] = make_float2(0.f, 0.f);
                    auto rhs = [&](int j) {
                        const T2 p = sxy[j];
                        const float2 dx = __fadd2_rn(make_float2(p.x, p.x), nvx);
                        const float2 dy = __fadd2_rn(make_float2(p.y, p.y), nvy);
                        const float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                        const float2 g = __fmul2_rn(w, __ffma2_rn(c2v, dy, __ffma2_rn(c1v, dx, c0v)));
#pragma unroll
                        for (int k = 0; k < DC; ++k) {
                            const float q = sq[j * QE + k];
                            acc2[k] = __ffma2_rn(g, make_float2(q, q), acc2[k]);
                        }
                    };
#if MDC_SIMT_STATIC
                    if (cnt == NT) {
#pragma unroll 4
                        for (int j = 0; j < NT; ++j) rhs(j);
                    } else
#endif
                    {
#pragma unroll 2
                        for (int j = 0; j < cnt; ++j) rhs(j);
                    }
#pragma unroll
                    for (int k = 0; k < DC; ++k) {
                        tacc[0][k] += acc2[k].x;
                        tacc[1][k] += acc2[k].y;
                    }
                } else {
#pragma unroll SIMT_P2U
                    for (int j = 0; j < cnt; ++j) {
                        T2 p = sxy[j];
                        T qv[DC];
#pragma unroll
                        for (int k = 0; k < DC; ++k) qv[k] = sq[j * QE + k];
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            T dx = p.x - vx[r], dy = p.y - vy[r];
                            T w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                            T g = w * (c0[r] + c1[r] * dx + c2[r] * dy);
#pragma unroll
                            for (int k = 0; k < DC; ++k) acc[r][k] += g * qv[k];
                        }
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int k = 0; k < DC; ++k) run_flush(acc[r][k], tacc[r][k]);
                }
            });
            // epilogue: add back qm, write, bands
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!active[r]) continue;
                int64_t p = tile_base + r * NT + tid;
                int64_t row = p / a.width;
                int64_t col = p - row * a.width;
                int64_t lr = row - a.row0;
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    int ch = c0ch + k;
                    if (ch >= a.d) break;
                    T f = to_t<T>((tacc[r][k] + (double)acc[r][k]) + a.qm[ch]);
                    reinterpret_cast<T *>(a.out)[ch * a.out_cs + lr * a.out_rs + col * a.out_ps] = f;
                    if (!isfinite((double)f)) bad[r] = true;
                    store_band(a, ch, lr, col, (double)f);
                }
            }
        }
        if (a.nonfinite) {
            int cnt = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) cnt += (active[r] && bad[r]) ? 1 : 0;
            if (cnt) atomicAdd(a.nonfinite, cnt);
        }
    } else if constexpr (VAR == MDC_MEAN) {
        // f_k = v_axis + sum w dq_k / sum w   (_kernels.py:52-67), chunked.
        bool bad[R];
#pragma unroll
        for (int r = 0; r < R; ++r) bad[r] = false;
        for (int c0ch = 0; c0ch < a.d; c0ch += DC) {
            T acc[R][DC], sw[R];
            double tacc[R][DC], tsw[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                sw[r] = T(0);
                tsw[r] = 0.0;
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    acc[r][k] = T(0);
                    tacc[r][k] = 0.0;
                }
            }
            stream_controls(c0ch, true, [&](const T *sq, int cnt) {
                if constexpr (PK) {
                    const float2 nvx = make_float2(-vx[0], -vx[1]), nvy = make_float2(-vy[0], -vy[1]);
                    float2 sw2 = make_float2(0.f, 0.f), acc2[DC];
#pragma unroll
                    for (int k = 0; k < DC; ++k) acc2[k] = sw2;
#pragma unroll 2
                    for (int j = 0; j < cnt; ++j) {
                        const T2 p = sxy[j];
                        const float2 dx = __fadd2_rn(make_float2(p.x, p.x), nvx);
                        const float2 dy = __fadd2_rn(make_float2(p.y, p.y), nvy);
                        const float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                        sw2 = __fadd2_rn(sw2, w);
#pragma unroll
                        for (int k = 0; k < DC; ++k) {
                            const float q = sq[j * QE + k];
                            acc2[k] = __ffma2_rn(w, make_float2(q, q), acc2[k]);
                        }
                    }
                    tsw[0] += sw2.x;
                    tsw[1] += sw2.y;
#pragma unroll
                    for (int k = 0; k < DC; ++k) {
                        tacc[0][k] += acc2[k].x;
                        tacc[1][k] += acc2[k].y;
                    }
                } else {
#pragma unroll 2
                    for (int j = 0; j < cnt; ++j) {
                        T2 p = sxy[j];
                        T qv[DC];
#pragma unroll
                        for (int k = 0; k < DC; ++k) qv[k] = sq[j * QE + k];
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            T dx = p.x - vx[r], dy = p.y - vy[r];
                            T w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                            sw[r] += w;
#pragma unroll
                            for (int k = 0; k < DC; ++k) acc[r][k] += w * qv[k];
                        }
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        run_flush(sw[r], tsw[r]);
#pragma unroll
                        for (int k = 0; k < DC; ++k) run_flush(acc[r][k], tacc[r][k]);
                    }
                }
            });
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (!active[r]) continue;
                int64_t p = tile_base + r * NT + tid;
                int64_t row = p / a.width;
                int64_t col = p - row * a.width;
                int64_t lr = row - a.row0;
#pragma unroll
                for (int k = 0; k < DC; ++k) {
                    int ch = c0ch + k;
                    if (ch >= a.d) break;
                    double v = a.axis[ch] == 0 ? vxg[r] : vyg[r];
                    T f = to_t<T>((v + (tacc[r][k] + (double)acc[r][k]) / (tsw[r] + (double)sw[r])) + a.qm[ch]);
                    reinterpret_cast<T *>(a.out)[ch * a.out_cs + lr * a.out_rs + col * a.out_ps] = f;
                    if (!isfinite((double)f)) bad[r] = true;
                    store_band(a, ch, lr, col, (double)f);
                }
            }
        }
        if (a.nonfinite) {
            int cnt = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) cnt += (active[r] && bad[r]) ? 1 : 0;
            if (cnt) atomicAdd(a.nonfinite, cnt);
        }
    } else {
        // Rigid (_kernels.py:127-175), 2 channels, one pass, pixel-local frame.
        T sw[R], mx[R], my[R], bqx[R], bqy[R], b00[R], b01[R], b10[R], b11[R];
        double t_[9][R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            sw[r] = mx[r] = my[r] = bqx[r] = bqy[r] = b00[r] = b01[r] = b10[r] = b11[r] = T(0);
#pragma unroll
            for (int i = 0; i < 9; ++i) t_[i][r] = 0.0;
        }
        stream_controls(0, true, [&](const T *sq, int cnt) {
            if constexpr (PK) {
                const float2 nvx = make_float2(-vx[0], -vx[1]), nvy = make_float2(-vy[0], -vy[1]);
                float2 v[9];
#pragma unroll
                for (int i = 0; i < 9; ++i) v[i] = make_float2(0.f, 0.f);
#pragma unroll 2
                for (int j = 0; j < cnt; ++j) {
                    const T2 p = sxy[j];
                    const float2 qx = make_float2(sq[j * QE + 0], sq[j * QE + 0]);
                    const float2 qy = make_float2(sq[j * QE + 1], sq[j * QE + 1]);
                    const float2 dx = __fadd2_rn(make_float2(p.x, p.x), nvx);
                    const float2 dy = __fadd2_rn(make_float2(p.y, p.y), nvy);
                    const float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                    const float2 wdx = __fmul2_rn(w, dx), wdy = __fmul2_rn(w, dy);
                    v[0] = __fadd2_rn(v[0], w);
                    v[1] = __fadd2_rn(v[1], wdx);
                    v[2] = __fadd2_rn(v[2], wdy);
                    v[3] = __ffma2_rn(w, qx, v[3]);
                    v[4] = __ffma2_rn(w, qy, v[4]);
                    v[5] = __ffma2_rn(wdx, qx, v[5]);
                    v[6] = __ffma2_rn(wdx, qy, v[6]);
                    v[7] = __ffma2_rn(wdy, qx, v[7]);
                    v[8] = __ffma2_rn(wdy, qy, v[8]);
                }
#pragma unroll
                for (int i = 0; i < 9; ++i) {
                    t_[i][0] += v[i].x;
                    t_[i][1] += v[i].y;
                }
            } else {
#pragma unroll 2
                for (int j = 0; j < cnt; ++j) {
                    T2 p = sxy[j];
                    T qx = sq[j * QE + 0], qy = sq[j * QE + 1];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        T dx = p.x - vx[r], dy = p.y - vy[r];
                        T w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                        T wdx = w * dx, wdy = w * dy;
                        sw[r] += w;
                        mx[r] += wdx;
                        my[r] += wdy;
                        bqx[r] += w * qx;
                        bqy[r] += w * qy;
                        b00[r] += wdx * qx;
                        b01[r] += wdx * qy;
                        b10[r] += wdy * qx;
                        b11[r] += wdy * qy;
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    run_flush(sw[r], t_[0][r]);
                    run_flush(mx[r], t_[1][r]);
                    run_flush(my[r], t_[2][r]);
                    run_flush(bqx[r], t_[3][r]);
                    run_flush(bqy[r], t_[4][r]);
                    run_flush(b00[r], t_[5][r]);
                    run_flush(b01[r], t_[6][r]);
                    run_flush(b10[r], t_[7][r]);
                    run_flush(b11[r], t_[8][r]);
                }
            }
        });
        int cnt_bad = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (!active[r]) continue;
            double s = t_[0][r] + (double)sw[r];
            const double Mx = t_[1][r] + (double)mx[r], My = t_[2][r] + (double)my[r];
            double psx = Mx / s, psy = My / s;  // delta*
            double qsx = (t_[3][r] + (double)bqx[r]) / s, qsy = (t_[4][r] + (double)bqy[r]) / s;
            double c00 = (t_[5][r] + (double)b00[r]) - qsx * Mx;
            double c01 = (t_[6][r] + (double)b01[r]) - qsy * Mx;
            double c10 = (t_[7][r] + (double)b10[r]) - qsx * My;
            double c11 = (t_[8][r] + (double)b11[r]) - qsy * My;
            double ss = c00 + c11, dd = c10 - c01;
            double dx = -psx, dy = -psy;  // v - p*
            double fx = dx * ss + dy * dd;
            double fy = dy * ss - dx * dd;
            double norm = hypot(fx, fy);
            double ox_, oy_;
            if (norm < 1e-12) {
                // mean-blend fallback vx + (mq - mp)/sw (_kernels.py:168-171);
                // with p* = v + delta* this is q* - delta*.
                ox_ = qsx - psx;
                oy_ = qsy - psy;
            } else {
                double rr = hypot(dx, dy) / norm;
                ox_ = fx * rr + qsx;
                oy_ = fy * rr + qsy;
            }
            T f0 = to_t<T>(ox_ + a.qm[0]), f1 = to_t<T>(oy_ + a.qm[1]);
            int64_t p = tile_base + r * NT + tid;
            int64_t row = p / a.width;
            int64_t col = p - row * a.width;
            int64_t lr = row - a.row0;
            T *o = reinterpret_cast<T *>(a.out);
            o[lr * a.out_rs + col * a.out_ps] = f0;
            o[a.out_cs + lr * a.out_rs + col * a.out_ps] = f1;
            store_band(a, 0, lr, col, (double)f0);
            store_band(a, 1, lr, col, (double)f1);
            if (!isfinite((double)f0) || !isfinite((double)f1)) ++cnt_bad;
        }
        if (a.nonfinite && cnt_bad) atomicAdd(a.nonfinite, cnt_bad);
    }
}

template <typename T, int DC>
static size_t smem_bytes() {
    constexpr int QE = Stager<T, DC>::QV * 16 / (int)sizeof(T);
    return NT * sizeof(typename V2<T>::type) + 2 * (size_t)NT * QE * sizeof(T);
}

template <typename T, int VAR, int AM, int DC, int R>
static int launch_t(const KArgs &k, cudaStream_t s) {
    auto fn = mls_kernel<T, VAR, AM, DC, R>;
    size_t smem = smem_bytes<T, DC>();
    MDC_CHECK_CUDA(ensure_dynamic_smem((const void *)fn, (int)smem));
    KArgs kk = k;
    const int64_t tile = NT * R;
    kk.tile0 = kk.p_begin / tile;
    int64_t blocks = (kk.p_end + tile - 1) / tile - kk.tile0;
    if (blocks > 0) fn<<<(unsigned)blocks, NT, smem, s>>>(kk);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

template <typename T, int VAR, int AM>
static int dispatch_dc(const KArgs &k, cudaStream_t s) {
    // channel chunk: smallest instantiated DC >= d (cap 8 for f32, 16 for f64)
    constexpr bool F32 = sizeof(T) == 4;
    constexpr int R = 2;
    int d = k.d;
    if (VAR == MDC_RIGID) return launch_t<T, VAR, AM, 2, R>(k, s);
    if (d <= 1) return launch_t<T, VAR, AM, 1, R>(k, s);
    if (d <= 2) return launch_t<T, VAR, AM, 2, R>(k, s);
    if (d <= 4) return launch_t<T, VAR, AM, 4, R>(k, s);
    if (d <= 8) return launch_t<T, VAR, AM, 8, R>(k, s);
    if constexpr (F32) {
        // fp32 keeps fp64 run totals per channel in registers: chunks of 8
        return launch_t<T, VAR, AM, 8, R>(k, s);
    } else {
#if MDC_F64_DC32
        if (VAR == MDC_AFFINE && d > 16 && k.ldq >= ((d + 31) / 32) * 32)
            return launch_t<T, VAR, AM, 32, MDC_F64_DC32>(k, s);
#endif
        return launch_t<T, VAR, AM, 16, R>(k, s);
    }
}

template <typename T, int VAR>
static int dispatch_alpha(const KArgs &k, cudaStream_t s) {
    switch (alpha_mode(k.alpha)) {
        case A_ONE: return dispatch_dc<T, VAR, A_ONE>(k, s);
        case A_THREE_HALVES: return dispatch_dc<T, VAR, A_THREE_HALVES>(k, s);
        case A_HALF: return dispatch_dc<T, VAR, A_HALF>(k, s);
        case A_TWO: return dispatch_dc<T, VAR, A_TWO>(k, s);
        default: return dispatch_dc<T, VAR, A_GENERIC>(k, s);
    }
}

// Padded channel stride the stager requires (elements).
static int required_chunk(int dtype, int d, int variant) {
    if (variant == MDC_RIGID) return 2;
    int cap = dtype == MDC_F32 ? 32 : 16;
    int dc = 1;
    while (dc < d && dc < cap) dc *= 2;
    return dc;
}

// ---------------------------------------------------------------------------
// Snap: four stream-ordered passes over the controls (field.py:388-412).
struct SnapArgs {
    int width, row0, row1, height;
    double x0, y1, sx, sy, eps;
    int rx, ry;
    int64_t n;
    int d, dtype;
    const double *pos, *tvals;
    void *out;
    int64_t out_cs, out_rs, out_ps;
    int32_t *bands;
    int64_t band_cs, band_rs;
    const double *spacing;
    int32_t *nonfinite;
    uint32_t *rgba;
    const uint32_t *palette;
    int32_t palette_n;
    unsigned long long *best_d2;
    unsigned *best_idx;
};

template <int PASS>
__global__ void snap_kernel(SnapArgs a) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    double px = a.pos[2 * i], py = a.pos[2 * i + 1];
    double pxf = dsub(__ddiv_rn(dsub(px, a.x0), a.sx), 0.5);
    double pyf = dsub(__ddiv_rn(dsub(a.y1, py), a.sy), 0.5);
    // int(round(x)) on np.float64: round half to even == rint.
    long long cx = (long long)rint(pxf), cy = (long long)rint(pyf);
    long long ylo = max(cy - a.ry, (long long)max(0, a.row0));
    long long yhi = min(cy + a.ry + 1, (long long)a.row1);
    long long xlo = max(cx - a.rx, 0LL), xhi = min(cx + a.rx + 1, (long long)a.width);
    for (long long yy = ylo; yy < yhi; ++yy) {
        double ys = dsub(a.y1, dmul((double)yy + 0.5, a.sy));
        double ey = dsub(ys, py);
        double ey2 = dmul(ey, ey);
        for (long long xx = xlo; xx < xhi; ++xx) {
            double xs = dadd(a.x0, dmul((double)xx + 0.5, a.sx));
            double ex = dsub(xs, px);
            double d2 = dadd(dmul(ex, ex), ey2);
            if (!(d2 < a.eps)) continue;
            int64_t lr = yy - a.row0;
            int64_t pix = lr * a.width + xx;
            unsigned long long key = (unsigned long long)__double_as_longlong(d2);
            if (PASS == 0) {
                atomicMin(&a.best_d2[pix], key);
            } else if (PASS == 1) {
                if (a.best_d2[pix] == key) atomicMin(&a.best_idx[pix], (unsigned)i);
            } else if (PASS == 2) {
                if (a.best_idx[pix] != (unsigned)i) continue;
                bool was_bad = false;
                for (int k = 0; k < a.d; ++k) {
                    int64_t off = k * a.out_cs + lr * a.out_rs + xx * a.out_ps;
                    double v = a.tvals[i * a.d + k];
                    if (a.dtype == MDC_F32) {
                        float *o = reinterpret_cast<float *>(a.out);
                        if (!isfinite(o[off])) was_bad = true;
                        o[off] = (float)v;
                        v = (double)(float)v;
                    } else {
                        double *o = reinterpret_cast<double *>(a.out);
                        if (!isfinite(o[off])) was_bad = true;
                        o[off] = v;
                    }
                    store_band(a, k, lr, xx, v);
                }
                if (was_bad && a.nonfinite) atomicSub(a.nonfinite, 1);
            } else {
                a.best_d2[pix] = ~0ULL;
                a.best_idx[pix] = ~0U;
            }
        }
    }
}

size_t mls_tc_workspace_bytes(int d, int64_t n);
int launch_mls_tc(const KArgs &k, void *ws, cudaStream_t s);
size_t mls_tc2_workspace_bytes(int d, int64_t n);
int launch_mls_tc2(const KArgs &k, void *ws, cudaStream_t s);

// Two-pass kernel (mls_tc.cu) by default; MDC_FLAG_TC_ONEPASS selects the
// experimental one-pass kernel (mls_tc2.cu) for A/B comparisons.
static size_t tc_ws_bytes(const MdcMlsArgs *a) {
    return (a->flags & MDC_FLAG_TC_ONEPASS) ? mls_tc2_workspace_bytes(a->d, a->n) : mls_tc_workspace_bytes(a->d, a->n);
}

static bool tc_eligible(const MdcMlsArgs *a) {
#ifndef MDC_TC_MIN_D
#define MDC_TC_MIN_D 8
#endif
    return a->dtype == MDC_F32 && a->variant == MDC_AFFINE && a->d >= MDC_TC_MIN_D && !(a->flags & MDC_FLAG_NO_TC);
}

}  // namespace mdc

using namespace mdc;

extern "C" size_t mdc_mls_workspace_bytes(const MdcMlsArgs *a) {
    if (!a || !tc_eligible(a)) return 0;
    return tc_ws_bytes(a);
}

extern "C" int mdc_mls_field(const MdcMlsArgs *a, void *stream) {
    MDC_REQUIRE(a != nullptr, "null args");
    MDC_REQUIRE(a->variant == MDC_MEAN || a->variant == MDC_AFFINE || a->variant == MDC_RIGID,
                "variant must be MDC_MEAN, MDC_AFFINE or MDC_RIGID");
    MDC_REQUIRE(a->dtype == MDC_F32 || a->dtype == MDC_F64, "dtype must be MDC_F32 or MDC_F64");
    MDC_REQUIRE(a->width > 0 && a->height > 0, "width/height must be positive");
    MDC_REQUIRE(0 <= a->row0 && a->row0 <= a->row1 && a->row1 <= a->height, "bad row band");
    MDC_REQUIRE(a->n > 0, "need at least one control");
    MDC_REQUIRE(a->d >= 1, "need at least one channel");
    MDC_REQUIRE(a->variant != MDC_RIGID || a->d == 2, "rigid MLS needs exactly 2 channels");
    MDC_REQUIRE(a->variant != MDC_MEAN || a->axis != nullptr, "mean variant needs axis[]");
    MDC_REQUIRE(a->pc && a->q && a->qm && a->out, "null device pointer");
    MDC_REQUIRE(a->bands == nullptr || a->spacing != nullptr, "bands need spacing[]");
    MDC_REQUIRE(a->rgba == nullptr || (a->spacing != nullptr && a->palette != nullptr && a->palette_n > 0),
                "rgba shading needs spacing[] and a non-empty palette");
    size_t es = a->dtype == MDC_F32 ? 4 : 8;
    int chunk = required_chunk(a->dtype, a->d, a->variant);
    int64_t need = ((a->d + chunk - 1) / chunk) * chunk;
    MDC_REQUIRE(a->ldq >= need && (a->ldq * es) % 16 == 0,
                "ldq must cover d rounded up to the channel chunk and be 16-byte aligned");
    MDC_REQUIRE(((uintptr_t)a->q % 16) == 0 && ((uintptr_t)a->pc % 16) == 0,
                "q and pc must be 16-byte aligned");
    KArgs k;
    k.width = a->width;
    k.row0 = a->row0;
    k.nrows = a->row1 - a->row0;
    k.npix = (int64_t)k.nrows * a->width;
    k.p_begin = (int64_t)a->row0 * a->width;
    k.p_end = (int64_t)a->row1 * a->width;
    k.p_total = (int64_t)a->height * a->width;
    k.tile0 = 0;
    k.x0 = a->x0;
    k.y1 = a->y1;
    k.sx = a->sx;
    k.sy = a->sy;
    k.pmx = a->pmx;
    k.pmy = a->pmy;
    k.pm_dev = a->pm;
    k.n = a->n;
    k.d = a->d;
    k.ldq = a->ldq;
    k.alpha = a->alpha;
    k.reg_eps = a->reg_eps;
    k.pc = a->pc;
    k.q = a->q;
    k.qm = a->qm;
    k.axis = a->axis;
    k.out = a->out;
    k.out_cs = a->out_cs;
    k.out_rs = a->out_rs;
    k.out_ps = a->out_ps;
    k.bands = a->bands;
    k.band_cs = a->band_cs;
    k.band_rs = a->band_rs;
    k.spacing = a->spacing;
    k.nonfinite = a->nonfinite;
    k.rgba = a->rgba;
    k.palette = a->palette;
    k.palette_n = a->palette_n;
    if (k.npix == 0) return MDC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (tc_eligible(a) && a->workspace && a->workspace_bytes >= tc_ws_bytes(a) && ((uintptr_t)a->workspace % 16) == 0)
        return (a->flags & MDC_FLAG_TC_ONEPASS) ? launch_mls_tc2(k, a->workspace, s) : launch_mls_tc(k, a->workspace, s);
    if (a->dtype == MDC_F32) {
        switch (a->variant) {
            case MDC_MEAN: return dispatch_alpha<float, MDC_MEAN>(k, s);
            case MDC_AFFINE: return dispatch_alpha<float, MDC_AFFINE>(k, s);
            default: return dispatch_alpha<float, MDC_RIGID>(k, s);
        }
    }
    switch (a->variant) {
        case MDC_MEAN: return dispatch_alpha<double, MDC_MEAN>(k, s);
        case MDC_AFFINE: return dispatch_alpha<double, MDC_AFFINE>(k, s);
        default: return dispatch_alpha<double, MDC_RIGID>(k, s);
    }
}

extern "C" size_t mdc_snap_workspace_bytes(int32_t width, int32_t rows) {
    return (size_t)width * (size_t)rows * (sizeof(unsigned long long) + sizeof(unsigned));
}

extern "C" int mdc_mls_snap(const MdcMlsArgs *a, const double *pos, const double *tvals, double eps,
                            void *workspace, void *stream) {
    MDC_REQUIRE(a && pos && tvals && workspace, "null pointer");
    MDC_REQUIRE(eps > 0, "eps must be positive");
    MDC_REQUIRE(a->rgba == nullptr || (a->spacing != nullptr && a->palette != nullptr && a->palette_n > 0),
                "rgba shading needs spacing[] and a non-empty palette");
    MDC_REQUIRE(0 <= a->row0 && a->row0 <= a->row1 && a->row1 <= a->height, "bad row band");
    SnapArgs s;
    s.width = a->width;
    s.row0 = a->row0;
    s.row1 = a->row1;
    s.height = a->height;
    s.x0 = a->x0;
    s.y1 = a->y1;
    s.sx = a->sx;
    s.sy = a->sy;
    s.eps = eps;
    // field.py:398-399: r = int(ceil(sqrt(eps) / s)) + 1
    s.rx = (int)ceil(sqrt(eps) / a->sx) + 1;
    s.ry = (int)ceil(sqrt(eps) / a->sy) + 1;
    s.n = a->n;
    s.d = a->d;
    s.dtype = a->dtype;
    s.pos = pos;
    s.tvals = tvals;
    s.out = a->out;
    s.out_cs = a->out_cs;
    s.out_rs = a->out_rs;
    s.out_ps = a->out_ps;
    s.bands = a->bands;
    s.band_cs = a->band_cs;
    s.band_rs = a->band_rs;
    s.spacing = a->spacing;
    s.nonfinite = a->nonfinite;
    s.rgba = a->rgba;
    s.palette = a->palette;
    s.palette_n = a->palette_n;
    int64_t npix = (int64_t)(a->row1 - a->row0) * a->width;
    s.best_d2 = reinterpret_cast<unsigned long long *>(workspace);
    s.best_idx = reinterpret_cast<unsigned *>(s.best_d2 + npix);
    if (npix == 0 || a->n == 0) return MDC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned blocks = (unsigned)((a->n + 127) / 128);
    snap_kernel<0><<<blocks, 128, 0, st>>>(s);
    snap_kernel<1><<<blocks, 128, 0, st>>>(s);
    snap_kernel<2><<<blocks, 128, 0, st>>>(s);
    snap_kernel<3><<<blocks, 128, 0, st>>>(s);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}
