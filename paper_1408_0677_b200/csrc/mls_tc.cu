// mls_tc.cu -- affine MLS with the pass-2 contraction on the 5th-gen tensor
// cores (tcgen05, kind::tf32, 3xTF32 split, A operand and accumulators in TMEM).
//
// Same mathematics as mls.cu (SURVEY.md §8a M6'; reference _kernels.py:70-124):
//   pass 1 (SIMT, packed f32x2 on the FP32 pipe): 6 pixel-local moments
//           -> c = A_reg^{-1} e0 (fp64 solve)
//   pass 2: F[p, k] = sum_j G[p, j] Q[j, k],  G[p, j] = w_pj (c0 + c1 dx + c2 dy)
// Pass 2 is a dense (pixels x N) . (N x d) contraction (north_star: "tensor
// cores ... only for the global-support weight case").  The SIMT threads
// evaluate G (one weight per pair), split it hi + lo and write it straight
// into TMEM with tcgen05.st (thread = pixel = TMEM lane), so the A operand
// never touches shared memory; one elected thread issues tcgen05.mma
// (M = 128 pixels, N = channels, K = 8 controls) x 3 (hi*hi + hi*lo + lo*hi,
// ~fp32-accurate) per K step with B = the target tile.  A two-stage ring
// (mbarrier armed by tcgen05.commit) overlaps the tensor core with the SIMT
// evaluation of the next tile.  The target block Q is pre-arranged once per
// call into the UMMA core-matrix layout (hi/lo), one bulk copy per K tile.
//
// Accuracy at scale: G has both signs (affine weights), so F is a sum with
// heavy cancellation; a single fp32 accumulator over 100k controls misses
// the 1e-4 fp32 contract by ~5x.  Both passes therefore accumulate in fp32
// only over bounded runs (pass 1: one staging round; pass 2: FLUSH K tiles
// in TMEM) and add the runs into fp64 totals (registers / shared memory).
//
// Tile geometry (A/B-tuned): CTA = 128 pixels (one M = 128 MMA tile) + an
// issuer warp, K tile = 16 controls, 2-stage ring, 4 CTAs per SM (TMEM).
#include <cuda_bf16.h>
#include <type_traits>

#include "mls_common.cuh"
#include "tcgen05.cuh"

namespace mdc {
namespace tc {

constexpr int TPB = 128;          // compute threads == pixels per CTA == MMA M
#ifndef MDC_TC_XYR
#define MDC_TC_XYR 256
#endif
constexpr int XYR = MDC_TC_XYR;   // controls per position staging round
#ifndef MDC_TC_KT
#define MDC_TC_KT 16
#endif
#ifndef MDC_TC_STAGES
#define MDC_TC_STAGES 2
#endif
#ifndef MDC_TC_MINB
#define MDC_TC_MINB 4
#endif
#ifndef MDC_TC_SLEEPC
#define MDC_TC_SLEEPC 0  // compute warps park (1) or spin (0) on the ring's empty barriers
#endif
#ifndef MDC_TC_TRUNC
#define MDC_TC_TRUNC 1  // pass-2 G split: truncated hi (1, +5 %) or round-to-nearest hi (0)
#endif
#ifndef MDC_TC_P1STATIC
#define MDC_TC_P1STATIC 32  // pass-1 unroll factor for full staging rounds (0: dynamic loop only)
#endif
#ifndef MDC_TC_FLUSH
#define MDC_TC_FLUSH 32  // K tiles accumulated in TMEM before the fp64 flush (512 controls)
#endif
constexpr int KT = MDC_TC_KT;          // controls per K tile (multiple of 8 = tcgen05 tf32 K)
constexpr int STAGES = MDC_TC_STAGES;  // ring depth
constexpr int FLUSH = MDC_TC_FLUSH;
constexpr int P1U = MDC_TC_P1STATIC > 0 ? MDC_TC_P1STATIC : 1;
constexpr int A_SBO = (KT / 4) * 128;  // bytes between 8-row core-matrix groups of a Q tile
static_assert(KT % 8 == 0 && XYR % KT == 0, "K tiles are whole tf32 K steps and tile a staging round");
constexpr int NC_MAX = 32;             // channels per pass-2 chunk (fp64 totals in shared memory)
#ifndef MDC_TC_SPLIT
#define MDC_TC_SPLIT 1  // compute threads per pixel (2: each half takes half of every round / K tile)
#endif
#ifndef MDC_TC_P1_TRACE
#define MDC_TC_P1_TRACE 1  // alpha = 3/2: accumulate sum 1/r instead of sum w dy^2 (13 FP32 lane-ops per pass-1 pair)
#endif
#ifndef MDC_TC_WIDE
#define MDC_TC_WIDE 64  // d > 32: 64-channel chunks (0: 32-channel chunks only)
#endif
#ifndef MDC_TC_WIDE2
#define MDC_TC_WIDE2 128  // d > 64: 128-channel chunks (0: 64-channel chunks)
#endif
#ifndef MDC_TC_MIXED
#define MDC_TC_MIXED 1  // wide chunks: tf32 main product + bf16 correction products (2 instead of 3 tf32 passes)
#endif
#ifndef MDC_TC_MIXED_MIN
#define MDC_TC_MIXED_MIN 64  // smallest chunk width using the mixed split
#endif
#ifndef MDC_TC_TOT32
#define MDC_TC_TOT32 1  // wide chunks keep their run totals in fp32 (RN adds) instead of fp64
#endif
// CTAs per SM the register allocation targets: 64-channel chunks need 64 KB
// of fp64 totals per CTA, so two CTAs share an SM.
// Run totals: fp64 for chunks of up to 32 channels; wide chunks use fp32
// totals (round-to-nearest adds of the fp32 runs -- the truncating tensor-core
// accumulation stays bounded by the run length) so that their shared memory
// (NC x 128 x 4 B) does not cap the CTAs per SM.
// Wide chunks are tensor-bound (N = 64/128 at 3 MMAs per K step), so they
// use the mixed split: G_hi . Q_hi on kind::tf32 plus [G_hi | G_lo] .
// [Q_lo ; Q_hi] on kind::f16 with bf16 operands (the correction products
// are 2^-11 of the main one; 8 significant bits carry them).
template <int NC>
__host__ __device__ constexpr bool mixed() { return MDC_TC_MIXED && NC >= MDC_TC_MIXED_MIN; }
static_assert(!MDC_TC_MIXED || MDC_TC_SPLIT == 1, "the mixed split's bf16 pairs assume one thread per pixel");

template <int NC>
struct TotOf {
    using T = typename std::conditional<(NC > NC_MAX && MDC_TC_TOT32), float, double>::type;
};
// CTAs per SM the register allocation targets: TMEM (NC + 64 columns, power
// of two) and the totals' shared memory set the real limit.
template <int NC>
__host__ __device__ constexpr int minb() {
    return NC > 2 * NC_MAX ? 2 : (NC > NC_MAX ? (MDC_TC_TOT32 ? MDC_TC_MINB : 2) : (MDC_TC_SPLIT > 1 ? 3 : MDC_TC_MINB));
}

// ---------------------------------------------------------------------------
// Q -> tiled core-matrix image, hi/lo split.  img[(chunk * ntiles + t)][hi|lo]
// each half = NC rows (channels) x KT controls = NC * KT * 4 bytes.
// mixed: the tile is [tf32 hi: NC x KT core matrices (8 x 4) | bf16 lo | bf16
// hi: NC x KT core matrices (8 x 8 bf16)] -- the same NC * KT * 8 bytes.
__global__ void q_image_kernel(const float *q, int64_t n, int ldq, int d, int nc, int nchunk, int64_t ntiles,
                               float *img, int mixed_layout) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)nchunk * ntiles * nc * KT;
    if (e >= total) return;
    int k = (int)(e % KT);
    int64_t r = e / KT;
    int ch = (int)(r % nc);
    r /= nc;
    int64_t t = r % ntiles;
    int chunk = (int)(r / ntiles);
    int64_t j = t * KT + k;
    int gch = chunk * nc + ch;
    float v = (j < n && gch < d) ? q[j * ldq + gch] : 0.0f;
    float hi = __uint_as_float(tf32_hi_bits(v));
    float lo = v - hi;
    size_t tile_bytes = (size_t)nc * KT * 4;
    char *base = reinterpret_cast<char *>(img) + ((size_t)chunk * ntiles + t) * 2 * tile_bytes;
    uint32_t off = (uint32_t)((ch >> 3) * A_SBO + (k >> 2) * 128 + (ch & 7) * 16 + (k & 3) * 4);
    *reinterpret_cast<float *>(base + off) = hi;
    if (!mixed_layout) {
        *reinterpret_cast<float *>(base + tile_bytes + off) = lo;
        return;
    }
    const size_t bf_bytes = (size_t)nc * KT * 2;
    const uint32_t boff = (uint32_t)((ch >> 3) * (KT / 8) * 128 + (k >> 3) * 128 + (ch & 7) * 16 + (k & 7) * 2);
    *reinterpret_cast<__nv_bfloat16 *>(base + tile_bytes + boff) = __float2bfloat16_rn(lo);
    *reinterpret_cast<__nv_bfloat16 *>(base + tile_bytes + bf_bytes + boff) = __float2bfloat16_rn(hi);
}

// Warp roles: warps 0..3 (128 threads, one pixel each) evaluate moments and
// G tiles; warp 4 is the issuer: lane 0 waits for a full stage (4 warp
// arrivals + the bulk-copied Q tile's bytes), issues the MMAs and commits
// them to the stage's "empty" barrier.  No block-wide barrier per K tile;
// compute warps only wait when the ring wraps onto a stage whose MMAs are
// still in flight, and at each fp64 flush.
constexpr int SP = MDC_TC_SPLIT;
constexpr int CT = SP * TPB;             // compute threads
constexpr int CWARPS = CT / 32;          // compute warps
constexpr int THREADS = CT + 32;         // + one issuer warp
static_assert((XYR / 2) % SP == 0 && KT % (2 * SP) == 0, "halves take whole control pairs");

__device__ __forceinline__ void compute_bar_sync() {  // named barrier over the compute threads
    asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
}

template <int AM, int NC>
__global__ void __launch_bounds__(THREADS, minb<NC>()) mls_tc_kernel(KArgs a, const float *qimg, int64_t ntiles, int nchunk) {
    constexpr int B_HALF = NC * KT * 4;
    constexpr int B_STAGE = 2 * B_HALF;
    // TMEM columns: accumulators (NC) then the G ring ({hi, lo} x KT per stage)
    constexpr int ACOL = NC;
    constexpr int COLS = ACOL + STAGES * 2 * KT;
    constexpr int TMEM_COLS = COLS <= 32 ? 32 : (COLS <= 64 ? 64 : (COLS <= 128 ? 128 : (COLS <= 256 ? 256 : 512)));
    constexpr int NPAIR = XYR / 2;                     // staged control pairs per round
    constexpr int PPT = (NPAIR + CT - 1) / CT;         // pairs staged per thread
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *sB = smem;                                          // STAGES x B_STAGE
    using TotT = typename TotOf<NC>::T;
    TotT *tot = reinterpret_cast<TotT *>(sB + STAGES * B_STAGE);       // NC x TPB run totals
    float2 *sxy = reinterpret_cast<float2 *>(tot + NC * TPB);         // 2 x XYR controls
    double *red = reinterpret_cast<double *>(sxy + 2 * XYR);          // SP > 1: 6 x TPB moment totals
    float *cbuf = reinterpret_cast<float *>(red + (SP > 1 ? 6 * TPB : 0));  // SP > 1: 3 x TPB
    unsigned char *sbad = reinterpret_cast<unsigned char *>(cbuf + (SP > 1 ? 3 * TPB : 0));  // SP > 1: TPB
    uint64_t *full = reinterpret_cast<uint64_t *>(sbad + (SP > 1 ? TPB : 0));               // STAGES: G + Q ready
    uint64_t *empty = full + STAGES;                                   // STAGES: MMAs retired
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(empty + STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool issuer = warp == CWARPS;
    const int64_t tile_base = (a.tile0 + blockIdx.x) * (int64_t)TPB;
    const float neg_alpha = (float)(-a.alpha);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], CWARPS + 1);  // compute-warp arrivals + 1 expect_tx arrival
            mbar_init(&empty[s], 1);          // tcgen05.commit
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (issuer) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_tf32(NC);
    const uint32_t idesc_bf = idesc_bf16(NC);

    if (issuer) {
        // ------------------------------ MMA issuer --------------------------
        if (lane == 0) {
            uint32_t ring = 0;
            for (int chunk = 0; chunk < nchunk; ++chunk) {
                for (int64_t t = 0; t < ntiles; ++t, ++ring) {
                    const int s = ring % STAGES;
                    mbar_wait_sleep(&full[s], (ring / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t b_hi = smem_u32(sB + s * B_STAGE), b_lo = b_hi + B_HALF;
                    if constexpr (mixed<NC>()) {
                        // stage A: [G_hi tf32 (KT cols) | G_hi bf16 pairs (KT/2) | G_lo bf16 pairs (KT/2)]
                        // stage B: [Q_hi tf32 | Q_lo bf16 | Q_hi bf16]
                        const uint32_t ta = tmem + ACOL + s * 2 * KT;
#pragma unroll
                        for (int kk = 0; kk < KT / 8; ++kk)
                            mma_tf32_ts(tmem, ta + kk * 8, umma_desc(b_hi + kk * 256, 128, A_SBO), idesc,
                                        (t % FLUSH != 0 || kk > 0) ? 1u : 0u);
                        constexpr uint32_t BF_SBO = (KT / 8) * 128, BF_BYTES = NC * KT * 2;
                        mma_bf16_ts(tmem, ta + KT, umma_desc(b_lo, 128, BF_SBO), idesc_bf, 1u);
                        mma_bf16_ts(tmem, ta + KT + KT / 2, umma_desc(b_lo + BF_BYTES, 128, BF_SBO), idesc_bf, 1u);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < KT / 8; ++kk) {
                            const uint32_t koff = kk * 256;
                            // a fresh fp32 run after every fp64 flush
                            const uint32_t acc = (t % FLUSH != 0 || kk > 0) ? 1u : 0u;
                            const uint64_t dbh = umma_desc(b_hi + koff, 128, A_SBO);
                            const uint64_t dbl = umma_desc(b_lo + koff, 128, A_SBO);
                            const uint32_t ta = tmem + ACOL + s * 2 * KT + kk * 8;
                            mma_tf32_ts(tmem, ta, dbh, idesc, acc);
                            mma_tf32_ts(tmem, ta, dbl, idesc, 1u);
                            mma_tf32_ts(tmem, ta + KT, dbh, idesc, 1u);
                        }
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            smem_u32(&empty[s]))
                        : "memory");
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------ compute warps ------------------------
        double ox, oy;
        {
            int64_t mid = tile_base + TPB / 2;
            if (mid >= a.p_total) mid = a.p_total - 1;
            pixel_xy(a, mid, ox, oy);
        }
        const int pix = SP > 1 ? tid % TPB : tid, hh = SP > 1 ? tid / TPB : 0;  // pixel (TMEM lane), control half
        int64_t p = tile_base + pix;
        const bool active = p >= a.p_begin && p < a.p_end;
        if (!active) p = p < a.p_begin ? a.p_begin : a.p_end - 1;
        double vxg, vyg;
        pixel_xy(a, p, vxg, vyg);
        const float vx = (float)(vxg - ox), vy = (float)(vyg - oy);
        const int64_t n = a.n;
        const int64_t nxy = (n + XYR - 1) / XYR;
        const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;  // this warp's TMEM lanes

        // Control positions stream through a double-buffered staging area,
        // one named barrier per round.  Controls past n are parked far away
        // (weight underflows to 0, G stays finite) and their Q rows are zero:
        // full tiles, no masking.
        // Staging layout: one float4 per control PAIR, {x0, x1, y0, y1}, so
        // a 128-bit load yields packed (x0, x1) / (y0, y1) operands for the
        // f32x2 arithmetic below.  Each thread stages whole pairs.
        double2 pre[2 * PPT];
        auto fetch = [&](int64_t r) {
#pragma unroll
            for (int e = 0; e < PPT; ++e) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pi = e * CT + tid;
                    int64_t j = r * XYR + 2 * pi + h;
                    pre[2 * e + h] = (pi < NPAIR && r < nxy && j < n) ? reinterpret_cast<const double2 *>(a.pc)[j]
                                                                     : make_double2(1e300, 1e300);
                }
            }
        };
        auto store = [&](int64_t r) {
            float4 *buf = reinterpret_cast<float4 *>(sxy + (r & 1) * XYR);
#pragma unroll
            for (int e = 0; e < PPT; ++e) {
                if (e * CT + tid >= NPAIR) break;
                float x[2], y[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2 v = pre[2 * e + h];
                    x[h] = v.x == 1e300 ? 1e18f : (float)(v.x - ox);
                    y[h] = v.x == 1e300 ? 1e18f : (float)(v.y - oy);
                }
                buf[e * CT + tid] = make_float4(x[0], x[1], y[0], y[1]);
            }
        };
        auto xy_init = [&]() {
            compute_bar_sync();
            fetch(0);
            store(0);
            fetch(1);
        };
        auto xy_step = [&](int64_t r) {  // make round r readable, stage r + 1, prefetch r + 2
            compute_bar_sync();
            if (r + 1 < nxy) store(r + 1);
            fetch(r + 2);
        };

        // ---------------- pass 1: moments (SIMT, packed f32x2) ----------------
        constexpr bool TRACE = MDC_TC_P1_TRACE && AM == A_THREE_HALVES;
        // Lane 0 of each float2 accumulates the even controls, lane 1 the odd
        // ones.  The fp32 partials cover one staging round (XYR controls) and
        // are then added into fp64 totals, so the rounding error is bounded by
        // the round length instead of growing with N (100k-control frames
        // otherwise exceed the 1e-4 fp32 contract).
        const float2 nvx = make_float2(-vx, -vx), nvy = make_float2(-vy, -vy);
        double tw = 0.0, tmx = 0.0, tmy = 0.0, txx = 0.0, txy = 0.0, tyy = 0.0;
        xy_init();
        for (int64_t r = 0; r < nxy; ++r) {
            xy_step(r);
            const float4 *s4 = reinterpret_cast<const float4 *>(sxy + (r & 1) * XYR);
            const int cnt = (int)min((int64_t)XYR, n - r * XYR);
            float2 sw2 = make_float2(0.f, 0.f), mx2 = sw2, my2 = sw2, sxx2 = sw2, sxy2 = sw2, syy2 = sw2;
            auto acc = [&](const float4 pp, bool odd_tail) {
                const float2 dx = __fadd2_rn(make_float2(pp.x, pp.y), nvx);
                const float2 dy = __fadd2_rn(make_float2(pp.z, pp.w), nvy);
                if constexpr (TRACE) {
                    // alpha = 3/2: w r^2 = 1/r = y, so sum w dy^2 = sum y - sum w dx^2
                    // (the last moment becomes a plain sum: one FMUL2 less per pair)
                    const float2 d2 = __ffma2_rn(dy, dy, __fmul2_rn(dx, dx));
                    float2 y = make_float2(rsqrt_approx(d2.x), rsqrt_approx(d2.y));
                    float2 w = __fmul2_rn(__fmul2_rn(y, y), y);
                    if (odd_tail) w.y = y.y = 0.f;
                    const float2 wdx = __fmul2_rn(w, dx);
                    sw2 = __fadd2_rn(sw2, w);
                    mx2 = __fadd2_rn(mx2, wdx);
                    my2 = __ffma2_rn(w, dy, my2);
                    sxx2 = __ffma2_rn(wdx, dx, sxx2);
                    sxy2 = __ffma2_rn(wdx, dy, sxy2);
                    syy2 = __fadd2_rn(syy2, y);  // sum y (= sum w r^2)
                    return;
                }
                float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                if (odd_tail) w.y = 0.f;  // parked control (alpha < 1 does not underflow)
                const float2 wdx = __fmul2_rn(w, dx), wdy = __fmul2_rn(w, dy);
                sw2 = __fadd2_rn(sw2, w);
                mx2 = __fadd2_rn(mx2, wdx);
                my2 = __fadd2_rn(my2, wdy);
                sxx2 = __ffma2_rn(wdx, dx, sxx2);
                sxy2 = __ffma2_rn(wdx, dy, sxy2);
                syy2 = __ffma2_rn(wdy, dy, syy2);
            };
            constexpr int HP = NPAIR / SP;  // pairs per half
            const int jlo = hh * HP;
#if MDC_TC_P1STATIC
            if (cnt == XYR) {  // full round: static trip count
#pragma unroll (P1U)
                for (int j2 = 0; j2 < HP; ++j2) acc(s4[jlo + j2], false);
            } else
#endif
            {
                const int jhi = min(jlo + HP, cnt >> 1);
#pragma unroll 4
                for (int j2 = jlo; j2 < jhi; ++j2) acc(s4[j2], false);
                if ((cnt & 1) && (cnt >> 1) >= jlo && (cnt >> 1) < jlo + HP) acc(s4[cnt >> 1], true);
            }
            tw += (double)sw2.x + (double)sw2.y;
            tmx += (double)mx2.x + (double)mx2.y;
            tmy += (double)my2.x + (double)my2.y;
            txx += (double)sxx2.x + (double)sxx2.y;
            txy += (double)sxy2.x + (double)sxy2.y;
            tyy += (double)syy2.x + (double)syy2.y;
        }
        float c0 = 0.f, c1 = 0.f, c2 = 0.f;
        if (SP > 1) {  // halves' moment totals -> half 0 (fixed order: half 0 + half 1)
            if (hh == 1) {
                red[0 * TPB + pix] = tw, red[1 * TPB + pix] = tmx, red[2 * TPB + pix] = tmy;
                red[3 * TPB + pix] = txx, red[4 * TPB + pix] = txy, red[5 * TPB + pix] = tyy;
            }
            compute_bar_sync();
            if (hh == 0) {
                tw += red[0 * TPB + pix], tmx += red[1 * TPB + pix], tmy += red[2 * TPB + pix];
                txx += red[3 * TPB + pix], txy += red[4 * TPB + pix], tyy += red[5 * TPB + pix];
            }
        }
        if (hh == 0) {
            double s = tw, m0 = tmx, m1 = tmy;
            if (TRACE) tyy -= txx;  // sum w dy^2 = sum w r^2 - sum w dx^2
            double a00 = txx - m0 * m0 / s;
            double a01 = txy - m0 * m1 / s;
            double a11 = tyy - m1 * m1 / s;
            double reg = a.reg_eps * (a00 + a11);
            a00 += reg;
            a11 += reg;
            double det = a00 * a11 - a01 * a01;
            double u0 = (a11 * m0 - a01 * m1) / det;
            double u1 = (a00 * m1 - a01 * m0) / det;
            c0 = (float)(1.0 / s + (m0 * u0 + m1 * u1) / (s * s));
            c1 = (float)(-u0 / s);
            c2 = (float)(-u1 / s);
            if (SP > 1) cbuf[pix] = c0, cbuf[TPB + pix] = c1, cbuf[2 * TPB + pix] = c2;
        }
        if (SP > 1) {
            compute_bar_sync();
            c0 = cbuf[pix], c1 = cbuf[TPB + pix], c2 = cbuf[2 * TPB + pix];
        }

        // ---------------- pass 2: G tiles -> TMEM ring -> tcgen05 ----------------
        bool bad = false;
        uint32_t ring = 0;
        const float2 c0v = make_float2(c0, c0), c1v = make_float2(c1, c1), c2v = make_float2(c2, c2);
        const int64_t row = p / a.width;
        const int64_t col = p - row * a.width;
        const int64_t lr = row - a.row0;
        constexpr int TPR = XYR / KT;  // K tiles per staging round
        // Read the TMEM accumulator run (after its last MMA retired) into the
        // fp64 totals; `init` starts a chunk's totals.
        auto flush = [&](bool init) {
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int c8 = hh * (NC / 8 / SP); c8 < (hh + 1) * (NC / 8 / SP); ++c8) {  // this half's columns
                uint32_t v[8];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                    : "r"(tmem + lane_addr + c8 * 8));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    TotT &t = tot[(c8 * 8 + e) * TPB + pix];
                    t = (init ? TotT(0) : t) + (TotT)__uint_as_float(v[e]);
                }
            }
            // the next run's first MMA (accumulate = 0) overwrites these
            // columns only after this warp's next arrival
            asm volatile("tcgen05.fence::before_thread_sync;");
        };
        for (int chunk = 0; chunk < nchunk; ++chunk) {
            const char *qchunk = reinterpret_cast<const char *>(qimg) + (size_t)chunk * ntiles * B_STAGE;
            xy_init();
            for (int64_t t = 0; t < ntiles; ++t, ++ring) {
                const int tin = (int)(t % TPR);
                const int64_t round = t / TPR;
                if (tin == 0) xy_step(round);
                const int s = ring % STAGES;
                if (ring >= STAGES) {
#if MDC_TC_SLEEPC
                    mbar_wait_sleep(&empty[s], ((ring - STAGES) / STAGES) & 1);
#else
                    mbar_wait(&empty[s], ((ring - STAGES) / STAGES) & 1);
#endif
                }
                asm volatile("tcgen05.fence::after_thread_sync;");  // the stage's MMAs retired
                if (tid == 0) {  // Q tile: one bulk copy, completion counted on full[s]
                    mbar_arrive_tx(&full[s], B_STAGE);
                    bulk_g2s(sB + s * B_STAGE, qchunk + (size_t)t * B_STAGE, B_STAGE, &full[s]);
                }
                constexpr int KH = KT / SP;  // controls of the K tile this thread evaluates
                const float4 *buf = reinterpret_cast<const float4 *>(sxy + (round & 1) * XYR + tin * KT) + hh * (KH / 2);
                uint32_t ghi[KH], glo[KH];
#pragma unroll
                for (int h = 0; h < KH / 2; ++h) {
                    const float4 pp = buf[h];
                    const float2 dx = __fadd2_rn(make_float2(pp.x, pp.y), nvx);
                    const float2 dy = __fadd2_rn(make_float2(pp.z, pp.w), nvy);
                    const float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                    const float2 g = __fmul2_rn(w, __ffma2_rn(c2v, dy, __ffma2_rn(c1v, dx, c0v)));
#if MDC_TC_TRUNC
                    // truncated hi (one LOP per value): the residual stays exact in fp32
                    const float2 gh = make_float2(__uint_as_float(__float_as_uint(g.x) & 0xFFFFE000u),
                                                  __uint_as_float(__float_as_uint(g.y) & 0xFFFFE000u));
#else
                    const float2 gh = make_float2(__uint_as_float(tf32_hi_bits(g.x)), __uint_as_float(tf32_hi_bits(g.y)));
#endif
                    const float2 gl = __ffma2_rn(gh, make_float2(-1.f, -1.f), g);  // g - hi, exact
                    ghi[2 * h] = __float_as_uint(gh.x);
                    ghi[2 * h + 1] = __float_as_uint(gh.y);
                    if constexpr (mixed<NC>()) {  // [hi bf16 pairs | lo bf16 pairs]
                        glo[h] = pack_bf16(gh.x, gh.y);
                        glo[KH / 2 + h] = pack_bf16(gl.x, gl.y);
                    } else {
                        glo[2 * h] = __float_as_uint(gl.x);
                        glo[2 * h + 1] = __float_as_uint(gl.y);
                    }
                }
                // this warp's 32 rows (TMEM lanes) of the stage's G tile
                const uint32_t ta = tmem + lane_addr + ACOL + s * 2 * KT + hh * KH;
                tmem_st<KH>(ta, ghi);
                tmem_st<KH>(ta + KT, glo);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (t % FLUSH == FLUSH - 1 || t == ntiles - 1) {
                    // the run ends with this tile: MMAs retire in order
                    mbar_wait(&empty[s], (ring / STAGES) & 1);
                    flush(t < FLUSH);
                }
            }
            if (active) {
#pragma unroll 4
                for (int c = hh * (NC / SP); c < (hh + 1) * (NC / SP); ++c) {
                    const int ch = chunk * NC + c;
                    if (ch < a.d) {
                        float f = (float)((double)tot[c * TPB + pix] + a.qm[ch]);
                        reinterpret_cast<float *>(a.out)[ch * a.out_cs + lr * a.out_rs + col * a.out_ps] = f;
                        if (!isfinite(f)) bad = true;
                        store_band(a, ch, lr, col, (double)f);
                    }
                }
            }
        }
        if (SP > 1 && a.nonfinite) {  // one count per pixel (the snap pass decrements per pixel)
            if (hh == 1) sbad[pix] = bad;
            compute_bar_sync();
            if (hh == 0) bad = bad || sbad[pix];
        }
        if (a.nonfinite && active && bad && hh == 0) atomicAdd(a.nonfinite, 1);
    }
    __syncthreads();
    if (issuer) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
}

#ifndef MDC_TC_ONEPASS
#define MDC_TC_ONEPASS 0
#endif
#if MDC_TC_ONEPASS
// One-pass form (A/B experiment, DESIGN.md "Next" item 0).  Pass 2 depends on
// pass 1 only through c, so F_k = sum_m c_m T_mk with T_m = (w phi_m) . Q,
// phi = [1, dx, dy]: one sweep accumulates the 6 moments (SIMT) and the three
// contractions T_0..T_2 (tcgen05, A = {w, w dx, w dy} hi/lo per control); the
// epilogue solves for c in fp64 and combines the fp64 run totals.
template <int AM, int NC>
__global__ void __launch_bounds__(THREADS, 2) mls_tc1_kernel(KArgs a, const float *qimg, int64_t ntiles, int nchunk) {
    constexpr int B_HALF = NC * KT * 4;
    constexpr int B_STAGE = 2 * B_HALF;
    constexpr int ACOL = 3 * NC;  // T_0 | T_1 | T_2
    constexpr int GST = 6 * KT;   // ring columns per stage: {w, w dx, w dy} x {hi, lo}
    constexpr int COLS = ACOL + STAGES * GST;
    constexpr int TMEM_COLS = COLS <= 32 ? 32 : (COLS <= 64 ? 64 : (COLS <= 128 ? 128 : (COLS <= 256 ? 256 : 512)));
    constexpr int PER = XYR / TPB;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *sB = smem;
    double *tot = reinterpret_cast<double *>(sB + STAGES * B_STAGE);  // 3 NC x TPB
    float2 *sxy = reinterpret_cast<float2 *>(tot + 3 * NC * TPB);
    uint64_t *full = reinterpret_cast<uint64_t *>(sxy + 2 * XYR);
    uint64_t *empty = full + STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(empty + STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool issuer = warp == CWARPS;
    const int64_t tile_base = (a.tile0 + blockIdx.x) * (int64_t)TPB;
    const float neg_alpha = (float)(-a.alpha);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], CWARPS + 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (issuer) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_tf32(NC);

    if (issuer) {
        if (lane == 0) {
            uint32_t ring = 0;
            for (int chunk = 0; chunk < nchunk; ++chunk) {
                for (int64_t t = 0; t < ntiles; ++t, ++ring) {
                    const int s = ring % STAGES;
                    mbar_wait_sleep(&full[s], (ring / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t b_hi = smem_u32(sB + s * B_STAGE), b_lo = b_hi + B_HALF;
#pragma unroll
                    for (int kk = 0; kk < KT / 8; ++kk) {
                        const uint32_t koff = kk * 256;
                        const uint32_t acc = (t % FLUSH != 0 || kk > 0) ? 1u : 0u;
                        const uint64_t dbh = umma_desc(b_hi + koff, 128, A_SBO);
                        const uint64_t dbl = umma_desc(b_lo + koff, 128, A_SBO);
#pragma unroll
                        for (int m = 0; m < 3; ++m) {
                            const uint32_t ta = tmem + ACOL + s * GST + m * 2 * KT + kk * 8;
                            const uint32_t td = tmem + m * NC;
                            mma_tf32_ts(td, ta, dbh, idesc, acc);
                            mma_tf32_ts(td, ta, dbl, idesc, 1u);
                            mma_tf32_ts(td, ta + KT, dbh, idesc, 1u);
                        }
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            smem_u32(&empty[s]))
                        : "memory");
                }
            }
        }
        __syncwarp();
    } else {
        double ox, oy;
        {
            int64_t mid = tile_base + TPB / 2;
            if (mid >= a.p_total) mid = a.p_total - 1;
            pixel_xy(a, mid, ox, oy);
        }
        int64_t p = tile_base + tid;
        const bool active = p >= a.p_begin && p < a.p_end;
        if (!active) p = p < a.p_begin ? a.p_begin : a.p_end - 1;
        double vxg, vyg;
        pixel_xy(a, p, vxg, vyg);
        const float vx = (float)(vxg - ox), vy = (float)(vyg - oy);
        const int64_t n = a.n;
        const int64_t nxy = (n + XYR - 1) / XYR;
        const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
        static_assert(PER % 2 == 0, "controls are staged in pairs");
        double2 pre[PER];
        auto fetch = [&](int64_t r) {
#pragma unroll
            for (int e = 0; e < PER / 2; ++e) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    int64_t j = r * XYR + 2 * (e * TPB + tid) + h;
                    pre[2 * e + h] = (r < nxy && j < n) ? reinterpret_cast<const double2 *>(a.pc)[j]
                                                        : make_double2(1e300, 1e300);
                }
            }
        };
        auto store = [&](int64_t r) {
            float4 *buf = reinterpret_cast<float4 *>(sxy + (r & 1) * XYR);
#pragma unroll
            for (int e = 0; e < PER / 2; ++e) {
                float x[2], y[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2 v = pre[2 * e + h];
                    x[h] = v.x == 1e300 ? 1e18f : (float)(v.x - ox);
                    y[h] = v.x == 1e300 ? 1e18f : (float)(v.y - oy);
                }
                buf[e * TPB + tid] = make_float4(x[0], x[1], y[0], y[1]);
            }
        };
        auto xy_init = [&]() {
            compute_bar_sync();
            fetch(0);
            store(0);
            fetch(1);
        };
        auto xy_step = [&](int64_t r) {
            compute_bar_sync();
            if (r + 1 < nxy) store(r + 1);
            fetch(r + 2);
        };
        const float2 nvx = make_float2(-vx, -vx), nvy = make_float2(-vy, -vy);
        const int64_t row = p / a.width;
        const int64_t col = p - row * a.width;
        const int64_t lr = row - a.row0;
        constexpr int TPR = XYR / KT;
        auto flush = [&](bool init) {
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int c8 = 0; c8 < 3 * NC / 8; ++c8) {
                uint32_t v[8];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                    : "r"(tmem + lane_addr + c8 * 8));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    double &tt = tot[(c8 * 8 + e) * TPB + tid];
                    tt = (init ? 0.0 : tt) + (double)__uint_as_float(v[e]);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
        };
        bool bad = false;
        uint32_t ring = 0;
        for (int chunk = 0; chunk < nchunk; ++chunk) {
            const char *qchunk = reinterpret_cast<const char *>(qimg) + (size_t)chunk * ntiles * B_STAGE;
            double tw = 0.0, tmx = 0.0, tmy = 0.0, txx = 0.0, txy = 0.0, tyy = 0.0;
            float2 sw2 = make_float2(0.f, 0.f), mx2 = sw2, my2 = sw2, sxx2 = sw2, sxy2 = sw2, syy2 = sw2;
            auto fold = [&]() {  // fp32 run of one staging round -> fp64 totals
                tw += (double)sw2.x + (double)sw2.y;
                tmx += (double)mx2.x + (double)mx2.y;
                tmy += (double)my2.x + (double)my2.y;
                txx += (double)sxx2.x + (double)sxx2.y;
                txy += (double)sxy2.x + (double)sxy2.y;
                tyy += (double)syy2.x + (double)syy2.y;
                sw2 = make_float2(0.f, 0.f);
                mx2 = sw2, my2 = sw2, sxx2 = sw2, sxy2 = sw2, syy2 = sw2;
            };
            xy_init();
            for (int64_t t = 0; t < ntiles; ++t, ++ring) {
                const int tin = (int)(t % TPR);
                const int64_t round = t / TPR;
                if (tin == 0) {
                    if (t > 0) fold();
                    xy_step(round);
                }
                const int s = ring % STAGES;
                if (ring >= STAGES) mbar_wait(&empty[s], ((ring - STAGES) / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (tid == 0) {
                    mbar_arrive_tx(&full[s], B_STAGE);
                    bulk_g2s(sB + s * B_STAGE, qchunk + (size_t)t * B_STAGE, B_STAGE, &full[s]);
                }
                const float4 *buf = reinterpret_cast<const float4 *>(sxy + (round & 1) * XYR + tin * KT);
                const int64_t jt = t * KT;  // first control of the tile
                uint32_t ahi[3][KT], alo[3][KT];
#pragma unroll
                for (int h = 0; h < KT / 2; ++h) {
                    const float4 pp = buf[h];
                    const float2 dx = __fadd2_rn(make_float2(pp.x, pp.y), nvx);
                    const float2 dy = __fadd2_rn(make_float2(pp.z, pp.w), nvy);
                    float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                    if (jt + 2 * h + 1 >= n) {  // parked controls (alpha < 1 does not underflow)
                        if (jt + 2 * h >= n) w.x = 0.f;
                        w.y = 0.f;
                    }
                    const float2 wdx = __fmul2_rn(w, dx), wdy = __fmul2_rn(w, dy);
                    sw2 = __fadd2_rn(sw2, w);
                    mx2 = __fadd2_rn(mx2, wdx);
                    my2 = __fadd2_rn(my2, wdy);
                    sxx2 = __ffma2_rn(wdx, dx, sxx2);
                    sxy2 = __ffma2_rn(wdx, dy, sxy2);
                    syy2 = __ffma2_rn(wdy, dy, syy2);
                    const float2 av[3] = {w, wdx, wdy};
#pragma unroll
                    for (int m = 0; m < 3; ++m) {
                        const float2 gh =
                            make_float2(__uint_as_float(tf32_hi_bits(av[m].x)), __uint_as_float(tf32_hi_bits(av[m].y)));
                        const float2 gl = __ffma2_rn(gh, make_float2(-1.f, -1.f), av[m]);
                        ahi[m][2 * h] = __float_as_uint(gh.x);
                        ahi[m][2 * h + 1] = __float_as_uint(gh.y);
                        alo[m][2 * h] = __float_as_uint(gl.x);
                        alo[m][2 * h + 1] = __float_as_uint(gl.y);
                    }
                }
                const uint32_t ta = tmem + lane_addr + ACOL + s * GST;
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    tmem_st<KT>(ta + m * 2 * KT, ahi[m]);
                    tmem_st<KT>(ta + m * 2 * KT + KT, alo[m]);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                if (t % FLUSH == FLUSH - 1 || t == ntiles - 1) {
                    mbar_wait(&empty[s], (ring / STAGES) & 1);
                    flush(t < FLUSH);
                }
            }
            fold();
            double c0, c1, c2;
            {
                double s = tw, m0 = tmx, m1 = tmy;
                double a00 = txx - m0 * m0 / s;
                double a01 = txy - m0 * m1 / s;
                double a11 = tyy - m1 * m1 / s;
                double reg = a.reg_eps * (a00 + a11);
                a00 += reg;
                a11 += reg;
                double det = a00 * a11 - a01 * a01;
                double u0 = (a11 * m0 - a01 * m1) / det;
                double u1 = (a00 * m1 - a01 * m0) / det;
                c0 = 1.0 / s + (m0 * u0 + m1 * u1) / (s * s);
                c1 = -u0 / s;
                c2 = -u1 / s;
            }
            if (active) {
#pragma unroll 4
                for (int c = 0; c < NC; ++c) {
                    const int ch = chunk * NC + c;
                    if (ch < a.d) {
                        const double F = c0 * tot[c * TPB + tid] + c1 * tot[(NC + c) * TPB + tid] +
                                         c2 * tot[(2 * NC + c) * TPB + tid];
                        float f = (float)(F + a.qm[ch]);
                        reinterpret_cast<float *>(a.out)[ch * a.out_cs + lr * a.out_rs + col * a.out_ps] = f;
                        if (!isfinite(f)) bad = true;
                        store_band(a, ch, lr, col, (double)f);
                    }
                }
            }
        }
        if (a.nonfinite && active && bad) atomicAdd(a.nonfinite, 1);
    }
    __syncthreads();
    if (issuer) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
}
constexpr int TOT_SETS = 3;
#else
constexpr int TOT_SETS = 1;
#endif

template <int NC>
static size_t tc_smem_bytes() {
    return STAGES * (size_t)(2 * NC * KT * 4) + (size_t)TOT_SETS * NC * TPB * sizeof(typename TotOf<NC>::T) +
           2 * XYR * sizeof(float2) + (SP > 1 ? TPB * (6 * sizeof(double) + 3 * sizeof(float) + 1) : 0) +
           2 * STAGES * sizeof(uint64_t) + 16;
}

static int pick_nc(int d) {
    if (d <= 16) return 16;
    if (d <= NC_MAX || !MDC_TC_WIDE) return NC_MAX;
    if (d <= MDC_TC_WIDE || !MDC_TC_WIDE2) return MDC_TC_WIDE;
    return MDC_TC_WIDE2;
}

}  // namespace tc

size_t mls_tc_workspace_bytes(int d, int64_t n) {
    int nc = tc::pick_nc(d);
    int nchunk = (d + nc - 1) / nc;
    int64_t ntiles = (n + tc::KT - 1) / tc::KT;
    return (size_t)nchunk * ntiles * 2 * nc * tc::KT * 4 + 256;
}

template <int AM, int NC>
static int launch_tc_nc(const KArgs &k, void *ws, cudaStream_t s) {
    using namespace tc;
    const int nchunk = (k.d + NC - 1) / NC;
    const int64_t ntiles = (k.n + KT - 1) / KT;
    float *img = reinterpret_cast<float *>(ws);
    int64_t total = (int64_t)nchunk * ntiles * NC * KT;
    q_image_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(reinterpret_cast<const float *>(k.q), k.n,
                                                                   k.ldq, k.d, NC, nchunk, ntiles, img,
                                                                   mixed<NC>() ? 1 : 0);
#if MDC_TC_ONEPASS
    auto fn = mls_tc1_kernel<AM, NC>;
#else
    auto fn = mls_tc_kernel<AM, NC>;
#endif
    size_t smem = tc_smem_bytes<NC>();
    MDC_CHECK_CUDA(ensure_dynamic_smem((const void *)fn, (int)smem));
    KArgs kk = k;
    kk.tile0 = kk.p_begin / TPB;
    int64_t blocks = (kk.p_end + TPB - 1) / TPB - kk.tile0;
    if (blocks > 0) fn<<<(unsigned)blocks, THREADS, smem, s>>>(kk, img, ntiles, nchunk);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

template <int AM>
static int launch_tc_am(const KArgs &k, void *ws, cudaStream_t s) {
    switch (tc::pick_nc(k.d)) {
        case 16: return launch_tc_nc<AM, 16>(k, ws, s);
#if MDC_TC_WIDE
        case MDC_TC_WIDE: return launch_tc_nc<AM, MDC_TC_WIDE>(k, ws, s);
#endif
#if MDC_TC_WIDE2
        case MDC_TC_WIDE2: return launch_tc_nc<AM, MDC_TC_WIDE2>(k, ws, s);
#endif
        default: return launch_tc_nc<AM, tc::NC_MAX>(k, ws, s);
    }
}

int launch_mls_tc(const KArgs &k, void *ws, cudaStream_t s) {
    switch (alpha_mode(k.alpha)) {
        case A_ONE: return launch_tc_am<A_ONE>(k, ws, s);
        case A_THREE_HALVES: return launch_tc_am<A_THREE_HALVES>(k, ws, s);
        case A_HALF: return launch_tc_am<A_HALF>(k, ws, s);
        case A_TWO: return launch_tc_am<A_TWO>(k, ws, s);
        default: return launch_tc_am<A_GENERIC>(k, ws, s);
    }
}

}  // namespace mdc
