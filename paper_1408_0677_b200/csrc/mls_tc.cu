// mls_tc.cu -- affine MLS with the pass-2 contraction on the 5th-gen tensor
// cores (tcgen05, kind::tf32, 3xTF32 split, accumulators in TMEM).
//
// Same mathematics as mls.cu (SURVEY.md §8a M6'; reference _kernels.py:70-124):
//   pass 1 (SIMT, fp32 FMA pipe): 6 pixel-local moments -> c = A_reg^{-1} e0
//   pass 2: F[p, k] = sum_j G[p, j] Q[j, k],  G[p, j] = w_pj (c0 + c1 dx + c2 dy)
// Pass 2 is a dense (pixels x N) . (N x d) contraction (north_star: "tensor
// cores ... only for the global-support weight case").  The SIMT threads only
// evaluate G (one weight per pair) and store it, split hi + lo, straight into
// shared memory in the UMMA K-major core-matrix layout; one elected thread
// issues tcgen05.mma (M = 128 pixels, N = channels, K = 8 controls) x 3
// (hi*hi + hi*lo + lo*hi, ~fp32-accurate) per K step, accumulating in TMEM.
// A two-stage ring (mbarrier armed by tcgen05.commit) overlaps the tensor
// core with the SIMT evaluation of the next tile.  The target block Q is
// pre-arranged once per call into the same core-matrix layout (hi/lo), so its
// tiles are plain contiguous cp.async copies.
//
// Tile geometry (A/B-tuned): CTA = 128 pixels (one M = 128 MMA tile) + an
// issuer warp, K tile = 16 controls, 2-stage ring, 5 CTAs per SM.
#include "mls_common.cuh"
#include "tcgen05.cuh"

namespace mdc {
namespace tc {

#ifndef MDC_TC_TPB
#define MDC_TC_TPB 128
#endif
constexpr int TPB = MDC_TC_TPB;   // compute threads == pixels per CTA (multiple of 128)
constexpr int MT = TPB / 128;     // M = 128 MMA tiles per CTA
constexpr int XYR = 256;          // controls per position staging round
#ifndef MDC_TC_KT
#define MDC_TC_KT 16
#endif
#ifndef MDC_TC_STAGES
#define MDC_TC_STAGES 2
#endif
#ifndef MDC_TC_MINB
#define MDC_TC_MINB 5
#endif
constexpr int KT = MDC_TC_KT;          // controls per K tile (multiple of 8 = tcgen05 tf32 K)
constexpr int STAGES = MDC_TC_STAGES;  // ring depth
constexpr int A_SBO = (KT / 4) * 128;                  // bytes between 8-row core-matrix groups
constexpr int A_HALF = (TPB / 8) * A_SBO;              // one of hi/lo: TPB rows x KT
constexpr int A_STAGE = 2 * A_HALF;

// byte offset of (row m, k) in a K-major core-matrix tile with SBO = A_SBO
__device__ __forceinline__ uint32_t cm_off(int m, int k) {
    return (uint32_t)((m >> 3) * A_SBO + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4);
}

// ---------------------------------------------------------------------------
// Q -> tiled core-matrix image, hi/lo split.  img[(chunk * ntiles + t)][hi|lo]
// each half = NC rows (channels) x KT controls = NC * KT * 4 bytes.
__global__ void q_image_kernel(const float *q, int64_t n, int ldq, int d, int nc, int nchunk, int64_t ntiles,
                               float *img) {
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
    *reinterpret_cast<float *>(base + tile_bytes + off) = lo;
}

// Warp roles: warps 0..7 (256 threads, one pixel each) evaluate moments and
// G tiles; warp 8 is the producer/issuer: lane 0 waits for a full stage
// (8 warp arrivals + the bulk-copied Q tile's bytes), issues the MMAs and
// commits them to the stage's "empty" barrier.  No block-wide barrier per
// K tile; compute warps only wait when the ring wraps onto a stage whose
// MMAs are still in flight.
constexpr int CWARPS = TPB / 32;        // compute warps
constexpr int THREADS = TPB + 32;       // + one issuer warp

__device__ __forceinline__ void compute_bar_sync() {  // named barrier over the 256 compute threads
    asm volatile("bar.sync 1, %0;" ::"n"(TPB) : "memory");
}

template <int AM, int NC>
__global__ void __launch_bounds__(THREADS, MDC_TC_MINB) mls_tc_kernel(KArgs a, const float *qimg, int64_t ntiles, int nchunk) {
    constexpr int B_HALF = NC * KT * 4;
    constexpr int B_STAGE = 2 * B_HALF;
    constexpr int COLS = MT * NC;
    constexpr int TMEM_COLS = COLS <= 32 ? 32 : (COLS <= 64 ? 64 : (COLS <= 128 ? 128 : 256));
    constexpr int PER = XYR / TPB;  // staged controls per thread per round
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *sA = smem;                                          // STAGES x A_STAGE
    unsigned char *sB = sA + STAGES * A_STAGE;                         // STAGES x B_STAGE
    float2 *sxy = reinterpret_cast<float2 *>(sB + STAGES * B_STAGE);  // 2 x XYR controls
    uint64_t *full = reinterpret_cast<uint64_t *>(sxy + 2 * XYR);     // STAGES: G + Q ready
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

    if (issuer) {
        // ------------------------------ MMA issuer --------------------------
        if (lane == 0) {
            uint32_t ring = 0;
#ifdef MDC_TC_PASS1_ONLY
            nchunk = 0;
#endif
            for (int chunk = 0; chunk < nchunk; ++chunk) {
                for (int64_t t = 0; t < ntiles; ++t, ++ring) {
                    const int s = ring % STAGES;
                    mbar_wait(&full[s], (ring / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    unsigned char *as = sA + s * A_STAGE;
                    unsigned char *bs = sB + s * B_STAGE;
                    const uint32_t a_hi = smem_u32(as), a_lo = smem_u32(as + A_HALF);
                    const uint32_t b_hi = smem_u32(bs), b_lo = smem_u32(bs + B_HALF);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        const uint32_t dcol = tmem + mt * NC;
                        const uint32_t moff = mt * (128 / 8) * A_SBO;
#pragma unroll
                        for (int kk = 0; kk < KT / 8; ++kk) {
                            const uint32_t koff = kk * 256;
                            const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
                            const uint64_t dah = umma_desc(a_hi + moff + koff, 128, A_SBO);
                            const uint64_t dal = umma_desc(a_lo + moff + koff, 128, A_SBO);
                            const uint64_t dbh = umma_desc(b_hi + koff, 128, A_SBO);
                            const uint64_t dbl = umma_desc(b_lo + koff, 128, A_SBO);
                            mma_tf32(dcol, dah, dbh, idesc, acc);
                            mma_tf32(dcol, dah, dbl, idesc, 1u);
                            mma_tf32(dcol, dal, dbh, idesc, 1u);
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
        int64_t p = tile_base + tid;
        const bool active = p >= a.p_begin && p < a.p_end;
        if (!active) p = p < a.p_begin ? a.p_begin : a.p_end - 1;
        double vxg, vyg;
        pixel_xy(a, p, vxg, vyg);
        const float vx = (float)(vxg - ox), vy = (float)(vyg - oy);
        const int64_t n = a.n;
        const int64_t nxy = (n + XYR - 1) / XYR;

        // Control positions stream through a double-buffered staging area,
        // one named barrier per round.  Controls past n are parked far away
        // (weight underflows to 0, G stays finite) and their Q rows are zero:
        // full tiles, no masking.
        double2 pre[PER];
        auto fetch = [&](int64_t r) {
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                int64_t j = r * XYR + e * TPB + tid;
                pre[e] = (r < nxy && j < n) ? reinterpret_cast<const double2 *>(a.pc)[j] : make_double2(1e300, 1e300);
            }
        };
        auto store = [&](int64_t r) {
            float2 *buf = sxy + (r & 1) * XYR;
#pragma unroll
            for (int e = 0; e < PER; ++e)
                buf[e * TPB + tid] = pre[e].x == 1e300 ? make_float2(1e18f, 1e18f)
                                                       : make_float2((float)(pre[e].x - ox), (float)(pre[e].y - oy));
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

        // ---------------- pass 1: moments (SIMT) ----------------
        float sw = 0.f, mx = 0.f, my = 0.f, sxx = 0.f, sxy_ = 0.f, syy = 0.f;
        xy_init();
        for (int64_t r = 0; r < nxy; ++r) {
            xy_step(r);
            const float2 *buf = sxy + (r & 1) * XYR;
            const int cnt = (int)min((int64_t)XYR, n - r * XYR);
            const float4 *s4 = reinterpret_cast<const float4 *>(buf);
            int j = 0;
#pragma unroll 4
            for (; j + 1 < cnt; j += 2) {
                float4 pp = s4[j >> 1];
                {
                    float dx = pp.x - vx, dy = pp.y - vy;
                    float w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                    float wdx = w * dx, wdy = w * dy;
                    sw += w; mx += wdx; my += wdy;
                    sxx += wdx * dx; sxy_ += wdx * dy; syy += wdy * dy;
                }
                {
                    float dx = pp.z - vx, dy = pp.w - vy;
                    float w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                    float wdx = w * dx, wdy = w * dy;
                    sw += w; mx += wdx; my += wdy;
                    sxx += wdx * dx; sxy_ += wdx * dy; syy += wdy * dy;
                }
            }
            if (j < cnt) {
                float2 pp = buf[j];
                float dx = pp.x - vx, dy = pp.y - vy;
                float w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                float wdx = w * dx, wdy = w * dy;
                sw += w; mx += wdx; my += wdy;
                sxx += wdx * dx; sxy_ += wdx * dy; syy += wdy * dy;
            }
        }
        float c0, c1, c2;
        {
            double s = sw, m0 = mx, m1 = my;
            double a00 = (double)sxx - m0 * m0 / s;
            double a01 = (double)sxy_ - m0 * m1 / s;
            double a11 = (double)syy - m1 * m1 / s;
            double reg = a.reg_eps * (a00 + a11);
            a00 += reg;
            a11 += reg;
            double det = a00 * a11 - a01 * a01;
            double u0 = (a11 * m0 - a01 * m1) / det;
            double u1 = (a00 * m1 - a01 * m0) / det;
            c0 = (float)(1.0 / s + (m0 * u0 + m1 * u1) / (s * s));
            c1 = (float)(-u0 / s);
            c2 = (float)(-u1 / s);
        }

        // ---------------- pass 2: G tiles -> ring -> tcgen05 ----------------
#ifdef MDC_TC_PASS1_ONLY
        if (c0 == 12345.f) a.nonfinite[0] = 1;  // keep pass 1 alive
        nchunk = 0;
#endif
        bool bad = false;
        uint32_t ring = 0;
        const int64_t row = p / a.width;
        const int64_t col = p - row * a.width;
        const int64_t lr = row - a.row0;
        constexpr int TPR = XYR / KT;  // K tiles per staging round
        for (int chunk = 0; chunk < nchunk; ++chunk) {
            const char *qchunk = reinterpret_cast<const char *>(qimg) + (size_t)chunk * ntiles * B_STAGE;
            xy_init();
            for (int64_t t = 0; t < ntiles; ++t, ++ring) {
                const int tin = (int)(t % TPR);
                const int64_t round = t / TPR;
                if (tin == 0) xy_step(round);
                const int s = ring % STAGES;
                if (ring >= STAGES) mbar_wait(&empty[s], ((ring - STAGES) / STAGES) & 1);
                unsigned char *as = sA + s * A_STAGE;
                if (tid == 0) {  // Q tile: one bulk copy, completion counted on full[s]
                    mbar_arrive_tx(&full[s], B_STAGE);
                    bulk_g2s(sB + s * B_STAGE, qchunk + (size_t)t * B_STAGE, B_STAGE, &full[s]);
                }
                const float2 *buf = sxy + (round & 1) * XYR + tin * KT;
#pragma unroll
                for (int q4 = 0; q4 < KT / 4; ++q4) {
                    const float4 *s4 = reinterpret_cast<const float4 *>(buf + q4 * 4);
                    float g[4];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float4 pp = s4[h];
                        float dx = pp.x - vx, dy = pp.y - vy;
                        float w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                        g[2 * h] = w * (c0 + c1 * dx + c2 * dy);
                        dx = pp.z - vx;
                        dy = pp.w - vy;
                        w = weight<AM>(dx * dx + dy * dy, neg_alpha);
                        g[2 * h + 1] = w * (c0 + c1 * dx + c2 * dy);
                    }
                    uint4 hi, lo;
                    uint32_t *hp = &hi.x, *lp = &lo.x;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uint32_t hb = tf32_hi_bits(g[e]);
                        hp[e] = hb;
                        lp[e] = __float_as_uint(g[e] - __uint_as_float(hb));
                    }
                    const uint32_t off = cm_off(tid, q4 * 4);
                    *reinterpret_cast<uint4 *>(as + off) = hi;
                    *reinterpret_cast<uint4 *>(as + A_HALF + off) = lo;
                }
                // make this warp's generic-proxy stores visible to the tensor core
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
            // drain: the chunk's last MMAs retire in order
            {
                const uint32_t last = ring - 1;
                mbar_wait(&empty[last % STAGES], (last / STAGES) & 1);
            }
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
            const uint32_t col0 = tmem + (warp >> 2) * NC;
#pragma unroll
            for (int c8 = 0; c8 < NC / 8; ++c8) {
                uint32_t v[8];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                    : "r"(lane_base + col0 + c8 * 8));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (active) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int ch = chunk * NC + c8 * 8 + e;
                        if (ch < a.d) {
                            float f = (float)((double)__uint_as_float(v[e]) + a.qm[ch]);
                            reinterpret_cast<float *>(a.out)[ch * a.out_cs + lr * a.out_rs + col * a.out_ps] = f;
                            if (!isfinite(f)) bad = true;
                            if (a.bands)
                                a.bands[ch * a.band_cs + lr * a.band_rs + col] =
                                    (int32_t)floor((double)f / a.spacing[ch]);
                        }
                    }
                }
            }
            // TMEM is re-used by the next chunk's first MMA, which the issuer
            // only starts after every compute warp has arrived on that tile
            // (i.e. after these tcgen05.ld completed).
            asm volatile("tcgen05.fence::before_thread_sync;");
        }
        if (a.nonfinite && active && bad) atomicAdd(a.nonfinite, 1);
    }
    __syncthreads();
    if (issuer) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
}

template <int NC>
static size_t tc_smem_bytes() {
    return STAGES * (size_t)A_STAGE + STAGES * (size_t)(2 * NC * KT * 4) + 2 * XYR * sizeof(float2) +
           2 * STAGES * sizeof(uint64_t) + 16;
}

static int pick_nc(int d) { return d <= 16 ? 16 : (d <= 32 ? 32 : 64); }

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
                                                                   k.ldq, k.d, NC, nchunk, ntiles, img);
    auto fn = mls_tc_kernel<AM, NC>;
    size_t smem = tc_smem_bytes<NC>();
    static bool attr = false;
    if (!attr) {
        MDC_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
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
        case 32: return launch_tc_nc<AM, 32>(k, ws, s);
        default: return launch_tc_nc<AM, 64>(k, ws, s);
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
