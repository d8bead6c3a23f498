// mls_tc2.cu -- one-pass affine MLS on the 5th-gen tensor cores with the
// basis expansion on the B side (default fp32 affine path for d >= 8).
//
// Same field as mls.cu / mls_tc.cu (SURVEY.md §8a M6'; reference
// _kernels.py:70-124).  In a frame centred on the CTA's 16x8 pixel tile,
// with X_j, Y_j the control coordinates and (a, b) the pixel offset, the
// pixel-local basis is phi = [1, X - a, Y - b], so every per-pixel sum the
// affine solve needs is a contraction of the weight row w[p, :] with a
// per-CONTROL column block that does not depend on the pixel:
//     B_j = [ q_j | X_j q_j | Y_j q_j | 1, X_j, Y_j, X_j^2, X_j Y_j, Y_j^2 ]
//     T[p, :] = sum_j w_pj B_j        (pixels x N) . (N x (3 NC + 6))
// and the epilogue shifts the tile-frame moments / right-hand sides to the
// pixel frame in fp64, solves the 3x3 system and forms
//     f_k = c0 T0k + c1 (TXk - a T0k) + c2 (TYk - b T0k).
// The SIMT side is the weight alone (one MUFU, ~6.5 issue slots per pair);
// the tensor cores carry the 6 moments and the 3 NC right-hand sides.
//
// Precision (3-term split, mixed kinds): w = w_hi + w_lo (w_hi = tf32
// truncation), B = B_hi + B_lo (likewise),
//     T += w_hi . B_hi                    tcgen05 kind::tf32
//        + [w_hi | w_lo] . [B_lo ; B_hi]  tcgen05 kind::f16 (bf16 operands)
// The two correction products only need ~8 significant bits (they are
// 2^-11 of the main term), so bf16 carries them at twice the tf32 rate:
// 2 tf32-equivalent MMA passes per pair instead of 3.  A numpy model of this
// exact scheme on a config-3 frame gives 4.6e-6 normwise (3xTF32: 3.0e-6;
// dropping w_lo: 2e-4, over the 1e-4 contract).
// fp32 accumulation runs are FLUSH K tiles long; the runs are added into fp64
// registers (two accumulator regions in TMEM, so the pixel warps drain run r
// while the tensor cores fill run r + 1).
//
// Warp roles (1 CTA per SM, 384 threads):
//   warps 0..7   pixel warps: thread = (pixel row m of the tile = TMEM lane,
//                half h = control half of each K tile / channel half of the
//                epilogue).  Weights -> tcgen05.st into the A ring in TMEM.
//   warps 8..10  builders: stage positions (fp64 -> tile-centred fp32) and
//                targets (bulk copy) per 256-control round; build the B tile
//                (tf32 + bf16 hi/lo, UMMA K-major core matrices) per K tile.
//   warp 11      MMA issuer (one elected thread).
#include "mls_common.cuh"
#include "tcgen05.cuh"

namespace mdc {
namespace tc2 {
using namespace ::mdc::tc;

constexpr int TW = 16, TH = 8, TP = TW * TH;  // pixel tile = MMA M
#ifndef MDC_TC2_KQ
#define MDC_TC2_KQ 1  // K tile = 16 KQ controls (each pixel warp half: 8 KQ per tile)
#endif
constexpr int KQ = MDC_TC2_KQ;
constexpr int KT = 16 * KQ;                   // controls per K tile
constexpr int XYR = 256;                      // controls per staging round
constexpr int TPR = XYR / KT;                 // K tiles per round
#ifndef MDC_TC2_STAGES
#define MDC_TC2_STAGES 8
#endif
#ifndef MDC_TC2_FLUSH
#define MDC_TC2_FLUSH 16
#endif
#ifndef MDC_TC2_NACC
#define MDC_TC2_NACC 2
#endif
#ifndef MDC_TC2_LAG
#define MDC_TC2_LAG (MDC_TC2_STAGES + 2)
#endif
#ifndef MDC_TC2_EXP
#define MDC_TC2_EXP 0  // timing experiments only (bit mask): 1 no B build, 2 no weights, 4 no MMAs
#endif
#ifndef MDC_TC2_PROF
#define MDC_TC2_PROF 0  // experiments: per-role cycle breakdown printed by CTA 0
#endif
#if MDC_TC2_PROF
struct Prof {
    long long c[8];
};
#define PDECL Prof P = {}
#define PBEGIN(v) long long v = clock64()
#define PEND(i, v) P.c[i] += clock64() - v
#define PREPORT(name)                                                                                           \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)                                                             \
        printf("%s w%d: %lld %lld %lld %lld %lld %lld\n", name, threadIdx.x >> 5, P.c[0], P.c[1], P.c[2], P.c[3], \
               P.c[4], P.c[5])
#else
#define PDECL do {} while (0)
#define PBEGIN(v) do {} while (0)
#define PEND(i, v) do {} while (0)
#define PREPORT(name) do {} while (0)
#endif
#ifndef MDC_TC2_PARK
#define MDC_TC2_PARK 1  // pixel / builder warps park (suspend-hinted try_wait) instead of spinning on the ring
#endif
constexpr int STAGES = MDC_TC2_STAGES;
constexpr int FLUSH = MDC_TC2_FLUSH;  // K tiles per fp32 accumulation run
constexpr int NACC = MDC_TC2_NACC;    // accumulator regions in TMEM (runs in flight)
constexpr int LAG = MDC_TC2_LAG;      // pixel warps drain run r after tile LAG of run r + 1
static_assert(LAG < (NACC - 1) * FLUSH, "a region is drained before the tensor cores reuse it");
constexpr int PW = 8, BW = 3;         // pixel / builder warps (12 warps: 3 per SMSP -> 168 registers)
constexpr int THREADS = (PW + BW + 1) * 32;
constexpr int BT = BW * 32;           // builder threads
constexpr int ASTAGE = 32 * KQ;       // TMEM columns per A stage: per half [tf32 8KQ | bf16 hi 4KQ | bf16 lo 4KQ]
constexpr int GSBO = 512 * KQ;        // bytes per 8-row core-matrix group of one B operand part
constexpr int QSTRIDE = XYR + 4;      // staged targets: channel-major rows, padded (conflict-free LDS.128)

template <int NC>
struct Geo {
    static constexpr int NCOL = ((3 * NC + 6) + 15) / 16 * 16;  // MMA N
    static constexpr int G = NCOL / 8;                          // 8-row core-matrix groups
    static constexpr int PART = G * GSBO;                       // bytes of one operand part per stage
    static constexpr int BSTAGE = 2 * PART;                     // tf32 part + bf16 part
    static constexpr int ACC = 0;                               // accumulator regions [0, 2 NCOL)
    static constexpr int ARING = NACC * NCOL;
    static constexpr int COLS = ARING + STAGES * ASTAGE;
    static_assert(COLS <= 512, "TMEM budget");
    static constexpr int QBYTES = NC * QSTRIDE * 4;  // one round of staged targets
    static constexpr size_t SMEM = (size_t)STAGES * BSTAGE + 2 * (size_t)QBYTES + 2 * XYR * sizeof(float2) +
                                   (2 * STAGES + 6 + 2 * NACC) * sizeof(uint64_t) + 16 + TP;
};

__device__ __forceinline__ void ring_wait(uint64_t *bar, uint32_t parity) {
#if MDC_TC2_PARK
    mbar_wait_sleep(bar, parity);
#else
    mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[N]);
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// Byte offsets inside one B stage.  tf32 part: rows n (MMA N) x KT controls,
// core matrices of 8 rows x 4 controls; bf16 part: rows n x 2 KT "k" slots in
// 8-slot k-blocks, per pixel-warp half h: KQ blocks of B_lo then KQ blocks of
// B_hi for its 8 KQ controls (lo_block / hi_block below).
__device__ __forceinline__ uint32_t tf_off(int n, int k) { return (n >> 3) * GSBO + (k >> 2) * 128 + (n & 7) * 16; }
template <int PART>
__device__ __forceinline__ uint32_t bf_off(int n, int kb, int kin) {
    return PART + (n >> 3) * GSBO + kb * 128 + (n & 7) * 16 + kin * 2;
}
// 8-control block kb8 (0 .. 2 KQ - 1) of a K tile: its half and bf16 k-blocks
__device__ __forceinline__ int lo_block(int kb8) { return 2 * KQ * (kb8 / KQ) + kb8 % KQ; }
__device__ __forceinline__ int hi_block(int kb8) { return 2 * KQ * (kb8 / KQ) + KQ + kb8 % KQ; }

// Targets, chunk-major, channel-major within a staging round and zero-padded
// to whole rounds: img[((chunk * nr + r) * nc + c) * QSTRIDE + jl] =
// q[r * XYR + jl][chunk * nc + c]  (one bulk copy per round).
__global__ void q2_image_kernel(const float *q, int64_t n, int ldq, int d, int nc, int nchunk, int64_t nr,
                                float *img) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t total = (int64_t)nchunk * nr * nc * QSTRIDE;
    if (e >= total) return;
    int jl = (int)(e % QSTRIDE);
    int64_t rc = e / QSTRIDE;  // (chunk * nr + r) * nc + c
    int c = (int)(rc % nc);
    int64_t R = rc / nc;
    int64_t r = R % nr;
    int chunk = (int)(R / nr);
    int64_t j = r * XYR + jl;
    int ch = chunk * nc + c;
    img[e] = (jl < XYR && j < n && ch < d) ? q[j * ldq + ch] : 0.0f;
}

__device__ __forceinline__ void pixel_xy_rc(const KArgs &a, int64_t row, int64_t col, double &vx, double &vy) {
    double xs = dadd(a.x0, dmul((double)col + 0.5, a.sx));
    double ys = dsub(a.y1, dmul((double)row + 0.5, a.sy));
    const double pmx = a.pm_dev ? __ldg(a.pm_dev) : a.pmx, pmy = a.pm_dev ? __ldg(a.pm_dev + 1) : a.pmy;
    vx = dsub(xs, pmx);
    vy = dsub(ys, pmy);
}

struct Args2 {
    int tiles_x, ty0;
    int64_t ntiles, nr;  // K tiles / staging rounds per chunk
    int nchunk;
};

template <int AM, int NC>
__global__ void __launch_bounds__(THREADS, 1) mls_tc2_kernel(KArgs a, const float *qimg, Args2 g2) {
    using GE = Geo<NC>;
    constexpr int NCOL = GE::NCOL, PART = GE::PART, BSTAGE = GE::BSTAGE;
    constexpr int NH = NC / 2;  // channels per half
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *sB = smem;
    float *sq = reinterpret_cast<float *>(sB + STAGES * BSTAGE);            // 2 x NC x QSTRIDE
    float4 *sxy = reinterpret_cast<float4 *>(sq + 2 * NC * QSTRIDE);        // 2 x XYR/2 pairs
    uint64_t *full = reinterpret_cast<uint64_t *>(sxy + XYR);               // STAGES
    uint64_t *empty = full + STAGES;                                        // STAGES
    uint64_t *xy_full = empty + STAGES, *xy_empty = xy_full + 2, *q_full = xy_empty + 2;
    uint64_t *acc_full = q_full + 2, *acc_free = acc_full + NACC;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_free + NACC);
    unsigned char *sbad = reinterpret_cast<unsigned char *>(tmem_slot + 4);  // TP flags

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tx = (int)(blockIdx.x % g2.tiles_x);
    const int ty = g2.ty0 + (int)(blockIdx.x / g2.tiles_x);
    const int64_t n = a.n;
    const int ntiles = (int)g2.ntiles, nr = (int)g2.nr;
    const int nchunk = g2.nchunk;
    constexpr int QROUND = NC * QSTRIDE;  // floats per staged round
    // tile frame origin (fp64): the tile's centre
    const double pmx = a.pm_dev ? __ldg(a.pm_dev) : a.pmx, pmy = a.pm_dev ? __ldg(a.pm_dev + 1) : a.pmy;
    const double cx = dsub(dadd(a.x0, dmul((double)(tx * TW + TW / 2), a.sx)), pmx);
    const double cy = dsub(dsub(a.y1, dmul((double)(ty * TH + TH / 2), a.sy)), pmy);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], PW + BW);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&xy_full[b], BW);
            mbar_init(&xy_empty[b], PW);
            mbar_init(&q_full[b], 1);
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_free[b], PW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == PW + BW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp >= PW && warp < PW + BW) {
        // zero every stage once: the pad rows (3 NC + 6 .. NCOL) are never written again
        const int bt = tid - PW * 32;
        for (int e = bt; e < STAGES * BSTAGE / 16; e += BT) reinterpret_cast<float4 *>(sB)[e] = make_float4(0, 0, 0, 0);
        fence_async_smem();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == PW + BW) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            const uint32_t id_tf = idesc_tf32(NCOL), id_bf = idesc_bf16(NCOL);
            const uint32_t sb0 = smem_u32(sB);
            int s = 0;
            uint32_t ph = 0;
            int run = 0;  // global accumulation run
            PDECL;
            PBEGIN(tall);
            for (int chunk = 0; chunk < nchunk; ++chunk) {
                int tr = 0;  // tile within the run
                for (int t = 0; t < ntiles; ++t) {
                    const uint32_t d = tmem + (uint32_t)((run % NACC) * NCOL);
                    PBEGIN(t0);
                    if (tr == 0 && run >= NACC) mbar_wait_sleep(&acc_free[run % NACC], (uint32_t)((run / NACC - 1) & 1));
                    PEND(0, t0);
                    PBEGIN(t1);
#if MDC_TC2_ISSUER_SPIN
                    mbar_wait(&full[s], ph);
#else
                    mbar_wait_sleep(&full[s], ph);
#endif
                    PEND(1, t1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t bs = sb0 + s * BSTAGE;
                    const uint32_t ta = tmem + GE::ARING + s * ASTAGE;
#pragma unroll
                    for (int h = 0; h < 2 * !(MDC_TC2_EXP & 4); ++h) {
#pragma unroll
                        for (int j = 0; j < KQ; ++j)
                            mma_tf32_ts(d, ta + (ASTAGE / 2) * h + 8 * j,
                                        umma_desc(bs + (2 * KQ * h + 2 * j) * 128, 128, GSBO), id_tf,
                                        (tr | h | j) ? 1u : 0u);
#pragma unroll
                        for (int c = 0; c < KQ; ++c)
                            mma_bf16_ts(d, ta + (ASTAGE / 2) * h + 8 * KQ + 8 * c,
                                        umma_desc(bs + PART + (2 * KQ * h + 2 * c) * 128, 128, GSBO), id_bf, 1u);
                    }
                    commit(&empty[s]);
                    if (++s == STAGES) s = 0, ph ^= 1;
                    if (++tr == FLUSH || t == ntiles - 1) {
                        commit(&acc_full[run % NACC]);
                        tr = 0;
                        ++run;
                    }
                }
            }
            PEND(5, tall);
            PREPORT("issuer   accfree full - - - total");
        }
        __syncwarp();
    } else if (warp >= PW) {
        // ------------------------------ builders ------------------------------
        // Fixed roles: (channel c, control half kh) -> rows c, NC + c, 2 NC + c
        // (q, X q, Y q) of 8 controls; or (moment m, kh) -> row 3 NC + m.
        const int bt = tid - PW * 32;
        constexpr int NB8 = 2 * KQ;  // 8-control blocks per K tile
        const int total_rounds = nchunk * nr;
        auto stage_round = [&](int R) {  // global round R -> buffer R & 1
            if (R >= total_rounds) return;
            const int b = R & 1;
            if (R >= 2) mbar_wait_sleep(&xy_empty[b], (uint32_t)(((R - 2) >> 1) & 1));
            named_sync(2, BT);  // every builder is done reading the buffer's previous round
            const int r = R % nr;
            if (bt == 0) {
                fence_async_smem();
                mbar_arrive_tx(&q_full[b], GE::QBYTES);
                bulk_g2s(sq + b * QROUND, qimg + (size_t)R * QROUND, GE::QBYTES, &q_full[b]);
            }
            for (int pi = bt; pi < XYR / 2; pi += BT) {
                float x[2], y[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t j = (int64_t)r * XYR + 2 * pi + e;
                    if (j < n) {
                        const double2 v = reinterpret_cast<const double2 *>(a.pc)[j];
                        x[e] = (float)(v.x - cx);
                        y[e] = (float)(v.y - cy);
                    } else {
                        x[e] = 1e18f;  // parked: tiny weight, zero B rows
                        y[e] = 1e18f;
                    }
                }
                sxy[b * (XYR / 2) + pi] = make_float4(x[0], x[1], y[0], y[1]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&xy_full[b]);
        };
        PDECL;
        PBEGIN(tall);
        stage_round(0);
        int s = 0;
        uint32_t ph = 0;
        bool warm = false;
        int R = 0;
        for (int chunk = 0; chunk < nchunk; ++chunk) {
            int tin = 0;
            for (int t = 0; t < ntiles; ++t) {
                const int b = R & 1;
                {  // stage the next round mid-way through this one (or at its last tile if shorter)
                    const int last = min(TPR, ntiles - (t - tin)) - 1;
                    PBEGIN(b0);
                    if (tin == min(TPR / 2, last)) stage_round(R + 1);
                    PEND(0, b0);
                }
                PBEGIN(b1);
                if (tin == 0) {
                    ring_wait(&xy_full[b], (uint32_t)((R >> 1) & 1));
                    ring_wait(&q_full[b], (uint32_t)((R >> 1) & 1));
                }
                PEND(1, b1);
                PBEGIN(b2);
                if (warm) ring_wait(&empty[s], ph ^ 1);
                PEND(2, b2);
                PBEGIN(b3);
                unsigned char *st = sB + s * BSTAGE;
                // items: (channel c, 8-control block kb8) -> rows c, NC + c, 2 NC + c; then
                // (moment m, kb8) -> row 3 NC + m
                constexpr int NQI = NC * NB8, NITEM = NQI + 6 * NB8;
#pragma unroll 1
                for (int it = bt; it < NITEM; it += BT) {
                    const bool role_q = it < NQI;
                    const int c = role_q ? it % NC : 0;
                    const int mm = role_q ? 0 : (it - NQI) % 6;
                    const int kb8 = role_q ? it / NC : (it - NQI) / 6;
                    const float4 *xy = sxy + b * (XYR / 2) + tin * (KT / 2) + 4 * kb8;
                    float X[8], Y[8];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const float4 pp = xy[p];
                        X[2 * p] = pp.x, X[2 * p + 1] = pp.y, Y[2 * p] = pp.z, Y[2 * p + 1] = pp.w;
                    }
                    const int hb = hi_block(kb8), lb = lo_block(kb8);
                    auto emit = [&](int nrw, const float (&v)[8]) {
                        float hi[8], lo[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            hi[e] = trunc_tf32(v[e]);
                            lo[e] = v[e] - hi[e];
                        }
                        *reinterpret_cast<float4 *>(st + tf_off(nrw, 8 * kb8)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                        *reinterpret_cast<float4 *>(st + tf_off(nrw, 8 * kb8 + 4)) =
                            make_float4(hi[4], hi[5], hi[6], hi[7]);
                        *reinterpret_cast<uint4 *>(st + bf_off<PART>(nrw, hb, 0)) =
                            make_uint4(pack_bf16(hi[0], hi[1]), pack_bf16(hi[2], hi[3]), pack_bf16(hi[4], hi[5]),
                                       pack_bf16(hi[6], hi[7]));
                        *reinterpret_cast<uint4 *>(st + bf_off<PART>(nrw, lb, 0)) =
                            make_uint4(pack_bf16(lo[0], lo[1]), pack_bf16(lo[2], lo[3]), pack_bf16(lo[4], lo[5]),
                                       pack_bf16(lo[6], lo[7]));
                    };
                    if (MDC_TC2_EXP & 1) {
                    } else if (role_q) {
                        const float *qrow = sq + b * QROUND + c * QSTRIDE + tin * KT + 8 * kb8;
                        const float4 q0 = *reinterpret_cast<const float4 *>(qrow);
                        const float4 q1 = *reinterpret_cast<const float4 *>(qrow + 4);
                        const float q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};  // zero past n
                        float v[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) v[e] = q[e];
                        emit(c, v);
#pragma unroll
                        for (int e = 0; e < 8; ++e) v[e] = X[e] * q[e];
                        emit(NC + c, v);
#pragma unroll
                        for (int e = 0; e < 8; ++e) v[e] = Y[e] * q[e];
                        emit(2 * NC + c, v);
                    } else {
                        const bool uX = mm == 1 || mm == 3 || mm == 4, uY = mm == 2 || mm == 5;
                        const bool wX = mm == 3, wY = mm == 4 || mm == 5;
                        const bool tail = (int64_t)(t + 1) * KT > n;
                        float v[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float u = uX ? X[e] : (uY ? Y[e] : 1.f);
                            const float w = wX ? X[e] : (wY ? Y[e] : 1.f);
                            v[e] = (tail && (int64_t)t * KT + 8 * kb8 + e >= n) ? 0.f : u * w;
                        }
                        emit(3 * NC + mm, v);
                    }
                }
                PEND(3, b3);
                PBEGIN(b4);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
                PEND(4, b4);
                if (++s == STAGES) s = 0, ph ^= 1, warm = true;
                if (++tin == TPR) tin = 0, ++R;
            }
            if (tin != 0) ++R;  // a chunk's short last round
        }
        PEND(5, tall);
        PREPORT("builder  stage xyq empty build fence total");
    } else {
        // ------------------------------ pixel warps ------------------------------
        const int q4 = warp & 3, h = warp >> 2;
        const int m = q4 * 32 + lane;  // tile pixel = TMEM lane
        const int64_t row = (int64_t)ty * TH + m / TW;
        const int64_t col = (int64_t)tx * TW + m % TW;
        const bool active = row >= a.row0 && row < a.row0 + a.nrows && col < a.width;
        double vxg, vyg;
        pixel_xy_rc(a, row, col, vxg, vyg);
        const float ax = (float)(vxg - cx), by = (float)(vyg - cy);
        const float2 nax = make_float2(-ax, -ax), nby = make_float2(-by, -by);
        const float neg_alpha = (float)(-a.alpha);
        const uint32_t lane_addr = (uint32_t)(q4 * 32) << 16;
        const uint32_t a_base = tmem + lane_addr + GE::ARING + (ASTAGE / 2) * h;
        double T0[NH], TX[NH], TY[NH], M6[6];
        bool bad = false;
        int s = 0;
        uint32_t ph = 0;
        bool warm = false;
        int R = 0;
        int run0 = 0;  // global index of the chunk's first run
        for (int chunk = 0; chunk < nchunk; ++chunk) {
#pragma unroll
            for (int i = 0; i < NH; ++i) T0[i] = TX[i] = TY[i] = 0.0;
#pragma unroll
            for (int i = 0; i < 6; ++i) M6[i] = 0.0;
            const int nruns = (ntiles + FLUSH - 1) / FLUSH;
            int next = 0;                 // chunk-local run to drain next
            int drain_at = FLUSH + LAG;   // tile after which it is drained
            auto drain = [&](int lrun) {
                const int run = run0 + lrun;
                ring_wait(&acc_full[run % NACC], (uint32_t)((run / NACC) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t base = tmem + lane_addr + (uint32_t)((run % NACC) * NCOL);
                uint32_t v0[NH], v1[NH], v2[NH], v3[8];
                tmem_ld<NH>(base + NH * h, v0);
                tmem_ld<NH>(base + NC + NH * h, v1);
                tmem_ld<NH>(base + 2 * NC + NH * h, v2);
                tmem_ld<8>(base + 3 * NC, v3);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_free[run % NACC]);
#pragma unroll
                for (int i = 0; i < NH; ++i) {
                    T0[i] += (double)__uint_as_float(v0[i]);
                    TX[i] += (double)__uint_as_float(v1[i]);
                    TY[i] += (double)__uint_as_float(v2[i]);
                }
#pragma unroll
                for (int i = 0; i < 6; ++i) M6[i] += (double)__uint_as_float(v3[i]);
            };
            int tin = 0;
            PDECL;
            PBEGIN(tall);
            for (int t = 0; t < ntiles; ++t) {
                const int b = R & 1;
                PBEGIN(p0);
                if (tin == 0) ring_wait(&xy_full[b], (uint32_t)((R >> 1) & 1));
                PEND(0, p0);
                PBEGIN(p1);
                if (warm) ring_wait(&empty[s], ph ^ 1);
                PEND(1, p1);
                PBEGIN(p2);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const float4 *xy = sxy + b * (XYR / 2) + tin * (KT / 2) + (KT / 4) * h;
                uint32_t v[16 * KQ];
#pragma unroll
                for (int p = 0; p < 4 * KQ; ++p) {
                    // parked controls (past n) get a tiny finite weight against zero B rows
                    const float4 pp = xy[p];
                    const float2 dx = __fadd2_rn(make_float2(pp.x, pp.y), nax);
                    const float2 dy = __fadd2_rn(make_float2(pp.z, pp.w), nby);
                    const float2 w = weight2<AM>(__ffma2_rn(dy, dy, __fmul2_rn(dx, dx)), neg_alpha);
                    const float2 wh = make_float2(trunc_tf32(w.x), trunc_tf32(w.y));
                    const float2 wl = __ffma2_rn(wh, make_float2(-1.f, -1.f), w);
                    v[2 * p] = __float_as_uint(wh.x);
                    v[2 * p + 1] = __float_as_uint(wh.y);
                    v[8 * KQ + p] = pack_bf16(wh.x, wh.y);
                    v[12 * KQ + p] = pack_bf16(wl.x, wl.y);
                }
                if (MDC_TC2_EXP & 2) {
#pragma unroll
                    for (int e = 0; e < 16 * KQ; ++e) v[e] = 0x3f800000u;
                }
                PEND(2, p2);
                PBEGIN(p3);
                tmem_st<16 * KQ>(a_base + s * ASTAGE, v);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                const bool round_end = tin == TPR - 1 || t == ntiles - 1;
                if (lane == 0) {
                    mbar_arrive(&full[s]);
                    if (round_end) mbar_arrive(&xy_empty[b]);
                }
                PEND(3, p3);
                if (++s == STAGES) s = 0, ph ^= 1, warm = true;
                if (++tin == TPR) tin = 0, ++R;
                PBEGIN(p4);
                if (t == drain_at) {
                    drain(next++);
                    drain_at += FLUSH;
                }
                PEND(4, p4);
            }
            PEND(5, tall);
            PREPORT("pixel    xy empty math store+arrive drain total");
            if (tin != 0) ++R;
            while (next < nruns) drain(next++);
            run0 += nruns;
            // ---- epilogue: pixel-frame moments, fp64 solve, channels of this half ----
            const double A = (double)ax, B = (double)by;
            const double s0 = M6[0];
            const double sx = M6[1] - A * s0, sy = M6[2] - B * s0;
            const double sxx = M6[3] - 2.0 * A * M6[1] + A * A * s0;
            const double sxy = M6[4] - A * M6[2] - B * M6[1] + A * B * s0;
            const double syy = M6[5] - 2.0 * B * M6[2] + B * B * s0;
            double c0, c1, c2;
            {
                const double m0 = sx, m1 = sy;
                double a00 = sxx - m0 * m0 / s0;
                double a01 = sxy - m0 * m1 / s0;
                double a11 = syy - m1 * m1 / s0;
                const double reg = a.reg_eps * (a00 + a11);
                a00 += reg;
                a11 += reg;
                const double det = a00 * a11 - a01 * a01;
                const double u0 = (a11 * m0 - a01 * m1) / det;
                const double u1 = (a00 * m1 - a01 * m0) / det;
                c0 = 1.0 / s0 + (m0 * u0 + m1 * u1) / (s0 * s0);
                c1 = -u0 / s0;
                c2 = -u1 / s0;
            }
            if (active) {
                const int64_t lr = row - a.row0;
#pragma unroll
                for (int i = 0; i < NH; ++i) {
                    const int ch = chunk * NC + NH * h + i;
                    if (ch < a.d) {
                        const double F = c0 * T0[i] + c1 * (TX[i] - A * T0[i]) + c2 * (TY[i] - B * T0[i]);
                        const float f = (float)(F + a.qm[ch]);
                        reinterpret_cast<float *>(a.out)[ch * a.out_cs + lr * a.out_rs + col * a.out_ps] = f;
                        if (!isfinite(f)) bad = true;
                        store_band(a, ch, lr, col, (double)f);
                    }
                }
            }
        }
        // one non-finite count per pixel (the snap pass repairs and decrements per pixel)
        if (a.nonfinite) {
            if (h == 0) sbad[m] = bad;
            named_sync(1, PW * 32);
            if (h == 1 && active && (bad || sbad[m])) atomicAdd(a.nonfinite, 1);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == PW + BW) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    }
}

static int pick_nc(int d) { return d <= 16 ? 16 : 32; }

}  // namespace tc2

size_t mls_tc2_workspace_bytes(int d, int64_t n) {
    const int nc = tc2::pick_nc(d);
    const int nchunk = (d + nc - 1) / nc;
    const int64_t nr = (n + tc2::XYR - 1) / tc2::XYR;
    return (size_t)nchunk * nr * nc * tc2::QSTRIDE * 4 + 256;
}

template <int AM, int NC>
static int launch_tc2_nc(const KArgs &k, void *ws, cudaStream_t s) {
    using namespace tc2;
    Args2 g2;
    g2.nchunk = (k.d + NC - 1) / NC;
    g2.ntiles = (k.n + KT - 1) / KT;
    g2.nr = (k.n + XYR - 1) / XYR;
    g2.tiles_x = (k.width + TW - 1) / TW;
    g2.ty0 = k.row0 / TH;
    const int ty1 = (k.row0 + k.nrows + TH - 1) / TH;
    float *img = reinterpret_cast<float *>(ws);
    const int64_t total = (int64_t)g2.nchunk * g2.nr * NC * QSTRIDE;
    q2_image_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(reinterpret_cast<const float *>(k.q), k.n, k.ldq,
                                                                    k.d, NC, g2.nchunk, g2.nr, img);
    auto fn = mls_tc2_kernel<AM, NC>;
    const size_t smem = Geo<NC>::SMEM;
    MDC_CHECK_CUDA(ensure_dynamic_smem((const void *)fn, (int)smem));
    const int64_t blocks = (int64_t)g2.tiles_x * (ty1 - g2.ty0);
    if (blocks > 0) fn<<<(unsigned)blocks, THREADS, smem, s>>>(k, img, g2);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

template <int AM>
static int launch_tc2_am(const KArgs &k, void *ws, cudaStream_t s) {
    switch (tc2::pick_nc(k.d)) {
        case 16: return launch_tc2_nc<AM, 16>(k, ws, s);
        default: return launch_tc2_nc<AM, 32>(k, ws, s);
    }
}

int launch_mls_tc2(const KArgs &k, void *ws, cudaStream_t s) {
    switch (alpha_mode(k.alpha)) {
        case A_ONE: return launch_tc2_am<A_ONE>(k, ws, s);
        case A_THREE_HALVES: return launch_tc2_am<A_THREE_HALVES>(k, ws, s);
        case A_HALF: return launch_tc2_am<A_HALF>(k, ws, s);
        case A_TWO: return launch_tc2_am<A_TWO>(k, ws, s);
        default: return launch_tc2_am<A_GENERIC>(k, ws, s);
    }
}

}  // namespace mdc
