// ubench_tc.cu -- latency microbenchmarks for the pieces of the MLS pass-2
// K-tile round trip (tools only; not part of libmdc):
//   (1) tcgen05.st.32x32b.x16 x2 + tcgen05.wait::st            (G tile to TMEM)
//   (2) a chain of 6 tcgen05.mma kind::tf32 (TS form, M=128, N=32, K=8)
//       + tcgen05.commit -> mbarrier -> try_wait               (one K tile's MMAs)
//   (3) mbarrier arrive (4 warps) -> issuer try_wait wake-up     (publish -> issue)
// Run alone (grid 1) and with 1 / 2 / 4 CTAs per SM sharing the tensor core.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tc tools/ubench_tc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t clk() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            smem_u32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           ((uint64_t)1 << 46);
}

__global__ void __launch_bounds__(160) ubench(unsigned long long *out, int reps) {
    __shared__ __align__(128) unsigned char sB[2 * 32 * 16 * 4];
    __shared__ uint64_t bar_full, bar_mma;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < (int)sizeof(sB) / 4; i += blockDim.x) reinterpret_cast<float *>(sB)[i] = 0.f;
    if (tid == 0) {
        mbar_init(&bar_full, 4);
        mbar_init(&bar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    unsigned long long t_st = 0, t_pub = 0, t_mma = 0;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(1.0f + i);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    for (int r = 0; r < reps; ++r) {
        // (1) TMEM stores + wait (compute warps)
        if (warp < 4) {
            const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 32;
            uint64_t t0 = clk();
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + 16),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            uint64_t t1 = clk();
            t_st += t1 - t0;
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_full);
        } else if (lane == 0) {
            // (3) publish -> issuer wake-up, (2) 6 MMAs -> commit -> wait
            uint64_t t0 = clk();
            mbar_wait(&bar_full, r & 1);
            uint64_t t1 = clk();
            t_pub += t1 - t0;
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t b = smem_u32(sB);
            uint64_t t2 = clk();
            for (int kk = 0; kk < 2; ++kk) {
                const uint64_t db = desc(b + kk * 256, 128, 512);
                for (int m = 0; m < 3; ++m)
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                            tmem),
                        "r"(tmem + 32 + kk * 8), "l"(db), "r"(idesc), "r"(1u));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bar_mma))
                         : "memory");
            mbar_wait(&bar_mma, r & 1);
            uint64_t t3 = clk();
            t_mma += t3 - t2;
        }
        __syncthreads();
    }
    if (tid == 0 && blockIdx.x == 0) out[0] = t_st / reps;
    if (tid == 128 && blockIdx.x == 0) {
        out[1] = t_pub / reps;
        out[2] = t_mma / reps;
    }
    __syncthreads();
    if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
    unsigned long long *d, h[3];
    cudaMalloc(&d, sizeof(h));
    for (int ctas_per_sm : {0, 1, 2, 4}) {
    ubench<<<ctas_per_sm ? 148 * ctas_per_sm : 1, 160>>>(d, 1000);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"grid\": %d, \"tmem_st_x16x2_wait_cycles\": %llu, \"publish_to_issuer_wake_cycles\": %llu, "
           "\"six_mma_commit_wait_cycles\": %llu}\n",
           ctas_per_sm ? 148 * ctas_per_sm : 1, h[0], h[1], h[2]);
    }
    return 0;
}
