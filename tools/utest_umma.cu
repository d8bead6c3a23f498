// Micro-test of the tcgen05 operand layouts mls_tc2.cu relies on (A from TMEM,
// B from shared memory, K-major, no swizzle): one kind::tf32 MMA (M128 N112
// K8) and one kind::f16 bf16 MMA (M128 N112 K16), checked against a CPU
// product of the same rounded operands.  Experiments only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/utest_umma tools/utest_umma.cu
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>

#include "../paper_1408_0677_b200/csrc/tcgen05.cuh"
using namespace mdc::tc;

constexpr int M = 128, N = 112;

__device__ __forceinline__ uint32_t pack_bf16(float lo_k, float hi_k) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_k), "f"(lo_k));
    return r;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// mode 0: tf32 K=8; mode 1: bf16 K=16
__global__ void k_test(int mode, const float *A, const float *B, float *D) {
    __shared__ __align__(128) unsigned char sB[N * 16 * 4];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int K = mode == 0 ? 8 : 16;
    // B[n][k] into K-major core matrices
    for (int e = tid; e < N * K; e += blockDim.x) {
        int n = e / K, k = e % K;
        if (mode == 0) {
            uint32_t off = (n >> 3) * 512 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4;
            *reinterpret_cast<float *>(sB + off) = B[n * K + k];
        } else {
            uint32_t off = (n >> 3) * 512 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
            *reinterpret_cast<__nv_bfloat16 *>(sB + off) = __float2bfloat16_rn(B[n * K + k]);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    // A row m = thread (4 warps)
    const int m = tid;
    const uint32_t la = (uint32_t)(warp * 32) << 16;
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) {
        if (mode == 0)
            v[c] = __float_as_uint(A[m * 8 + c]);
        else
            v[c] = pack_bf16(A[m * 16 + 2 * c], A[m * 16 + 2 * c + 1]);
    }
    tmem_st<8>(tmem + la + 128, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
        uint64_t bd = umma_desc(smem_u32(sB), 128, 512);
        if (mode == 0) {
            mma_tf32_ts(tmem, tmem + 128, bd, idesc_tf32(N), 0u);
        } else {
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                "r"(tmem + 128), "l"(bd), "r"(idesc_bf16(N)), "r"(0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c8 = 0; c8 < N / 8; ++c8) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + la + c8 * 8));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int e = 0; e < 8; ++e) D[m * N + c8 * 8 + e] = __uint_as_float(r[e]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

static float tf32_trunc(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}
static float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

int main() {
    for (int mode = 0; mode < 2; ++mode) {
        const int K = mode == 0 ? 8 : 16;
        std::vector<float> A(M * K), B(N * K), D(M * N);
        srand(1);
        for (auto &x : A) x = (float)rand() / RAND_MAX - 0.5f;
        for (auto &x : B) x = (float)rand() / RAND_MAX - 0.5f;
        float *dA, *dB, *dD;
        cudaMalloc(&dA, A.size() * 4);
        cudaMalloc(&dB, B.size() * 4);
        cudaMalloc(&dD, D.size() * 4);
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        k_test<<<1, 128>>>(mode, dA, dB, dD);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0, worst_alt = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < K; ++k) {
                    float a = mode == 0 ? tf32_trunc(A[m * K + k]) : bf16r(A[m * K + k]);
                    float b = mode == 0 ? tf32_trunc(B[n * K + k]) : bf16r(B[n * K + k]);
                    s += (double)a * b;
                }
                worst = fmax(worst, fabs(s - D[m * N + n]));
            }
        printf("mode %s: err %s max |D - ref| = %.3e  (D[0][0]=%f)\n", mode == 0 ? "tf32" : "bf16",
               cudaGetErrorString(e), worst, D[0]);
        (void)worst_alt;
    }
    return 0;
}
