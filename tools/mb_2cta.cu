// Microbenchmark (dev tool): tcgen05.mma issue cost per 16 KB of weights
// for cta_group::1 (M=128 per SM) vs cta_group::2 (CTA pair, M=256 = 128
// rows from each SM's smem), N=48, K=16, back-to-back with no pipeline.
// Also checks the pair MMA's result against a host reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr tools/mb_2cta.cu -o tools/mb_2cta
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../paper_2602_16760_b200/csrc/sfg_tc.cuh"

using namespace sfg::tc;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <int M_, int N_>
__host__ __device__ constexpr uint32_t idesc() {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N_ >> 3) << 17) | (static_cast<uint32_t>(M_ >> 4) << 24);
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc<256, 48>()), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma1(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc<128, 48>()), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}

// units: number of 16 KB-per-SM weight units (4 x K16 MMAs each)
// pair=1: cluster of 2, leader issues cta_group::2; pair=0: each CTA cta_group::1
template <int PAIR>
__global__ void __launch_bounds__(128, 1) k(int units, const uint8_t* gA, const uint8_t* gB, float* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * 22528);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cta_rank() : 0;
    // stage 0: A = this CTA's 128 rows (gA + rank * 16 KB), B: pair -> this CTA's 24 rows, else 48
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = reinterpret_cast<const uint4*>(gA + (PAIR ? rank * 16384 : 0))[i];
    for (int i = threadIdx.x; i < 384; i += blockDim.x)
        reinterpret_cast<uint4*>(smem + 16384)[i] = reinterpret_cast<const uint4*>(gB + (PAIR ? rank * 3072 : 0))[i];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(128) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc(slot, 128);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0 && (PAIR == 0 || rank == 0)) {
        const uint32_t sa = smem_u32(smem);
        const uint64_t da = smem_desc(sa), db = smem_desc(sa + 16384);
        for (int u = 0; u < units; ++u)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (PAIR) mma2(tmem, da + 2 * kk, db + 2 * kk, (u > 0 || kk > 0));
                else mma1(tmem, da + 2 * kk, db + 2 * kk, (u > 0 || kk > 0));
            }
        if (PAIR) commit2(&bar[0]);
        else mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    if (out) {
        float v[48];
        const uint32_t ta = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        tmem_ld16(ta, v);
        tmem_ld16(ta + 16, v + 16);
        tmem_ld16(ta + 32, v + 32);
        tmem_wait_ld();
        for (int n = 0; n < 48; ++n) out[((blockIdx.x & 1) * 128 + warp * 32 + lane) * 48 + n] = v[n];
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();
    if (warp == 0) {
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
        else tmem_free(tmem, 128);
    }
}

static uint16_t bf(float x) {
    __nv_bfloat16 b = __float2bfloat16(x);
    uint16_t u;
    memcpy(&u, &b, 2);
    return u;
}
static float fb(uint16_t u) {
    uint32_t w = static_cast<uint32_t>(u) << 16;
    float f;
    memcpy(&f, &w, 4);
    return f;
}
static uint32_t swoff(int row, int kk) {
    return (row >> 3) * 1024 + (row & 7) * 128 + (((kk >> 3) ^ (row & 7)) << 4) + (kk & 7) * 2;
}

template <int PAIR>
void launch(int grid, int units, const uint8_t* dA, const uint8_t* dB, float* out) {
    const int smem = 8 * 22528 + 2048;
    cudaFuncSetAttribute(k<PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k<PAIR>, units, dA, dB, out);
}

int main() {
    // A: 256 rows (two CTAs x 128), B: 48 rows, stored as the per-CTA SW128 images
    std::vector<uint8_t> A(2 * 16384), B(6144), Bpair(6144);
    std::vector<float> Af(256 * 64), Bf(48 * 64);
    unsigned s = 7;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 65536.0f - 0.5f; };
    for (int r = 0; r < 256; ++r)
        for (int kk = 0; kk < 64; ++kk) {
            const uint16_t u = bf(rnd());
            Af[r * 64 + kk] = fb(u);
            memcpy(&A[(r / 128) * 16384 + swoff(r % 128, kk)], &u, 2);
        }
    for (int r = 0; r < 48; ++r)
        for (int kk = 0; kk < 64; ++kk) {
            const uint16_t u = bf(rnd());
            Bf[r * 64 + kk] = fb(u);
            memcpy(&B[swoff(r, kk)], &u, 2);
            // pair layout: CTA 0 holds rows 0..23, CTA 1 rows 24..47, each as its own SW128 image
            memcpy(&Bpair[(r / 24) * 3072 + swoff(r % 24, kk)], &u, 2);
        }
    uint8_t *dA, *dB, *dBp;
    float* dout;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dBp, Bpair.size());
    cudaMalloc(&dout, 256 * 48 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dBp, Bpair.data(), Bpair.size(), cudaMemcpyHostToDevice);
    // correctness of the pair MMA: one unit (K=64), grid 2
    launch<1>(2, 1, dA, dBp, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("pair check error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> h(256 * 48);
    cudaMemcpy(h.data(), dout, h.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < 48; ++n) {
            double ref = 0;
            for (int kk = 0; kk < 64; ++kk) ref += (double)Af[m * 64 + kk] * Bf[n * 64 + kk];
            mx = fmax(mx, fabs(h[m * 48 + n] - ref));
        }
    printf("pair MMA (M=256 over 2 CTAs, B split 24/24) max |D - ref| = %.3g\n", mx);
    {  // the same 1-SM kernel through a plain <<<>>> launch (no cluster attribute)
        const int U = 8192, smem = 8 * 22528 + 2048;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k<0><<<148, 128, smem>>>(U, dA, dB, nullptr);
        cudaEventRecord(e0);
        k<0><<<148, 128, smem>>>(U, dA, dB, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cta_group::1 via <<<>>>: %.0f ns per unit\n", ms * 1e6 / U);
        const int smem2 = 8 * 22528 + 2048 + 32768;
        cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
        k<0><<<148, 128, smem2>>>(U, dA, dB, nullptr);
        cudaEventRecord(e0);
        k<0><<<148, 128, smem2>>>(U, dA, dB, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cta_group::1 via <<<>>>, 214 KB smem: %.0f ns per unit\n", ms * 1e6 / U);
    }
    for (int pair : {0, 1}) {
        const int U = 8192;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        if (pair) launch<1>(148, U, dA, dBp, nullptr); else launch<0>(148, U, dA, dB, nullptr);
        cudaEventRecord(e0);
        if (pair) launch<1>(148, U, dA, dBp, nullptr); else launch<0>(148, U, dA, dB, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        e = cudaGetLastError();
        printf("%s: %.0f ns per 16 KB of weights per SM (%d units)%s\n",
               pair ? "cta_group::2 (M=256 pair)" : "cta_group::1 (M=128)", ms * 1e6 / U, U,
               e != cudaSuccess ? cudaGetErrorString(e) : "");
    }
    return 0;
}
