// Microbenchmark (dev tool): what slows the single-thread tcgen05.mma issue
// loop (M=128 N=48 K=16, 4 per 16 KB unit).  Variants add, one at a time, the
// megakernel loop's per-unit work to a tight back-to-back loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_issue.cu -o tools/mb_issue
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2602_16760_b200/csrc/sfg_tc.cuh"

using namespace sfg::tc;

// V bits: 1 rotate stages (descriptor per unit), 2 commit per unit, 4 try_wait per unit
// (already-complete barrier), 8 tcgen05 fence per unit, 16 issuer is warp 1 (else warp 0)
template <int V>
__global__ void __launch_bounds__(128, 1) k(int units, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * 22528);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * 22528 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(slot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) mbar_arrive(&bar[2]);  // a completed phase for the try_wait variant
    __syncthreads();
    const int issuer = (V & 16) ? 32 : 0;
    if (threadIdx.x == issuer) {
        int stage = 0;
        for (int u = 0; u < units; ++u) {
            if (V & 4) mbar_wait(&bar[2], 0);
            if (V & 8) tc_fence_after();
            const uint32_t sa = smem_u32(smem + ((V & 1) ? stage : 0) * 22528);
            const uint64_t da = smem_desc(sa), db = smem_desc(sa + 16384);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_bf16(tmem, da + 2 * kk, db + 2 * kk, (u > 0 || kk > 0));
            if (V & 2) mma_commit(&bar[1]);
            if (++stage == 8) stage = 0;
        }
        mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free(tmem, 128);
    if (threadIdx.x == 0) out[blockIdx.x] = 0;
}

template <int V>
void run(int U, unsigned long long* d) {
    const int smem = 8 * 22528 + 2048;
    cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<V><<<148, 128, smem>>>(U, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<V><<<148, 128, smem>>>(U, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    printf("V=%2d (rotate %d commit %d trywait %d fence %d warp1 %d): %.0f ns/unit %s\n", V, V & 1, (V >> 1) & 1,
           (V >> 2) & 1, (V >> 3) & 1, (V >> 4) & 1, ms * 1e6 / U, e ? cudaGetErrorString(e) : "");
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int U = 8192;
    run<0>(U, d);
    run<1>(U, d);
    run<2>(U, d);
    run<4>(U, d);
    run<8>(U, d);
    run<16>(U, d);
    run<3>(U, d);
    run<15>(U, d);
    run<31>(U, d);
    return 0;
}
