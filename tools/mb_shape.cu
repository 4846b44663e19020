// Microbenchmark (dev tool): tensor-pipe time of one tcgen05.mma kind::f16
// (bf16, K=16) by shape, back to back from one thread per SM, all 148 SMs.
// Question it answers: does a skinny decode GEMM consume weights faster as
// the A operand (M = 128 weight rows, N = 3 x rows) or as the B operand
// (M = 64 activation rows, N = 256 weight rows)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_shape.cu -o tools/mb_shape
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2602_16760_b200/csrc/sfg_tc.cuh"

using namespace sfg::tc;

__device__ __forceinline__ void mma_id(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__global__ void __launch_bounds__(128, 1) k(int iters, uint32_t idesc, int rot, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 4 * 32768 + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (5 * 32768) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        const unsigned long long t0 = clock64();
        for (int u = 0; u < iters; ++u) {
            const uint32_t sa = smem_u32(smem + (rot ? (u & 3) : 0) * 32768);
            const uint64_t da = smem_desc(sa), db = smem_desc(smem_u32(smem + 4 * 32768));
            mma_id(tmem, da, db, idesc, u > 0);
        }
        mma_commit(&bar[0]);
        mbar_wait(&bar[0], 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free(tmem, 512);
}

static uint32_t idesc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 5 * 32768 + 2048;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int shapes[][2] = {{128, 16}, {128, 32}, {128, 48}, {128, 64}, {128, 96}, {128, 128}, {128, 192},
                             {128, 256}, {64, 16}, {64, 48}, {64, 64}, {64, 128}, {64, 192}, {64, 256}};
    const int iters = 20000;
    for (auto& s : shapes) {
        const int M = s[0], N = s[1];
        k<<<148, 128, smem>>>(100, idesc(M, N), 1, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<148, 128, smem>>>(iters, idesc(M, N), 1, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc[148];
        cudaMemcpy(cyc, d, sizeof(cyc), cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        // weight bytes one instruction consumes: the 128-row A side (M = 128)
        // or the N-row B side (M = 64: weights as B)
        const double wbytes = (M == 128 ? 128.0 : N) * 16 * 2;
        const double ns = ms * 1e6 / iters;
        printf("M=%3d N=%3d: %.1f ns/instr (%.0f cycles), %.1f ns per 16 KB of weights %s\n", M, N, ns,
               static_cast<double>(cyc[0]) / iters, ns * 16384.0 / wbytes, e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
