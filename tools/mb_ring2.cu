// Microbenchmark (dev tool): the megakernel's per-unit pipeline without
// memory traffic, with its warp roles added one at a time, to find what
// makes the in-kernel rate (~400 ns / 16 KB unit) slower than the bare
// ring + MMA (~200 ns).  One CTA per SM, 320 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_ring2.cu -o tools/mb_ring2
// feature bits: 1 loader warp arrives too (full count 2), 2 epilogue warps
// drain the accumulator per tile (TMEM loads), 4 three warps poll a global
// flag (like attention warps waiting), 8 loader polls 32 flags per 32 units,
// 16 tiles of 64 units (else one tile), 32 producer uses nanosleep spin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2602_16760_b200/csrc/sfg_tc.cuh"

using namespace sfg::tc;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(320, 1) k2(int units, int feat, unsigned* gflag, unsigned* flags,
                                            unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int S = 8;
    const int stage_bytes = 16384 + 6144;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* empty = full + 16;
    uint64_t* tfull = empty + 16;
    uint64_t* tempty = tfull + 2;
    uint32_t* slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile_units = (feat & 16) ? 64 : units;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], (feat & 1) ? 2 : 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(slot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const unsigned long long t0 = clock64();
    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t ph = 0;
            for (int u = 0; u < units; ++u) {
                mbar_wait(&empty[stage], ph ^ 1);
                mbar_arrive(&full[stage]);
                if (++stage == S) { stage = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int u0 = 0; u0 < units; u0 += tile_units) {
                if (feat & 2) mbar_wait(&tempty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * 64;
                for (int u = u0; u < u0 + tile_units && u < units; ++u) {
                    mbar_wait(&full[stage], ph);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * stage_bytes);
                    const uint64_t da = smem_desc(sa), db = smem_desc(sa + 16384);
#pragma unroll
                    for (int k = 0; k < 4; ++k) mma_bf16(d, da + 2 * k, db + 2 * k, (u > u0 || k > 0) ? 1u : 0u);
                    mma_commit(&empty[stage]);
                    if (++stage == S) { stage = 0; ph ^= 1; }
                }
                if (feat & 2) mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gflag + blockIdx.x), "r"(1u) : "memory");
        }
    } else if (warp < 6) {
        if (feat & 2) {
            const int q = warp & 3;
            int acc = 0;
            uint32_t aph = 0;
            float sink = 0;
            for (int u0 = 0; u0 < units; u0 += tile_units) {
                mbar_wait(&tfull[acc], aph);
                tc_fence_after();
                float v[48];
                const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * 64;
                tmem_ld16(ta, v);
                tmem_ld16(ta + 16, v + 16);
                tmem_ld16(ta + 32, v + 32);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                for (int i = 0; i < 48; ++i) sink += v[i];
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
            if (sink == 12345.f) out[1000] = 1;
        }
    } else if (warp == 6) {
        if (feat & 1) {
            int stage = 0;
            uint32_t ph = 0;
            int ready = 0;
            for (int u = 0; u < units; ++u) {
                if ((feat & 8) && u >= ready) {
                    const bool ok = ld_acq(flags + ((u + lane) & 1023)) >= 1u;
                    const unsigned mk = __ballot_sync(0xffffffffu, ok);
                    ready += (mk == 0xffffffffu) ? 32 : 1;
                }
                if (lane == 0) {
                    mbar_wait(&empty[stage], ph ^ 1);
                    mbar_arrive(&full[stage]);
                }
                if (++stage == S) { stage = 0; ph ^= 1; }
            }
        }
    } else {
        if ((feat & 4) && lane == 0) {
            unsigned long long spins = 0;
            while (ld_acq(gflag + blockIdx.x) == 0u && ++spins < (1ull << 24)) __nanosleep(32);
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free(tmem, 128);
}

int main() {
    unsigned *gflag, *flags;
    cudaMalloc(&gflag, 4 * 148);
    cudaMalloc(&flags, 4096);
    cudaMemset(flags, 0xff, 4096);
    unsigned long long* d_out;
    cudaMalloc(&d_out, 2000 * sizeof(unsigned long long));
    const int smem = 8 * (16384 + 6144) + 2048;
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int U = 4096;
    for (int feat : {0, 1, 2, 16 | 2, 4, 1 | 8, 1 | 2 | 16, 1 | 2 | 8 | 16, 1 | 2 | 4 | 8 | 16}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaMemset(gflag, 0, 4 * 148);
        k2<<<148, 320, smem>>>(U, feat, gflag, flags, d_out);
        cudaMemset(gflag, 0, 4 * 148);
        cudaEventRecord(e0);
        k2<<<148, 320, smem>>>(U, feat, gflag, flags, d_out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("feat=%2d: %.0f ns/unit (kernel %.1f us)\n", feat, ms * 1e6 / U, ms * 1000.0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    }
    return 0;
}
