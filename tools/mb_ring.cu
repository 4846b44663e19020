// Microbenchmark (dev tool): per-unit cost of the megakernel's smem ring
// (producer arrive -> tcgen05.mma issue -> commit -> empty) without memory
// traffic, for several MMA shapes / issue patterns.  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_ring.cu -o /tmp/mb_ring
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2602_16760_b200/csrc/sfg_tc.cuh"

using namespace sfg::tc;

template <int N_>
__device__ __forceinline__ void mma_n(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N_ >> 3) << 17) |
                               (static_cast<uint32_t>(128 >> 4) << 24);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

// mode 0: ring with producer arrive (no load) + MMA (4 x K16) + commit per stage
// mode 1: MMA issue only, no barriers (4 x K16 per unit, commit every 8 units)
// mode 2: ring, producer does a 16 KB bulk copy from a small L2-resident buffer
template <int N_>
__global__ void __launch_bounds__(128, 1) ring_kernel(int units, int mode, int S, const uint8_t* src,
                                                     unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = 16384 + 6144;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* empty = full + 16;
    uint64_t* done = empty + 16;
    uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (mode >= 6)  // valid (zero) operands instead of uninitialised shared memory
        for (int i = threadIdx.x; i < S * stage_bytes / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (mode >= 6) mode -= 6;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(slot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    unsigned long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        if (mode != 1 && mode < 3) {
            int stage = 0;
            uint32_t ph = 0;
            for (int u = 0; u < units; ++u) {
                mbar_wait(&empty[stage], ph ^ 1);
                if (mode == 2) {
                    mbar_expect_tx(&full[stage], 16384);
                    bulk_g2s(smem + stage * stage_bytes, src + (size_t)(blockIdx.x * 8 + (u & 7)) * 16384, 16384, &full[stage]);
                } else {
                    mbar_arrive(&full[stage]);
                }
                if (++stage == S) { stage = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        int stage = 0;
        uint32_t ph = 0;
        for (int u = 0; u < units; ++u) {
            if (mode != 1 && mode < 3) mbar_wait(&full[stage], ph);
            if (mode != 3 && mode != 5) tc_fence_after();
            const uint32_t sa = smem_u32(smem + ((mode == 4 || mode == 5) ? 0 : stage) * stage_bytes);
            const uint64_t da = smem_desc(sa), db = smem_desc(sa + 16384);
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_n<N_>(tmem, da + 2 * k, db + 2 * k, (u > 0 || k > 0) ? 1u : 0u);
            if (mode != 1 && mode < 3) mma_commit(&empty[stage]);
            if (++stage == S) { stage = 0; ph ^= 1; }
        }
        mma_commit(done);
        mbar_wait(done, 0);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free(tmem, 128);
}

template <int N_>
void run(int mode, int S, int units, const uint8_t* src, unsigned long long* d_out) {
    const int smem = S * (16384 + 6144) + 1024 + 512 + 32768;  // slack: wide-N B reads past the stage
    cudaFuncSetAttribute(ring_kernel<N_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    ring_kernel<N_><<<148, 128, smem>>>(units, mode, S, src, d_out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ring_kernel<N_><<<148, 128, smem>>>(units, mode, S, src, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("N=%3d mode=%d S=%d units=%d: %.1f cycles/unit (max CTA), kernel %.1f us -> %.0f ns/unit%s\n", N_, mode,
           S, units, (double)mx / units, ms * 1000.0, ms * 1e6 / units,
           mode == 2 ? "  (16 KB L2 bulk copy per unit)" : "");
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
    uint8_t* src;
    cudaMalloc(&src, 148 * 8 * 16384);
    cudaMemset(src, 0, 148 * 8 * 16384);
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
    const int U = 4096;
    for (int mode : {1, 3, 4, 5, 7, 11, 6}) run<48>(mode, 8, U, src, d_out);
    for (int mode : {1, 0, 2}) {
        run<48>(mode, 8, U, src, d_out);
        run<16>(mode, 8, U, src, d_out);
        run<128>(mode, 8, U, src, d_out);
        run<256>(mode, 8, U, src, d_out);
    }
    run<48>(0, 4, U, src, d_out);
    run<48>(0, 2, U, src, d_out);
    run<48>(2, 4, U, src, d_out);
    return 0;
}
