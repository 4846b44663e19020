// Microbenchmark (dev tool): cost of the publish fences the megakernel's
// epilogue uses after its stores (MEMBAR.GPU via __threadfence, and
// fence.proxy.async.global before a bulk-copy consumer reads the bytes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_fence.cu -o tools/mb_fence
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void kf(float* buf, int mode, int nst, unsigned long long* out) {
    const int t = threadIdx.x;
    float* p = buf + (size_t)blockIdx.x * 65536;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int r = 0; r < nst; ++r) p[r * 4096 + t] = r + t;
    const unsigned long long t1 = clock64();
    if (mode & 1) __threadfence();
    if (mode & 2) asm volatile("fence.proxy.async.global;" ::: "memory");
    if (mode & 4) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const unsigned long long t2 = clock64();
    __syncthreads();
    const unsigned long long t3 = clock64();
    if (t == 0) {
        out[blockIdx.x * 3 + 0] = t1 - t0;
        out[blockIdx.x * 3 + 1] = t2 - t1;
        out[blockIdx.x * 3 + 2] = t3 - t0;
    }
}

int main() {
    float* buf;
    cudaMalloc(&buf, 148ull * 65536 * 4);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 3 * 8);
    unsigned long long h[148 * 3];
    for (int nst : {0, 1, 16, 64}) {
        for (int mode : {0, 1, 2, 3, 4}) {
            kf<<<148, 128>>>(buf, mode, nst, d);
            kf<<<148, 128>>>(buf, mode, nst, d);
            cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double a = 0, b = 0, c = 0;
            for (int i = 0; i < 148; ++i) {
                a += h[3 * i];
                b += h[3 * i + 1];
                c += h[3 * i + 2];
            }
            printf("stores/thread %2d mode %d (%s): issue %.0f cyc, fence %.0f cyc, total to bar %.0f cyc\n", nst, mode,
                   mode == 0 ? "none" : mode == 1 ? "threadfence" : mode == 2 ? "proxy.async.global"
                             : mode == 3 ? "both" : "acq_rel.gpu",
                   a / 148, b / 148, c / 148);
        }
    }
    return 0;
}
