// Microbenchmark + layout check (dev tool): weight tiles staged
// smem -> registers (LDS) -> TMEM (tcgen05.st) by four copier warps, and the
// MMA reading A from TMEM (tcgen05.mma ... [a_tmem], b_desc) instead of
// from shared memory.  Checks the A-in-TMEM layout against the SS MMA on the
// same random tile, then times the staged pipeline per 16 KB unit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_tmem.cu -o tools/mb_tmem
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../paper_2602_16760_b200/csrc/sfg_tc.cuh"

using namespace sfg::tc;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// copy row r (this thread's TMEM lane) of an SW128 K-major [128 x 64] bf16 tile
// into 32 TMEM columns: column j = bf16 pair (k = 2j, 2j + 1)
__device__ __forceinline__ void stage_row(const uint8_t* tile, int r, uint32_t taddr) {
    uint32_t v[32];
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // 16-byte chunk c of the logical row = k 8c..8c+7
        const uint4 q = *reinterpret_cast<const uint4*>(tile + (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
        v[4 * c + 0] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
    tmem_st32(taddr, v);
}

// check: D_ss = A(smem) x B and D_ts = A(TMEM, staged) x B for one 128 x 48 x 64 tile
__global__ void check_kernel(const uint8_t* gA, const uint8_t* gB, float* out_ss, float* out_ts) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 6144);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (16384 + 6144) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = i < 1024 ? reinterpret_cast<const uint4*>(gA)[i]
                                                     : reinterpret_cast<const uint4*>(gB)[i - 1024];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    // stage A into columns [128, 160) (all 4 warps: lane quarter = warp)
    stage_row(smem, warp * 32 + lane, tmem + (static_cast<uint32_t>(warp * 32) << 16) + 128);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t sa = smem_u32(smem);
        const uint64_t da = smem_desc(sa), db = smem_desc(sa + 16384);
        for (int k = 0; k < 4; ++k) mma_bf16(tmem + 0, da + 2 * k, db + 2 * k, k > 0);
        for (int k = 0; k < 4; ++k) mma_bf16_ts(tmem + 64, tmem + 128 + 8 * k, db + 2 * k, k > 0);
        mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    float v[48];
    const uint32_t ta = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    tmem_ld16(ta, v);
    tmem_ld16(ta + 16, v + 16);
    tmem_ld16(ta + 32, v + 32);
    tmem_wait_ld();
    for (int n = 0; n < 48; ++n) out_ss[(warp * 32 + lane) * 48 + n] = v[n];
    tmem_ld16(ta + 64, v);
    tmem_ld16(ta + 80, v + 16);
    tmem_ld16(ta + 96, v + 32);
    tmem_wait_ld();
    for (int n = 0; n < 48; ++n) out_ts[(warp * 32 + lane) * 48 + n] = v[n];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free(tmem, 256);
}

// pipeline: warp 0 producer (arrive, smem stage "full"), warps 4..7 copiers
// (stage -> TMEM slot, release smem stage), warp 1 MMA from TMEM slots.
// mode 0: copier path (A via TMEM); mode 1: plain SS MMA ring for reference.
constexpr int S = 8, NSLOT = 12;
__global__ void __launch_bounds__(256, 1) pipe_kernel(int units, int mode, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = 16384 + 6144;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* aready = empty + S;
    uint64_t* afree = aready + NSLOT;
    uint64_t* done = afree + NSLOT;
    uint32_t* slotp = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], (mode == 0 || mode == 3) ? 4 : 1);  // copier warps release the stage
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&aready[s], 4);
            mbar_init(&afree[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) tmem_alloc(slotp, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slotp;
    if (warp == 0 && lane == 0 && mode != 2) {
        int st = 0;
        uint32_t ph = 0;
        for (int u = 0; u < units; ++u) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive(&full[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        int st = 0, as = 0;
        uint32_t ph = 0, aph = 0;
        for (int u = 0; u < units; ++u) {
            if (mode == 3) break;
            if (mode == 0 || mode == 2) {
                if (mode == 0) mbar_wait(&aready[as], aph);
                tc_fence_after();
                const uint32_t sb = smem_u32(smem + st * stage_bytes + 16384);
                const uint64_t db = smem_desc(sb);
                for (int k = 0; k < 4; ++k) mma_bf16_ts(tmem, tmem + 128 + as * 32 + 8 * k, db + 2 * k, (u > 0 || k > 0));
                mma_commit(&afree[as]);
                if (++as == NSLOT) { as = 0; aph ^= 1; }
                if (++st == S) { st = 0; ph ^= 1; }
            } else {
                mbar_wait(&full[st], ph);
                tc_fence_after();
                const uint32_t sa = smem_u32(smem + st * stage_bytes);
                const uint64_t da = smem_desc(sa), db = smem_desc(sa + 16384);
                for (int k = 0; k < 4; ++k) mma_bf16(tmem, da + 2 * k, db + 2 * k, (u > 0 || k > 0));
                mma_commit(&empty[st]);
                if (++st == S) { st = 0; ph ^= 1; }
            }
        }
        mma_commit(done);
        mbar_wait(done, 0);
    } else if (warp >= 4 && (mode == 0 || mode == 3)) {
        const int q = warp & 3;
        int st = 0, as = 0;
        uint32_t ph = 0, aph = 0;
        for (int u = 0; u < units; ++u) {
            mbar_wait(&full[st], ph);
            if (mode == 0) mbar_wait(&afree[as], aph ^ 1);
            tc_fence_after();
            stage_row(smem + st * stage_bytes, q * 32 + lane, tmem + (static_cast<uint32_t>(q * 32) << 16) + 128 + as * 32);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[st]);   // NOTE: B stays in the stage in this bench (not reloaded)
                mbar_arrive(&aready[as]);
            }
            if (++as == NSLOT) { as = 0; aph ^= 1; }
            if (++st == S) { st = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = 0;
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_free(tmem, 512);
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

int main() {
    // layout check
    std::vector<uint8_t> A(16384), B(6144);
    std::vector<float> Af(128 * 64), Bf(48 * 64);
    unsigned s = 1;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 65536.0f - 0.5f; };
    for (int r = 0; r < 128; ++r)
        for (int k = 0; k < 64; ++k) {
            const uint16_t u = bf(rnd());
            Af[r * 64 + k] = fb(u);
            memcpy(&A[swoff(r, k)], &u, 2);
        }
    for (int r = 0; r < 48; ++r)
        for (int k = 0; k < 64; ++k) {
            const uint16_t u = bf(rnd());
            Bf[r * 64 + k] = fb(u);
            memcpy(&B[swoff(r, k)], &u, 2);
        }
    uint8_t *dA, *dB;
    float *dss, *dts;
    cudaMalloc(&dA, 16384);
    cudaMalloc(&dB, 6144);
    cudaMalloc(&dss, 128 * 48 * 4);
    cudaMalloc(&dts, 128 * 48 * 4);
    cudaMemcpy(dA, A.data(), 16384, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), 6144, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    check_kernel<<<1, 128, 32768>>>(dA, dB, dss, dts);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("check error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> hs(128 * 48), ht(128 * 48);
    cudaMemcpy(hs.data(), dss, hs.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht.data(), dts, ht.size() * 4, cudaMemcpyDeviceToHost);
    double mx_ss = 0, mx_ts = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 48; ++n) {
            double ref = 0;
            for (int k = 0; k < 64; ++k) ref += (double)Af[m * 64 + k] * Bf[n * 64 + k];
            mx_ss = fmax(mx_ss, fabs(hs[m * 48 + n] - ref));
            mx_ts = fmax(mx_ts, fabs(ht[m * 48 + n] - ref));
        }
    printf("layout check: max |D - ref| SS %.3g, TS (A staged to TMEM) %.3g\n", mx_ss, mx_ts);
    // timing
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * 8);
    const int smem = S * (16384 + 6144) + 2048;
    cudaFuncSetAttribute(pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode : {1, 0, 2, 3}) {
        const int U = 8192;
        pipe_kernel<<<148, 256, smem>>>(U, mode, d_out);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        pipe_kernel<<<148, 256, smem>>>(U, mode, d_out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        e = cudaGetLastError();
        const char* nm[] = {"TS (copier warps LDS->tcgen05.st, A from TMEM)", "SS ring (A from smem)",
                            "TS MMA only (no staging)", "copiers only (LDS->tcgen05.st, no MMA)"};
        printf("%s: %.0f ns per 16 KB unit%s\n", nm[mode],
               ms * 1e6 / U, e != cudaSuccess ? cudaGetErrorString(e) : "");
    }
    return 0;
}
