// FAST-mode masked GQA decode attention (tinyformer.cpp:450-489 semantics).
//
// One CTA per (batch row, kv head): the `group` query heads that share a KV
// head are scored together, so each K/V row is read once per group (the
// reference re-reads it per query head).  Visibility comes from the
// compacted run list of the row (mask entries {0,-inf} + additive values),
// expanded into a column list in shared memory; every reduction is over that
// compacted index space with a fixed partition (lane-per-key scores, warp-
// per-key-range value sums, fixed-order tree combines), so a row's output is
// deterministic and independent of the batch it rides in and of where its
// branch columns sit in the cache (batch invariance, test_metrics.cpp:187).
#include <cuda_runtime.h>

#include <algorithm>

#include "sfg_engine.h"
#include "sfg_expf.h"

namespace sfg {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxGroup = 8;

template <int HD>
__global__ void __launch_bounds__(kThreads) attn_fast_kernel(const float* __restrict__ q, const float* __restrict__ kc,
                                                             const float* __restrict__ vc,
                                                             const int32_t* __restrict__ row_off,
                                                             const MaskRun* __restrict__ runs, Dims d,
                                                             float* __restrict__ att, uint32_t* status, int cap) {
    extern __shared__ float4 smem4[];
    float* smem = reinterpret_cast<float*>(smem4);
    const int group = d.n_heads / d.n_kv;
    const int row = blockIdx.x / d.n_kv, kvh = blockIdx.x % d.n_kv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* qs = smem;                                     // [group][HD]
    float* red = qs + group * HD;                         // [kWarps][group][HD]
    // cap = the launch's bound on a row's visible keys (max_len, or the cache
    // length after this batch for prompt passes)
    int* cols = reinterpret_cast<int*>(red + kWarps * group * HD);      // [cap]
    float* mv = reinterpret_cast<float*>(cols + cap);                   // [cap]
    float* sc = mv + cap;                                               // [group][cap]
    __shared__ int run_off[65];
    __shared__ int n_s;
    __shared__ float stat[kWarps][kMaxGroup];
    __shared__ float mx_s[kMaxGroup], inv_s[kMaxGroup];

    for (int t = threadIdx.x; t < group * HD; t += kThreads)
        qs[t] = q[static_cast<size_t>(row) * d.qd + static_cast<size_t>(kvh * group) * HD + t];
    // expand the row's visibility runs into a compacted column list
    const int r0 = row_off[row], r1 = row_off[row + 1];
    for (int base = r0; base < r1; base += 64) {
        const int nr = min(64, r1 - base);
        if (threadIdx.x == 0) {
            int off = base == r0 ? 0 : run_off[64];
            for (int r = 0; r < nr; ++r) {
                run_off[r] = off;
                off += runs[base + r].end - runs[base + r].start;
            }
            run_off[64] = off;
        }
        __syncthreads();
        if (run_off[64] > cap) {  // fail loudly rather than overrun shared memory
            if (threadIdx.x == 0) atomicOr(status, ST_ATTN_CAP);
            return;
        }
        for (int r = 0; r < nr; ++r) {
            const MaskRun rr = runs[base + r];
            for (int j = rr.start + threadIdx.x; j < rr.end; j += kThreads) {
                cols[run_off[r] + j - rr.start] = j;
                mv[run_off[r] + j - rr.start] = rr.mval;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) n_s = r1 > r0 ? run_off[64] : 0;
    __syncthreads();
    const int n = n_s;
    const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(HD));
    const float* kb = kc + static_cast<size_t>(kvh) * d.max_len * HD;
    const float* vb = vc + static_cast<size_t>(kvh) * d.max_len * HD;

    // scores: one key per thread, all group heads at once
    float mx[kMaxGroup];
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) mx[g] = -INFINITY;
    for (int c = threadIdx.x; c < n; c += kThreads) {
        const float4* kr = reinterpret_cast<const float4*>(kb + static_cast<size_t>(cols[c]) * HD);
        float acc[kMaxGroup];
#pragma unroll
        for (int g = 0; g < kMaxGroup; ++g) acc[g] = 0.0f;
#pragma unroll 4
        for (int t = 0; t < HD / 4; ++t) {
            const float4 k4 = __ldg(kr + t);
#pragma unroll
            for (int g = 0; g < kMaxGroup; ++g) {
                if (g >= group) break;
                const float4 q4 = reinterpret_cast<const float4*>(qs + g * HD)[t];
                acc[g] += q4.x * k4.x + q4.y * k4.y + q4.z * k4.z + q4.w * k4.w;
            }
        }
#pragma unroll
        for (int g = 0; g < kMaxGroup; ++g) {
            if (g >= group) break;
            const float s = acc[g] * inv_sqrt_hd + mv[c];
            sc[g * cap + c] = s;
            mx[g] = fmaxf(mx[g], s);
        }
    }
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
        float m = mx[g];
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) stat[warp][g] = m;
    }
    __syncthreads();
    if (threadIdx.x < group) {
        float m = stat[0][threadIdx.x];
        for (int w = 1; w < kWarps; ++w) m = fmaxf(m, stat[w][threadIdx.x]);
        mx_s[threadIdx.x] = m;
    }
    __syncthreads();
    bool empty = false;
    for (int g = 0; g < group; ++g) empty |= mx_s[g] == -INFINITY;
    if (empty) {  // tinyformer.cpp:467-469
        if (threadIdx.x == 0) atomicOr(status, ST_EMPTY_ROW);
        return;
    }
    // exp + denominators (fixed per-thread assignment, fixed tree)
    float sum[kMaxGroup];
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) sum[g] = 0.0f;
    for (int c = threadIdx.x; c < n; c += kThreads)
#pragma unroll
        for (int g = 0; g < kMaxGroup; ++g) {
            if (g >= group) break;
            const float s = sc[g * cap + c];
            const float e = s == -INFINITY ? 0.0f : sfg_expf(s - mx_s[g]);
            sc[g * cap + c] = e;
            sum[g] += e;
        }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
        float s = sum[g];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) stat[warp][g] = s;
    }
    __syncthreads();
    if (threadIdx.x < group) {
        float s = 0.0f;
        for (int w = 0; w < kWarps; ++w) s += stat[w][threadIdx.x];
        inv_s[threadIdx.x] = 1.0f / s;
    }
    // value sums: warp w owns a contiguous key range, lane owns dims lane + 32i
    constexpr int DPL = HD / 32;
    float acc[kMaxGroup][DPL];
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g)
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[g][i] = 0.0f;
    const int chunk = (n + kWarps - 1) / kWarps;
    const int c0 = warp * chunk, c1 = min(n, c0 + chunk);
    for (int c = c0; c < c1; ++c) {
        const float* vr = vb + static_cast<size_t>(cols[c]) * HD;
        float v[DPL];
#pragma unroll
        for (int i = 0; i < DPL; ++i) v[i] = __ldg(vr + lane + 32 * i);
#pragma unroll
        for (int g = 0; g < kMaxGroup; ++g) {
            if (g >= group) break;
            const float p = sc[g * cap + c];
#pragma unroll
            for (int i = 0; i < DPL; ++i) acc[g][i] += p * v[i];
        }
    }
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) {
        if (g >= group) break;
#pragma unroll
        for (int i = 0; i < DPL; ++i) red[(warp * group + g) * HD + lane + 32 * i] = acc[g][i];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < group * HD; t += kThreads) {
        const int g = t / HD, dd = t % HD;
        float o = 0.0f;
        for (int w = 0; w < kWarps; ++w) o += red[(w * group + g) * HD + dd];
        att[static_cast<size_t>(row) * d.qd + static_cast<size_t>(kvh * group + g) * HD + dd] = o * inv_s[g];
    }
}

template <int HD>
int launch_hd(const float* q, const float* kc, const float* vc, const int32_t* row_off, const MaskRun* runs, int rows,
              const Dims& d, float* att, uint32_t* status, cudaStream_t s, int cap) {
    const int group = d.n_heads / d.n_kv;  // shared memory sized by the real GQA group
    const size_t smem = sizeof(float) * (static_cast<size_t>(group) * HD + static_cast<size_t>(kWarps) * group * HD) +
                        static_cast<size_t>(cap) * (sizeof(int) + sizeof(float)) +
                        sizeof(float) * static_cast<size_t>(d.n_heads / d.n_kv) * cap;
    // opt in even near 48 KB: static smem counts against the default limit
    if (smem > 220 * 1024) throw Error(Kind::config, "max_seq_len too large for the FAST attention kernel");
    ensure_smem_attr(reinterpret_cast<const void*>(attn_fast_kernel<HD>), smem);
    attn_fast_kernel<HD><<<rows * d.n_kv, kThreads, smem, s>>>(q, kc, vc, row_off, runs, d, att, status, cap);
    return 1;
}

}  // namespace

int launch_attention_fast(const float* q, const float* kcache, const float* vcache, const int32_t* row_off,
                          const MaskRun* runs, int rows, const Dims& d, float* att, uint32_t* status, cudaStream_t s,
                          int kv_cap) {
    const int cap = kv_cap > 0 ? std::min(kv_cap, d.max_len) : d.max_len;
    if (d.n_heads / d.n_kv > kMaxGroup) throw Error(Kind::config, "GQA group > 8 not supported by FAST attention");
    switch (d.hd) {
        case 64: return launch_hd<64>(q, kcache, vcache, row_off, runs, rows, d, att, status, s, cap);
        case 128: return launch_hd<128>(q, kcache, vcache, row_off, runs, rows, d, att, status, s, cap);
        case 160: return launch_hd<160>(q, kcache, vcache, row_off, runs, rows, d, att, status, s, cap);
        case 32: return launch_hd<32>(q, kcache, vcache, row_off, runs, rows, d, att, status, s, cap);
        default:
            return launch_attention_exact(q, kcache, vcache, row_off, runs, rows, 0, d, att, status, s);
    }
}

}  // namespace sfg
