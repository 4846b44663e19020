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

// ── prompt (prefill) attention: tiled, K/V shared by a block of queries ──
// attn_fast_kernel reads every visible K/V row once per (query row, kv head):
// a 2048-token prompt moves ~16 GB per layer through L2.  Here a CTA takes 64
// queries (64 / G consecutive rows x the G q-heads of one kv head) and walks
// the keys in blocks of 64 at ABSOLUTE positions, staged in shared memory once
// for all 64 queries: S = Q K^T by a 4 x 4 register tile per thread, an online
// softmax per query in ascending block order, O += P V by a 4 x HD/16 tile.
// Only the prefix mask law applies (every row sees keys [0, lim): causal
// prompts, tinyformer.cpp:229-241); a row's result depends on its own query
// and keys only, never on the rows it is tiled with.
constexpr int kPQ = 64;   // queries per CTA
constexpr int kPK = 64;   // keys per block

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Shared memory: Q [kPQ][HD] and K [kPK][HD] with float4 column c of row r at
// c ^ (r & 7) (the 16 key rows a half-warp reads at once hit 8 bank groups),
// V [kPK][HD]; P [kPQ][kPK + 4] reuses K's space once the scores are taken.
// 96 KB at HD = 128: two CTAs per SM, so one CTA's K / V copies (cp.async,
// straight to shared memory) overlap the other's arithmetic.
template <int HD>
__global__ void __launch_bounds__(256, 2) attn_prompt_kernel(const float* __restrict__ q, const float* __restrict__ kc,
                                                             const float* __restrict__ vc,
                                                             const int32_t* __restrict__ row_off,
                                                             const MaskRun* __restrict__ runs, Dims d, int rows,
                                                             float* __restrict__ att, uint32_t* status) {
    constexpr int C4 = HD / 4;    // float4 columns per row
    constexpr int DPT = HD / 16;  // value dims per thread
    extern __shared__ float4 smem4[];
    float4* Q4 = smem4;                                // [kPQ][C4] swizzled
    float4* K4 = Q4 + kPQ * C4;                        // [kPK][C4] swizzled
    float* Vs = reinterpret_cast<float*>(K4) + kPK * (HD > kPK + 4 ? HD : kPK + 4);  // [kPK][HD]
    float* P = reinterpret_cast<float*>(K4);           // [kPQ][kPK + 4] (after the scores)
    __shared__ int lim_s[kPQ];
    const int G = d.n_heads / d.n_kv, RPB = kPQ / G;
    // the heaviest (latest, longest causal) row blocks are scheduled first
    const int rb0 = (gridDim.x - 1 - blockIdx.x) * RPB, kvh = blockIdx.y;
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    // query qi = g * RPB + r: row rb0 + r, head kvh * G + g
    for (int idx = tid; idx < kPQ * C4; idx += 256) {
        const int qi = idx / C4, c = idx % C4, r = qi % RPB, g = qi / RPB, row = rb0 + r;
        float4* dst = Q4 + qi * C4 + (c ^ (qi & 7));
        if (row < rows)
            cp_async16(dst, q + static_cast<size_t>(row) * d.qd + static_cast<size_t>(kvh * G + g) * HD + 4 * c);
        else
            *dst = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    cp_async_commit();
    if (tid < kPQ) {
        const int row = rb0 + tid % RPB;
        lim_s[tid] = row < rows ? runs[row_off[row]].end : 0;
    }
    __syncthreads();
    int kmax = 0;
    for (int i = 0; i < kPQ; ++i) kmax = max(kmax, lim_s[i]);
    int lim[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) lim[i] = lim_s[4 * ty + i];
    const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(HD));
    const float* kb = kc + static_cast<size_t>(kvh) * d.max_len * HD;
    const float* vb = vc + static_cast<size_t>(kvh) * d.max_len * HD;
    float m[4], l[4], o[4][DPT];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.0f;
#pragma unroll
        for (int c = 0; c < DPT; ++c) o[i][c] = 0.0f;
    }
    for (int k0 = 0; k0 < kmax; k0 += kPK) {
        const int nk = min(kPK, kmax - k0);
        __syncthreads();  // the previous block's P / V are consumed
        for (int idx = tid; idx < nk * C4; idx += 256) {
            const int kk = idx / C4, c = idx % C4;
            cp_async16(K4 + kk * C4 + (c ^ (kk & 7)), kb + static_cast<size_t>(k0 + kk) * HD + 4 * c);
        }
        cp_async_commit();
        for (int idx = tid; idx < nk * C4; idx += 256)
            cp_async16(reinterpret_cast<float4*>(Vs) + idx, vb + static_cast<size_t>(k0) * HD + 4 * idx);
        cp_async_commit();
        cp_async_wait<1>();  // queries + K
        __syncthreads();
        // scores: queries 4ty + i, keys tx + 16 j (rows past nk are masked below)
        float sc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) sc[i][j] = 0.0f;
#pragma unroll 2
        for (int c = 0; c < C4; ++c) {
            float4 q4[4], k4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) q4[i] = Q4[(4 * ty + i) * C4 + (c ^ ((4 * ty + i) & 7))];
#pragma unroll
            for (int j = 0; j < 4; ++j) k4[j] = K4[(tx + 16 * j) * C4 + (c ^ (tx & 7))];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    sc[i][j] = fmaf(q4[i].x, k4[j].x, sc[i][j]);
                    sc[i][j] = fmaf(q4[i].y, k4[j].y, sc[i][j]);
                    sc[i][j] = fmaf(q4[i].z, k4[j].z, sc[i][j]);
                    sc[i][j] = fmaf(q4[i].w, k4[j].w, sc[i][j]);
                }
        }
        __syncthreads();  // K is consumed: P takes its space
        // online softmax per query (its 64 keys sit on the 16 tx lanes of its half-warp)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float bm = -INFINITY;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = k0 + tx + 16 * j;
                sc[i][j] = key < lim[i] ? sc[i][j] * inv_sqrt_hd : -INFINITY;
                bm = fmaxf(bm, sc[i][j]);
            }
            for (int off = 8; off > 0; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, off));
            const float mn = fmaxf(m[i], bm);
            const float alpha = m[i] == -INFINITY ? 0.0f : expf(m[i] - mn);
            float rs = 0.0f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float pj = sc[i][j] == -INFINITY ? 0.0f : expf(sc[i][j] - mn);
                P[(4 * ty + i) * (kPK + 4) + tx + 16 * j] = pj;
                rs += pj;
            }
            for (int off = 8; off > 0; off >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
            l[i] = l[i] * alpha + rs;
            m[i] = mn;
#pragma unroll
            for (int c = 0; c < DPT; ++c) o[i][c] *= alpha;
        }
        cp_async_wait<0>();  // V
        __syncthreads();
        // O += P V: rows 4ty..4ty+3, dims tx*DPT ..
#pragma unroll 2
        for (int kk = 0; kk < nk; ++kk) {
            float pv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pv[i] = P[(4 * ty + i) * (kPK + 4) + kk];
            const float2* vr = reinterpret_cast<const float2*>(Vs + kk * HD + tx * DPT);
#pragma unroll
            for (int c2 = 0; c2 < DPT / 2; ++c2) {
                const float2 v2 = vr[c2];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    o[i][2 * c2] = fmaf(pv[i], v2.x, o[i][2 * c2]);
                    o[i][2 * c2 + 1] = fmaf(pv[i], v2.y, o[i][2 * c2 + 1]);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int qi = 4 * ty + i, r = qi % RPB, g = qi / RPB, row = rb0 + r;
        if (row >= rows) continue;
        if (!(l[i] > 0.0f)) {  // tinyformer.cpp:467-469
            if (tx == 0) atomicOr(status, ST_EMPTY_ROW);
            continue;
        }
        float* dst = att + static_cast<size_t>(row) * d.qd + static_cast<size_t>(kvh * G + g) * HD + tx * DPT;
        const float inv = 1.0f / l[i];
#pragma unroll
        for (int c = 0; c < DPT; ++c) dst[c] = o[i][c] * inv;
    }
}

template <int HD>
int launch_prompt_hd(const float* q, const float* kc, const float* vc, const int32_t* row_off, const MaskRun* runs,
                     int rows, const Dims& d, float* att, uint32_t* status, cudaStream_t s) {
    // Q | K (then P) | V; P [kPQ][kPK + 4] fits in K's [kPK][HD] for HD >= 68
    const size_t smem = sizeof(float) * (static_cast<size_t>(kPQ) * HD + 2 * static_cast<size_t>(kPK) * std::max(HD, kPK + 4));
    ensure_smem_attr(reinterpret_cast<const void*>(attn_prompt_kernel<HD>), smem);
    const int rpb = kPQ / (d.n_heads / d.n_kv);
    const dim3 grid((rows + rpb - 1) / rpb, d.n_kv);
    attn_prompt_kernel<HD><<<grid, 256, smem, s>>>(q, kc, vc, row_off, runs, d, rows, att, status);
    return 1;
}

}  // namespace

// Prompt attention for masks of the prefix law (host-checked: every row one
// run [0, lim) with value 0); other shapes take launch_attention_fast.
bool attention_prompt_supported(const Dims& d) {
    const int G = d.n_heads / d.n_kv;
    return (d.hd == 64 || d.hd == 128 || d.hd == 160) && (G == 1 || G == 2 || G == 4 || G == 8);
}

int launch_attention_prompt(const float* q, const float* kcache, const float* vcache, const int32_t* row_off,
                            const MaskRun* runs, int rows, int keys, const Dims& d, float* att, uint32_t* status,
                            cudaStream_t s, void** scratch, size_t* scratch_bytes) {
    if (attention_prompt_tc_supported(d))
        return launch_attention_prompt_tc(q, kcache, vcache, row_off, runs, rows, keys, d, att, status, s, scratch,
                                          scratch_bytes);
    switch (d.hd) {
        case 64: return launch_prompt_hd<64>(q, kcache, vcache, row_off, runs, rows, d, att, status, s);
        case 128: return launch_prompt_hd<128>(q, kcache, vcache, row_off, runs, rows, d, att, status, s);
        default: return launch_prompt_hd<160>(q, kcache, vcache, row_off, runs, rows, d, att, status, s);
    }
}

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
