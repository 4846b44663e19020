// EXACT-mode layer executor kernels (CUDA cores, sm_100a).
//
// These reproduce the reference's fp32 arithmetic (tinyformer.cpp:33-65,
// 375-526) operation for operation: every multiply and add is an explicit
// IEEE round-to-nearest intrinsic (__fmul_rn / __fadd_rn, never contracted to
// FMA; this TU is also compiled with --fmad=false), every reduction runs in
// the reference's serial loop order, exp is the bit-exact glibc port
// (sfg_expf.h) and RoPE uses the host-libm cos/sin table.  Parallelism comes
// only from the reference's independent chains: output columns x batch rows
// for the projections, keys for the score dots, head dims for the value sum.
//
// Roofline: at B rows a projection with K inputs and N outputs streams
// K*N*sizeof(w) bytes once (HBM-bound) but needs K*N*B dependent-chain
// mul+add pairs on the FP32 pipe; for B >= ~6 this mode is FP32-issue-bound,
// by design — it is the bit-parity mode, FAST mode is the throughput mode.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sfg_expf.h"
#include "sfg_kernels.h"

namespace sfg {
namespace {

constexpr int kThreads = 128;
constexpr int kKC = 64;  // k-chunk of activations staged in shared memory

template <int WT>
struct WLoad;
template <>
struct WLoad<W_BF16> {
    // two adjacent output columns of one weight row
    static __device__ __forceinline__ void load2(const void* w, size_t off, float& a, float& b) {
        const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(
            reinterpret_cast<const __nv_bfloat16*>(w) + off);
        a = __low2float(v);
        b = __high2float(v);
    }
};
template <>
struct WLoad<W_F32> {
    static __device__ __forceinline__ void load2(const void* w, size_t off, float& a, float& b) {
        const float2 v = *reinterpret_cast<const float2*>(reinterpret_cast<const float*>(w) + off);
        a = v.x;
        b = v.y;
    }
};

// Core of matvec (tinyformer.cpp:41-49) for RB batch rows x 2 adjacent
// columns per thread: acc[r][c] = (((0 + x0 w0) + x1 w1) + ...) in k order.
// The reference skips x[i] == 0; that skip is provably a no-op for finite
// weights (acc starts at +0 and can never become -0 under RNE), so the loop
// is branch-free.  All threads of the CTA must call this (barriers inside).
template <int WT, int RB, int NM>
__device__ __forceinline__ void mv_core(const float* __restrict__ X, int ldx, int row0, int rows,
                                        int K, const void* const (&W)[NM], int ldw, int col,
                                        bool active, float (&acc)[NM][RB][2], float* xs) {
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[m][r][0] = acc[m][r][1] = 0.0f;
    for (int k0 = 0; k0 < K; k0 += kKC) {
        const int kc = min(kKC, K - k0);
        __syncthreads();
        for (int t = threadIdx.x; t < kc * RB; t += blockDim.x) {
            const int r = t / kc, k = t - r * kc;
            xs[k * RB + r] = (row0 + r < rows) ? X[(size_t)(row0 + r) * ldx + k0 + k] : 0.0f;
        }
        __syncthreads();
        if (active) {
#pragma unroll 8
            for (int k = 0; k < kc; ++k) {
                float w[NM][2];
#pragma unroll
                for (int m = 0; m < NM; ++m)
                    WLoad<WT>::load2(W[m], (size_t)(k0 + k) * ldw + col, w[m][0], w[m][1]);
#pragma unroll
                for (int r = 0; r < RB; ++r) {
                    const float xv = xs[k * RB + r];
#pragma unroll
                    for (int m = 0; m < NM; ++m) {
                        acc[m][r][0] = __fadd_rn(acc[m][r][0], __fmul_rn(xv, w[m][0]));
                        acc[m][r][1] = __fadd_rn(acc[m][r][1], __fmul_rn(xv, w[m][1]));
                    }
                }
            }
        }
    }
}

// rope_rotate (tinyformer.cpp:52-63) on the pair (2i, 2i+1):
// a' = a*c - b*s ; b' = a*s + b*c with separately rounded products.
__device__ __forceinline__ void rope_pair(float& a, float& b, float c, float s) {
    const float na = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
    const float nb = __fadd_rn(__fmul_rn(a, s), __fmul_rn(b, c));
    a = na;
    b = nb;
}

// ── RMSNorm (tinyformer.cpp:33-38) ───────────────────────────────────────
// The sum of squares is one serial chain per row (reference loop order);
// the row is staged in shared memory so the chain never waits on L2.
__global__ void rmsnorm_exact_kernel(const float* __restrict__ h, const float* __restrict__ g,
                                     float* __restrict__ y, int H, float eps) {
    extern __shared__ float xrow[];
    __shared__ float scale_s;
    const float* x = h + (size_t)blockIdx.x * H;
    for (int i = threadIdx.x; i < H; i += blockDim.x) xrow[i] = x[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        float ss = 0.0f;
#pragma unroll 16
        for (int i = 0; i < H; ++i) ss = __fadd_rn(ss, __fmul_rn(xrow[i], xrow[i]));
        scale_s = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)H), eps)));
    }
    __syncthreads();
    const float sc = scale_s;
    float* yr = y + (size_t)blockIdx.x * H;
    for (int i = threadIdx.x; i < H; i += blockDim.x) yr[i] = __fmul_rn(__fmul_rn(xrow[i], sc), g[i]);
}

// ── Q/K/V projections + RoPE + KV append (tinyformer.cpp:416-448) ─────────
// blockIdx.x spans the concatenated output columns [q | k | v]; each thread
// owns 2 adjacent columns (one rotary pair) for RB rows.
template <int WT, int RB>
__global__ void __launch_bounds__(kThreads) qkv_exact_kernel(
    const float* __restrict__ xn, int rows, Dims d, const void* wq, const void* wk, const void* wv,
    const int32_t* __restrict__ pos, const float* __restrict__ rope_cos,
    const float* __restrict__ rope_sin, float* __restrict__ q, float* __restrict__ kc,
    float* __restrict__ vc, const int32_t* __restrict__ prior_ptr) {
    __shared__ __align__(16) float xs[kKC * RB];
    const int pairs_q = d.qd / 2, pairs_kv = d.kvd / 2;
    const int pair = blockIdx.x * kThreads + threadIdx.x;
    int seg, col;
    const void* w;
    int ldw;
    if (pair < pairs_q) {
        seg = 0; col = 2 * pair; w = wq; ldw = d.qd;
    } else if (pair < pairs_q + pairs_kv) {
        seg = 1; col = 2 * (pair - pairs_q); w = wk; ldw = d.kvd;
    } else {
        seg = 2; col = 2 * (pair - pairs_q - pairs_kv); w = wv; ldw = d.kvd;
    }
    const bool active = pair < pairs_q + 2 * pairs_kv;
    if (!active) { w = wq; ldw = d.qd; col = 0; }
    // Segment boundaries are multiples of 128 pairs only when qd, kvd are
    // multiples of 256; a CTA may straddle q|k|v, so each thread carries its
    // own weight pointer (warp-uniform in practice).
    const void* const W[1] = {w};
    float acc[1][RB][2];
    const int row0 = blockIdx.y * RB;
    mv_core<WT, RB, 1>(xn, d.H, row0, rows, d.H, W, ldw, col, active, acc, xs);
    if (!active) return;
    const int half = d.hd / 2;
    const int i = (col % d.hd) / 2;  // rotary pair index within the head
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        const int row = row0 + r;
        if (row >= rows) break;
        float a = acc[0][r][0], b = acc[0][r][1];
        if (seg != 2) {
            const int p = pos[row];
            rope_pair(a, b, rope_cos[(size_t)p * half + i], rope_sin[(size_t)p * half + i]);
        }
        if (seg == 0) {
            q[(size_t)row * d.qd + col] = a;
            q[(size_t)row * d.qd + col + 1] = b;
        } else {
            const int kvh = col / d.hd, dd = col % d.hd;
            float* dst = (seg == 1 ? kc : vc) + ((size_t)kvh * d.max_len + *prior_ptr + row) * d.hd + dd;
            dst[0] = a;
            dst[1] = b;
        }
    }
}

// ── masked softmax attention (tinyformer.cpp:450-489) ────────────────────
// One CTA per (row, head).  Scores in parallel over visible keys (each dot a
// serial chain over head_dim), max (order-free), exp (glibc port), then the
// reference's two serial reductions: the denominator over keys (thread 0)
// and the weighted value sum over keys (one chain per head dim).
constexpr int kAttnThreads = 256;

__global__ void __launch_bounds__(kAttnThreads) attention_exact_kernel(
    const float* __restrict__ q, const float* __restrict__ kc, const float* __restrict__ vc,
    const int32_t* __restrict__ row_off, const MaskRun* __restrict__ runs, Dims d,
    float* __restrict__ att, uint32_t* status) {
    extern __shared__ float smem[];
    const int row = blockIdx.x / d.n_heads, head = blockIdx.x % d.n_heads;
    const int kvh = head / (d.n_heads / d.n_kv);
    float* qh = smem;                        // [hd]
    float* sc = qh + d.hd;                   // [max_len] scores then exp
    float* wg = sc + d.max_len;              // [max_len] weights
    int* cols = reinterpret_cast<int*>(wg + d.max_len);  // [max_len]
    float* mv = reinterpret_cast<float*>(cols + d.max_len);  // [max_len]
    __shared__ float red[kAttnThreads / 32];
    __shared__ int n_s;
    __shared__ float inv_s;

    for (int t = threadIdx.x; t < d.hd; t += blockDim.x)
        qh[t] = q[(size_t)row * d.qd + (size_t)head * d.hd + t];
    if (threadIdx.x == 0) {
        int n = 0;
        for (int r = row_off[row]; r < row_off[row + 1]; ++r)
            for (int j = runs[r].start; j < runs[r].end; ++j) {
                cols[n] = j;
                mv[n] = runs[r].mval;
                ++n;
            }
        n_s = n;
    }
    __syncthreads();
    const int n = n_s;
    const float inv_sqrt_hd = __fdiv_rn(1.0f, __fsqrt_rn((float)d.hd));
    const float* kbase = kc + (size_t)kvh * d.max_len * d.hd;
    const float* vbase = vc + (size_t)kvh * d.max_len * d.hd;

    float mx = -INFINITY;
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const float4* kj = reinterpret_cast<const float4*>(kbase + (size_t)cols[c] * d.hd);
        float dot = 0.0f;
        for (int t = 0; t < d.hd / 4; ++t) {
            const float4 k4 = kj[t];
            dot = __fadd_rn(dot, __fmul_rn(qh[4 * t + 0], k4.x));
            dot = __fadd_rn(dot, __fmul_rn(qh[4 * t + 1], k4.y));
            dot = __fadd_rn(dot, __fmul_rn(qh[4 * t + 2], k4.z));
            dot = __fadd_rn(dot, __fmul_rn(qh[4 * t + 3], k4.w));
        }
        const float s = __fadd_rn(__fmul_rn(dot, inv_sqrt_hd), mv[c]);
        sc[c] = s;
        mx = fmaxf(mx, s);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = red[0];
        for (int w = 1; w < kAttnThreads / 32; ++w) m = fmaxf(m, red[w]);
        red[0] = m;
    }
    __syncthreads();
    mx = red[0];
    if (mx == -INFINITY) {  // tinyformer.cpp:467-469
        if (threadIdx.x == 0) atomicOr(status, ST_EMPTY_ROW);
        return;
    }
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const float s = sc[c];
        sc[c] = (s == -INFINITY) ? 0.0f : sfg_expf(__fsub_rn(s, mx));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float den = 0.0f;
        // masked-by-value entries carry 0 and adding +0 to den (>= +0) is a no-op
        for (int c = 0; c < n; ++c) den = __fadd_rn(den, sc[c]);
        inv_s = __fdiv_rn(1.0f, den);
    }
    __syncthreads();
    const float inv = inv_s;
    for (int c = threadIdx.x; c < n; c += blockDim.x) wg[c] = __fmul_rn(sc[c], inv);
    __syncthreads();
    for (int t = threadIdx.x; t < d.hd; t += blockDim.x) {
        float o = 0.0f;
        for (int c = 0; c < n; ++c) {
            const float w = wg[c];
            if (w == 0.0f) continue;
            o = __fadd_rn(o, __fmul_rn(w, vbase[(size_t)cols[c] * d.hd + t]));
        }
        att[(size_t)row * d.qd + (size_t)head * d.hd + t] = o;
    }
}

// ── O-proj / down-proj with residual (tinyformer.cpp:491-493, 499-500) ──
template <int WT, int RB>
__global__ void __launch_bounds__(kThreads) mv_residual_exact_kernel(const float* __restrict__ x,
                                                                     int rows, int K, const void* w,
                                                                     int N, float* __restrict__ h) {
    __shared__ __align__(16) float xs[kKC * RB];
    const int col = 2 * (blockIdx.x * kThreads + threadIdx.x);
    const bool active = col < N;
    const void* const W[1] = {w};
    float acc[1][RB][2];
    const int row0 = blockIdx.y * RB;
    mv_core<WT, RB, 1>(x, K, row0, rows, K, W, N, active ? col : 0, active, acc, xs);
    if (!active) return;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        if (row0 + r >= rows) break;
        float* hr = h + (size_t)(row0 + r) * N + col;
        hr[0] = __fadd_rn(hr[0], acc[0][r][0]);
        hr[1] = __fadd_rn(hr[1], acc[0][r][1]);
    }
}

// plain store (LM head logits, tinyformer.cpp:520-524)
template <int WT, int RB>
__global__ void __launch_bounds__(kThreads) mv_store_exact_kernel(const float* __restrict__ x,
                                                                  int rows, int K, const void* w,
                                                                  int N, float* __restrict__ out) {
    __shared__ __align__(16) float xs[kKC * RB];
    const int col = 2 * (blockIdx.x * kThreads + threadIdx.x);
    const bool active = col < N;
    const void* const W[1] = {w};
    float acc[1][RB][2];
    const int row0 = blockIdx.y * RB;
    mv_core<WT, RB, 1>(x, K, row0, rows, K, W, N, active ? col : 0, active, acc, xs);
    if (!active) return;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        if (row0 + r >= rows) break;
        out[(size_t)(row0 + r) * N + col] = acc[0][r][0];
        out[(size_t)(row0 + r) * N + col + 1] = acc[0][r][1];
    }
}

// SwiGLU (tinyformer.cpp:495-498): gate and up share the column loop;
// act = silu(g) * u with silu(g) = g / (1 + expf(-g)).
template <int WT, int RB>
__global__ void __launch_bounds__(kThreads) gateup_exact_kernel(const float* __restrict__ xn,
                                                                int rows, int H, int F,
                                                                const void* wg, const void* wu,
                                                                float* __restrict__ act) {
    __shared__ __align__(16) float xs[kKC * RB];
    const int col = 2 * (blockIdx.x * kThreads + threadIdx.x);
    const bool active = col < F;
    const void* const W[2] = {wg, wu};
    float acc[2][RB][2];
    const int row0 = blockIdx.y * RB;
    mv_core<WT, RB, 2>(xn, H, row0, rows, H, W, F, active ? col : 0, active, acc, xs);
    if (!active) return;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        if (row0 + r >= rows) break;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float g = acc[0][r][c];
            const float silu = __fdiv_rn(g, __fadd_rn(1.0f, sfg_expf(-g)));
            act[(size_t)(row0 + r) * F + col + c] = __fmul_rn(silu, acc[1][r][c]);
        }
    }
}

constexpr int kRB = 4;

inline dim3 mv_grid(int N, int rows) {
    return dim3((unsigned)((N / 2 + kThreads - 1) / kThreads), (unsigned)((rows + kRB - 1) / kRB));
}

}  // namespace

int launch_rmsnorm_exact(const float* h, const float* g, float* y, int rows, int H, float eps,
                         cudaStream_t s) {
    rmsnorm_exact_kernel<<<rows, 256, H * sizeof(float), s>>>(h, g, y, H, eps);
    return 1;
}

int launch_qkv_exact(const float* xn, int rows, const Dims& d, int wt, const void* wq,
                     const void* wk, const void* wv, const int32_t* pos, const float* rope_cos,
                     const float* rope_sin, float* q, float* kcache, float* vcache, const int32_t* prior,
                     cudaStream_t s) {
    const int pairs = (d.qd + 2 * d.kvd) / 2;
    dim3 grid((pairs + kThreads - 1) / kThreads, (rows + kRB - 1) / kRB);
    if (wt == W_BF16)
        qkv_exact_kernel<W_BF16, kRB><<<grid, kThreads, 0, s>>>(xn, rows, d, wq, wk, wv, pos, rope_cos,
                                                               rope_sin, q, kcache, vcache, prior);
    else
        qkv_exact_kernel<W_F32, kRB><<<grid, kThreads, 0, s>>>(xn, rows, d, wq, wk, wv, pos, rope_cos,
                                                              rope_sin, q, kcache, vcache, prior);
    return 1;
}

int launch_attention_exact(const float* q, const float* kcache, const float* vcache,
                           const int32_t* row_off, const MaskRun* runs, int rows, int kv_len,
                           const Dims& d, float* att, uint32_t* status, cudaStream_t s) {
    (void)kv_len;
    const size_t smem = sizeof(float) * (size_t)d.hd + (size_t)d.max_len * (4 * sizeof(float));
    ensure_smem_attr(reinterpret_cast<const void*>(attention_exact_kernel), 200 * 1024);
    attention_exact_kernel<<<rows * d.n_heads, kAttnThreads, smem, s>>>(q, kcache, vcache, row_off,
                                                                        runs, d, att, status);
    return 1;
}

int launch_matvec_residual_exact(const float* x, int rows, int K, int wt, const void* w, int N,
                                 float* h, cudaStream_t s) {
    if (wt == W_BF16)
        mv_residual_exact_kernel<W_BF16, kRB><<<mv_grid(N, rows), kThreads, 0, s>>>(x, rows, K, w, N, h);
    else
        mv_residual_exact_kernel<W_F32, kRB><<<mv_grid(N, rows), kThreads, 0, s>>>(x, rows, K, w, N, h);
    return 1;
}

int launch_matvec_store_exact(const float* x, int rows, int K, int wt, const void* w, int N,
                              float* out, cudaStream_t s) {
    if (wt == W_BF16)
        mv_store_exact_kernel<W_BF16, kRB><<<mv_grid(N, rows), kThreads, 0, s>>>(x, rows, K, w, N, out);
    else
        mv_store_exact_kernel<W_F32, kRB><<<mv_grid(N, rows), kThreads, 0, s>>>(x, rows, K, w, N, out);
    return 1;
}

int launch_gateup_exact(const float* xn, int rows, int H, int F, int wt, const void* wg,
                        const void* wu, float* act, cudaStream_t s) {
    if (wt == W_BF16)
        gateup_exact_kernel<W_BF16, kRB><<<mv_grid(F, rows), kThreads, 0, s>>>(xn, rows, H, F, wg, wu, act);
    else
        gateup_exact_kernel<W_F32, kRB><<<mv_grid(F, rows), kThreads, 0, s>>>(xn, rows, H, F, wg, wu, act);
    return 1;
}

}  // namespace sfg
