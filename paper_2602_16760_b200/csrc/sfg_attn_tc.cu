// FAST-mode causal prompt attention on the tensor cores (sm_100a), head_dim 128.
//
// tinyformer.cpp:442-489 for prompts (prefix mask law: row r sees keys
// [0, lim_r), server.cpp:203-224).  A CTA owns 128 queries = (128 / G) rows x
// the G q-heads of one kv head and walks the keys in 64-key blocks:
//
//   S  = Q K^T    tcgen05.mma, A = Q (smem, M = 128 queries), B = K block (smem, N = 64)
//   P  = exp(S - m)   online softmax, one query per thread (TMEM lane), P written
//                     back into TMEM as the A operand of
//   O += P V      tcgen05.mma, A = P (TMEM), B = V^T block (smem, N = 128 dims)
//
// fp32 operands are split into three bf16 pieces (hi | mid | lo) and every
// product of the six leading piece pairs (hh hm mh hl mm lh) is accumulated in
// fp32 TMEM, so S and O carry ~fp32 accuracy (the dropped terms are 2^-32
// relative), the same bar as the FAST GEMMs.  When a block raises a query's
// running max, its O row is rescaled in TMEM (tcgen05.ld / st) before the
// next PV MMA accumulates into it.
//
// Warp roles (288 threads, one CTA per SM: 192 KB of shared memory, 512 TMEM
// columns):
//   warps 0-3  softmax + output: thread = query = TMEM lane;
//   warps 4-7  producer: Q once, then per block the K pieces ([key][dim],
//              K-major) and the V^T pieces ([dim][key], K-major) from the
//              fp32 KV cache, split on the fly;
//   warp 8     MMA issuer (one thread).
// mbarriers: k_ready / v_ready (producer -> MMA), s_full (MMA -> softmax and
// producer: K consumed), s_free (softmax -> MMA: S read), p_ready (softmax ->
// MMA), pv_done (MMA -> softmax: O final for the block, P and V consumed).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "sfg_engine.h"
#include "sfg_tc.cuh"

namespace sfg {
namespace {

using namespace tc;

constexpr int kHD = 128;
constexpr int kQ = 128;       // queries per CTA (TMEM lanes)
constexpr int kKB = 64;       // keys per block
constexpr int kThreadsTC = 288;
// shared memory: Q pieces 3 x [2 k-blocks][128 rows][128 B] | K pieces 3 x [2][64][128 B] | V^T pieces 3 x [128 dims][128 B]
constexpr int kQBytes = 3 * 2 * 128 * 128;  // 96 KB
constexpr int kKBytes = 3 * 2 * 64 * 128;   // 48 KB
constexpr int kVBytes = 3 * 128 * 128;      // 48 KB
constexpr int kSmemTC = 1024 + kQBytes + kKBytes + kVBytes + 256;
// TMEM columns
constexpr uint32_t kColS = 0;    // S [128 q][64 keys] fp32
constexpr uint32_t kColP = 64;   // P pieces 3 x 32 columns (bf16 pairs)
constexpr uint32_t kColO = 256;  // O [128 q][128 dims] fp32

__host__ __device__ constexpr uint32_t idesc_mn(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
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

// bounded mbarrier wait (traps instead of hanging on a protocol bug)
// (try_wait suspends the thread in hardware between polls: the 257 waiting
// threads do not flood the shared-memory pipe the way test_wait spinning does)
__device__ __forceinline__ void bwait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    unsigned long long spins = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
        if (done) return;
        if (++spins > (1ull << 26)) asm volatile("trap;");
    }
}

// three bf16 pieces of x
struct Split3 {
    __nv_bfloat16 h, m, l;
};
__device__ __forceinline__ Split3 split3(float x) {
    Split3 s;
    s.h = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(s.h);
    s.m = __float2bfloat16_rn(r1);
    s.l = __float2bfloat16_rn(r1 - __bfloat162float(s.m));
    return s;
}
__device__ __forceinline__ uint32_t pack2(__nv_bfloat16 a, __nv_bfloat16 b) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(a)) | (static_cast<uint32_t>(__bfloat16_as_ushort(b)) << 16);
}
// 4 consecutive K elements (k % 4 == 0) of row r: three 8-byte stores into
// SW128 K-major tiles (piece p at base + p * pstride, k-block at + (k / 64) * kbstride)
__device__ __forceinline__ void put3x4(uint8_t* base, uint32_t pstride, uint32_t kbstride, int r, int k, float a0,
                                       float a1, float a2, float a3) {
    const Split3 s0 = split3(a0), s1 = split3(a1), s2 = split3(a2), s3 = split3(a3);
    uint8_t* t = base + (k >> 6) * kbstride + sw128_off(r, k & 63);
    *reinterpret_cast<uint2*>(t) = make_uint2(pack2(s0.h, s1.h), pack2(s2.h, s3.h));
    *reinterpret_cast<uint2*>(t + pstride) = make_uint2(pack2(s0.m, s1.m), pack2(s2.m, s3.m));
    *reinterpret_cast<uint2*>(t + 2 * pstride) = make_uint2(pack2(s0.l, s1.l), pack2(s2.l, s3.l));
}

__global__ void __launch_bounds__(kThreadsTC, 1) attn_prompt_tc_kernel(const float* __restrict__ q, const float* __restrict__ kc,
                                                                        const float* __restrict__ vc,
                                                                        const int32_t* __restrict__ row_off,
                                                                        const MaskRun* __restrict__ runs, Dims d, int rows,
                                                                        float* __restrict__ att, uint32_t* status) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + kQBytes;
    uint8_t* sV = sK + kKBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVBytes);
    uint64_t *k_ready = bars, *v_ready = bars + 1, *s_full = bars + 2, *s_free = bars + 3, *p_ready = bars + 4,
             *pv_done = bars + 5;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
    __shared__ int lim_s[kQ];
    __shared__ int kmax_s;
    const int G = d.n_heads / d.n_kv, RB = kQ / G;
    // heaviest (latest, longest causal) row blocks first
    const int r0 = (gridDim.x - 1 - blockIdx.x) * RB, kvh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < kQ) {  // query qi = r * G + g: row r0 + r, head kvh * G + g
        const int row = r0 + threadIdx.x / G;
        lim_s[threadIdx.x] = row < rows ? runs[row_off[row]].end : 0;
    }
    if (threadIdx.x == 0) {
        mbar_init(k_ready, 128);
        mbar_init(v_ready, 128);
        mbar_init(s_full, 1);
        mbar_init(s_free, 128);
        mbar_init(p_ready, 128);
        mbar_init(pv_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        int km = 0;
        for (int i = 0; i < kQ; ++i) km = max(km, lim_s[i]);
        kmax_s = km;
    }
    __syncthreads();
    const uint32_t tmem = *tslot;
    const int nblk = (kmax_s + kKB - 1) / kKB;
    const float* kbase = kc + static_cast<size_t>(kvh) * d.max_len * kHD;
    const float* vbase = vc + static_cast<size_t>(kvh) * d.max_len * kHD;

    if (warp >= 4 && warp < 8) {
        // ── producer: Q once, then K / V^T pieces per block ──────────────
        const int pt = threadIdx.x - 128;
        for (int i = 0; i < 32; ++i) {  // 128 queries x 32 float4
            const int f = pt + 128 * i, qi = f >> 5, c = f & 31, row = r0 + qi / G, g = qi % G;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < rows)
                x = __ldg(reinterpret_cast<const float4*>(q + static_cast<size_t>(row) * d.qd +
                                                           static_cast<size_t>(kvh * G + g) * kHD) + c);
            put3x4(sQ, 32768, 16384, qi, 4 * c, x.x, x.y, x.z, x.w);
        }
        for (int b = 0; b < nblk; ++b) {
            const int k0 = b * kKB, nk = min(kKB, kmax_s - k0);
            float4 kx[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {  // 64 keys x 32 float4
                const int f = pt + 128 * i, r = f >> 5, c = f & 31;
                kx[i] = r < nk ? __ldg(reinterpret_cast<const float4*>(kbase + static_cast<size_t>(k0 + r) * kHD) + c)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            // V^T: this thread's dim = pt, keys 4j..4j+3 (lanes read consecutive dims: coalesced)
            float vx[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) vx[j] = j < nk ? __ldg(vbase + static_cast<size_t>(k0 + j) * kHD + pt) : 0.0f;
            if (b > 0) bwait(s_full, static_cast<uint32_t>((b - 1) & 1));  // S_{b-1} has consumed K
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int f = pt + 128 * i;
                put3x4(sK, 16384, 8192, f >> 5, 4 * (f & 31), kx[i].x, kx[i].y, kx[i].z, kx[i].w);
            }
            fence_proxy_async();
            mbar_arrive(k_ready);
            if (b > 0) bwait(pv_done, static_cast<uint32_t>((b - 1) & 1));  // PV_{b-1} has consumed V
#pragma unroll
            for (int j = 0; j < 64; j += 4) put3x4(sV, 16384, 0, pt, j, vx[j], vx[j + 1], vx[j + 2], vx[j + 3]);
            fence_proxy_async();
            mbar_arrive(v_ready);
        }
    } else if (warp == 8) {
        // ── MMA issuer ───────────────────────────────────────────────────
        if (lane == 0) {
            const uint32_t aq = smem_u32(sQ), bk = smem_u32(sK), bv = smem_u32(sV);
            const uint32_t idS = idesc_mn(128, 64), idO = idesc_mn(128, 128);
            // piece pairs (a, b): hh hm mh hl mm lh
            const int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
            for (int b = 0; b < nblk; ++b) {
                bwait(k_ready, static_cast<uint32_t>(b & 1));
                if (b > 0) bwait(s_free, static_cast<uint32_t>((b - 1) & 1));
                tc_fence_after();
                for (int kb = 0; kb < 2; ++kb)
                    for (int ks = 0; ks < 4; ++ks)
                        for (int e = 0; e < 6; ++e) {
                            const uint64_t a = smem_desc(aq + pa[e] * 32768 + kb * 16384) + 2 * ks;
                            const uint64_t bb = smem_desc(bk + pb[e] * 16384 + kb * 8192) + 2 * ks;
                            mma_ss(tmem + kColS, a, bb, idS, (kb | ks | e) ? 1u : 0u);
                        }
                mma_commit(s_full);
                bwait(p_ready, static_cast<uint32_t>(b & 1));
                bwait(v_ready, static_cast<uint32_t>(b & 1));
                tc_fence_after();
                for (int ks = 0; ks < 4; ++ks)
                    for (int e = 0; e < 6; ++e) {
                        const uint64_t bb = smem_desc(bv + pb[e] * 16384) + 2 * ks;
                        mma_ts(tmem + kColO, tmem + kColP + pa[e] * 32 + 8 * ks, bb, idO, (b | ks | e) ? 1u : 0u);
                    }
                mma_commit(pv_done);
            }
        }
    } else if (warp < 4) {
        // ── softmax + output: thread = query = TMEM lane ─────────────────
        const int qi = threadIdx.x;
        const int lim = lim_s[qi];
        const uint32_t lb = static_cast<uint32_t>(warp * 32) << 16;
        const float scale = 1.0f / sqrtf(static_cast<float>(kHD));
        float m = -INFINITY, l = 0.0f;
        for (int b = 0; b < nblk; ++b) {
            const int k0 = b * kKB;
            bwait(s_full, static_cast<uint32_t>(b & 1));
            tc_fence_after();
            uint32_t sr[2][32];
            tmem_ld32(tmem + lb + kColS, sr[0]);
            tmem_ld32(tmem + lb + kColS + 32, sr[1]);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(s_free);
            float s[64];
            float mb = -INFINITY;
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                s[j] = k0 + j < lim ? __uint_as_float(sr[j >> 5][j & 31]) * scale : -INFINITY;
                mb = fmaxf(mb, s[j]);
            }
            const float mn = fmaxf(m, mb);
            float rs = 0.0f;
            uint32_t ph[32], pm[32], pl[32];
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
                const float p0 = s[j] == -INFINITY ? 0.0f : expf(s[j] - mn);
                const float p1 = s[j + 1] == -INFINITY ? 0.0f : expf(s[j + 1] - mn);
                rs += p0 + p1;
                const Split3 a = split3(p0), c = split3(p1);
                ph[j >> 1] = pack2(a.h, c.h);
                pm[j >> 1] = pack2(a.m, c.m);
                pl[j >> 1] = pack2(a.l, c.l);
            }
            // PV_{b-1} must be done before P is overwritten and O rescaled
            if (b > 0) bwait(pv_done, static_cast<uint32_t>((b - 1) & 1));
            tc_fence_after();
            // rescale O rows whose max rose (tcgen05.ld / st are warp-collective:
            // the warp rescales together, alpha = 1 for the other lanes)
            const bool need = b > 0 && m != -INFINITY && mn > m;
            if (__any_sync(0xffffffffu, need)) {
                const float alpha = need ? expf(m - mn) : 1.0f;
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    uint32_t o[32];
                    tmem_ld32(tmem + lb + kColO + 32 * c4, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
                    tmem_st32(tmem + lb + kColO + 32 * c4, o);
                }
                l *= alpha;
            }
            tmem_st32(tmem + lb + kColP, ph);
            tmem_st32(tmem + lb + kColP + 32, pm);
            tmem_st32(tmem + lb + kColP + 64, pl);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_ready);
            l += rs;
            if (mn != -INFINITY) m = mn;
        }
        // output row
        const int row = r0 + qi / G, g = qi % G;
        if (nblk > 0) {
            bwait(pv_done, static_cast<uint32_t>((nblk - 1) & 1));
            tc_fence_after();
        }
        const bool ok = row < rows && l > 0.0f;
        if (row < rows && !(l > 0.0f)) atomicOr(status, ST_EMPTY_ROW);  // tinyformer.cpp:467-469
        float* dst = att + static_cast<size_t>(ok ? row : 0) * d.qd + static_cast<size_t>(kvh * G + g) * kHD;
        const float inv = ok ? 1.0f / l : 0.0f;
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {  // warp-collective loads, per-lane stores
            uint32_t o[32];
            tmem_ld32(tmem + lb + kColO + 32 * c4, o);
            tmem_wait_ld();
            if (ok)
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4*>(dst + 32 * c4 + j) =
                        make_float4(__uint_as_float(o[j]) * inv, __uint_as_float(o[j + 1]) * inv,
                                    __uint_as_float(o[j + 2]) * inv, __uint_as_float(o[j + 3]) * inv);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_free(tmem, 512);
    }
}

}  // namespace

// Tensor-core prompt attention: head_dim 128, GQA group dividing 128.
// SFG_PROMPT_ATTN=cuda forces the CUDA-core attn_prompt_kernel (A/B knob).
bool attention_prompt_tc_supported(const Dims& d) {
    static const bool off = [] {
        const char* v = getenv("SFG_PROMPT_ATTN");
        return v && std::strcmp(v, "cuda") == 0;
    }();
    const int G = d.n_heads / d.n_kv;
    return !off && d.hd == kHD && (G == 1 || G == 2 || G == 4 || G == 8);
}

int launch_attention_prompt_tc(const float* q, const float* kcache, const float* vcache, const int32_t* row_off,
                               const MaskRun* runs, int rows, const Dims& d, float* att, uint32_t* status,
                               cudaStream_t s) {
    ensure_smem_attr(reinterpret_cast<const void*>(attn_prompt_tc_kernel), kSmemTC);
    const int rb = kQ / (d.n_heads / d.n_kv);
    const dim3 grid((rows + rb - 1) / rb, d.n_kv);
    attn_prompt_tc_kernel<<<grid, kThreadsTC, kSmemTC, s>>>(q, kcache, vcache, row_off, runs, d, rows, att, status);
    return 1;
}

}  // namespace sfg
