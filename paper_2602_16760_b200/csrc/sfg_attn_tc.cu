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
// The fp32 queries and KV cache are split ONCE per layer by split_q_kernel /
// split_kv_kernel into bf16 pieces already in the MMA's SW128 K-major tile
// layout (Q [kv head][query block][piece][k-block][128 x 128 B], K [kv head][key
// block][piece][k-block][64 x 128 B], V^T [kv head][key block][piece][128 dims x
// 128 B]); the attention CTAs fetch them with one bulk copy per operand block
// (the ~32 query blocks reading a key block no longer re-split it).
// Warp roles (192 threads, one CTA per SM: 192 KB of shared memory, 512 TMEM
// columns):
//   warps 0-3  softmax + output: thread = query = TMEM lane;
//   warp 4     producer (one thread): bulk copies of Q once, then K / V^T per block;
//   warp 5     MMA issuer (one thread).
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
constexpr int kKeyBlk = 64;       // keys per block
constexpr int kThreadsTC = 192;
// shared memory: Q pieces 3 x [2 k-blocks][128 rows][128 B] | K pieces 3 x [2][64][128 B] | V^T pieces 3 x [128 dims][128 B]
constexpr int kQBytes = 3 * 2 * 128 * 128;  // 96 KB
constexpr int kKBytes = 3 * 2 * 64 * 128;   // 48 KB
constexpr int kVBytes = 3 * 128 * 128;      // 48 KB
constexpr int kSmemTC = 1024 + kQBytes + kKBytes + kVBytes + 256;
// TMEM columns
constexpr uint32_t kColS = 0;    // S [128 q][64 keys] fp32, two buffers (block parity): columns 0 / 64
constexpr uint32_t kColP = 128;  // P pieces 3 x 32 columns (bf16 pairs)
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

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
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

// the queries / K / V^T as bf16 pieces in the MMA tile layout (see the header)
__global__ void split_q_kernel(const float* __restrict__ q, Dims d, int rows, int nqb, uint8_t* __restrict__ Qp) {
    const int G = d.n_heads / d.n_kv, RB = kQ / G;
    const size_t n = static_cast<size_t>(d.n_kv) * nqb * kQ * 32;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i & 31), qi = static_cast<int>((i >> 5) % kQ);
        const size_t hb = i / (32 * kQ);  // kv head * nqb + query block
        const int qb = static_cast<int>(hb % nqb), h = static_cast<int>(hb / nqb);
        const int row = qb * RB + qi / G, g = qi % G;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < rows)
            x = __ldg(reinterpret_cast<const float4*>(q + static_cast<size_t>(row) * d.qd + static_cast<size_t>(h * G + g) * kHD) + c);
        put3x4(Qp + hb * kQBytes, 32768, 16384, qi, 4 * c, x.x, x.y, x.z, x.w);
    }
}
__global__ void split_kv_kernel(const float* __restrict__ kc, const float* __restrict__ vc, Dims d, int keys, int nkb,
                                uint8_t* __restrict__ Kp, uint8_t* __restrict__ Vp) {
    const size_t n = static_cast<size_t>(d.n_kv) * nkb * kKeyBlk * 32;  // per head: nkb*64 keys x 32 float4 (K); same count of V quads
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        {  // K: key j, dims 4c..4c+3
            const int c = static_cast<int>(i & 31);
            const size_t hj = i >> 5;
            const int j = static_cast<int>(hj % (static_cast<size_t>(nkb) * kKeyBlk)), h = static_cast<int>(hj / (static_cast<size_t>(nkb) * kKeyBlk));
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (j < keys) x = __ldg(reinterpret_cast<const float4*>(kc + (static_cast<size_t>(h) * d.max_len + j) * kHD) + c);
            put3x4(Kp + (static_cast<size_t>(h) * nkb + j / kKeyBlk) * kKBytes, 16384, 8192, j % kKeyBlk, 4 * c, x.x, x.y, x.z, x.w);
        }
        {  // V^T: dim dd, keys 4jq..4jq+3 (consecutive threads: consecutive dims, coalesced loads)
            const int dd = static_cast<int>(i % kHD);
            const size_t hq = i / kHD;
            const int jq = static_cast<int>(hq % (static_cast<size_t>(nkb) * kKeyBlk / 4)), h = static_cast<int>(hq / (static_cast<size_t>(nkb) * kKeyBlk / 4));
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = 4 * jq + u;
                v[u] = j < keys ? __ldg(vc + (static_cast<size_t>(h) * d.max_len + j) * kHD + dd) : 0.0f;
            }
            put3x4(Vp + (static_cast<size_t>(h) * nkb + (4 * jq) / kKeyBlk) * kVBytes, 16384, 0, dd, (4 * jq) % kKeyBlk, v[0], v[1], v[2], v[3]);
        }
    }
}

__global__ void __launch_bounds__(kThreadsTC, 1) attn_prompt_tc_kernel(const uint8_t* __restrict__ Qp,
                                                                        const uint8_t* __restrict__ Kp,
                                                                        const uint8_t* __restrict__ Vp, int nkb,
                                                                        const int32_t* __restrict__ row_off,
                                                                        const MaskRun* __restrict__ runs, Dims d, int rows,
                                                                        float* __restrict__ att, uint32_t* status) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + kQBytes;
    uint8_t* sV = sK + kKBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVBytes);
    // s_full / s_free: one pair per S buffer (block parity), so no waiter can
    // ever be two phases behind its barrier
    uint64_t *k_ready = bars, *v_ready = bars + 1, *s_full = bars + 2, *s_free = bars + 4, *p_ready = bars + 6,
             *pv_done = bars + 7;
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
        mbar_init(k_ready, 1);
        mbar_init(v_ready, 1);
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        mbar_init(&s_free[0], 128);
        mbar_init(&s_free[1], 128);
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
    const int nblk = (kmax_s + kKeyBlk - 1) / kKeyBlk;

    if (warp == 4) {
        // ── producer: bulk copies of the pre-split operand blocks ─────────
        if (lane == 0) {
            const uint8_t* qsrc = Qp + (static_cast<size_t>(kvh) * gridDim.x + (gridDim.x - 1 - blockIdx.x)) * kQBytes;
            for (int b = 0; b < nblk; ++b) {
                if (b > 0) bwait(&s_full[(b - 1) & 1], static_cast<uint32_t>(((b - 1) >> 1) & 1));  // S_{b-1} has consumed K
                mbar_expect_tx(k_ready, (b == 0 ? kQBytes : 0) + kKBytes);
                if (b == 0) bulk_g2s(sQ, qsrc, kQBytes, k_ready);
                bulk_g2s(sK, Kp + (static_cast<size_t>(kvh) * nkb + b) * kKBytes, kKBytes, k_ready);
                if (b > 0) bwait(pv_done, static_cast<uint32_t>((b - 1) & 1));  // PV_{b-1} has consumed V
                mbar_expect_tx(v_ready, kVBytes);
                bulk_g2s(sV, Vp + (static_cast<size_t>(kvh) * nkb + b) * kVBytes, kVBytes, v_ready);
            }
        }
    } else if (warp == 5) {
        // ── MMA issuer ───────────────────────────────────────────────────
        if (lane == 0) {
            const uint32_t aq = smem_u32(sQ), bk = smem_u32(sK), bv = smem_u32(sV);
            const uint32_t idS = idesc_mn(128, 64), idO = idesc_mn(128, 128);
            // piece pairs (a, b): hh hm mh hl mm lh
            const int pa[6] = {0, 0, 1, 0, 1, 2}, pb[6] = {0, 1, 0, 2, 1, 0};
            // software pipelined: S_{b+1} is issued before PV_b, so the tensor
            // pipe computes the next scores while the softmax warps work on block b
            auto issue_s = [&](int j) {
                bwait(k_ready, static_cast<uint32_t>(j & 1));
                if (j >= 2) bwait(&s_free[j & 1], static_cast<uint32_t>(((j - 2) >> 1) & 1));  // S_{j-2} read
                tc_fence_after();
                const uint32_t ds = tmem + kColS + 64 * (j & 1);
                for (int kb = 0; kb < 2; ++kb)
                    for (int ks = 0; ks < 4; ++ks)
                        for (int e = 0; e < 6; ++e) {
                            const uint64_t a = smem_desc(aq + pa[e] * 32768 + kb * 16384) + 2 * ks;
                            const uint64_t bb = smem_desc(bk + pb[e] * 16384 + kb * 8192) + 2 * ks;
                            mma_ss(ds, a, bb, idS, (kb | ks | e) ? 1u : 0u);
                        }
                mma_commit(&s_full[j & 1]);
            };
            if (nblk > 0) issue_s(0);
            for (int b = 0; b < nblk; ++b) {
                if (b + 1 < nblk) issue_s(b + 1);
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
        // scores live in the log2 domain: p = 2^(s * scale * log2(e) - m) (ex2.approx,
        // ~2^-22 relative), the same softmax as exp(s * scale - m')
        const float scale = 1.4426950408889634f / sqrtf(static_cast<float>(kHD));
        float m = -INFINITY, l = 0.0f;
        for (int b = 0; b < nblk; ++b) {
            const int k0 = b * kKeyBlk;
            bwait(&s_full[b & 1], static_cast<uint32_t>((b >> 1) & 1));
            tc_fence_after();
            uint32_t sr[2][32];
            tmem_ld32(tmem + lb + kColS + 64 * (b & 1), sr[0]);
            tmem_ld32(tmem + lb + kColS + 64 * (b & 1) + 32, sr[1]);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&s_free[b & 1]);
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
                const float p0 = s[j] == -INFINITY ? 0.0f : ex2(s[j] - mn);
                const float p1 = s[j + 1] == -INFINITY ? 0.0f : ex2(s[j + 1] - mn);
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
                const float alpha = need ? ex2(m - mn) : 1.0f;
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
                               const MaskRun* runs, int rows, int keys, const Dims& d, float* att, uint32_t* status,
                               cudaStream_t s, void** scratch, size_t* scratch_bytes) {
    const int G = d.n_heads / d.n_kv, rb = kQ / G;
    const int nqb = (rows + rb - 1) / rb, nkb = (keys + kKeyBlk - 1) / kKeyBlk;
    const size_t qb = static_cast<size_t>(d.n_kv) * nqb * kQBytes, kb = static_cast<size_t>(d.n_kv) * nkb * kKBytes;
    const size_t need = qb + 2 * kb;
    if (*scratch_bytes < need) {  // grow (rare): the previous user of the buffer must be done
        SFG_CUDA(cudaStreamSynchronize(s));
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        SFG_CUDA(cudaMalloc(scratch, need));
        *scratch_bytes = need;
    }
    uint8_t* Qp = static_cast<uint8_t*>(*scratch);
    uint8_t* Kp = Qp + qb;
    uint8_t* Vp = Kp + kb;
    const int nsm = device_sm_count();
    split_q_kernel<<<4 * nsm, 256, 0, s>>>(q, d, rows, nqb, Qp);
    split_kv_kernel<<<4 * nsm, 256, 0, s>>>(kcache, vcache, d, keys, nkb, Kp, Vp);
    ensure_smem_attr(reinterpret_cast<const void*>(attn_prompt_tc_kernel), kSmemTC);
    attn_prompt_tc_kernel<<<dim3(nqb, d.n_kv), kThreadsTC, kSmemTC, s>>>(Qp, Kp, Vp, nkb, row_off, runs, d, rows, att, status);
    return 3;
}

}  // namespace sfg
