// FAST-mode layer executor: weight-streaming skinny GEMMs on tcgen05 (sm_100a).
//
// Every projection of the lookahead step is Y[B x N] = X[B x K] . W[K x N]
// with B <= 16 token rows and N, K in the thousands — a dense contraction
// that is HBM-bound at ~16 flop/byte.  It runs "swap-AB" on the 5th-gen
// tensor core: D[128 features x 48] (TMEM, fp32) += W^T[128 x K] . Xs^T, where
// Xs stacks the fp32 activations as three bf16 pieces (hi | mid | lo, 16 rows
// each) so bf16 x bf16 products reconstruct ~fp32 activations exactly and
// only the weights are bf16 (their storage precision).
//
//   * weights are re-laid out once at load into the exact shared-memory image
//     of each [128 x 64] K-major SWIZZLE_128B stage (16 KB), so a stage is ONE
//     contiguous cp.async.bulk (TMA engine, UBLKCP) — no tensor maps;
//   * 8-stage smem ring, warp-specialised: warp 0 = bulk-copy producer, warp 1
//     = single-thread tcgen05.mma issuer, warps 2-5 = TMEM epilogue (two TMEM
//     accumulators so the epilogue of one tile overlaps the next);
//   * stream-K: the (tile, k-block) space is cut into gridDim.x (= #SMs)
//     contiguous equal ranges; tiles split between CTAs are finished by the
//     last arriving CTA, which sums the pieces in fixed k order — results are
//     deterministic and independent of B (batch invariance);
//   * epilogues fuse RoPE + KV-cache append (QKV), the residual add (O, down),
//     SiLU(gate)*up, and logits + per-tile argmax partials (LM head).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <initializer_list>
#include <string>
#include <type_traits>

#include "sfg_engine.h"
#include "sfg_expf.h"
#include "sfg_prof.h"

namespace sfg {
namespace fast {

constexpr int kRows = 16;            // token rows per pass
constexpr int kN = 3 * kRows;        // MMA N: hi | mid | lo
constexpr int kM = 128;              // output features per tile (MMA M)
constexpr int kKB = 64;              // K per stage: one 128-byte swizzle row of bf16
constexpr int kStages = 8;
constexpr int kABytes = kM * kKB * 2;  // 16 KB
constexpr int kBBytes = kN * kKB * 2;  // 6 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;
constexpr int kAccCols = 64;           // TMEM columns per accumulator (48 used)
constexpr int kTmemCols = 128;         // two accumulators
constexpr int kMaxPieces = 16;
// Prompt passes: one launch feeds each weight stage to NC 16-row chunks (NC
// accumulators of N = 48 in TMEM), so a prompt streams the weights once per
// NC chunks instead of once per chunk.  Each chunk's MMAs and k order are
// those of the one-chunk kernel, so results are bitwise the same.
constexpr int kPromptChunks = 5;
template <int NC> constexpr int stage_bytes() { return kABytes + NC * kBBytes; }
template <int NC> constexpr int n_stages() { return NC == 1 ? kStages : (200 * 1024) / stage_bytes<NC>(); }
template <int NC> constexpr int acc_cols() { return NC == 1 ? kAccCols : 256; }
template <int NC> constexpr int tmem_cols() { return 2 * acc_cols<NC>(); }
static_assert(kPromptChunks * kN <= 256, "prompt chunks must fit one 256-column accumulator");

enum Epi : int { EPI_RESID = 0, EPI_QKV = 1, EPI_GATEUP = 2, EPI_HEAD = 3 };

struct GemmArgs {
    const uint8_t* W;   // tiled, swizzled [tiles][KB][kABytes]
    const uint8_t* X;   // swizzled [KB][kBBytes]
    int tiles, KB;
    int n_out;          // real output features (EPI_GATEUP: F, gate/up pairs)
    float* partials;    // [tiles][kMaxPieces][kRows][kM]
    int* counters;      // [tiles]
    int rows, row0;     // valid rows of this pass, global row offset
    // EPI_RESID: out[(row0+r)*ld + f] += y   (store_only: = y, a tensor-parallel
    // rank's partial that the all-reduce adds to rank 0's h + partial)
    int store_only;
    // EPI_GATEUP: out[(row0+r)*ld + f] = silu(g)*u
    // EPI_HEAD: out (nullable) logits [(row0+r)*ld + f]
    float* out;
    int ld;
    // EPI_QKV
    int qd, kvd, hd, max_len;
    const int32_t* prior;  // device: cache length before this batch
    const int32_t* pos;
    const float* rope_cos;
    const float* rope_sin;
    float* kc;
    float* vc;
    // EPI_HEAD
    float* amax_val;    // [rows_total][tiles]
    int32_t* amax_idx;
    // multi-chunk launches: chunk j >= 1 reads X2 + (j-1)*KB*kBBytes and keeps its
    // stream-K partials / counters at partials2 + (j-1)*tiles*kMaxPieces*kRows*kM,
    // counters2 + (j-1)*tiles
    const uint8_t* X2;
    float* partials2;
    int* counters2;
};

// ── PTX wrappers ──────────────────────────────────────────────────────────
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
    d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm100)
    d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M x N.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kN >> 3) << 17) |
                            (static_cast<uint32_t>(kM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Byte offset of element (row, kk) inside a [rows x 64] K-major SW128 tile.
__host__ __device__ __forceinline__ uint32_t sw128_off(int row, int kk) {
    return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + (((kk >> 3) ^ (row & 7)) << 4) + (kk & 7) * 2);
}

// ── epilogues ─────────────────────────────────────────────────────────────
// Thread = one output feature m of the tile (TMEM lane); y[r] for r < 16.
template <int EPI>
__device__ __forceinline__ void final_epilogue(const GemmArgs& a, int tile, int m, const float (&y)[kRows],
                                               float* xch) {
    const int f = tile * kM + m;
    if constexpr (EPI == EPI_RESID) {
        if (f < a.n_out)
#pragma unroll
            for (int r = 0; r < kRows; ++r)
                if (r < a.rows) {
                    float* o = a.out + static_cast<size_t>(a.row0 + r) * a.ld + f;
                    *o = a.store_only ? y[r] : *o + y[r];
                }
    } else if constexpr (EPI == EPI_QKV) {
        // features: [0,qd) q | [qd, qd+kvd) k | [qd+kvd, qd+2kvd) v; RoPE pairs
        // (2i, 2i+1) sit on adjacent lanes of the same warp.
        const bool valid = f < a.qd + 2 * a.kvd;
        const int seg = f < a.qd ? 0 : (f < a.qd + a.kvd ? 1 : 2);
        const int fl = seg == 0 ? f : (seg == 1 ? f - a.qd : f - a.qd - a.kvd);
        const int d = fl % a.hd, half = a.hd >> 1, i = d >> 1;
        const bool odd = (m & 1) != 0;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const float partner = __shfl_xor_sync(0xffffffffu, y[r], 1);
            if (!valid || r >= a.rows) continue;
            float v = y[r];
            const int row = a.row0 + r;
            if (seg != 2) {
                const int p = a.pos[row];
                const float c = a.rope_cos[static_cast<size_t>(p) * half + i];
                const float s = a.rope_sin[static_cast<size_t>(p) * half + i];
                v = odd ? __fadd_rn(__fmul_rn(partner, s), __fmul_rn(v, c))
                        : __fsub_rn(__fmul_rn(v, c), __fmul_rn(partner, s));
            }
            if (seg == 0) {
                a.out[static_cast<size_t>(row) * a.qd + fl] = v;
            } else {
                const int kvh = fl / a.hd;
                float* dst = (seg == 1 ? a.kc : a.vc) +
                             (static_cast<size_t>(kvh) * a.max_len + *a.prior + row) * a.hd + d;
                *dst = v;
            }
        }
    } else if constexpr (EPI == EPI_GATEUP) {
        // tile rows 0-63: gate features, 64-127: the matching up features
        float* ub = xch;  // [64][kRows]
        if (m >= 64)
            for (int r = 0; r < kRows; ++r) ub[(m - 64) * kRows + r] = y[r];
        named_sync(1, 128);
        if (m < 64) {
            const int fg = tile * 64 + m;
            if (fg < a.n_out)
#pragma unroll
                for (int r = 0; r < kRows; ++r)
                    if (r < a.rows) {
                        const float g = y[r];
                        const float silu = __fdiv_rn(g, __fadd_rn(1.0f, sfg_expf(-g)));
                        a.out[static_cast<size_t>(a.row0 + r) * a.ld + fg] = __fmul_rn(silu, ub[m * kRows + r]);
                    }
        }
        named_sync(1, 128);
    } else {  // EPI_HEAD: logits + (max, argmax) per row over this tile
        float* sv = xch;                                    // [4][kRows]
        int* si = reinterpret_cast<int*>(xch + 4 * kRows);  // [4][kRows]
        const int wq = (threadIdx.x >> 5) & 3;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            float v = f < a.n_out ? y[r] : -INFINITY;
            int idx = f < a.n_out ? f : 0x7fffffff;
            if (a.out && f < a.n_out && r < a.rows) a.out[static_cast<size_t>(a.row0 + r) * a.ld + f] = y[r];
            for (int o = 16; o > 0; o >>= 1) {
                const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
                if (v2 > v || (v2 == v && i2 < idx)) {
                    v = v2;
                    idx = i2;
                }
            }
            if ((threadIdx.x & 31) == 0) {
                sv[wq * kRows + r] = v;
                si[wq * kRows + r] = idx;
            }
        }
        named_sync(1, 128);
        if (m < a.rows) {
            const int r = m;
            float v = sv[r];
            int idx = si[r];
            for (int w = 1; w < 4; ++w) {
                const float v2 = sv[w * kRows + r];
                const int i2 = si[w * kRows + r];
                if (v2 > v || (v2 == v && i2 < idx)) {
                    v = v2;
                    idx = i2;
                }
            }
            a.amax_val[static_cast<size_t>(a.row0 + r) * a.tiles + tile] = v;
            a.amax_idx[static_cast<size_t>(a.row0 + r) * a.tiles + tile] = idx;
        }
        named_sync(1, 128);
    }
}

// ── the kernel ────────────────────────────────────────────────────────────
// One accumulated piece [lo, hi) of tile t for one 16-row chunk: a whole tile
// goes straight to the epilogue; a split tile deposits its partial and the
// last arriver reduces the pieces in k order.
template <int EPI>
__device__ __forceinline__ void finish_piece(const GemmArgs& a, int t, int lo, int hi, const float (&y)[kRows],
                                             float* xch, int* flag, int G, long long U, int c, int m, int et) {
    if (lo == 0 && hi == a.KB) {
        final_epilogue<EPI>(a, t, m, y, xch);
        return;
    }
    const long long first_u = static_cast<long long>(t) * a.KB;
    const int c_first = static_cast<int>(((first_u + 1) * G - 1) / U);
    const int piece = c - c_first;
    const long long last_u = first_u + a.KB - 1;
    const int n_pieces = static_cast<int>(((last_u + 1) * G - 1) / U) - c_first + 1;
    float* slot = a.partials + (static_cast<size_t>(t) * kMaxPieces + piece) * kRows * kM;
#pragma unroll
    for (int r = 0; r < kRows; ++r) slot[r * kM + m] = y[r];
    __threadfence();
    named_sync(1, 128);
    if (et == 0) {
        const int old = atomicAdd(&a.counters[t], 1);
        *flag = (old == n_pieces - 1) ? 1 : 0;
        if (old == n_pieces - 1) a.counters[t] = 0;  // reset for the next launch
    }
    named_sync(1, 128);
    if (*flag) {
        __threadfence();
        float s[kRows];
        const float* p0 = a.partials + static_cast<size_t>(t) * kMaxPieces * kRows * kM;
#pragma unroll
        for (int r = 0; r < kRows; ++r) s[r] = __ldcg(p0 + r * kM + m);
        for (int p = 1; p < n_pieces; ++p)
#pragma unroll
            for (int r = 0; r < kRows; ++r) s[r] = s[r] + __ldcg(p0 + (static_cast<size_t>(p) * kRows + r) * kM + m);
        final_epilogue<EPI>(a, t, m, s, xch);
    }
    named_sync(1, 128);
}

template <int EPI, int NC = 1>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmArgs a) {
    constexpr int kSt = n_stages<NC>(), kSB = stage_bytes<NC>(), kAcc = acc_cols<NC>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kSB);
    uint64_t* empty = full + kSt;
    uint64_t* tfull = empty + kSt;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* flag = reinterpret_cast<int*>(tmem_slot + 4);
    float* xch = reinterpret_cast<float*>(flag + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSt; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tmem_cols<NC>())
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const long long U = static_cast<long long>(a.tiles) * a.KB;
    const int G = gridDim.x, c = blockIdx.x;
    const long long start = c * U / G, end = (c + 1) * U / G;

    if (warp == 0) {
        if (lane == 0) {  // ── producer: bulk copies into the smem ring
            int stage = 0;
            uint32_t phase = 0;
            for (long long u = start; u < end;) {
                const int t = static_cast<int>(u / a.KB);
                const int lo = static_cast<int>(u - static_cast<long long>(t) * a.KB);
                const int hi = static_cast<int>(min(end - static_cast<long long>(t) * a.KB, static_cast<long long>(a.KB)));
                for (int kb = lo; kb < hi; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * kSB;
                    mbar_expect_tx(&full[stage], kSB);
                    bulk_g2s(sa, a.W + (static_cast<size_t>(t) * a.KB + kb) * kABytes, kABytes, &full[stage]);
                    bulk_g2s(sa + kABytes, a.X + static_cast<size_t>(kb) * kBBytes, kBBytes, &full[stage]);
#pragma unroll
                    for (int j = 1; j < NC; ++j)
                        bulk_g2s(sa + kABytes + j * kBBytes,
                                 a.X2 + (static_cast<size_t>(j - 1) * a.KB + kb) * kBBytes, kBBytes, &full[stage]);
                    if (++stage == kSt) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                u = static_cast<long long>(t) * a.KB + hi;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ── MMA issuer
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (long long u = start; u < end;) {
                const int t = static_cast<int>(u / a.KB);
                const int lo = static_cast<int>(u - static_cast<long long>(t) * a.KB);
                const int hi = static_cast<int>(min(end - static_cast<long long>(t) * a.KB, static_cast<long long>(a.KB)));
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * kAcc;
                for (int kb = lo; kb < hi; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * kSB);
                    const uint64_t da = smem_desc(sa);
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        const uint64_t db = smem_desc(sa + kABytes + j * kBBytes);
#pragma unroll
                        for (int k = 0; k < kKB / 16; ++k)  // +32 bytes per K=16 step inside the swizzle row
                            mma_bf16(d + j * kN, da + 2 * k, db + 2 * k, (kb > lo || k > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == kSt) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                u = static_cast<long long>(t) * a.KB + hi;
            }
        }
    } else {  // ── epilogue warps 2..5 (TMEM lane quadrant = warp % 4)
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const int et = threadIdx.x - 64;  // 0..127
        int acc = 0;
        uint32_t acc_phase = 0;
        for (long long u = start; u < end;) {
            const int t = static_cast<int>(u / a.KB);
            const int lo = static_cast<int>(u - static_cast<long long>(t) * a.KB);
            const int hi = static_cast<int>(min(end - static_cast<long long>(t) * a.KB, static_cast<long long>(a.KB)));
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * kAcc;
            if constexpr (NC == 1) {
                float v[kN];
                tmem_ld16(ta, v);
                tmem_ld16(ta + 16, v + 16);
                tmem_ld16(ta + 32, v + 32);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                float y[kRows];
#pragma unroll
                for (int r = 0; r < kRows; ++r) y[r] = (v[r] + v[kRows + r]) + v[2 * kRows + r];
                finish_piece<EPI>(a, t, lo, hi, y, xch, flag, G, U, c, m, et);
            } else {
                for (int j = 0; j < NC; ++j) {
                    float v[kN];
                    tmem_ld16(ta + j * kN, v);
                    tmem_ld16(ta + j * kN + 16, v + 16);
                    tmem_ld16(ta + j * kN + 32, v + 32);
                    tmem_wait_ld();
                    if (j == NC - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[acc]);
                    }
                    if (j * kRows >= a.rows) continue;  // uniform: no valid row in this chunk
                    float y[kRows];
#pragma unroll
                    for (int r = 0; r < kRows; ++r) y[r] = (v[r] + v[kRows + r]) + v[2 * kRows + r];
                    if (j == 0) {
                        GemmArgs ac = a;
                        ac.rows = min(kRows, a.rows);
                        finish_piece<EPI>(ac, t, lo, hi, y, xch, flag, G, U, c, m, et);
                    } else {
                        GemmArgs ac = a;
                        ac.rows = min(kRows, a.rows - j * kRows);
                        ac.row0 = a.row0 + j * kRows;
                        ac.partials = a.partials2 + static_cast<size_t>(j - 1) * a.tiles * kMaxPieces * kRows * kM;
                        ac.counters = a.counters2 + static_cast<size_t>(j - 1) * a.tiles;
                        finish_piece<EPI>(ac, t, lo, hi, y, xch, flag, G, U, c, m, et);
                    }
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
            u = static_cast<long long>(t) * a.KB + hi;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols<NC>())
                     : "memory");
    }
}

// ── prompt GEMM: (weight tile x 128-token tile) items, whole K, no split-K ──
// A prompt of P tokens has P/128 token tiles; every (weight tile t, token tile
// j) item is one CTA that streams the tile's weights (16 KB per k-block, L2
// hits for all but the first of the tile's P/128 items, which run side by
// side) against the token tile's activation image and accumulates D[128
// features x 128 tokens] in TMEM: per k-block and K=16 step, the hi, mid and
// lo bf16 pieces of the activations are three N = 128 MMAs into the SAME
// accumulator (fixed order hi, mid, lo) — so a 2048-token prompt reads each
// weight byte from HBM once instead of 26 times, runs N = 128 MMAs instead of
// N = 48 ones, and needs no stream-K fixups.  Results differ from the decode
// kernels only in summation order (deterministic; FAST tolerance vs the
// reference, tests/test_gpu_fast.py, test_gpu_long_context.py).
constexpr int kPT = 128;                     // tokens per tile (MMA N)
constexpr int kPBBytes = kPT * kKB * 2;      // one piece of a k-block: 16 KB
constexpr int kPTiles = 2;                   // weight tiles per item: they share every activation stage
constexpr int kPStage = kPTiles * kABytes + 3 * kPBBytes;  // 80 KB
constexpr int kPStages = 2;
constexpr uint32_t kPIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kPT >> 3) << 17) |
                             (static_cast<uint32_t>(kM >> 4) << 24);
constexpr size_t pgemm_smem_bytes() { return 1024 + static_cast<size_t>(kPStages) * kPStage + 2 * kPStages * 8 + 4 * 8 + 16 + (64 * kRows + 8 * kRows) * 4; }

struct PgArgs {
    GemmArgs g;           // weights, tiles, KB, n_out and the epilogue operands (row0/rows set per block)
    int tpi;              // weight tiles per item (1 or kPTiles): 2 when there are enough items to fill the SMs
    const uint8_t* X;     // [TT][KB][3][kPT x 64] bf16 SW128 (hi | mid | lo)
    int TT;               // token tiles
    int total_rows;       // prompt rows of this pass
};

__device__ __forceinline__ void mma_bf16_n128(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kPIdesc), "r"(accum)
        : "memory");
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1) pgemm_kernel(const __grid_constant__ PgArgs pa) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPStages * kPStage);
    uint64_t* empty = full + kPStages;
    uint64_t* tfull = empty + kPStages;   // [2] accumulator ready
    uint64_t* tempty = tfull + 2;         // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* xch = reinterpret_cast<float*>(tmem_slot + 4);
    const GemmArgs& a = pa.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent: item i = (weight tile pair i / TT, token tile i % TT); items
    // of one CTA alternate between two TMEM accumulators so one item's
    // epilogue overlaps the next item's MMAs
    const int tpi = pa.tpi;
    const int items = ((a.tiles + tpi - 1) / tpi) * pa.TT;
    constexpr uint32_t kAccW = kPTiles * kPT;  // TMEM columns per accumulator
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * kAccW)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {  // ── producer
            int stage = 0;
            uint32_t phase = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                const int t0 = (it / pa.TT) * tpi, j = it % pa.TT, nt = min(tpi, a.tiles - t0);
                for (int kb = 0; kb < a.KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * kPStage;
                    mbar_expect_tx(&full[stage], nt * kABytes + 3 * kPBBytes);
                    for (int i = 0; i < nt; ++i)
                        bulk_g2s(sa + i * kABytes, a.W + (static_cast<size_t>(t0 + i) * a.KB + kb) * kABytes, kABytes,
                                 &full[stage]);
                    bulk_g2s(sa + kPTiles * kABytes, pa.X + (static_cast<size_t>(j) * a.KB + kb) * 3 * kPBBytes,
                             3 * kPBBytes, &full[stage]);
                    if (++stage == kPStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ── MMA issuer: hi, mid, lo into one accumulator per K=16 step
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_ph = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                const int t0 = (it / pa.TT) * tpi, nt = min(tpi, a.tiles - t0);
                mbar_wait(&tempty[acc], acc_ph ^ 1);
                tc_fence_after();
                const uint32_t d0 = tmem + acc * kAccW;
                for (int kb = 0; kb < a.KB; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * kPStage);
#pragma unroll
                    for (int i = 0; i < kPTiles; ++i) {
                        if (i >= nt) break;
                        const uint64_t da = smem_desc(sa + i * kABytes);
#pragma unroll
                        for (int k = 0; k < kKB / 16; ++k)
#pragma unroll
                            for (int pc = 0; pc < 3; ++pc)
                                mma_bf16_n128(d0 + i * kPT, da + 2 * k,
                                              smem_desc(sa + kPTiles * kABytes + pc * kPBBytes) + 2 * k,
                                              (kb > 0 || k > 0 || pc > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);
                    if (++stage == kPStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_ph ^= 1;
                }
            }
        }
    } else {  // ── epilogue: 16-token blocks of the tile through the decode epilogues
        const int q = warp & 3;
        const int m = q * 32 + lane;
        int acc = 0;
        uint32_t acc_ph = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            const int t0 = (it / pa.TT) * tpi, j = it % pa.TT, nt = min(tpi, a.tiles - t0);
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            for (int i = 0; i < nt; ++i) {
                const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * kAccW + i * kPT;
                for (int b = 0; b < kPT / kRows; ++b) {
                    const int row0 = j * kPT + b * kRows;
                    if (row0 >= pa.total_rows) break;  // uniform over the epilogue warps
                    float y[kRows];
                    tmem_ld16(ta + b * kRows, y);
                    tmem_wait_ld();
                    GemmArgs ab = a;
                    ab.row0 = a.row0 + row0;
                    ab.rows = min(kRows, pa.total_rows - row0);
                    final_epilogue<EPI>(ab, t0 + i, m, y, xch);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_ph ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccW) : "memory");
    }
}

// [RMSNorm] + 3-way split of prompt rows into the token-tiled image: one CTA
// per row (rows beyond `rows` of the last tile are written as zeros).
__global__ void __launch_bounds__(256) pprep_kernel(const float* __restrict__ x, int ldx, int K, int rows,
                                                    const float* __restrict__ gain, float eps,
                                                    uint8_t* __restrict__ xs) {
    const int row = blockIdx.x, j = row / kPT, r = row % kPT, KB = K / kKB;
    const bool live = row < rows;
    const float* xr = x + static_cast<size_t>(live ? row : 0) * ldx;
    float scale = 1.0f;
    if (gain && live) {
        __shared__ float red[8];
        float ss = 0.0f;
        for (int i = threadIdx.x; i < K; i += 256) ss += xr[i] * xr[i];
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
            float tt = 0.0f;
            for (int w = 0; w < 8; ++w) tt += red[w];
            red[0] = 1.0f / sqrtf(tt / static_cast<float>(K) + eps);
        }
        __syncthreads();
        scale = red[0];
    }
    for (int k8 = threadIdx.x * 8; k8 < K; k8 += 256 * 8) {
        __align__(16) __nv_bfloat16 hi[8], mid[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float v = live ? xr[k8 + e] : 0.0f;
            if (gain) v = (v * scale) * gain[k8 + e];
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            const float r1 = v - __bfloat162float(h);
            const __nv_bfloat16 mm = __float2bfloat16_rn(r1);
            hi[e] = h;
            mid[e] = mm;
            lo[e] = __float2bfloat16_rn(r1 - __bfloat162float(mm));
        }
        const int kb = k8 / kKB, kk = k8 % kKB;
        uint8_t* base = xs + (static_cast<size_t>(j) * KB + kb) * 3 * kPBBytes;
        *reinterpret_cast<uint4*>(base + sw128_off(r, kk)) = *reinterpret_cast<uint4*>(hi);
        *reinterpret_cast<uint4*>(base + kPBBytes + sw128_off(r, kk)) = *reinterpret_cast<uint4*>(mid);
        *reinterpret_cast<uint4*>(base + 2 * kPBBytes + sw128_off(r, kk)) = *reinterpret_cast<uint4*>(lo);
    }
}

template <int EPI>
void launch_pgemm(const PgArgs& pa, cudaStream_t s) {
    ensure_smem_attr(reinterpret_cast<const void*>(pgemm_kernel<EPI>), pgemm_smem_bytes());
    PgArgs p = pa;
    const int nsm = device_sm_count();
    // two weight tiles per item when that still leaves >= one item per SM
    p.tpi = ((pa.g.tiles + kPTiles - 1) / kPTiles) * pa.TT >= nsm ? kPTiles : 1;
    const int items = ((pa.g.tiles + p.tpi - 1) / p.tpi) * pa.TT;
    pgemm_kernel<EPI><<<std::min(items, nsm), kThreads, pgemm_smem_bytes(), s>>>(p);
}

// ── activation prologue: [RMSNorm] + 3-way bf16 split into the swizzled B image
// One CTA per row of the pass; rows beyond `rows` keep stale values, which
// only feed their own (ignored) MMA columns.
constexpr int kPrepThreads = 256;
__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const float* __restrict__ x, int ldx, int K,
                                                            const float* __restrict__ gain, float eps,
                                                            uint8_t* __restrict__ xs,
                                                            uint8_t* __restrict__ xs2 = nullptr,
                                                            size_t chunk_bytes = 0) {
    // block b = row b of the pass; rows 16j.. go to chunk j's image (prompt passes)
    const int b = blockIdx.x, chunk = b / kRows, r = b % kRows;
    const float* xr = x + static_cast<size_t>(b) * ldx;
    if (chunk > 0) xs = xs2 + static_cast<size_t>(chunk - 1) * chunk_bytes;
    float scale = 1.0f;
    if (gain) {
        __shared__ float red[kPrepThreads / 32];
        float ss = 0.0f;
        for (int i = threadIdx.x; i < K; i += kPrepThreads) ss += xr[i] * xr[i];
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
            float t = 0.0f;
            for (int w = 0; w < kPrepThreads / 32; ++w) t += red[w];
            red[0] = 1.0f / sqrtf(t / static_cast<float>(K) + eps);
        }
        __syncthreads();
        scale = red[0];
    }
    // each thread handles 8 consecutive k (one 16-byte chunk per piece)
    for (int k8 = threadIdx.x * 8; k8 < K; k8 += kPrepThreads * 8) {
        __align__(16) __nv_bfloat16 hi[8], mid[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float v = xr[k8 + e];
            if (gain) v = (v * scale) * gain[k8 + e];
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            const float r1 = v - __bfloat162float(h);
            const __nv_bfloat16 mm = __float2bfloat16_rn(r1);
            hi[e] = h;
            mid[e] = mm;
            lo[e] = __float2bfloat16_rn(r1 - __bfloat162float(mm));
        }
        const int kb = k8 / kKB, kk = k8 % kKB;
        uint8_t* base = xs + static_cast<size_t>(kb) * kBBytes;
        *reinterpret_cast<uint4*>(base + sw128_off(r, kk)) = *reinterpret_cast<uint4*>(hi);
        *reinterpret_cast<uint4*>(base + sw128_off(kRows + r, kk)) = *reinterpret_cast<uint4*>(mid);
        *reinterpret_cast<uint4*>(base + sw128_off(2 * kRows + r, kk)) = *reinterpret_cast<uint4*>(lo);
    }
}

// argmax over the per-tile partials (first maximum wins)
__global__ void head_argmax_kernel(const float* __restrict__ val, const int32_t* __restrict__ idx, int tiles,
                                   int32_t* __restrict__ out) {
    const int r = blockIdx.x;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) {
        const float v = val[static_cast<size_t>(r) * tiles + t];
        const int i = idx[static_cast<size_t>(r) * tiles + t];
        if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v2 > bv || (v2 == bv && i2 < bi)) {
            bv = v2;
            bi = i2;
        }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = bv;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
            if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
                bv = sv[w];
                bi = si[w];
            }
        out[r] = bi == 0x7fffffff ? 0 : bi;
    }
}

// ── weight re-layout: reference [K x N] (row-major, in x out) -> tiled SW128 W^T
// kind 0: plain (feature f = tile*128 + m from src0 with ld n0)
// kind 1: q|k|v concat   kind 2: gate/up interleave (64 + 64 per tile)
// s0/s1/s2 are [K x ld] reference-layout matrices; the first n columns are
// taken (ld > n: a tensor-parallel column slice, the pointer pre-offset)
__global__ void relayout_kernel(const __nv_bfloat16* __restrict__ s0, const __nv_bfloat16* __restrict__ s1,
                                const __nv_bfloat16* __restrict__ s2, int n0, int n1, int n2, int ld0, int ld1,
                                int ld2, int kind, int K, int tiles, uint8_t* __restrict__ dst) {
    const int KB = K / kKB;
    const size_t total = static_cast<size_t>(tiles) * KB * kM * kKB;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        // e enumerates (tile, kb, kk, m) with m fastest so reads of a weight row coalesce
        const int m = static_cast<int>(e % kM);
        size_t rest = e / kM;
        const int kk = static_cast<int>(rest % kKB);
        rest /= kKB;
        const int kb = static_cast<int>(rest % KB);
        const int t = static_cast<int>(rest / KB);
        const int k = kb * kKB + kk;
        __nv_bfloat16 v = __float2bfloat16_rn(0.0f);
        if (kind == 0) {
            const int f = t * kM + m;
            if (f < n0) v = s0[static_cast<size_t>(k) * ld0 + f];
        } else if (kind == 1) {
            const int f = t * kM + m;
            if (f < n0) v = s0[static_cast<size_t>(k) * ld0 + f];
            else if (f < n0 + n1) v = s1[static_cast<size_t>(k) * ld1 + (f - n0)];
            else if (f < n0 + n1 + n2) v = s2[static_cast<size_t>(k) * ld2 + (f - n0 - n1)];
        } else {
            const int f = t * 64 + (m & 63);
            if (f < n0) v = (m < 64 ? s0 : s1)[static_cast<size_t>(k) * ld0 + f];
        }
        uint8_t* tileb = dst + (static_cast<size_t>(t) * KB + kb) * kABytes;
        *reinterpret_cast<__nv_bfloat16*>(tileb + sw128_off(m, kk)) = v;
    }
}

template <int NC = 1>
constexpr size_t smem_bytes() {
    return 1024 + static_cast<size_t>(n_stages<NC>()) * stage_bytes<NC>() + 2 * n_stages<NC>() * 8 + 4 * 8 + 16 + 16 +
           (64 * kRows + 8 * kRows) * 4;
}

template <int EPI, int NC = 1>
void launch_gemm(const GemmArgs& a, int grid, cudaStream_t s) {
    ensure_smem_attr(reinterpret_cast<const void*>(gemm_kernel<EPI, NC>), smem_bytes<NC>());
    gemm_kernel<EPI, NC><<<grid, kThreads, smem_bytes<NC>(), s>>>(a);
}

int num_sms() { return device_sm_count(); }

int tiles_for(int n) { return (n + kM - 1) / kM; }

}  // namespace fast

using namespace fast;

// ── workspace layout inside Workspace::fast ───────────────────────────────
namespace {
struct FastWs {
    uint8_t* xs;       // [KBmax][kBBytes]
    float* partials;   // [tiles_max][kMaxPieces][kRows][kM]
    int* counters;     // [tiles_max]
    float* amax_val;   // [rows][tiles_head]
    int32_t* amax_idx;
    uint8_t* xs2;      // prompt chunks 1..kPromptChunks-1: [chunk][KBmax][kBBytes]
    float* partials2;  // [chunk][layer_tiles_max][kMaxPieces][kRows][kM]
    int* counters2;    // [chunk][layer_tiles_max]
};
size_t max_layer_tiles(const ModelCfg& c) {
    const int qkv = tiles_for(c.q_dim() + 2 * c.kv_dim());
    const int gu = (c.ffn_dim + 63) / 64;
    return static_cast<size_t>(std::max({qkv, gu, tiles_for(c.hidden_dim)}));
}
size_t max_tiles(const ModelCfg& c) {
    const int qkv = tiles_for(c.q_dim() + 2 * c.kv_dim());
    const int gu = (c.ffn_dim + 63) / 64;
    const int hv = tiles_for(c.vocab_size);
    return static_cast<size_t>(std::max({qkv, gu, hv, tiles_for(c.hidden_dim)}));
}
size_t max_kb(const ModelCfg& c) {
    return static_cast<size_t>(std::max({c.hidden_dim, c.q_dim(), c.ffn_dim}) / kKB);
}
FastWs carve(const ModelCfg& c, Workspace& ws, int rows) {
    FastWs f;
    uint8_t* p = static_cast<uint8_t*>(ws.fast);
    auto take = [&](size_t bytes) {
        uint8_t* r = p;
        p += (bytes + 1023) & ~size_t(1023);
        return r;
    };
    f.xs = take(max_kb(c) * kBBytes);
    f.partials = reinterpret_cast<float*>(take(max_tiles(c) * kMaxPieces * kRows * kM * sizeof(float)));
    f.counters = reinterpret_cast<int*>(take(max_tiles(c) * sizeof(int)));
    f.amax_val = reinterpret_cast<float*>(take(static_cast<size_t>(rows) * tiles_for(c.vocab_size) * sizeof(float)));
    f.amax_idx = reinterpret_cast<int32_t*>(take(static_cast<size_t>(rows) * tiles_for(c.vocab_size) * sizeof(int32_t)));
    const size_t extra = kPromptChunks - 1;
    f.xs2 = take(extra * max_kb(c) * kBBytes);
    f.partials2 = reinterpret_cast<float*>(take(extra * max_layer_tiles(c) * kMaxPieces * kRows * kM * sizeof(float)));
    f.counters2 = reinterpret_cast<int*>(take(extra * max_layer_tiles(c) * sizeof(int)));
    return f;
}
}  // namespace

float* fast_partials(const ModelCfg& c, Workspace& ws) { return carve(c, ws, ws.cap_rows).partials; }
int* fast_counters(const ModelCfg& c, Workspace& ws) { return carve(c, ws, ws.cap_rows).counters; }

size_t fast_workspace_bytes(const ModelCfg& c, int rows) {
    const size_t extra = kPromptChunks - 1;
    return max_kb(c) * kBBytes + max_tiles(c) * kMaxPieces * kRows * kM * sizeof(float) + max_tiles(c) * sizeof(int) +
           2 * static_cast<size_t>(rows) * tiles_for(c.vocab_size) * sizeof(float) +
           extra * (max_kb(c) * kBBytes + max_layer_tiles(c) * (kMaxPieces * kRows * kM * sizeof(float) + sizeof(int))) +
           16 * 1024;
}

static void check_fast_shape(const ModelCfg& c) {
    if (c.hidden_dim % kKB || c.q_dim() % kKB || c.ffn_dim % kKB)
        throw Error(Kind::config, "FAST math needs hidden_dim, q_dim and ffn_dim to be multiples of 64");
}

static void* relayout(Engine& e, const void* s0, const void* s1, const void* s2, int n0, int n1, int n2, int kind,
                      int K, int tiles, cudaStream_t s, int ld0 = 0, int ld1 = 0, int ld2 = 0) {
    void* dst = nullptr;
    const size_t bytes = static_cast<size_t>(tiles) * (K / kKB) * kABytes;
    SFG_CUDA(cudaMalloc(&dst, bytes));
    relayout_kernel<<<2048, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(s0), static_cast<const __nv_bfloat16*>(s1),
                                         static_cast<const __nv_bfloat16*>(s2), n0, n1, n2, ld0 ? ld0 : n0,
                                         ld1 ? ld1 : n1, ld2 ? ld2 : n2, kind, K, tiles, static_cast<uint8_t*>(dst));
    SFG_CUDA(cudaGetLastError());
    e.adopt(dst, bytes);
    return dst;
}

// Tensor parallelism: QKV and gate|up are split by output columns (whole
// heads / FFN columns), O and down by input rows; rank r takes slice r.
void fast_build_layer(Engine& e, LayerWeights& L, cudaStream_t s) {
    const ModelCfg& c = e.cfg();
    check_fast_shape(c);
    const int H = c.hidden_dim, qd = c.q_dim(), kvd = c.kv_dim(), F = c.ffn_dim;
    const int t = e.tp_size(), r = e.tp_rank();
    const int ql = qd / t, kl = kvd / t, fl = F / t;
    const auto* wq = static_cast<const __nv_bfloat16*>(L.wq) + static_cast<size_t>(r) * ql;
    const auto* wk = static_cast<const __nv_bfloat16*>(L.wk) + static_cast<size_t>(r) * kl;
    const auto* wv = static_cast<const __nv_bfloat16*>(L.wv) + static_cast<size_t>(r) * kl;
    const auto* wo = static_cast<const __nv_bfloat16*>(L.wo) + static_cast<size_t>(r) * ql * H;
    const auto* wg = static_cast<const __nv_bfloat16*>(L.w_gate) + static_cast<size_t>(r) * fl;
    const auto* wu = static_cast<const __nv_bfloat16*>(L.w_up) + static_cast<size_t>(r) * fl;
    const auto* wd = static_cast<const __nv_bfloat16*>(L.w_down) + static_cast<size_t>(r) * fl * H;
    L.f_qkv = relayout(e, wq, wk, wv, ql, kl, kl, 1, H, tiles_for(ql + 2 * kl), s, qd, kvd, kvd);
    L.f_o = relayout(e, wo, nullptr, nullptr, H, 0, 0, 0, ql, tiles_for(H), s);
    L.f_gu = relayout(e, wg, wu, nullptr, fl, 0, 0, 2, H, (fl + 63) / 64, s, F);
    L.f_down = relayout(e, wd, nullptr, nullptr, H, 0, 0, 0, fl, tiles_for(H), s);
}

void* fast_build_head(Engine& e, const void* lm_head, cudaStream_t s) {
    const ModelCfg& c = e.cfg();
    check_fast_shape(c);
    return relayout(e, lm_head, nullptr, nullptr, c.vocab_size, 0, 0, 0, c.hidden_dim, tiles_for(c.vocab_size), s);
}

// Stream-K grid: every CTA gets >= ceil((KB-1)/(kMaxPieces-1)) k-blocks so
// no tile is split into more than kMaxPieces pieces.
static int grid_for(int tiles, int KB) {
    const long long U = static_cast<long long>(tiles) * KB;
    const int min_units = (KB - 1 + kMaxPieces - 2) / (kMaxPieces - 1);
    long long g = min_units > 0 ? U / min_units : U;
    g = std::min<long long>(g, num_sms());
    return static_cast<int>(std::max<long long>(g, 1));
}

// Prompt passes (rows > 16): the (weight tile x 128-token tile) GEMMs.
// SFG_PROMPT=chunks selects the older five-chunk stream-K passes (A/B).
static bool prompt_tiles() {
    static const bool on = [] {
        const char* v = getenv("SFG_PROMPT");
        return !(v && std::string(v) == "chunks");
    }();
    return on;
}

static int fast_forward_layer_prompt(Engine& e, Bank& b, int layer, int rows, Workspace& ws, int prior,
                                     cudaStream_t s) {
    const ModelCfg& c = e.cfg();
    const Dims d = e.dims();
    const LayerWeights& L = e.layer(layer);
    float* kc = b.kslab(layer);
    float* vc = b.vslab(layer);
    const int TT = (rows + kPT - 1) / kPT;
    const size_t img = static_cast<size_t>(TT) * max_kb(c) * 3 * kPBBytes;
    if (img > ws.pimg_bytes) {
        SFG_CUDA(cudaDeviceSynchronize());
        if (ws.pimg) cudaFree(ws.pimg);
        ws.pimg = nullptr;
        SFG_CUDA(cudaMalloc(&ws.pimg, img));
        ws.pimg_bytes = img;
    }
    uint8_t* X = static_cast<uint8_t*>(ws.pimg);
    int n = 0;
    const double R = rows;
    auto pprep = [&](const float* x, int ld, int K, const float* gain, float eps) {
        pprep_kernel<<<TT * kPT, 256, 0, s>>>(x, ld, K, rows, gain, eps, X);
        ++n;
    };
    auto args = [&]() {
        PgArgs pa{};
        pa.X = X;
        pa.TT = TT;
        pa.total_rows = rows;
        pa.g.row0 = 0;
        pa.g.rows = rows;
        return pa;
    };
    {  // attention-input RMSNorm + split, fused QKV + RoPE + KV append
        pprep(ws.h, d.H, d.H, L.attn_norm, d.eps);
        PgArgs pa = args();
        GemmArgs& a = pa.g;
        a.W = static_cast<const uint8_t*>(L.f_qkv);
        a.tiles = tiles_for(d.qd + 2 * d.kvd);
        a.KB = d.H / kKB;
        a.n_out = d.qd + 2 * d.kvd;
        a.out = ws.q;
        a.qd = d.qd;
        a.kvd = d.kvd;
        a.hd = d.hd;
        a.max_len = d.max_len;
        a.prior = ws.meta;
        a.pos = ws.pos;
        a.rope_cos = e.rope_cos();
        a.rope_sin = e.rope_sin();
        a.kc = kc;
        a.vc = vc;
        ProfScope ps(K_QKV, s, 2.0 * d.H * a.n_out + 4.0 * R * (d.H + a.n_out), 2.0 * R * d.H * a.n_out);
        launch_pgemm<EPI_QKV>(pa, s);
        ++n;
    }
    {
        const double kvb = 2.0 * 4.0 * d.kvd * (prior + rows);
        ProfScope ps(K_ATTN, s, kvb + 8.0 * R * d.qd, 4.0 * R * d.qd * (prior + rows));
        if (ws.prefix_mask && attention_prompt_supported(d)) {
            n += launch_attention_prompt(ws.q, kc, vc, ws.row_off, ws.runs, rows, prior + rows, d, ws.att, ws.status, s,
                                         &ws.apieces, &ws.apieces_bytes);
        } else {
            int cap = 0;  // prompt passes are never graph-captured: size by the cache length
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            SFG_CUDA(cudaStreamIsCapturing(s, &cs));
            if (cs == cudaStreamCaptureStatusNone) cap = prior + rows;
            n += launch_attention_fast(ws.q, kc, vc, ws.row_off, ws.runs, rows, d, ws.att, ws.status, s, cap);
        }
    }
    {  // O-proj + residual
        pprep(ws.att, d.qd, d.qd, nullptr, 0.f);
        PgArgs pa = args();
        GemmArgs& a = pa.g;
        a.W = static_cast<const uint8_t*>(L.f_o);
        a.tiles = tiles_for(d.H);
        a.KB = d.qd / kKB;
        a.n_out = d.H;
        a.out = ws.h;
        a.ld = d.H;
        a.store_only = e.tp_rank() > 0;
        ProfScope ps(K_OPROJ, s, 2.0 * d.qd * d.H + 4.0 * R * (d.qd + 2.0 * d.H), 2.0 * R * d.qd * d.H);
        launch_pgemm<EPI_RESID>(pa, s);
        ++n;
    }
    e.tp_allreduce(ws.h, static_cast<size_t>(rows) * d.H, s);
    {  // FFN RMSNorm + split, gate|up + SiLU*up
        pprep(ws.h, d.H, d.H, L.ffn_norm, d.eps);
        PgArgs pa = args();
        GemmArgs& a = pa.g;
        a.W = static_cast<const uint8_t*>(L.f_gu);
        a.tiles = (d.F + 63) / 64;
        a.KB = d.H / kKB;
        a.n_out = d.F;
        a.out = ws.act;
        a.ld = d.F;
        ProfScope ps(K_GATEUP, s, 4.0 * d.H * d.F + 4.0 * R * (d.H + d.F), 4.0 * R * d.H * d.F);
        launch_pgemm<EPI_GATEUP>(pa, s);
        ++n;
    }
    {  // down + residual
        pprep(ws.act, d.F, d.F, nullptr, 0.f);
        PgArgs pa = args();
        GemmArgs& a = pa.g;
        a.W = static_cast<const uint8_t*>(L.f_down);
        a.tiles = tiles_for(d.H);
        a.KB = d.F / kKB;
        a.n_out = d.H;
        a.out = ws.h;
        a.ld = d.H;
        a.store_only = e.tp_rank() > 0;
        ProfScope ps(K_DOWN, s, 2.0 * d.F * d.H + 4.0 * R * (d.F + 2.0 * d.H), 2.0 * R * d.F * d.H);
        launch_pgemm<EPI_RESID>(pa, s);
        ++n;
    }
    e.tp_allreduce(ws.h, static_cast<size_t>(rows) * d.H, s);
    SFG_CUDA(cudaGetLastError());
    return n;
}

// One layer of forward_layers (tinyformer.cpp:412-504) in FAST math.
int fast_forward_layer(Engine& e, Bank& b, int layer, int rows, Workspace& ws, int prior, cudaStream_t s) {
    if (rows > kRows && prompt_tiles()) return fast_forward_layer_prompt(e, b, layer, rows, ws, prior, s);
    const ModelCfg& c = e.cfg();
    const Dims d = e.dims();
    const LayerWeights& L = e.layer(layer);
    FastWs f = carve(c, ws, ws.cap_rows);
    float* kc = b.kslab(layer);
    float* vc = b.vslab(layer);
    int n = 0;
    const double R = rows;
    // A pass covers one 16-row chunk, or (prompts: rows > 16) up to
    // kPromptChunks chunks that share every weight stage.  Each projection runs
    // GEMM-outer over the passes, so its weights (QKV 50 MB, O 32 MB at 7B)
    // can be re-read from L2 (ncu: little reuse in practice; the L2 is split
    // over the two dies).  Passes touch disjoint rows.
    const int step = rows > kRows ? kRows * kPromptChunks : kRows;
    auto pass_args = [&](int p0, int pr) {
        GemmArgs a{};
        a.X = f.xs;
        a.partials = f.partials;
        a.counters = f.counters;
        a.X2 = f.xs2;
        a.partials2 = f.partials2;
        a.counters2 = f.counters2;
        a.rows = pr;
        a.row0 = p0;
        return a;
    };
    // [RMSNorm] + 3-way split of the pass's rows into the chunk images
    auto prep = [&](const float* x, int ld, int K, const float* gain, float eps, int p0, int pr) {
        prep_kernel<<<pr, kPrepThreads, 0, s>>>(x + static_cast<size_t>(p0) * ld, ld, K, gain, eps, f.xs, f.xs2,
                                                static_cast<size_t>(K / kKB) * kBBytes);
        ++n;
    };
    auto gemm = [&](auto epi, const GemmArgs& a) {
        constexpr int EPI = decltype(epi)::value;
        if (a.rows > kRows)
            launch_gemm<EPI, kPromptChunks>(a, grid_for(a.tiles, a.KB), s);
        else
            launch_gemm<EPI>(a, grid_for(a.tiles, a.KB), s);
        ++n;
    };
    using QKV = std::integral_constant<int, EPI_QKV>;
    using RESID = std::integral_constant<int, EPI_RESID>;
    using GATEUP = std::integral_constant<int, EPI_GATEUP>;
    for (int p0 = 0; p0 < rows; p0 += step) {  // attention-input RMSNorm + split, fused QKV + RoPE + KV append
        const int pr = std::min(step, rows - p0);
        GemmArgs a = pass_args(p0, pr);
        prep(ws.h, d.H, d.H, L.attn_norm, d.eps, p0, pr);
        a.W = static_cast<const uint8_t*>(L.f_qkv);
        a.tiles = tiles_for(d.qd + 2 * d.kvd);
        a.KB = d.H / kKB;
        a.n_out = d.qd + 2 * d.kvd;
        a.out = ws.q;
        a.qd = d.qd;
        a.kvd = d.kvd;
        a.hd = d.hd;
        a.max_len = d.max_len;
        a.prior = ws.meta;
        a.pos = ws.pos;
        a.rope_cos = e.rope_cos();
        a.rope_sin = e.rope_sin();
        a.kc = kc;
        a.vc = vc;
        {
            ProfScope ps(K_QKV, s, 2.0 * d.H * a.n_out + 4.0 * pr * (d.H + a.n_out), 2.0 * pr * d.H * a.n_out);
            gemm(QKV{}, a);
        }
    }
    {
        const double kvb = 2.0 * 4.0 * d.kvd * (prior + rows);
        ProfScope ps(K_ATTN, s, kvb + 8.0 * R * d.qd, 4.0 * R * d.qd * (prior + rows));
        // prompt passes (never graph-captured) size the launch by the cache
        // length after this batch instead of max_seq_len: more resident CTAs
        int cap = 0;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        SFG_CUDA(cudaStreamIsCapturing(s, &cs));
        if (rows > kRows && cs == cudaStreamCaptureStatusNone) cap = prior + rows;
        n += launch_attention_fast(ws.q, kc, vc, ws.row_off, ws.runs, rows, d, ws.att, ws.status, s, cap);
    }
    for (int p0 = 0; p0 < rows; p0 += step) {  // O-proj + residual
        const int pr = std::min(step, rows - p0);
        GemmArgs a = pass_args(p0, pr);
        prep(ws.att, d.qd, d.qd, nullptr, 0.f, p0, pr);
        a.W = static_cast<const uint8_t*>(L.f_o);
        a.tiles = tiles_for(d.H);
        a.KB = d.qd / kKB;
        a.n_out = d.H;
        a.out = ws.h;
        a.ld = d.H;
        a.store_only = e.tp_rank() > 0;  // rank 0 adds the residual, the others their partial
        {
            ProfScope ps(K_OPROJ, s, 2.0 * d.qd * d.H + 4.0 * pr * (d.qd + 2.0 * d.H), 2.0 * pr * d.qd * d.H);
            gemm(RESID{}, a);
        }
    }
    e.tp_allreduce(ws.h, static_cast<size_t>(rows) * d.H, s);
    for (int p0 = 0; p0 < rows; p0 += step) {  // FFN RMSNorm + split, gate|up + SiLU*up
        const int pr = std::min(step, rows - p0);
        GemmArgs a = pass_args(p0, pr);
        prep(ws.h, d.H, d.H, L.ffn_norm, d.eps, p0, pr);
        a.W = static_cast<const uint8_t*>(L.f_gu);
        a.tiles = (d.F + 63) / 64;
        a.KB = d.H / kKB;
        a.n_out = d.F;
        a.out = ws.act;
        a.ld = d.F;
        {
            ProfScope ps(K_GATEUP, s, 4.0 * d.H * d.F + 4.0 * pr * (d.H + d.F), 4.0 * pr * d.H * d.F);
            gemm(GATEUP{}, a);
        }
    }
    for (int p0 = 0; p0 < rows; p0 += step) {  // down + residual
        const int pr = std::min(step, rows - p0);
        GemmArgs a = pass_args(p0, pr);
        prep(ws.act, d.F, d.F, nullptr, 0.f, p0, pr);
        a.W = static_cast<const uint8_t*>(L.f_down);
        a.tiles = tiles_for(d.H);
        a.KB = d.F / kKB;
        a.n_out = d.H;
        a.out = ws.h;
        a.ld = d.H;
        a.store_only = e.tp_rank() > 0;
        {
            ProfScope ps(K_DOWN, s, 2.0 * d.F * d.H + 4.0 * pr * (d.F + 2.0 * d.H), 2.0 * pr * d.F * d.H);
            gemm(RESID{}, a);
        }
    }
    e.tp_allreduce(ws.h, static_cast<size_t>(rows) * d.H, s);
    SFG_CUDA(cudaGetLastError());
    return n;
}

// finalize (tinyformer.cpp:510-526) + argmax_row in FAST math: final RMSNorm
// + split, LM-head GEMM with logits/argmax-partial epilogue, partial reduce.
int fast_head(Engine& e, const void* f_lm_head, const float* final_norm, int rows, Workspace& ws, bool want_logits,
              cudaStream_t s) {
    const ModelCfg& c = e.cfg();
    FastWs f = carve(c, ws, ws.cap_rows);
    const int tiles = tiles_for(c.vocab_size);
    int n = 0;
    for (int p0 = 0; p0 < rows; p0 += kRows) {
        const int pr = std::min(kRows, rows - p0);
        prep_kernel<<<pr, kPrepThreads, 0, s>>>(ws.h + static_cast<size_t>(p0) * c.hidden_dim, c.hidden_dim,
                                                c.hidden_dim, final_norm, c.rms_eps, f.xs);
        GemmArgs a{};
        a.W = static_cast<const uint8_t*>(f_lm_head);
        a.X = f.xs;
        a.tiles = tiles;
        a.KB = c.hidden_dim / kKB;
        a.n_out = c.vocab_size;
        a.partials = f.partials;
        a.counters = f.counters;
        a.rows = pr;
        a.row0 = p0;
        a.out = want_logits ? ws.logits : nullptr;
        a.ld = c.vocab_size;
        a.amax_val = f.amax_val;
        a.amax_idx = f.amax_idx;
        {
            ProfScope ps(K_HEAD, s, 2.0 * c.hidden_dim * c.vocab_size + 4.0 * pr * (c.hidden_dim + c.vocab_size),
                         2.0 * pr * c.hidden_dim * c.vocab_size);
            launch_gemm<EPI_HEAD>(a, grid_for(a.tiles, a.KB), s);
        }
        n += 2;
    }
    head_argmax_kernel<<<rows, 256, 0, s>>>(f.amax_val, f.amax_idx, tiles, ws.argmax);
    SFG_CUDA(cudaGetLastError());
    return n + 1;
}

}  // namespace sfg
