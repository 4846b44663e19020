// FAST-mode layer-stack megakernel (sm_100a): forward_layers over a whole
// layer range in ONE cooperative launch.
//
// Why: a lookahead step streams 12 GB of weights through 28 x 4 dependent
// skinny GEMMs.  With one kernel per GEMM every boundary costs a launch, a
// TMEM/barrier prologue and a DRAM-latency ramp, and HBM idles meanwhile.
// Here one CTA per SM (320 threads) runs the whole stack:
//
//   warp 0      weight producer: walks the CTA's stream-K share of every GEMM
//               of every layer and keeps the 8-stage smem ring full with
//               cp.async.bulk weight tiles — never waits on activations, so
//               the next GEMM's weights arrive while the current one drains
//               and while attention / grid barriers are in flight;
//   warp 1      tcgen05.mma issuer (one thread), TMEM double accumulator;
//   warps 2-5   TMEM epilogue: RoPE + KV append (QKV), residual add + per-tile
//               sum-of-squares partials (O, down), SiLU*up (gate|up), stream-K
//               fixup (last arriver sums the pieces in fixed k order); each
//               output is also stored as the NEXT GEMM's input image (3-way
//               bf16 split, times the RMSNorm gain, in the MMA's swizzled
//               layout), and the 1/rms row scale is applied to the consuming
//               GEMM's accumulator;
//   warp 6      activation loader (one thread): after the phase's grid
//               barrier, one 6 KB bulk copy of the image per stage;
//   warps 2-9   attention phase between QKV and O (flash-decode style, fixed
//               key partition -> deterministic, batch invariant).
//
// Dependent phases are separated by a monotonic grid barrier (all CTAs are
// co-resident: cooperative launch, one CTA per SM); the last CTA to exit
// resets it for the next launch.  Arithmetic matches sfg_fast.cu (same
// split, same stream-K fixup order) within the stated tolerance; results
// are deterministic and independent of the batch composition.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <string>

#include "sfg_engine.h"
#include "sfg_prof.h"
#include "sfg_tc.cuh"

namespace sfg {
namespace mega {

using namespace tc;

constexpr int kMaxStages = 8;
constexpr int kThreads = 320;
constexpr int kAccCols = 64;
constexpr int kTmemCols = 128;
constexpr int kMaxPieces = 16;
constexpr int kMaxGroup = 8;
constexpr int kMaxBanks = 16;  // sessions per launch (one row each at least)
// Rows per launch: R = 16 (one session's lookahead batch) or 32 (several
// sessions' batches in one weight pass).  The MMA N is 3R (hi | mid | lo bf16
// pieces of every row) and costs the same for N = 48 and N = 96 (it is issue
// bound below N = 128, tools/mb_ring.cu), so a 32-row pass streams the same
// weights with the same tensor-core time; epilogues work in 16-row blocks.
constexpr int kMaxRows = 32;
enum Phase : int { P_QKV = 0, P_O = 1, P_GU = 2, P_DOWN = 3 };

struct LayerDesc {
    const uint8_t* w[4];     // tiled W^T images: qkv, o, gate|up, down
    const float* attn_norm;
    const float* ffn_norm;
    const float* next_attn_norm;  // the following layer's attn_norm (nullptr for the last)
    float* kc;               // this layer's K slab [n_kv][max_len][hd]
    float* vc;
};

struct MegaArgs {
    const LayerDesc* layers;
    int nlayers, rows, stages;
    int R;             // row capacity of this launch (16 or 32): image / partial / sum-of-squares row stride
    int stage_bytes;   // kABytes + xbytes
    int xbytes;        // one k-block of the activation image: 3R rows x 64 bf16
    int acc_cols;      // TMEM columns per accumulator (>= 3R)
    int tmem_cols;     // TMEM columns allocated (2 accumulators)
    uint32_t idesc;    // kind::f16 instruction descriptor, N = 3R
    int H, qd, kvd, F, hd, n_heads, n_kv, max_len;
    float eps;
    float* h;        // [16][H] residual stream, in/out
    float* q;        // [16][qd]
    float* att;      // [16][qd]
    float* act;      // [16][F]
    float* ss_d;     // [tilesH][16] sum-of-squares partials of h (input / after down)
    float* ss_o;     // [tilesH][16] after O-proj
    const int32_t* pos;
    const float* rope_cos;
    const float* rope_sin;
    const int32_t* prior;
    const int32_t* row_off;
    const MaskRun* runs;
    float* partials;   // 2 x [tiles_max][kMaxPieces][16][128] (by phase parity)
    int* counters;     // 2 x [tiles_max]
    size_t part_stride;  // floats between the two partial buffers
    int cnt_stride;      // ints between the two counter arrays
    unsigned* flags;   // dataflow completion flags (see fptr), zeroed by the last CTA out
    int nflags;
    unsigned* bar;     // per-barrier arrival counters + exit counter
    uint32_t* status;
    int pf;            // L2 prefetch distance in weight units (0: off)
    int evict_first;   // stream weights with an L2 evict-first policy
    int spin_mma;      // dev knob: MMA issuer spins on test_wait instead of try_wait
    int bpf;           // bubble L2 prefetch depth in units (0: off)
    int noload;        // dev knob (timing experiments only, WRONG results): bit 0 no weight bytes, bit 1 no activation bytes, bit 2 no input flag polls
    int G[4];          // per phase: CTAs sharing its stream-K split (phase_ctas)
    int W[4];          // per phase: whole tiles per CTA after the split part (whole_tiles)
    int fl_base, fl_lay, fl_off[6];  // dataflow flag layout (see fptr)
    long long bpf_cycles;  // ring-full wait (SM cycles) that counts as a bubble
    uint8_t* xim[4];   // per phase: the GEMM's input as [KB][48 x 64] split bf16 images (put_split)
    int attn_rows;     // 1: per-(row, kv head) attention; 0: key-chunked, rows share K/V (long contexts)
    // KV caches: rows may belong to different sessions (cross-session batching):
    // bank b's K slab of launch layer l is kbank[b] + l * slab_stride; row r
    // appends at rowinfo[3r + 1] and sees rowinfo[3r + 2] cached keys of bank
    // rowinfo[3r] (rowinfo == nullptr: one bank, slot = prior + r)
    float* kbank[kMaxBanks];
    float* vbank[kMaxBanks];
    size_t slab_stride;
    const int32_t* rowinfo;
    // tensor parallelism (TP = 2): O / down partial tiles are exchanged with the
    // peer GPU through its inbox (CUDA IPC over NVLink) inside the epilogue
    int tp, tp_rank;
    float* inbox;          // mine, written by the peer
    unsigned* inflag;      // mine: epoch flags per (layer, O|down, tile)
    float* peer_inbox;     // the peer's (mapped)
    unsigned* peer_inflag;
    unsigned* epoch_ptr;   // launch counter
    float* apart;      // attention chunk partials [n_kv][ceil(max_len/kAttnMinKC)][128 queries][hd + 2]
    unsigned* acnt;    // [n_kv] chunk arrival counters (reset by the merging chunk)
    // optional [G][kBarSlots][kTraceW] (tools/trace_mega.py): per CTA and
    // barrier id, globaltimer stamps and wait totals (see tslot users)
    unsigned long long* trace;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int kTraceW = 20;
// slot k of (CTA c, barrier id): 0 X start, 1 X done, 2 arrive, 3/4/5 ns waited by
// X loader (empty) / MMA (full) / producer (empty), 6 last accumulator ready,
// 7 epilogue done; last fixup: 8 partials fenced, 9 counter, 10 loads, 11 epi_final;
// MMA issuer: 16 first MMA issued, 17 last commit, 18 ns waited on a free accumulator
__device__ __forceinline__ unsigned long long* tslot(const MegaArgs& a, int c, int id, int k) {
    return a.trace + (static_cast<size_t>(c) * 256 + id) * kTraceW + k;
}

struct Geo {
    int tiles, KB, G;  // G: CTAs sharing this GEMM's stream-K split (see split_ctas)
    int W;             // whole tiles per CTA, processed after its stream-K piece
    __device__ __forceinline__ int split_units() const { return (tiles - W * G) * KB; }
};
// Stream-K split width: at most gridDim.x CTAs, each with at least
// ceil((KB-1)/(kMaxPieces-1)) k-blocks so a tile never has more than
// kMaxPieces pieces; CTAs >= G get no units in this phase.
__host__ __device__ __forceinline__ int split_ctas(int tiles, int KB, int grid) {
    const int U = tiles * KB;
    const int min_units = (KB - 1 + kMaxPieces - 2) / (kMaxPieces - 1);
    int g = min_units > 0 ? U / min_units : U;
    if (g > grid) g = grid;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}
__device__ __forceinline__ Geo geom(const MegaArgs& a, int p) {
    int t, kb;
    switch (p) {
        case P_QKV: t = (a.qd + 2 * a.kvd + kM - 1) / kM; kb = a.H / kKB; break;
        case P_O: t = (a.H + kM - 1) / kM; kb = a.qd / kKB; break;
        case P_GU: t = a.F / 64; kb = a.H / kKB; break;
        default: t = (a.H + kM - 1) / kM; kb = a.F / kKB; break;
    }
    return {t, kb, a.G[p], a.W[p]};  // host: phase_ctas / whole_tiles
}
// CTAs of a phase's split.  A tile-aligned split is used when it keeps at
// least align_pct % of the grid busy: every CTA then gets exactly one 1/P piece
// of one tile (tiles <= grid, P | KB) or k whole tiles (tiles > grid, k |
// tiles) -- one accumulator and at most one fixup per CTA, while the idle CTAs'
// producers already stream the next GEMM's weights.  Otherwise stream-K over
// the whole grid (split_ctas).
inline int phase_ctas(int tiles, int KB, int grid, int align_pct) {
    if (align_pct > 0) {
        int ga = 0;
        if (tiles <= grid) {
            for (int P = std::min(kMaxPieces, grid / tiles); P >= 1; --P)
                if (KB % P == 0) {
                    ga = tiles * P;
                    break;
                }
        } else {
            for (int k = (tiles + grid - 1) / grid; k <= tiles; ++k)
                if (tiles % k == 0) {
                    ga = tiles / k;
                    break;
                }
        }
        if (ga * 100 >= align_pct * grid) return ga;
    }
    return split_ctas(tiles, KB, grid);
}

// Phases with more tiles than CTAs: every CTA also owns W whole tiles, and
// only the remaining tiles are split stream-K.  A CTA runs its split piece
// FIRST and its whole tiles last, so the split tiles' fixups (partial
// stores, arrival counter, reduction) overlap the whole tiles' weight
// streaming and the phase ends with plain epilogues.  The remainder must
// keep every split tile within kMaxPieces pieces.
inline int whole_tiles(int tiles, int KB, int G) {
    if (G < 1 || tiles < G) return 0;
    const int W = tiles / G;
    const int rem = tiles - W * G;
    if (rem == 0) return W;
    const int min_units = (rem * KB) / G;  // smallest piece of a split tile
    if (min_units < 1 || (KB + min_units - 1) / min_units + 1 > kMaxPieces) return 0;
    return W;
}
// this CTA's units of a phase as segments: seg 0 = its piece of the split
// tiles [0, tiles - W*G), seg 1 = its whole tiles (empty when W == 0; both
// empty when c >= g.G).  32-bit unit math (tiles x k-blocks < 2^31).
__device__ __forceinline__ void unit_seg(const Geo& g, int c, int seg, int& st, int& en) {
    if (c >= g.G) {
        st = en = 0;
        return;
    }
    if (seg == 0) {
        const int U = g.split_units();
        st = c * U / g.G;
        en = (c + 1) * U / g.G;
    } else {
        const int t0 = g.tiles - g.W * g.G + c * g.W;
        st = t0 * g.KB;
        en = (t0 + g.W) * g.KB;
    }
}
__device__ __forceinline__ void unit_range(const Geo& g, int c, int& st, int& en) { unit_seg(g, c, 0, st, en); }

// ── grid barrier ──────────────────────────────────────────────────────────
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_arrive(unsigned* bar) {
    __threadfence();
    atomicAdd(bar, 1u);
}
__device__ __forceinline__ void grid_wait(const unsigned* bar, unsigned target) {
    unsigned long long spins = 0;
    while (ld_acquire(bar) < target) {
        __nanosleep(64);
        if (++spins > (1ull << 27)) asm volatile("trap;");  // never hang the GPU
    }
    __threadfence();
}
// barrier ids: 0 = input stats; layer i: 1+5i QKV, 2+5i attention, 3+5i O, 4+5i gate|up, 5+5i down.
// One counter per id (a single monotonic counter is wrong: CTAs with no
// work in a phase may arrive for later barriers before others arrive for
// the current one); bar[kBarSlots] counts exits, the last CTA out zeroes all.
constexpr int kBarSlots = 256;
__device__ __forceinline__ void arrive_id(unsigned* bar, int id) { grid_arrive(bar + id); }
__device__ __forceinline__ void wait_id(unsigned* bar, int id, int G) { grid_wait(bar + id, static_cast<unsigned>(G)); }
__device__ __forceinline__ int input_barrier(int layer, int p) {
    switch (p) {
        case P_QKV: return layer == 0 ? 0 : 5 * (layer - 1) + 5;
        case P_O: return 5 * layer + 2;
        case P_GU: return 5 * layer + 3;
        default: return 5 * layer + 4;
    }
}

// ── dataflow completion flags (replace grid barriers between phases) ─────
// A consumer waits only for the producer tiles its own units need: the
// activation loader for the k-blocks of its range, attention for the 6 QKV
// tiles of its kv head, and the RMSNorm scale for "all tiles of the
// producing phase" (a per-phase tile counter).  Kinds: statistics of the
// input rows (layer -1), then per layer QKV tiles, attention kv heads, O, gate|up, down.
enum FlagKind : int { K_STATS = 0, K_QKV, K_ATT, K_O, K_GU, K_DOWN };
__device__ __forceinline__ int kind_tiles(const MegaArgs& a, int k) {
    switch (k) {
        case K_QKV: return (a.qd + 2 * a.kvd + kM - 1) / kM;
        case K_ATT: return a.n_kv;
        case K_GU: return a.F / 64;
        default: return (a.H + kM - 1) / kM;  // stats, O, down: 128-feature tiles of H
    }
}
// flag of tile t (t == kind_tiles: the kind's completed-tile counter)
// offsets precomputed on the host (flag_layout): a.fl_off[k] within a layer
// block of a.fl_lay flags that starts after the statistics flags
__device__ __forceinline__ unsigned* fptr(const MegaArgs& a, int l, int k, int t) {
    if (k == K_STATS) return a.flags + t;
    return a.flags + a.fl_base + l * a.fl_lay + a.fl_off[k] + t;
}
__device__ __forceinline__ void red_add(unsigned* f, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ void signal_add(unsigned* f, unsigned v) {
    __threadfence();
    atomicAdd(f, v);
}
__device__ __forceinline__ void wait_ge(const unsigned* f, unsigned v) {
    unsigned long long spins = 0;
    while (ld_acquire(f) < v) {
        __nanosleep(32);
        if (++spins > (1ull << 27)) asm volatile("trap;");  // never hang the GPU
    }
}
// is the input k-block kb of phase p (layer l) produced?  (acquire load)
__device__ __forceinline__ bool xblock_ready(const MegaArgs& a, int l, int p, int kb) {
    switch (p) {
        case P_QKV: return ld_acquire(l == 0 ? fptr(a, 0, K_STATS, kb >> 1) : fptr(a, l - 1, K_DOWN, kb >> 1)) >= 1u;
        case P_O: {
            const int group = a.n_heads / a.n_kv;
            const int h0 = (kb * kKB) / a.hd / group, h1 = (kb * kKB + kKB - 1) / a.hd / group;
            for (int h = h0; h <= h1; ++h)
                if (ld_acquire(fptr(a, l, K_ATT, h)) < static_cast<unsigned>(a.rows * group)) return false;
            return true;
        }
        case P_GU: return ld_acquire(fptr(a, l, K_O, kb >> 1)) >= 1u;
        default: return ld_acquire(fptr(a, l, K_GU, kb)) >= 1u;
    }
}

// kind::f16 MMA with a runtime instruction descriptor (N = 3R of the launch)
__device__ __forceinline__ void mma_bf16_id(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

// bounded mbarrier wait (traps instead of hanging on a protocol bug)
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t parity) {
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

// long waits (the lent ring): poll with back-off so the waiting thread does
// not compete with the attention warps for the shared-memory pipe
__device__ __forceinline__ void mwait_sleep(uint64_t* b, uint32_t parity) {
    unsigned long long spins = 0;
    while (!mbar_test(b, parity)) {
        __nanosleep(256);
        if (++spins > (1ull << 24)) asm volatile("trap;");
    }
}

// mwait that also accumulates the time spent waiting when tracing
__device__ __forceinline__ void mwait_acc(uint64_t* b, uint32_t parity, bool tr, unsigned long long& acc) {
    if (!tr) {
        mwait(b, parity);
        return;
    }
    const unsigned long long t0 = gtimer();
    mwait(b, parity);
    acc += gtimer() - t0;
}

// Deterministic sum over the 128 epilogue threads (feature m = 32*quad + lane)
// of v[r]^2 for 16 rows -> out[r]: warp butterfly, then a fixed 4-way combine.
__device__ __forceinline__ void tile_sumsq(const float (&v)[kRows], float* red, float* out, int et) {
    const int quad = et >> 5, lane = et & 31;
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
        float s = v[r] * v[r];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[quad * kRows + r] = s;
    }
    named_sync(1, 128);
    if (et < kRows) out[et] = (red[et] + red[kRows + et]) + (red[2 * kRows + et] + red[3 * kRows + et]);
    named_sync(1, 128);
}

// generic-proxy global writes <-> cp.async.bulk reads of the same bytes
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Store x as its 3-way bf16 split (hi | mid | lo rows of the B operand) at
// feature k, row r of a phase's global activation image: [KB][48 x 64] bf16
// K-major SW128 blocks, the exact smem layout the MMA reads, so a stage's
// activations arrive with one 6 KB bulk copy.
template <int R>  // rows per launch (image row stride)
__device__ __forceinline__ void put_split(uint8_t* img, int k, int r, float x) {
    uint8_t* blk = img + static_cast<size_t>(k >> 6) * (static_cast<size_t>(R) * 384);
    const int kk = k & 63;
    const __nv_bfloat16 hb = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(hb);
    const __nv_bfloat16 mb = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lb = __float2bfloat16_rn(r1 - __bfloat162float(mb));
    *reinterpret_cast<__nv_bfloat16*>(blk + sw128_off(r, kk)) = hb;
    *reinterpret_cast<__nv_bfloat16*>(blk + sw128_off(R + r, kk)) = mb;
    *reinterpret_cast<__nv_bfloat16*>(blk + sw128_off(2 * R + r, kk)) = lb;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// per-launch constants staged in shared memory at kernel entry (the layer
// table too: the epilogue dereferences it on the critical path of every tile)
constexpr int kMaxMegaLayers = 64;
__shared__ int sh_pos[kMaxRows];
__shared__ int sh_prior;
__shared__ int sh_row_bank[kMaxRows], sh_row_slot[kMaxRows], sh_row_prior[kMaxRows];
__shared__ LayerDesc sh_layers[kMaxMegaLayers];
// per row: compacted visible-key count and its tail slots (columns >= prior)
__shared__ int sh_ncols[kMaxRows];
__shared__ unsigned sh_epoch;
__shared__ int sh_tail[kMaxRows][kRows];  // a row's own tail slots (<= 16 per session)

// ── epilogues (thread = feature m of the tile; y[r] for 16 rows) ─────────
// RMSNorm is split across the two sides of the GEMM: the producing epilogue
// stores split(h * gain) (gain is per input feature), and the consuming
// epilogue scales its accumulator by the per-row 1/rms (rs[r]), which needs
// the whole row's sum of squares and so is only known after the barrier.
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float ld_relaxed_sys(const float* p) {
    float v;
    asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

// rows rb .. rb+15 of the launch (one 16-row block of its R rows)
template <int R>
__device__ void epi_final(const MegaArgs& a, const LayerDesc& L, int l, int p, int tile, int m, int et,
                          const float (&yin)[kRows], float* xch, const float* rs, const float* ropeT,
                          const float* hpre, int rb) {
    float y[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) y[r] = (p == P_QKV || p == P_GU) ? yin[r] * rs[rb + r] : yin[r];
    if (p == P_QKV) {
        const int f = tile * kM + m;
        const bool valid = f < a.qd + 2 * a.kvd;
        const int seg = f < a.qd ? 0 : (f < a.qd + a.kvd ? 1 : 2);
        const int fl = seg == 0 ? f : (seg == 1 ? f - a.qd : f - a.qd - a.kvd);
        const int d = fl % a.hd, half = a.hd >> 1, i = d >> 1;
        const bool odd = (m & 1) != 0;
        // the rows' cos/sin: staged in shared memory at kernel entry for
        // 16-row launches, read from the (L2-resident) host-libm tables otherwise
        float cs[kRows], sn[kRows];
        if constexpr (R == kRows) {
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                cs[r] = ropeT[r * a.hd + i];
                sn[r] = ropeT[r * a.hd + half + i];
            }
        } else {
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                const size_t o = static_cast<size_t>(rb + r < a.rows ? sh_pos[rb + r] : 0) * half + i;
                cs[r] = __ldg(a.rope_cos + o);
                sn[r] = __ldg(a.rope_sin + o);
            }
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            const float partner = __shfl_xor_sync(0xffffffffu, y[r], 1);
            if (!valid || rb + r >= a.rows) continue;
            float v = y[r];
            if (seg != 2) {
                const float c = cs[r], s = sn[r];
                v = odd ? __fadd_rn(__fmul_rn(partner, s), __fmul_rn(v, c))
                        : __fsub_rn(__fmul_rn(v, c), __fmul_rn(partner, s));
            }
            if (seg == 0) {
                a.q[static_cast<size_t>(rb + r) * a.qd + fl] = v;
            } else {
                const int b = sh_row_bank[rb + r];
                float* dst = (seg == 1 ? a.kbank[b] : a.vbank[b]) + static_cast<size_t>(l) * a.slab_stride +
                             (static_cast<size_t>(fl / a.hd) * a.max_len + sh_row_slot[rb + r]) * a.hd + d;
                *dst = v;
            }
        }
    } else if (p == P_GU) {
        float* ub = xch;  // [64][16]
        if (m >= 64)
#pragma unroll
            for (int r = 0; r < kRows; ++r) ub[(m - 64) * kRows + r] = y[r];
        named_sync(1, 128);
        if (m < 64) {
            const int fg = tile * 64 + m;
            if (fg < a.F)
#pragma unroll
                for (int r = 0; r < kRows; ++r)
                    if (rb + r < a.rows) {
                        const float g = y[r];
                        const float silu = g / (1.0f + expf(-g));
                        const float v = silu * ub[m * kRows + r];
                        a.act[static_cast<size_t>(rb + r) * a.F + fg] = v;
                        put_split<R>(a.xim[P_DOWN], fg, rb + r, v);
                    }
        }
        named_sync(1, 128);
    } else {  // residual add + sum-of-squares partials for the next RMSNorm
        const int f = tile * kM + m;
        if (a.tp > 1) {
            // row-parallel output: swap partial tiles with the peer over NVLink
            // and sum them in rank order (bitwise identical on both GPUs).  Every
            // value travels as ONE 64-bit word {launch epoch, f32 bits}: the
            // receiver polls its own words until they carry this launch's epoch,
            // so no system-scope fence or flag is needed (a __threadfence_system
            // per tile cost 7-10 us: tools/trace_mega_tp.py)
            const int tilesH = (a.H + kM - 1) / kM;
            const size_t slot = (static_cast<size_t>(l) * 2 + (p == P_O ? 0 : 1)) * tilesH + tile;
            const int xid = (p == P_O ? 240 : 248) + (l & 7);  // trace ids of the exchange
            if (a.trace && et == 0) *tslot(a, blockIdx.x, xid, 0) = gtimer();
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(a.peer_inbox) + slot * kRows * kM;
            const unsigned long long tag = static_cast<unsigned long long>(sh_epoch) << 32;
#pragma unroll
            for (int r = 0; r < kRows; ++r)  // static bound: y[] stays in registers
                if (r < a.rows) st_relaxed_sys_u64(dst + r * kM + m, tag | __float_as_uint(y[r]));
            if (a.trace && et == 0) *tslot(a, blockIdx.x, xid, 1) = gtimer();
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.inbox) + slot * kRows * kM;
            float other[kRows];
            unsigned pending = 0;
#pragma unroll
            for (int r = 0; r < kRows; ++r) {
                other[r] = 0.0f;
                if (r < a.rows) {
                    const unsigned long long v = ld_relaxed_sys_u64(src + r * kM + m);
                    if ((v >> 32) == sh_epoch) other[r] = __uint_as_float(static_cast<unsigned>(v));
                    else pending |= 1u << r;
                }
            }
            unsigned long long spins = 0;
            while (pending) {
                __nanosleep(32);
                if (++spins > (1ull << 27)) asm volatile("trap;");  // peer gone: fail, do not hang
#pragma unroll
                for (int r = 0; r < kRows; ++r)
                    if ((pending >> r) & 1u) {
                        const unsigned long long v = ld_relaxed_sys_u64(src + r * kM + m);
                        if ((v >> 32) == sh_epoch) {
                            other[r] = __uint_as_float(static_cast<unsigned>(v));
                            pending &= ~(1u << r);
                        }
                    }
            }
            if (a.trace && et == 0) *tslot(a, blockIdx.x, xid, 3) = gtimer();
#pragma unroll
            for (int r = 0; r < kRows; ++r)
                if (r < a.rows) y[r] = a.tp_rank == 0 ? y[r] + other[r] : other[r] + y[r];
            if (a.trace && et == 0) *tslot(a, blockIdx.x, xid, 4) = gtimer();
        }
        // the next GEMM's input image: split(h * gain) of ffn_norm (after O)
        // or of the next layer's attn_norm (after down; none after the last)
        const float* gn = p == P_O ? L.ffn_norm : L.next_attn_norm;
        uint8_t* img = p == P_O ? a.xim[P_GU] : a.xim[P_QKV];
        cp_async_wait_all();
        const float gf = (gn && f < a.H) ? hpre[R * kM + m] : 0.0f;  // prefetched with the residual
        // residual rows were prefetched into shared memory (cp.async) while
        // the accumulator was still being produced
        cp_async_wait_all();
        if (a.trace && et == 0) *tslot(a, blockIdx.x, input_barrier(l, p), 12) = gtimer();
        float hn[kRows];
#pragma unroll
        for (int r = 0; r < kRows; ++r) hn[r] = (f < a.H && rb + r < a.rows) ? hpre[(rb + r) * kM + m] : 0.0f;
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            if (f < a.H && rb + r < a.rows) {
                hn[r] += y[r];
                a.h[static_cast<size_t>(rb + r) * a.H + f] = hn[r];
                if (gn) put_split<R>(img, f, rb + r, hn[r] * gf);
            }
        }
        float* ss = (p == P_O ? a.ss_o : a.ss_d) + static_cast<size_t>(tile) * R + rb;
        if (a.trace && et == 0) *tslot(a, blockIdx.x, input_barrier(l, p), 13) = gtimer();
        tile_sumsq(hn, xch + 64 * kRows, ss, et);
        if (a.trace && et == 0) *tslot(a, blockIdx.x, input_barrier(l, p), 14) = gtimer();
    }
}

// ── attention for one (row, kv head): flash-decode over the row's visible
// keys with a fixed key partition (chunk i of 32 keys -> warp i % 8).
template <int HD, int GR, int R>  // GR: compile-time bound on the GQA group (register arrays); R: rows per launch
__device__ void attention_row_item(const MegaArgs& a, const LayerDesc& L, int l, int row, int kvh, int at, float* qs,
                               float* wst, float* ocomb, int* cols) {
    const int group = a.n_heads / a.n_kv;
    const int warp = at >> 5, lane = at & 31;
    for (int t = at; t < group * HD; t += 256)
        qs[t] = __ldcg(a.q + static_cast<size_t>(row) * a.qd + static_cast<size_t>(kvh * group) * HD + t);
    // the row's visible keys in compacted order: cache slots [0, prior) then
    // its own tail slots (staged per launch in sh_tail / sh_ncols; the host
    // guarantees every row sees the whole cached prefix, mega_mask_ok)
    const int prior = sh_row_prior[row];
    const int n = sh_ncols[row];
    named_sync(3, 256);  // queries staged
    // NOTE: frame masks carry mval == 0 for every visible column; additive
    // masks (seam 2) take the per-GEMM path (see mega_supported()).
    const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(HD));
    const float* kb = a.kbank[sh_row_bank[row]] + static_cast<size_t>(l) * a.slab_stride +
                      static_cast<size_t>(kvh) * a.max_len * HD;
    const float* vb = a.vbank[sh_row_bank[row]] + static_cast<size_t>(l) * a.slab_stride +
                      static_cast<size_t>(kvh) * a.max_len * HD;
    // A warp takes 8 keys per iteration: 4 lanes per key split the score dot
    // (HD/4 dims each, one batch of loads), then all 32 lanes sweep head
    // dims for the value sum with the 8 value rows loaded up front.
    constexpr int DPL = HD / 32;
    constexpr int Q4 = HD / 16;  // float4 loads per lane per key
    float mrun[GR], lrun[GR], o[GR][DPL];
#pragma unroll
    for (int g = 0; g < GR; ++g) {
        mrun[g] = -INFINITY;
        lrun[g] = 0.0f;
#pragma unroll
        for (int i = 0; i < DPL; ++i) o[g][i] = 0.0f;
    }
    const int kk = lane >> 2, sub = lane & 3;
    const int nchunks = (n + 7) / 8;
    for (int ch = warp; ch < nchunks; ch += 8) {
        const int c = ch * 8 + kk;
        const bool live = c < n;
        const int col = !live ? 0 : (c < prior ? c : sh_tail[row][c - prior]);
        // lane `sub` of a key owns the key's float4 columns sub, sub+4, ...:
        // the 4 lanes of a key read 64 contiguous bytes per load (not 4
        // scattered 16-byte pieces), and their query reads hit 4 banks groups
        const float4* kr = reinterpret_cast<const float4*>(kb + static_cast<size_t>(col) * HD) + sub;
        float4 k4[Q4];
#pragma unroll
        for (int t = 0; t < Q4; ++t) k4[t] = __ldcg(kr + 4 * t);
        float s[GR];
#pragma unroll
        for (int g = 0; g < GR; ++g) {
            s[g] = 0.0f;
            if (g >= group) continue;
            const float4* q4 = reinterpret_cast<const float4*>(qs + g * HD) + sub;
#pragma unroll
            for (int t = 0; t < Q4; ++t) {
                const float4 qq = q4[4 * t];
                s[g] += qq.x * k4[t].x + qq.y * k4[t].y + qq.z * k4[t].z + qq.w * k4[t].w;
            }
            s[g] += __shfl_xor_sync(0xffffffffu, s[g], 1);
            s[g] += __shfl_xor_sync(0xffffffffu, s[g], 2);
        }
        // value rows of the chunk's 8 keys (coalesced over lanes, one batch)
        float v[8][DPL];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int cj = __shfl_sync(0xffffffffu, col, 4 * j);
            const bool lj = ch * 8 + j < n;
#pragma unroll
            for (int i = 0; i < DPL; ++i) v[j][i] = lj ? __ldcg(vb + static_cast<size_t>(cj) * HD + lane + 32 * i) : 0.0f;
        }
#pragma unroll
        for (int g = 0; g < GR; ++g) {
            if (g >= group) break;
            const float sv = live ? s[g] * inv_sqrt_hd : -INFINITY;
            float cm = sv;
            for (int off = 16; off > 2; off >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
            const float mn = fmaxf(mrun[g], cm);
            const float scale_old = mrun[g] == -INFINITY ? 0.0f : expf(mrun[g] - mn);
            const float pr = live ? expf(sv - mn) : 0.0f;
            float ps = sub == 0 ? pr : 0.0f;
            for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
            lrun[g] = lrun[g] * scale_old + ps;
            mrun[g] = mn;
#pragma unroll
            for (int i = 0; i < DPL; ++i) o[g][i] *= scale_old;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float pj = __shfl_sync(0xffffffffu, pr, 4 * j);
#pragma unroll
                for (int i = 0; i < DPL; ++i) o[g][i] += pj * v[j][i];
            }
        }
    }
    // combine the 8 warps in fixed order
#pragma unroll
    for (int g = 0; g < GR; ++g) {
        if (g >= group) break;
        if (lane == 0) {
            wst[(warp * kMaxGroup + g) * 2] = mrun[g];
            wst[(warp * kMaxGroup + g) * 2 + 1] = lrun[g];
        }
#pragma unroll
        for (int i = 0; i < DPL; ++i) ocomb[(warp * group + g) * HD + lane + 32 * i] = o[g][i];
    }
    named_sync(3, 256);
    for (int t = at; t < group * HD; t += 256) {
        const int g = t / HD, dd = t % HD;
        float mx = -INFINITY;
        for (int w = 0; w < 8; ++w) mx = fmaxf(mx, wst[(w * kMaxGroup + g) * 2]);
        float l = 0.0f, acc = 0.0f;
        for (int w = 0; w < 8; ++w) {
            const float mw = wst[(w * kMaxGroup + g) * 2];
            const float sc = mw == -INFINITY ? 0.0f : expf(mw - mx);
            l += wst[(w * kMaxGroup + g) * 2 + 1] * sc;
            acc += ocomb[(w * group + g) * HD + dd] * sc;
        }
        if (mx == -INFINITY) atomicOr(a.status, ST_EMPTY_ROW);
        const int f = (kvh * group + g) * HD + dd;
        const float o = acc / l;
        a.att[static_cast<size_t>(row) * a.qd + f] = o;
        put_split<R>(a.xim[P_O], f, row, o);
    }
    fence_proxy_async_global();
    named_sync(3, 256);
}

template <int R>
__device__ __forceinline__ void attention_rows_dispatch(const MegaArgs& a, const LayerDesc& L, int l, int row, int kvh,
                                                   int at, float* qs, float* wst, float* ocomb, int* cols) {
    const int group = a.n_heads / a.n_kv;
    {  // wait for this kv head's QKV tiles: its q heads, K and V
        const int q0 = kvh * group * a.hd / kM, q1 = ((kvh + 1) * group * a.hd - 1) / kM;
        const int kt = (a.qd + kvh * a.hd) / kM, kt1 = (a.qd + kvh * a.hd + a.hd - 1) / kM;
        const int vt = (a.qd + a.kvd + kvh * a.hd) / kM, vt1 = (a.qd + a.kvd + kvh * a.hd + a.hd - 1) / kM;
        const int nq = q1 - q0 + 1, nk = kt1 - kt + 1, nv = vt1 - vt + 1;
        if (at < nq + nk + nv) {
            const int t = at < nq ? q0 + at : (at < nq + nk ? kt + at - nq : vt + at - nq - nk);
            wait_ge(fptr(a, l, K_QKV, t), 1u);
        }
        named_sync(3, 256);
    }
    if (group <= 4) {
        switch (a.hd) {
            case 64: attention_row_item<64, 4, R>(a, L, l, row, kvh, at, qs, wst, ocomb, cols); break;
            case 128: attention_row_item<128, 4, R>(a, L, l, row, kvh, at, qs, wst, ocomb, cols); break;
            case 160: attention_row_item<160, 4, R>(a, L, l, row, kvh, at, qs, wst, ocomb, cols); break;
            default: attention_row_item<32, 4, R>(a, L, l, row, kvh, at, qs, wst, ocomb, cols); break;
        }
    } else {
        switch (a.hd) {
            case 64: attention_row_item<64, 8, R>(a, L, l, row, kvh, at, qs, wst, ocomb, cols); break;
            default: attention_row_item<32, 8, R>(a, L, l, row, kvh, at, qs, wst, ocomb, cols); break;
        }
    }
    if (at == 0) signal_add(fptr(a, l, K_ATT, kvh), static_cast<unsigned>(a.n_heads / a.n_kv));  // the row's queries are published
}

// ── attention over the KV cache for long contexts (SFG_ATTN=chunked) ─────
// Work item = (kv head, chunk of KC keys in COMPACTED order, group of up to
// 64 queries = rows x the head group's q heads).  The CTA's weight ring is
// idle during the attention phase -- the producer drains it and lends it
// (see lend_ring) -- so an item stages its whole chunk in the ring's shared
// memory with all 256 attention threads issuing cp.async at once (K, the
// queries and the rows' tail slots in one group, V in a second that lands
// while the scores are computed).  K/V are read ONCE per head for all of its
// queries.
//   scores: warp w owns item queries 8w..8w+7, lane owns keys lane + 32j (an
//           8 x KC/32 register tile; K float4 columns XOR-swizzled by key so
//           the 32 lanes' rows hit distinct banks, queries are broadcast);
//   softmax per query over the chunk: fixed butterfly over the lanes;
//   P^T [key][64 queries] overwrites the queries; PV: warp w, lane = head
//           dims lane + 32d, keys in compacted order.
// Compacted index i < prior is cache slot i (shared by every row); i >= prior
// is the row's own tail slot, read from a per-row K/V row with the SAME fmaf
// sequence, so a row's result depends only on its own compacted key list:
// lookahead == sequential bitwise, independent of the batch.  Chunks of a
// head merge in chunk order (last arriver).
template <int HD>
__host__ __device__ constexpr int attn_kc() { return HD <= 128 ? 128 : 64; }
constexpr int kAttnMinKC = 64;  // chunk-slot stride of the partials buffer (smallest KC)
// shared-memory floats an item needs inside the lent ring
__host__ __device__ constexpr int attn_lend_floats(int hd, int kc) {
    return 2 * kc * hd + (64 * hd > kc * 64 ? 64 * hd : kc * 64) + 2 * kRows * hd;
}
// packed fp32 FMA (sm_100 FFMA2): (d0, d1) += (a0, a1) * (b0, b1), each lane an IEEE fma
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{\n.reg .b64 ra, rb, rd;\n"
        "mov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rd, {%0, %1};\n"
        "fma.rn.f32x2 rd, ra, rb, rd;\nmov.b64 {%0, %1}, rd;\n}"
        : "+f"(d0), "+f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// score partials over a float4 of head dims: even dims into se, odd into so
// (the dot product is se + so at the end; one fixed order for every path)
__device__ __forceinline__ void dot4x2(float& se, float& so, const float4 q, const float4 k) {
    ffma2(se, so, q.x, q.y, k.x, k.y);
    ffma2(se, so, q.z, q.w, k.z, k.w);
}

// the kernel's dynamic shared memory, named here so the attention phase
// (a separate, non-inlined function) addresses the lent ring as SHARED
// memory (LDS / STS) instead of through generic pointers
extern __shared__ __align__(1024) uint8_t mega_dyn_smem[];
__device__ __forceinline__ float* ring_base() {
    // 1024-byte aligned (SW128 operands); pointer arithmetic keeps the address space
    const uint32_t mis = static_cast<uint32_t>(__cvta_generic_to_shared(mega_dyn_smem)) & 1023u;
    return reinterpret_cast<float*>(mega_dyn_smem + ((1024u - mis) & 1023u));
}

// publish an item's (m, l, o) rows: one chunk -> the final attention rows and
// O-projection image; several -> partials, then the chunks of this (kv head,
// query group) merge in chunk order, each CTA a slice of the queries
template <int HD, bool kContig = false>  // kContig: lane owns head dims 4 lane .. 4 lane + 3 (else lane + 32 d)
__device__ __forceinline__ void attn_publish(const MegaArgs& a, int l, int kvh, int chunk, int nchunks, int qg, int at,
                                             float* part, float* scratch, const float (&mx)[8], const float (&sm)[8],
                                             const float (&o)[8][HD / 32]) {
    constexpr int DPL = HD / 32;
    const int group = a.n_heads / a.n_kv;
    const int NQ = a.rows * group;
    const int qbase = qg * 64, nq = min(64, NQ - qbase);
    const int warp = at >> 5, lane = at & 31;
    const int q0 = warp * 8;
    const bool wq = q0 < nq;
    // publish: one chunk -> final values; several -> partials, the last chunk merges
    const int cpk = (a.max_len + attn_kc<HD>() - 1) / attn_kc<HD>();  // chunk slots per kv head
    constexpr size_t qstride = HD + 2;
    int qa = 0, qb = nq;  // item queries this CTA finishes
    if (nchunks > 1) {
        // every chunk publishes (m, l, o) partials; once all chunks of this
        // (kv head, query group) have arrived, chunk c merges queries
        // [c * per, (c + 1) * per) over the chunks in chunk order (the merge is
        // spread over the head's CTAs, which all run concurrently: items per
        // head <= grid, mega_supported)
        float* p0 = part + static_cast<size_t>(kvh) * cpk * 128 * qstride;
        float* pc = p0 + static_cast<size_t>(chunk) * 128 * qstride;
        if (wq)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (q0 + i >= nq) continue;
                float* dst = pc + static_cast<size_t>(qbase + q0 + i) * qstride;
                if (lane == 0) {
                    dst[0] = mx[i];
                    dst[1] = sm[i];
                }
#pragma unroll
                for (int d = 0; d < DPL; ++d) dst[2 + (kContig ? 4 * lane + d : lane + 32 * d)] = o[i][d];
            }
        named_sync(3, 256);
        unsigned* cnt = fptr(a, l, K_ATT, a.n_kv + 1 + 2 * kvh + qg);
        if (at == 0) {
            __threadfence();  // cumulative over the CTA's partial stores ordered by the barrier
            atomicAdd(cnt, 1u);
            if (a.trace) *tslot(a, blockIdx.x, 230 + l, 6) = gtimer();
            wait_ge(cnt, static_cast<unsigned>(nchunks));
            if (a.trace) *tslot(a, blockIdx.x, 230 + l, 7) = gtimer();
        }
        named_sync(3, 256);
        const int per = (nq + nchunks - 1) / nchunks;
        qa = min(nq, chunk * per);
        qb = min(nq, qa + per);
        const int nm = qb - qa;
        if (nm > 0) {
            // this thread's first batch of partial o values (<= 2 outputs x 32
            // chunks) is requested BEFORE the (m, l) staging below, so both
            // travel in the same L2 round trip
            float t32[2][32];
            auto load_batch = [&](int t0, int ch0) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int t = t0 + 256 * u, qi = min(t, nm * HD - 1) / HD, dd = t % HD;
                    const float* src = p0 + static_cast<size_t>(qbase + qa + qi) * qstride + 2 + dd;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        t32[u][j] = ch0 + j < nchunks ? __ldcg(src + static_cast<size_t>(ch0 + j) * 128 * qstride) : 0.0f;
                }
            };
            load_batch(at, 0);
            // (m, l) of the merged queries x chunks -> per-chunk weights (the ring is still lent)
            // small scratch outside the ring (nm * nchunks < nq + nchunks <= 128): the
            // tensor-core path has already given the ring back to the producer
            float* sw = scratch;              // [nm][nchunks] (m, then the chunk weights)
            float* sll = sw + 128;            // [nm][nchunks] l
            float* sl = sll + 128;            // [nm] sums
            for (int t = at; t < nm * nchunks; t += 256) {
                const int qi = t / nchunks, ch = t % nchunks;
                const float* src = p0 + (static_cast<size_t>(ch) * 128 + qbase + qa + qi) * qstride;
                sw[t] = __ldcg(src);
                sll[t] = __ldcg(src + 1);
            }
            named_sync(3, 256);
            if (a.trace && at == 0) *tslot(a, blockIdx.x, 230 + l, 9) = gtimer();
            for (int qi = warp; qi < nm; qi += 8) {  // warp per query, lane = chunk (and chunk + 32)
                const int c0 = lane, c1 = lane + 32;
                const float m0 = c0 < nchunks ? sw[qi * nchunks + c0] : -INFINITY;
                const float m1 = c1 < nchunks ? sw[qi * nchunks + c1] : -INFINITY;
                float M = fmaxf(m0, m1);
                for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                const float w0 = m0 == -INFINITY ? 0.0f : expf(m0 - M);
                const float w1 = m1 == -INFINITY ? 0.0f : expf(m1 - M);
                // fixed butterfly over chunk lanes; chunks past the row's keys add exact zeros
                float lsum = fmaf(c0 < nchunks ? sll[qi * nchunks + c0] : 0.0f, w0,
                                  (c1 < nchunks ? sll[qi * nchunks + c1] : 0.0f) * w1);
                for (int off = 16; off > 0; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
                __syncwarp();
                if (c0 < nchunks) sw[qi * nchunks + c0] = w0;
                if (c1 < nchunks) sw[qi * nchunks + c1] = w1;
                if (lane == 0) sl[qi] = lsum;
            }
            named_sync(3, 256);
            if (a.trace && at == 0) *tslot(a, blockIdx.x, 230 + l, 10) = gtimer();
            for (int t0 = at; t0 < nm * HD; t0 += 512) {  // two outputs per thread, all their loads in flight
                float acc2[2] = {0.0f, 0.0f};
                for (int ch0 = 0; ch0 < nchunks; ch0 += 32) {  // chunk order
                    if (t0 != at || ch0 != 0) load_batch(t0, ch0);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int qi = min(t0 + 256 * u, nm * HD - 1) / HD;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (ch0 + j < nchunks) acc2[u] = fmaf(t32[u][j], sw[qi * nchunks + ch0 + j], acc2[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                const int t = t0 + 256 * u;
                if (t >= nm * HD) break;
                const int qi = t / HD, dd = t % HD, q = qbase + qa + qi;
                const float acc = acc2[u];
                const float lsum = sl[qi];
                const int r = q / group, g = q % group;
                if (dd == 0 && !(lsum > 0.0f)) atomicOr(a.status, ST_EMPTY_ROW);
                const float val = acc / lsum;
                const int f = (kvh * group + g) * HD + dd;
                a.att[static_cast<size_t>(r) * a.qd + f] = val;
                put_split<kRows>(a.xim[P_O], f, r, val);
                }
            }
        }
    } else if (wq) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (q0 + i < nq)
#pragma unroll
                for (int d = 0; d < DPL; ++d) {
                    const int q = qbase + q0 + i, r = q / group, g = q % group;
                    const float lsum = sm[i];
                    if (d == 0 && lane == 0 && !(lsum > 0.0f)) atomicOr(a.status, ST_EMPTY_ROW);
                    const float val = fmaf(o[i][d], 1.0f, 0.0f) / lsum;
                    const int f = (kvh * group + g) * HD + (kContig ? 4 * lane + d : lane + 32 * d);
                    a.att[static_cast<size_t>(r) * a.qd + f] = val;
                    put_split<kRows>(a.xim[P_O], f, r, val);
                }
    }
    if (a.trace && at == 0) *tslot(a, blockIdx.x, 230 + l, 11) = gtimer();
    fence_proxy_async_global();
    named_sync(3, 256);
    if (a.trace && at == 0) *tslot(a, blockIdx.x, 230 + l, 12) = gtimer();
    if (at == 0) {  // these queries of this kv head are published
        __threadfence();
        if (qb > qa) atomicAdd(fptr(a, l, K_ATT, kvh), static_cast<unsigned>(qb - qa));
        if (a.trace) *tslot(a, blockIdx.x, 230 + l, 8) = gtimer();
    }
}

template <int HD>
__device__ __noinline__ void attention_tile(const MegaArgs& a, int l, int kvh, int chunk, int nchunks, int qg, int at,
                                            float* part, int xoff) {
    float* ring = ring_base();
    float* sTS = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ring) + xoff);  // [64][16] tail scores (epilogue scratch)
    constexpr int KC = attn_kc<HD>();
    constexpr int KPL = KC / 32;  // keys per lane in the score tile
    constexpr int C4 = HD / 4;    // float4 columns per K / V / query row
    constexpr int DPL = HD / 32;  // head dims per lane in PV
    const int group = a.n_heads / a.n_kv;
    const int NQ = a.rows * group;  // item query q = row * group + g
    const int qbase = qg * 64, nq = min(64, NQ - qbase);
    const int warp = at >> 5, lane = at & 31;
    const int prior = sh_prior;
    const int ncmax = prior + a.rows;  // bound on every row's compacted key count
    const int k0 = chunk * KC, k1 = min(ncmax, k0 + KC);
    const int ns = max(0, min(k1, prior) - k0);  // shared-prefix keys [k0, k0 + ns)
    const int kt0 = max(k0, prior);              // tail indices [kt0, k1)
    float* sK = ring;                 // [KC][C4] float4, column c of key j at c ^ (j & 7)
    float* sV = sK + KC * HD;         // [KC][HD]
    float* sQ = sV + KC * HD;         // [64][HD] queries, then P^T [KC][64] (float4 chunk h of key j at h ^ (j & 15))
    float* sKt = sQ + (64 * HD > KC * 64 ? 64 * HD : KC * 64);  // tail slots prior.. : [kRows][HD]
    float* sVt = sKt + kRows * HD;
    const size_t hoff = static_cast<size_t>(l) * a.slab_stride + static_cast<size_t>(kvh) * a.max_len * HD;
    const float* kbase = a.kbank[0] + hoff;
    const float* vbase = a.vbank[0] + hoff;
    float4* sK4 = reinterpret_cast<float4*>(sK);
    float4* sQ4 = reinterpret_cast<float4*>(sQ);
    for (int t = at; t < ns * C4; t += 256) {
        const int j = t / C4, c4 = t % C4;
        cp_async16(sK4 + j * C4 + (c4 ^ (j & 7)), kbase + static_cast<size_t>(k0 + j) * HD + 4 * c4);
    }
    for (int t = at; t < nq * C4; t += 256) {
        const int qi = t / C4, c4 = t % C4, q = qbase + qi, r = q / group, g = q % group;
        cp_async16(sQ4 + qi * C4 + c4, a.q + static_cast<size_t>(r) * a.qd + static_cast<size_t>(kvh * group + g) * HD + 4 * c4);
    }
    if (k1 > prior)
        for (int t = at; t < a.rows * C4; t += 256) {
            const int j = t / C4, c4 = t % C4;
            cp_async16(reinterpret_cast<float4*>(sKt) + j * C4 + (c4 ^ (j & 7)), kbase + static_cast<size_t>(prior + j) * HD + 4 * c4);
            cp_async16(reinterpret_cast<float4*>(sVt) + t, vbase + static_cast<size_t>(prior + j) * HD + 4 * c4);
        }
    cp_async_commit();
    for (int t = at; t < ns * C4; t += 256)
        cp_async16(reinterpret_cast<float4*>(sV) + t, vbase + static_cast<size_t>(k0) * HD + 4 * t);
    cp_async_commit();
    const bool tr = a.trace && at == 0;
    if (tr) *tslot(a, blockIdx.x, 230 + l, 0) = gtimer();
    cp_async_wait_1();
    named_sync(3, 256);
    if (tr) *tslot(a, blockIdx.x, 230 + l, 1) = gtimer();
    const int q0 = warp * 8;  // this warp's item queries
    const bool wq = q0 < nq;
    float s[8][KPL];
    float mx[8], sm[8];
    if (wq) {
        // shared keys: every query of the warp against the lane's KPL keys
        float so[8][KPL];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < KPL; ++j) s[i][j] = so[i][j] = 0.0f;
#pragma unroll 2
        for (int c = 0; c < C4; ++c) {
            float4 k4[KPL];
#pragma unroll
            for (int j = 0; j < KPL; ++j) k4[j] = sK4[(lane + 32 * j) * C4 + (c ^ (lane & 7))];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float4 q4 = sQ4[(q0 + i) * C4 + c];
#pragma unroll
                for (int j = 0; j < KPL; ++j) dot4x2(s[i][j], so[i][j], q4, k4[j]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < KPL; ++j) s[i][j] += so[i][j];
    }
    // tail keys (compacted indices >= prior, row-specific K rows): every (query,
    // tail) pair by all 256 threads, the SAME dot4x2 sequence as a shared key
    const int ntail = k1 - kt0;
    if (ntail > 0) {
        const float4* sKt4 = reinterpret_cast<const float4*>(sKt);
        for (int pi = at; pi < nq * ntail; pi += 256) {
            const int qi = pi / ntail, t = pi % ntail;
            const int ts = sh_tail[(qbase + qi) / group][min(kt0 - prior + t, kRows - 1)] - prior;  // K rows swizzled by ts
            float acc = 0.0f, acco = 0.0f;
#pragma unroll 4
            for (int c = 0; c < C4; ++c) dot4x2(acc, acco, sQ4[qi * C4 + c], sKt4[ts * C4 + (c ^ (ts & 7))]);
            sTS[qi * 16 + t] = acc + acco;
        }
        named_sync(3, 256);
    }
    if (wq) {
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int ki = k0 + lane + 32 * j;
            if (ki >= kt0 && ki < k1)
#pragma unroll
                for (int i = 0; i < 8; ++i) s[i][j] = sTS[(q0 + i) * 16 + (ki - kt0)];
        }
        const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(HD));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int q = qbase + q0 + i;
            const int nc = q < NQ ? sh_ncols[q / group] : 0;  // the row's compacted key count
            float m = -INFINITY;
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                const int ki = k0 + lane + 32 * j;
                s[i][j] = (ki < k1 && ki < nc) ? s[i][j] * inv_sqrt_hd : -INFINITY;
                m = fmaxf(m, s[i][j]);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
            float sum = 0.0f;
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                const float p = s[i][j] == -INFINITY ? 0.0f : expf(s[i][j] - m);
                s[i][j] = p;
                sum += p;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
            mx[i] = m;
            sm[i] = sum;
        }
    }
    named_sync(3, 256);  // every warp is done with the queries: P^T overwrites them
    if (tr) *tslot(a, blockIdx.x, 230 + l, 2) = gtimer();
    if (wq) {
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int key = lane + 32 * j, sw = key & 15;
            sQ4[key * 16 + ((q0 >> 2) ^ sw)] = make_float4(s[0][j], s[1][j], s[2][j], s[3][j]);
            sQ4[key * 16 + (((q0 >> 2) + 1) ^ sw)] = make_float4(s[4][j], s[5][j], s[6][j], s[7][j]);
        }
    }
    cp_async_wait_all();
    named_sync(3, 256);
    if (tr) *tslot(a, blockIdx.x, 230 + l, 3) = gtimer();
    float o[8][DPL];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int d = 0; d < DPL; ++d) o[i][d] = 0.0f;
    if (wq) {
#pragma unroll 4
        for (int j = 0; j < ns; ++j) {
            const float4 p0 = sQ4[j * 16 + ((q0 >> 2) ^ (j & 15))];
            const float4 p1 = sQ4[j * 16 + (((q0 >> 2) + 1) ^ (j & 15))];
            const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
            float v[DPL];
#pragma unroll
            for (int d = 0; d < DPL; ++d) v[d] = sV[j * HD + lane + 32 * d];
#pragma unroll
            for (int i = 0; i < 8; i += 2)
#pragma unroll
                for (int d = 0; d < DPL; ++d) ffma2(o[i][d], o[i + 1][d], pp[i], pp[i + 1], v[d], v[d]);
        }
        for (int ki = kt0; ki < k1; ++ki) {  // tail keys: each query's own V row
            const int j = ki - k0;
            const float4 p0 = sQ4[j * 16 + ((q0 >> 2) ^ (j & 15))];
            const float4 p1 = sQ4[j * 16 + (((q0 >> 2) + 1) ^ (j & 15))];
            const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = min(qbase + q0 + i, NQ - 1) / group;
                const float* vr = sVt + (sh_tail[r][min(ki - prior, kRows - 1)] - prior) * HD;
#pragma unroll
                for (int d = 0; d < DPL; ++d) o[i][d] = fmaf(pp[i], vr[lane + 32 * d], o[i][d]);
            }
        }
    }
    if (tr) *tslot(a, blockIdx.x, 230 + l, 5) = gtimer();
    attn_publish<HD>(a, l, kvh, chunk, nchunks, qg, at, part, sTS, mx, sm, o);
}

// ── chunked attention, HD = 128: scores on the tensor cores ───────────────
// S^T [128 keys][64 queries] = K Q^T as tcgen05.mma kind::f16 with BOTH
// operands split into three bf16 pieces (hi | mid | lo, ~fp32 accuracy):
// A = the chunk's K pieces (M = 128 key rows), B = the queries' pieces stacked
// along N (rows 0-63 hi, 64-127 mid, 128-191 lo); per K=16 step
//   A_hi x B[hi|mid|lo] (N = 192), A_mid x B[hi|mid] (N = 128), A_lo x B[hi] (N = 64)
// so the three TMEM column blocks hold hi-, mid- and lo-query products and
// S = (blk0 + blk1) + blk2 drops only the 2^-32-scale cross terms.  The
// rows' tail keys (row-specific slots) go through a SECOND pass of the same
// MMAs with the tail K rows in rows 0..15 of the A tile: every (key, query)
// score is the same tensor-core arithmetic whatever the key's position, so a
// row's result still depends only on its own compacted key list.  Softmax
// per query over the chunk (4 threads per query, fixed order) and PV on the
// CUDA cores in compacted key order, as in attention_tile.
// Lent-ring layout: [0, 96 KB) K pieces, later V (fp32) + tail V; [96, 144 KB)
// query pieces, later per-query (m, l); [144, 176 KB) S^T / P^T (float4 chunk
// h of key j at h ^ (j & 15)).
constexpr int kTmS = 128;  // TMEM columns [128, 320): the chunk's score pieces
constexpr int kTmT = 320;  // [320, 512): the tail keys' score pieces
__host__ __device__ constexpr uint32_t attn_idesc(int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}
__shared__ uint32_t sh_attph;  // phase of the attention MMA barrier

// three bf16 pieces of 4 consecutive features (k % 4 == 0) of row r into SW128
// K-major tiles: piece p at base + p * pstride, k-block k / 64 at + kbstride
__device__ __forceinline__ void put3x4(uint8_t* base, uint32_t pstride, uint32_t kbstride, int r, int k, float4 x) {
    const float v[4] = {x.x, x.y, x.z, x.w};
    uint32_t h[2], m[2], lo[2];
#pragma unroll
    for (int e = 0; e < 4; e += 2) {
        __nv_bfloat16 hb[2], mb[2], lb[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            hb[u] = __float2bfloat16_rn(v[e + u]);
            const float r1 = v[e + u] - __bfloat162float(hb[u]);
            mb[u] = __float2bfloat16_rn(r1);
            lb[u] = __float2bfloat16_rn(r1 - __bfloat162float(mb[u]));
        }
        h[e / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(hb[0])) | (static_cast<uint32_t>(__bfloat16_as_ushort(hb[1])) << 16);
        m[e / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(mb[0])) | (static_cast<uint32_t>(__bfloat16_as_ushort(mb[1])) << 16);
        lo[e / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(lb[0])) | (static_cast<uint32_t>(__bfloat16_as_ushort(lb[1])) << 16);
    }
    uint8_t* t = base + (k >> 6) * kbstride + sw128_off(r, k & 63);
    *reinterpret_cast<uint2*>(t) = make_uint2(h[0], h[1]);
    *reinterpret_cast<uint2*>(t + pstride) = make_uint2(m[0], m[1]);
    *reinterpret_cast<uint2*>(t + 2 * pstride) = make_uint2(lo[0], lo[1]);
}

// issue the score MMAs of one pass (thread 0) and wait for them
__device__ __forceinline__ void attn_score_mma(uint32_t kp, uint32_t qp, uint32_t tcol, uint64_t* attb) {
    tc_fence_after();
#pragma unroll
    for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bq = smem_desc(qp + kb * 24576) + 2 * ks;
            const uint64_t ah = smem_desc(kp + kb * 16384) + 2 * ks;
            mma_bf16_id(tcol, ah, bq, attn_idesc(192), (kb | ks) ? 1u : 0u);
            mma_bf16_id(tcol, ah + (32768 >> 4), bq, attn_idesc(128), 1u);
            mma_bf16_id(tcol, ah + (65536 >> 4), bq, attn_idesc(64), 1u);
        }
    mma_commit(attb);
    mwait(attb, sh_attph & 1u);
    ++sh_attph;
}

// wait for kv head kvh's QKV tiles of layer l: its q heads, K and V (all 256 attention threads)
__device__ __forceinline__ void wait_head_qkv(const MegaArgs& a, int l, int kvh, int at) {
    const int group = a.n_heads / a.n_kv;
    const int q0 = kvh * group * a.hd / kM, q1 = ((kvh + 1) * group * a.hd - 1) / kM;
    const int kt = (a.qd + kvh * a.hd) / kM, kt1 = (a.qd + kvh * a.hd + a.hd - 1) / kM;
    const int vt = (a.qd + a.kvd + kvh * a.hd) / kM, vt1 = (a.qd + a.kvd + kvh * a.hd + a.hd - 1) / kM;
    const int nq = q1 - q0 + 1, nk = kt1 - kt + 1, nv = vt1 - vt + 1;
    if (at < nq + nk + nv) {
        const int t = at < nq ? q0 + at : (at < nq + nk ? kt + at - nq : vt + at - nq - nk);
        wait_ge(fptr(a, l, K_QKV, t), 1u);
    }
    named_sync(3, 256);
}

__device__ __noinline__ void attention_tile_tc(const MegaArgs& a, int l, int kvh, int chunk, int nchunks, int qg, int at,
                                               float* part, int xoff, uint32_t tmem, uint64_t* attb, uint64_t* retb,
                                               bool last) {
    constexpr int HD = 128, KC = 128, C4 = 32, DPL = 4;
    uint8_t* ringb = reinterpret_cast<uint8_t*>(ring_base());
    uint8_t* sKp = ringb;                                        // 3 x [2 k-blocks][128 rows][128 B]
    uint8_t* sQp = ringb + 98304;                                // [2 k-blocks][192 rows][128 B]
    float* sV = reinterpret_cast<float*>(ringb);                 // after the MMAs: V [KC][HD] | tail V [kRows][HD]
    float* sVt = sV + KC * HD;
    float* sML = reinterpret_cast<float*>(sQp);                  // after the MMAs: (m, l) per item query
    float4* sP4 = reinterpret_cast<float4*>(ringb + 147456);     // S^T / P^T [KC][16] float4 (swizzled)
    float* sTS = reinterpret_cast<float*>(ringb + xoff);         // [16][64] tail scores (epilogue scratch)
    const int group = a.n_heads / a.n_kv;
    const int NQ = a.rows * group;
    const int qbase = qg * 64, nq = min(64, NQ - qbase);
    const int warp = at >> 5, lane = at & 31;
    const int prior = sh_prior;
    const int ncmax = prior + a.rows;
    const int k0 = chunk * KC, k1 = min(ncmax, k0 + KC);
    const int ns = max(0, min(k1, prior) - k0);
    const int kt0 = max(k0, prior);
    const int ntail = k1 - kt0;
    const size_t hoff = static_cast<size_t>(l) * a.slab_stride + static_cast<size_t>(kvh) * a.max_len * HD;
    const float* kbase = a.kbank[0] + hoff;
    const float* vbase = a.vbank[0] + hoff;
    const bool tr = a.trace && at == 0;
    if (tr) *tslot(a, blockIdx.x, 230 + l, 0) = gtimer();
    // K rows, queries (and tail K rows) into registers, all loads in flight, then
    // split.  (Loading the cached K before this step's QKV tiles are done was
    // measured slower: the loads compete with the QKV weight stream for HBM.)
    wait_head_qkv(a, l, kvh, at);
    if (tr) *tslot(a, blockIdx.x, 230 + l, 14) = gtimer();  // this step's q / K / V tiles are published
    {
        float4 kx[16], qx[8], tx2[2];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int f = at + 256 * i, r = f >> 5, c = f & 31;
            kx[i] = r < ns ? __ldcg(reinterpret_cast<const float4*>(kbase + static_cast<size_t>(k0 + r) * HD) + c)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int f = at + 256 * i;
            put3x4(sKp, 32768, 16384, f >> 5, 4 * (f & 31), kx[i]);
        }
        if (tr) *tslot(a, blockIdx.x, 230 + l, 15) = gtimer();  // thread 0's K rows loaded and split
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int f = at + 256 * i, qi = f >> 5, c = f & 31, q = qbase + qi;
            qx[i] = qi < nq ? __ldcg(reinterpret_cast<const float4*>(a.q + static_cast<size_t>(q / group) * a.qd +
                                                                     static_cast<size_t>(kvh * group + q % group) * HD) + c)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int f = at + 256 * i, r = f >> 5, c = f & 31;
            tx2[i] = ntail > 0 && r < a.rows
                         ? __ldcg(reinterpret_cast<const float4*>(kbase + static_cast<size_t>(prior + r) * HD) + c)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // query qi: B rows qi (hi), 64 + qi (mid), 128 + qi (lo)
            const int f = at + 256 * i;
            put3x4(sQp, 64 * 128, 24576, f >> 5, 4 * (f & 31), qx[i]);
        }
        fence_proxy_async();
        named_sync(3, 256);
        if (tr) *tslot(a, blockIdx.x, 230 + l, 1) = gtimer();
        if (at == 0) attn_score_mma(smem_u32(sKp), smem_u32(sQp), tmem + kTmS, attb);
        named_sync(3, 256);
        if (ntail > 0) {  // second pass: the tail slots' K rows in rows 0..15 of the A tile
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int f = at + 256 * i;
                put3x4(sKp, 32768, 16384, f >> 5, 4 * (f & 31), tx2[i]);
            }
            fence_proxy_async();
            named_sync(3, 256);
            if (at == 0) attn_score_mma(smem_u32(sKp), smem_u32(sQp), tmem + kTmT, attb);
            named_sync(3, 256);
        }
    }
    // V (and the tail V rows) stream in while the scores are read out
    for (int t = at; t < ns * C4; t += 256) cp_async16(reinterpret_cast<float4*>(sV) + t, vbase + static_cast<size_t>(k0) * HD + 4 * t);
    if (ntail > 0)
        for (int t = at; t < a.rows * C4; t += 256)
            cp_async16(reinterpret_cast<float4*>(sVt) + t, vbase + static_cast<size_t>(prior) * HD + 4 * t);
    cp_async_commit();
    tc_fence_after();
    {  // S^T rows: the warp's TMEM lane quadrant = keys, half the queries
        const int quad = (warp + 2) & 3, qh = warp >> 2, key = 32 * quad + lane;
        const uint32_t lb = static_cast<uint32_t>(32 * quad) << 16;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float vh[16], vm[16], vl[16];
            const int qc = 32 * qh + 16 * h;
            tmem_ld16(tmem + lb + kTmS + qc, vh);
            tmem_ld16(tmem + lb + kTmS + 64 + qc, vm);
            tmem_ld16(tmem + lb + kTmS + 128 + qc, vl);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 4; ++c)
                sP4[key * 16 + ((qc / 4 + c) ^ (key & 15))] =
                    make_float4((vh[4 * c] + vm[4 * c]) + vl[4 * c], (vh[4 * c + 1] + vm[4 * c + 1]) + vl[4 * c + 1],
                                (vh[4 * c + 2] + vm[4 * c + 2]) + vl[4 * c + 2], (vh[4 * c + 3] + vm[4 * c + 3]) + vl[4 * c + 3]);
        }
        if (ntail > 0 && quad == 0) {  // tail slot `lane`'s scores (tcgen05.ld is warp-collective)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float vh[16], vm[16], vl[16];
                const int qc = 32 * qh + 16 * h;
                tmem_ld16(tmem + lb + kTmT + qc, vh);
                tmem_ld16(tmem + lb + kTmT + 64 + qc, vm);
                tmem_ld16(tmem + lb + kTmT + 128 + qc, vl);
                tmem_wait_ld();
                if (lane < kRows)
#pragma unroll
                    for (int c = 0; c < 16; ++c) sTS[lane * 64 + qc + c] = (vh[c] + vm[c]) + vl[c];
            }
        }
    }
    tc_fence_before();
    named_sync(3, 256);
    if (ntail > 0) {  // place each query's tail scores at its compacted positions
        for (int pi = at; pi < nq * ntail; pi += 256) {
            const int qi = pi / ntail, t = pi % ntail;
            const int ts = sh_tail[(qbase + qi) / group][min(kt0 - prior + t, kRows - 1)] - prior;
            const int key = ns + t;
            reinterpret_cast<float*>(sP4 + key * 16 + ((qi >> 2) ^ (key & 15)))[qi & 3] = sTS[ts * 64 + qi];
        }
        named_sync(3, 256);
    }
    if (tr) *tslot(a, blockIdx.x, 230 + l, 2) = gtimer();
    {  // softmax: 4 threads per query, keys part + 4 t (fixed order)
        const int qi = at >> 2, part = at & 3, q = qbase + qi;
        const int nc = qi < nq ? sh_ncols[q / group] : 0;
        const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(HD));
        float* sPf = reinterpret_cast<float*>(sP4);
        float sv[32];
        float m = -INFINITY;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int key = part + 4 * t, ki = k0 + key;
            const float x = sPf[(key * 16 + ((qi >> 2) ^ (key & 15))) * 4 + (qi & 3)];
            sv[t] = (ki < k1 && ki < nc) ? x * inv_sqrt_hd : -INFINITY;
            m = fmaxf(m, sv[t]);
        }
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
        float sum = 0.0f;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const int key = part + 4 * t;
            const float p = sv[t] == -INFINITY ? 0.0f : expf(sv[t] - m);
            sPf[(key * 16 + ((qi >> 2) ^ (key & 15))) * 4 + (qi & 3)] = p;
            sum += p;
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (part == 0) {
            sML[2 * qi] = m;
            sML[2 * qi + 1] = sum;
        }
    }
    cp_async_wait_all();
    named_sync(3, 256);
    if (tr) *tslot(a, blockIdx.x, 230 + l, 3) = gtimer();
    const int q0 = warp * 8;
    const bool wq = q0 < nq;
    float mx[8], sm[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        mx[i] = sML[2 * (q0 + i)];
        sm[i] = sML[2 * (q0 + i) + 1];
    }
    float o[8][DPL];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int d = 0; d < DPL; ++d) o[i][d] = 0.0f;
    if (wq) {
#pragma unroll 4
        for (int j = 0; j < ns; ++j) {
            const float4 p0 = sP4[j * 16 + ((q0 >> 2) ^ (j & 15))];
            const float4 p1 = sP4[j * 16 + (((q0 >> 2) + 1) ^ (j & 15))];
            const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
            const float4 v4 = reinterpret_cast<const float4*>(sV + j * HD)[lane];  // dims 4 lane .. + 3
            const float v[DPL] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int i = 0; i < 8; i += 2)
#pragma unroll
                for (int d = 0; d < DPL; ++d) ffma2(o[i][d], o[i + 1][d], pp[i], pp[i + 1], v[d], v[d]);
        }
        for (int ki = kt0; ki < k1; ++ki) {  // tail keys: each query's own V row
            const int j = ki - k0;
            const float4 p0 = sP4[j * 16 + ((q0 >> 2) ^ (j & 15))];
            const float4 p1 = sP4[j * 16 + (((q0 >> 2) + 1) ^ (j & 15))];
            const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = min(qbase + q0 + i, NQ - 1) / group;
                const float* vr = sVt + (sh_tail[r][min(ki - prior, kRows - 1)] - prior) * HD;
#pragma unroll
                for (int d = 0; d < DPL; ++d) o[i][d] = fmaf(pp[i], vr[4 * lane + d], o[i][d]);
            }
        }
    }
    if (tr) *tslot(a, blockIdx.x, 230 + l, 5) = gtimer();
    if (last) {  // the ring is free: give it back now, the merge below only needs the small scratch
        fence_proxy_async();
        named_sync(3, 256);
        if (at == 0) mbar_arrive(retb);
    }
    attn_publish<HD, true>(a, l, kvh, chunk, nchunks, qg, at, part, sTS, mx, sm, o);
}

__device__ __forceinline__ int attn_chunks(const MegaArgs& a) {
    const int kc = a.hd <= 128 ? attn_kc<128>() : attn_kc<160>();
    return (sh_prior + a.rows + kc - 1) / kc;
}
__device__ __forceinline__ int attention_items(const MegaArgs& a, int nchunks) {
    const int nqg = (a.rows * (a.n_heads / a.n_kv) + 63) / 64;
    return a.n_kv * nchunks * nqg;
}
__device__ __forceinline__ void attention_dispatch(const MegaArgs& a, int l, int item, int nchunks, int at, float* part,
                                                   int xoff, uint32_t tmem, uint64_t* attb, uint64_t* retb, bool last) {
    const int group = a.n_heads / a.n_kv;
    const int nqg = (a.rows * group + 63) / 64;
    const int kvh = item / (nchunks * nqg), rem = item % (nchunks * nqg), chunk = rem / nqg, qg = rem % nqg;
    if (a.hd == 128) {  // the tensor-core path stages the cached K before it waits for this step's QKV
        attention_tile_tc(a, l, kvh, chunk, nchunks, qg, at, part, xoff, tmem, attb, retb, last);
        return;
    }
    {  // wait for this kv head's QKV tiles: its q heads, K and V
        const int q0 = kvh * group * a.hd / kM, q1 = ((kvh + 1) * group * a.hd - 1) / kM;
        const int kt = (a.qd + kvh * a.hd) / kM, kt1 = (a.qd + kvh * a.hd + a.hd - 1) / kM;
        const int vt = (a.qd + a.kvd + kvh * a.hd) / kM, vt1 = (a.qd + a.kvd + kvh * a.hd + a.hd - 1) / kM;
        const int nq = q1 - q0 + 1, nk = kt1 - kt + 1, nv = vt1 - vt + 1;
        if (at < nq + nk + nv) {
            const int t = at < nq ? q0 + at : (at < nq + nk ? kt + at - nq : vt + at - nq - nk);
            wait_ge(fptr(a, l, K_QKV, t), 1u);
        }
        named_sync(3, 256);
    }
    switch (a.hd) {
        case 32: attention_tile<32>(a, l, kvh, chunk, nchunks, qg, at, part, xoff); break;
        case 64: attention_tile<64>(a, l, kvh, chunk, nchunks, qg, at, part, xoff); break;
        case 160: attention_tile<160>(a, l, kvh, chunk, nchunks, qg, at, part, xoff); break;
        default: attention_tile<128>(a, l, kvh, chunk, nchunks, qg, at, part, xoff); break;
    }
}
// the chunked design's attention phase of layer l for the attention threads
// (warps 2..9): wait for the lent ring, run this CTA's items, give it back
__device__ __forceinline__ void attention_phase_lent(const MegaArgs& a, int l, int at, uint64_t* lentb, uint64_t* retb,
                                                     int xoff, uint32_t tmem, uint64_t* attb) {
    if (at == 0) mwait(lentb, static_cast<uint32_t>(l & 1));
    named_sync(3, 256);
    const int nchunks = attn_chunks(a);
    const int items = attention_items(a, nchunks);
    bool returned = false;  // the tensor-core path returns the ring after its last item's PV
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const bool last = it + static_cast<int>(gridDim.x) >= items;
        attention_dispatch(a, l, it, nchunks, at, a.apart, xoff, tmem, attb, retb, last);
        returned = returned || (last && a.hd == 128);
    }
    if (!returned) {
        fence_proxy_async();  // generic-proxy ring accesses before the producer's bulk copies
        named_sync(3, 256);
        if (at == 0) mbar_arrive(retb);
    }
}

// A CTA's walk over its weight units: (layer, phase, unit) in stream order.
struct Cursor {
    int l, p;
    int u, en;
};
__device__ __forceinline__ void cursor_norm(const MegaArgs& a, int c, Cursor& k) {
    while (k.l < a.nlayers && k.u >= k.en) {
        if (++k.p == 4) {
            k.p = 0;
            ++k.l;
        }
        if (k.l >= a.nlayers) break;
        int st, en;
        unit_range(geom(a, k.p), c, st, en);
        k.u = st;
        k.en = en;
    }
}
__device__ __forceinline__ void cursor_begin(const MegaArgs& a, int c, Cursor& k) {
    k.l = 0;
    k.p = 0;
    unit_range(geom(a, 0), c, k.u, k.en);
    cursor_norm(a, c, k);
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// prefetch the cursor's unit into L2 and advance
__device__ __forceinline__ void cursor_prefetch_next(const MegaArgs& a, int c, Cursor& k) {
    if (k.l >= a.nlayers) return;
    prefetch_l2(a.layers[k.l].w[k.p] + static_cast<size_t>(k.u) * kABytes, kABytes);
    ++k.u;
    cursor_norm(a, c, k);
}

// shared-memory floats of the attention scratch: the larger of the two layouts
__host__ __device__ __forceinline__ int attn_scratch_floats(bool rows_attn, int hd, int group, int max_len) {
    // the chunked design stages its items in the lent weight ring (attention_tile)
    return rows_attn ? kMaxGroup * hd + 8 * kMaxGroup * 2 + 8 * group * hd : 0;
}

// ── the kernel ────────────────────────────────────────────────────────────
// 10 warps, one CTA per SM: 3 warps share an SM sub-partition's 16K
// registers, so 168 registers per thread is the ceiling
// kRowsAttn: which attention design this instantiation carries (MegaArgs::attn_rows)
// RR: rows per launch (16, or 32 for cross-session passes; compile time so the
// 16-row path keeps its constant-folded addressing)
template <bool kRowsAttn, int RR>
__global__ void __launch_bounds__(kThreads, 1) mega_kernel(const __grid_constant__ MegaArgs a) {
    uint8_t* smem = reinterpret_cast<uint8_t*>(ring_base());
    const int S = a.stages;
    const int SB = a.stage_bytes;  // [16 KB weights | 3R x 64 activation image] per stage
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * SB);
    uint64_t* empty = full + kMaxStages;
    uint64_t* tfull = empty + kMaxStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* lentb = tempty + 2;  // chunked attention: ring lent to the attention phase / given back
    uint64_t* retb = lentb + 1;
    uint64_t* attb = retb + 1;     // chunked attention: score MMAs complete
    // (one pad slot: the scratch below stays 16-byte aligned for float4 / cp.async)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(attb + 2);
    int* flag = reinterpret_cast<int*>(tmem_slot + 4);
    float* xch = reinterpret_cast<float*>(flag + 4);          // 64*16 gate|up + 4*16 sumsq
    float* rs = xch + 64 * kRows + 4 * kRows;                  // [kMaxRows] per-row 1/rms of the phase
    // attention scratch of the per-row design (the chunked design uses the lent ring)
    float* qs = rs + kMaxRows;                                 // per-row: [group][hd] queries
    float* wst = qs + kMaxGroup * a.hd;                        //   [8][kMaxGroup][2] warp stats
    float* ocomb = wst + 8 * kMaxGroup * 2;                    //   [8][group][hd] warp partials
    int* cols = reinterpret_cast<int*>(ocomb + 8 * (a.n_heads / a.n_kv) * a.hd);  //   [max_len]
    float* ropeT = rs + kMaxRows + attn_scratch_floats(kRowsAttn, a.hd, a.n_heads / a.n_kv, a.max_len);  // [16][hd] cos | sin (R = 16)
    float* hpre = ropeT + (RR == kRows ? kRows * a.hd : 0);     // [R][128] residual prefetch + gain row

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;
    if (threadIdx.x == 0 && (smem_u32(xch) & 15u)) asm volatile("trap;");  // float4 / cp.async scratch alignment
    if (threadIdx.x == 0 && a.trace) *tslot(a, c, kBarSlots - 1, 0) = gtimer();
    if (threadIdx.x < kMaxRows) sh_pos[threadIdx.x] = static_cast<int>(threadIdx.x) < a.rows ? a.pos[threadIdx.x] : 0;
    for (int i = threadIdx.x; RR == kRows && i < kRows * a.hd; i += blockDim.x) {  // RoPE table rows (host-libm values)
        const int r = i / a.hd, j = i % a.hd, half = a.hd >> 1;
        float v = j < half ? 1.0f : 0.0f;
        if (r < a.rows) {
            const size_t o = static_cast<size_t>(a.pos[r]) * half + (j < half ? j : j - half);
            v = j < half ? a.rope_cos[o] : a.rope_sin[o];
        }
        ropeT[i] = v;
    }
    if (threadIdx.x == 0) sh_prior = *a.prior;
    if (threadIdx.x == 0) sh_epoch = a.tp > 1 ? *a.epoch_ptr + 1u : 0u;
    for (int i = threadIdx.x; i < a.nlayers; i += blockDim.x) sh_layers[i] = a.layers[i];
    if (threadIdx.x < kMaxRows) {  // per-row cache, slot and compacted key list (mega_mask_ok)
        const int r = threadIdx.x;
        int prior = *a.prior, bank = 0, slot = prior + r;
        if (a.rowinfo && r < a.rows) {
            bank = a.rowinfo[3 * r];
            slot = a.rowinfo[3 * r + 1];
            prior = a.rowinfo[3 * r + 2];
        }
        sh_row_bank[r] = bank;
        sh_row_slot[r] = slot;
        sh_row_prior[r] = prior;
        int n = 0;
        if (r < a.rows)
            for (int i = a.row_off[r]; i < a.row_off[r + 1]; ++i) {
                const MaskRun rr = a.runs[i];
                for (int col = max(rr.start, prior); col < rr.end && n < kRows; ++col) sh_tail[r][n++] = col;
            }
        for (int j = n; j < kRows; ++j) sh_tail[r][j] = prior;
        sh_ncols[r] = r < a.rows ? prior + n : 0;
    }
    // the ring is walked in PAIRS of stages: one full / empty barrier per pair
    // (two consecutive units of a phase segment), so the MMA issuer waits and
    // commits once per 32 KB of weights instead of once per 16 KB (each wait +
    // commit costs the single issuing thread ~90 ns, tools/mb_issue.cu)
    const int NP = S / 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NP; ++s) {
            mbar_init(&full[s], 2);   // weight bytes + activation bytes (two expect_tx arrivals)
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        mbar_init(lentb, 1);
        mbar_init(retb, 1);
        mbar_init(attb, 1);
        sh_attph = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int tilesH = (a.H + kM - 1) / kM;

    if (warp == 0) {
        if (lane == 0) {  // ── weight producer
            int stage = 0;
            uint32_t ph = 0;
            // L2 prefetch cursor a.pf units ahead of the copies: while the
            // ring is full (grid barriers, attention, epilogue tails) HBM keeps
            // streaming upcoming weights into L2
            const uint64_t pol = l2_evict_first_policy();
            Cursor pf{0, 0, 0, 0};
            cursor_begin(a, c, pf);
            for (int i = 0; i < a.pf; ++i) cursor_prefetch_next(a, c, pf);
            // bubble prefetch: while the ring stays full for longer than a
            // steady-state refill (grid-wide dependencies, attention, epilogue
            // tails), prefetch the next units into L2 so HBM keeps streaming
            Cursor bp{0, 0, 0, 0};
            cursor_begin(a, c, bp);
            int n_cur = 0, n_bp = 0;
            for (int l = 0; l < a.nlayers; ++l)
                for (int p = 0; p < 4; ++p) {
                    const Geo g = geom(a, p);
                    const uint8_t* W = a.layers[l].w[p];
                    unsigned long long wacc = 0;
                    for (int sg = 0; sg < 2; ++sg) {
                    int st, en;
                    unit_seg(g, c, sg, st, en);
                    for (int u = st; u < en; u += 2, n_cur += 2) {
                        const int n = min(2, en - u);
                        if (a.bpf > 0) {
                            if (!mbar_test(&empty[stage], ph ^ 1)) {
                                const long long t0 = clock64();
                                unsigned long long spins = 0;
                                while (!mbar_test(&empty[stage], ph ^ 1)) {
                                    if (clock64() - t0 > a.bpf_cycles) {
                                        while (n_bp < n_cur && bp.l < a.nlayers) {  // already being loaded
                                            ++bp.u;
                                            cursor_norm(a, c, bp);
                                            ++n_bp;
                                        }
                                        if (n_bp < n_cur + a.bpf && bp.l < a.nlayers) {
                                            cursor_prefetch_next(a, c, bp);
                                            ++n_bp;
                                        }
                                    }
                                    __nanosleep(20);
                                    if (++spins > (1ull << 30)) asm volatile("trap;");
                                }
                            }
                        } else {
                            mwait_acc(&empty[stage], ph ^ 1, a.trace != nullptr, wacc);
                        }
                        if (a.noload & 1) {
                            mbar_arrive(&full[stage]);
                        } else {
                            mbar_expect_tx(&full[stage], n * kABytes);
                            for (int h = 0; h < n; ++h) {
                                uint8_t* dst = smem + (2 * stage + h) * SB;
                                const uint8_t* src = W + static_cast<size_t>(u + h) * kABytes;
                                if (a.evict_first)
                                    bulk_g2s_stream(dst, src, kABytes, &full[stage], pol);
                                else
                                    bulk_g2s(dst, src, kABytes, &full[stage]);
                            }
                        }
                        for (int h = 0; h < n; ++h)
                            if (a.pf) cursor_prefetch_next(a, c, pf);
                        if (++stage == NP) {
                            stage = 0;
                            ph ^= 1;
                        }
                    }
                    }
                    if (a.trace) *tslot(a, c, input_barrier(l, p), 5) = wacc;
                    if (!kRowsAttn && p == P_QKV) {
                        // lend the whole ring to the attention phase: wait until
                        // every pair is consumed (no copy in flight), hand it
                        // over, and on its return complete the lent pairs with
                        // plain arrivals (the MMA issuer skips them)
                        int st2 = stage;
                        uint32_t ph2 = ph;
                        for (int i = 0; i < NP; ++i) {
                            mwait(&empty[st2], ph2 ^ 1);
                            if (++st2 == NP) {
                                st2 = 0;
                                ph2 ^= 1;
                            }
                        }
                        mbar_arrive(lentb);
                        mwait_sleep(retb, static_cast<uint32_t>(l & 1));
                        for (int i = 0; i < NP; ++i) {
                            mbar_arrive(&full[stage]);
                            mbar_arrive(&full[stage]);
                            if (++stage == NP) {
                                stage = 0;
                                ph ^= 1;
                            }
                        }
                    }
                }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ── MMA issuer
            int stage = 0, acc = 0;
            uint32_t ph = 0, acc_ph = 0;
            const uint32_t ring0 = smem_u32(smem);
            for (int l = 0; l < a.nlayers; ++l)
                for (int p = 0; p < 4; ++p) {
                    const Geo g = geom(a, p);
                    unsigned long long wacc = 0, tacc = 0;
                    bool mfirst = false;
                    for (int sg = 0; sg < 2; ++sg) {
                    int st, en;
                    unit_seg(g, c, sg, st, en);
                    int t = st / max(g.KB, 1), kb = st - t * g.KB;
                    int lo = kb, hi = min(en - t * g.KB, g.KB);
                    for (int u = st; u < en; ++u) {
                        const int half = (u - st) & 1;
                        if (kb == lo) {  // a new tile: its accumulator must be drained
                            mwait_acc(&tempty[acc], acc_ph ^ 1, a.trace != nullptr, tacc);
                            if (a.trace && !mfirst) {
                                mfirst = true;
                                *tslot(a, c, input_barrier(l, p), 16) = gtimer();
                            }
                            tc_fence_after();
                        }
                        if (half == 0) {  // one wait per pair of units
                            if (a.spin_mma) {
                                unsigned long long sp = 0;
                                while (!mbar_test(&full[stage], ph))
                                    if (++sp > (1ull << 30)) asm volatile("trap;");
                            } else {
                                mwait_acc(&full[stage], ph, a.trace != nullptr, wacc);
                            }
                            tc_fence_after();
                        }
                        const uint32_t sa = ring0 + static_cast<uint32_t>((2 * stage + half) * SB);
                        const uint64_t da = smem_desc(sa), db = smem_desc(sa + kABytes);
                        const uint32_t d = tmem + acc * a.acc_cols;
#pragma unroll
                        for (int k = 0; k < kKB / 16; ++k) mma_bf16_id(d, da + 2 * k, db + 2 * k, a.idesc, (kb > lo || k > 0) ? 1u : 0u);
                        if (half == 1 || u + 1 == en) {  // the pair is consumed: release it
                            mma_commit(&empty[stage]);
                            if (++stage == NP) {
                                stage = 0;
                                ph ^= 1;
                            }
                        }
                        if (++kb == hi) {  // the tile's last unit of this range
                            mma_commit(&tfull[acc]);
                            if (++acc == 2) {
                                acc = 0;
                                acc_ph ^= 1;
                            }
                            ++t;
                            kb = lo = 0;
                            hi = min(en - t * g.KB, g.KB);
                        }
                    }
                    }
                    if (a.trace) {
                        *tslot(a, c, input_barrier(l, p), 4) = wacc;
                        *tslot(a, c, input_barrier(l, p), 17) = gtimer();
                        *tslot(a, c, input_barrier(l, p), 18) = tacc;
                    }
                    if (!kRowsAttn && p == P_QKV) {  // the lent pairs: nothing to multiply
                        for (int i = 0; i < NP; ++i) {
                            mwait_sleep(&full[stage], ph);
                            mbar_arrive(&empty[stage]);
                            if (++stage == NP) {
                                stage = 0;
                                ph ^= 1;
                            }
                        }
                    }
                }
        }
    } else if (warp < 6) {  // ── epilogue warps 2..5 (+ attention)
        const int q = warp & 3, m = q * 32 + lane, et = threadIdx.x - 64;
        // input statistics: sum-of-squares partials of h for the first RMSNorm,
        // and the first QKV GEMM's input image split(h * attn_norm)
        for (int t = c; t < tilesH; t += G) {
            const int f = t * kM + m;
            const float gf = f < a.H ? __ldg(sh_layers[0].attn_norm + f) : 0.0f;
            for (int rb = 0; rb < RR; rb += kRows) {  // 16-row blocks (every block: the ss rows of padding are 0)
                float hv[kRows];
#pragma unroll
                for (int r = 0; r < kRows; ++r) {
                    const bool ok = f < a.H && rb + r < a.rows;
                    hv[r] = ok ? __ldcg(a.h + static_cast<size_t>(rb + r) * a.H + f) : 0.0f;
                    if (ok) put_split<RR>(a.xim[P_QKV], f, rb + r, hv[r] * gf);
                }
                tile_sumsq(hv, xch + 64 * kRows, a.ss_d + static_cast<size_t>(t) * RR + rb, et);
            }
            fence_proxy_async_global();
            named_sync(1, 128);
            if (et == 0) {
                __threadfence();
                red_add(fptr(a, 0, K_STATS, t), 1u);
                red_add(fptr(a, 0, K_STATS, tilesH), 1u);
            }
        }
        if (a.trace && et == 0) *tslot(a, c, 0, 2) = gtimer();
        int acc = 0;
        uint32_t acc_ph = 0;
        int gp = 0;  // running phase index: stream-K partial buffers alternate by its parity
        for (int l = 0; l < a.nlayers; ++l) {
            const LayerDesc& L = sh_layers[l];
            for (int p = 0; p < 4; ++p, ++gp) {
                const Geo g = geom(a, p);
                const int U = g.split_units();  // stream-K part (seg 0)
                const int kind = K_QKV + (p == P_QKV ? 0 : p + 1);
                float* parts = a.partials + (gp & 1) * a.part_stride;
                int* cnts = a.counters + (gp & 1) * a.cnt_stride;
                int s0, e0, s1, e1;
                unit_seg(g, c, 0, s0, e0);
                unit_seg(g, c, 1, s1, e1);
                const bool any = s0 < e0 || s1 < e1;
                if ((p == P_QKV || p == P_GU) && any) {  // per-row 1/rms: needs every producer tile
                    if (et == 0)
                        wait_ge(p == P_QKV ? (l == 0 ? fptr(a, 0, K_STATS, tilesH) : fptr(a, l - 1, K_DOWN, tilesH))
                                           : fptr(a, l, K_O, tilesH),
                                static_cast<unsigned>(tilesH));
                    named_sync(1, 128);
                    for (int rb = 0; rb < RR; rb += kRows) {  // 8 threads per row, fixed-order combine
                        {
                            const float* ssb = p == P_QKV ? a.ss_d : a.ss_o;
                            const int r = et & 15, j = et >> 4;
                            float part = 0.0f;
                            for (int t = j; t < tilesH; t += 8) part += __ldcg(ssb + t * RR + rb + r);
                            xch[j * kRows + r] = part;
                        }
                        named_sync(1, 128);
                        if (et < kRows) {
                            float ss = 0.0f;
#pragma unroll
                            for (int j = 0; j < 8; ++j) ss += xch[j * kRows + et];
                            rs[rb + et] = 1.0f / sqrtf(ss / static_cast<float>(a.H) + a.eps);
                        }
                        named_sync(1, 128);
                    }
                }
                if ((p == P_O || p == P_DOWN) && any) {  // residual rows of this phase are final
                    if (et == 0) {
                        if (p == P_DOWN) wait_ge(fptr(a, l, K_O, tilesH), static_cast<unsigned>(tilesH));
                        else if (l > 0) wait_ge(fptr(a, l - 1, K_DOWN, tilesH), static_cast<unsigned>(tilesH));
                    }
                    named_sync(1, 128);
                }
                unsigned long long t_acc = 0;
                for (int sg = 0; sg < 2; ++sg) {
                const int st = sg ? s1 : s0, en = sg ? e1 : e0;
                for (int u = st; u < en;) {
                    const int t = static_cast<int>(u / g.KB);
                    const int lo = u - t * g.KB;
                    const int hi = min(en - t * g.KB, g.KB);
                    if (p == P_O || p == P_DOWN) {  // prefetch this tile's residual rows while the MMA runs
                        cp_async_wait_all();   // a previous (unused) prefetch must not land late
                        const int f = t * kM + m;
                        const float* gn = p == P_O ? L.ffn_norm : L.next_attn_norm;
                        if (f < a.H) {
                            for (int r = 0; r < a.rows; ++r) cp_async4(hpre + r * kM + m, a.h + static_cast<size_t>(r) * a.H + f);
                            if (gn) cp_async4(hpre + RR * kM + m, gn + f);
                        }
                        cp_async_commit();
                    }
                    mwait(&tfull[acc], acc_ph);
                    if (a.trace && et == 0) t_acc = gtimer();
                    tc_fence_after();
                    const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * a.acc_cols;
                    const int nblk = RR == kRows ? 1 : (a.rows + kRows - 1) / kRows;  // 16-row blocks that hold rows
                    // block rb of feature m: (hi + mid) + lo, the accumulator columns rb, R + rb, 2R + rb
                    auto load_block = [&](int rb, float (&y)[kRows]) {
                        float v[kN];
                        tmem_ld16(ta + rb, v);
                        tmem_ld16(ta + RR + rb, v + 16);
                        tmem_ld16(ta + 2 * RR + rb, v + 32);
                        tmem_wait_ld();
#pragma unroll
                        for (int r = 0; r < kRows; ++r) y[r] = (v[r] + v[kRows + r]) + v[2 * kRows + r];
                    };
                    auto release = [&]() {  // the accumulator is read: the MMA may reuse it
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[acc]);
                        if (++acc == 2) {
                            acc = 0;
                            acc_ph ^= 1;
                        }
                    };
                    bool done_tile = false;
                    if (lo == 0 && hi == g.KB) {
                        for (int bk = 0; bk < nblk; ++bk) {
                            float y[kRows];
                            load_block(bk * kRows, y);
                            if (bk == nblk - 1) release();
                            epi_final<RR>(a, L, l, p, t, m, et, y, xch, rs, ropeT, hpre, bk * kRows);
                        }
                        done_tile = true;
                    } else {  // stream-K fixup: last arriver sums the pieces in k order
                        const int first_u = t * g.KB;
                        const int c_first = static_cast<int>(((first_u + 1) * g.G - 1) / U);
                        const int piece = c - c_first;
                        const int n_pieces = static_cast<int>(((first_u + g.KB) * g.G - 1) / U) - c_first + 1;
                        float* slot = parts + (static_cast<size_t>(t) * kMaxPieces + piece) * RR * kM;
                        for (int bk = 0; bk < nblk; ++bk) {
                            float y[kRows];
                            load_block(bk * kRows, y);
#pragma unroll
                            for (int r = 0; r < kRows; ++r) slot[(bk * kRows + r) * kM + m] = y[r];
                        }
                        release();
                        __threadfence();
                        if (a.trace && et == 0) *tslot(a, c, input_barrier(l, p), 8) = gtimer();
                        named_sync(1, 128);
                        if (et == 0) {
                            const int old = atomicAdd(&cnts[t], 1);
                            *flag = (old == n_pieces - 1) ? 1 : 0;
                            if (old == n_pieces - 1) cnts[t] = 0;
                        }
                        named_sync(1, 128);
                        if (*flag) {
                            if (a.trace && et == 0) *tslot(a, c, input_barrier(l, p), 9) = gtimer();
                            __threadfence();
                            const float* p0 = parts + static_cast<size_t>(t) * kMaxPieces * RR * kM;
                            for (int bk = 0; bk < nblk; ++bk) {
                                const int rb = bk * kRows;
                                float sacc[kRows];
                                // pieces in k order; the loads of 4 pieces are in flight together
                                for (int pc0 = 0; pc0 < n_pieces; pc0 += 4) {
                                    float t4[4][kRows];
#pragma unroll
                                    for (int j = 0; j < 4; ++j)
#pragma unroll
                                        for (int r = 0; r < kRows; ++r)
                                            t4[j][r] = pc0 + j < n_pieces
                                                           ? __ldcg(p0 + (static_cast<size_t>(pc0 + j) * RR + rb + r) * kM + m)
                                                           : 0.0f;
#pragma unroll
                                    for (int j = 0; j < 4; ++j) {
                                        if (pc0 + j >= n_pieces) break;
#pragma unroll
                                        for (int r = 0; r < kRows; ++r) sacc[r] = (pc0 + j == 0) ? t4[j][r] : sacc[r] + t4[j][r];
                                    }
                                }
                                if (a.trace && et == 0) *tslot(a, c, input_barrier(l, p), 10) = gtimer();
                                epi_final<RR>(a, L, l, p, t, m, et, sacc, xch, rs, ropeT, hpre, rb);
                            }
                            if (a.trace && et == 0) *tslot(a, c, input_barrier(l, p), 11) = gtimer();
                            done_tile = true;
                        }
                    }
                    if (done_tile) {  // publish the tile: outputs, next input image, ss partials
                        fence_proxy_async_global();
                        named_sync(1, 128);
                        if (et == 0) {  // one fence publishes both the tile flag and the phase count
                            __threadfence();
                            red_add(fptr(a, l, kind, t), 1u);
                            red_add(fptr(a, l, kind, g.tiles), 1u);
                        }
                    } else {
                        named_sync(1, 128);
                    }
                    u = t * g.KB + hi;
                }
                }
                if (a.trace && et == 0) {
                    const int id = 5 * l + (p == P_QKV ? 1 : p + 2);
                    *tslot(a, c, input_barrier(l, p), 7) = gtimer();
                    *tslot(a, c, id, 2) = gtimer();
                    *tslot(a, c, input_barrier(l, p), 6) = t_acc;
                }
                if (p == P_QKV) {  // attention, shared with the activation warps
                    if constexpr (kRowsAttn) {
                        for (int it = c; it < a.rows * a.n_kv; it += G)
                            attention_rows_dispatch<RR>(a, L, l, it / a.n_kv, it % a.n_kv, threadIdx.x - 64, qs, wst,
                                                    ocomb, cols);
                    } else {
                        attention_phase_lent(a, l, threadIdx.x - 64, lentb, retb, static_cast<int>(reinterpret_cast<uint8_t*>(xch) - smem),
                                             tmem, attb);
                    }
                    if (a.trace && et == 0) *tslot(a, c, 5 * l + 2, 2) = gtimer();
                }
            }
        }
    } else {  // ── activation loader (warp 6) + attention (warps 6..9)
        const int xt = threadIdx.x - 192;
        int stage = 0;
        uint32_t ph = 0;
        for (int l = 0; l < a.nlayers; ++l) {
            const LayerDesc& L = sh_layers[l];
            for (int p = 0; p < 4; ++p) {
                if (warp == 6) {
                    // one bulk copy per stage of the unit's k-block of the prebuilt
                    // input image, as soon as the producer tiles of that block are
                    // published (the 32 lanes poll the next 32 units' flags at once)
                    const Geo g = geom(a, p);
                    const uint8_t* X = a.xim[p];
                    unsigned long long xwacc = 0;
                    bool first = true;
                    for (int sg = 0; sg < 2; ++sg) {
                    int st, en;
                    unit_seg(g, c, sg, st, en);
                    int ready = st;
                    for (int u = st; u < en; u += 2) {
                        const int n = min(2, en - u);
                        if (u + n > ready) {
                            unsigned long long spins = 0;
                            while (u + n > ready) {
                                const int uu = ready + lane;
                                const bool ok = uu >= en || (a.noload & 4) || xblock_ready(a, l, p, static_cast<int>(uu % g.KB));
                                const unsigned mk = __ballot_sync(0xffffffffu, ok);
                                const int k = mk == 0xffffffffu ? 32 : __ffs(~mk) - 1;
                                ready += k;
                                if (k == 0) {
                                    __nanosleep(32);
                                    if (++spins > (1ull << 27)) asm volatile("trap;");
                                }
                            }
                            if (lane == 0) fence_proxy_async_global();
                            if (first && a.trace && lane == 0) *tslot(a, c, input_barrier(l, p), 0) = gtimer();
                            first = false;
                        }
                        if (lane == 0) {
                            mwait_acc(&empty[stage], ph ^ 1, a.trace != nullptr, xwacc);
                            if (a.noload & 2) {
                                mbar_arrive(&full[stage]);
                            } else {
                                mbar_expect_tx(&full[stage], n * a.xbytes);
                                for (int h = 0; h < n; ++h)
                                    bulk_g2s(smem + (2 * stage + h) * SB + kABytes,
                                             X + static_cast<size_t>((u + h) % g.KB) * a.xbytes, a.xbytes, &full[stage]);
                            }
                        }
                        if (++stage == NP) {
                            stage = 0;
                            ph ^= 1;
                        }
                    }
                    }
                    if (a.trace && lane == 0) {
                        *tslot(a, c, input_barrier(l, p), 1) = gtimer();
                        *tslot(a, c, input_barrier(l, p), 3) = xwacc;
                    }
                    if (!kRowsAttn && p == P_QKV) ph ^= 1;  // the lent pairs (one whole wrap of the ring)
                    __syncwarp();
                }
                if (p == P_QKV) {  // join the attention phase
                    if constexpr (kRowsAttn) {
                        for (int it = c; it < a.rows * a.n_kv; it += G)
                            attention_rows_dispatch<RR>(a, L, l, it / a.n_kv, it % a.n_kv, threadIdx.x - 64, qs, wst,
                                                    ocomb, cols);
                    } else {
                        attention_phase_lent(a, l, threadIdx.x - 64, lentb, retb, static_cast<int>(reinterpret_cast<uint8_t*>(xch) - smem),
                                             tmem, attb);
                    }
                }
            }
        }
        (void)xt;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_free(tmem, a.tmem_cols);
    }
    // last CTA out resets the dataflow flags and the exit counter for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        *flag = atomicAdd(a.bar + kBarSlots, 1u) == static_cast<unsigned>(G) - 1 ? 1 : 0;
    }
    __syncthreads();
    if (*flag) {
        __threadfence();
        for (int i = threadIdx.x; i < a.nflags; i += blockDim.x) a.flags[i] = 0u;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (a.tp > 1) atomicAdd(a.epoch_ptr, 1u);  // next launch's exchange epoch
            atomicExch(a.bar + kBarSlots, 0u);
        }
    }
}

// dynamic shared memory available next to the kernel's static __shared__ data
size_t dyn_smem_budget(bool rows_attn) {
    static size_t budget[2] = {0, 0};
    if (!budget[rows_attn]) {
        cudaFuncAttributes fa{};
        if (rows_attn)
            cudaFuncGetAttributes(&fa, mega_kernel<true, kMaxRows>);
        else
            cudaFuncGetAttributes(&fa, mega_kernel<false, kRows>);
        budget[rows_attn] = 227 * 1024 - fa.sharedSizeBytes;
    }
    return budget[rows_attn];
}

// dynamic shared memory of a launch with row capacity R (must match the
// kernel's carve-up: ring | barriers | xch | rs | attention | ropeT | hpre)
size_t smem_bytes(bool rows_attn, int stages, int hd, int group, int max_len, int R = kRows) {
    return 1024 + static_cast<size_t>(stages) * (kABytes + 384 * R) + (2 * kMaxStages + 8) * 8 + 32 +
           sizeof(float) * (64 * kRows + 4 * kRows + kMaxRows + attn_scratch_floats(rows_attn, hd, group, max_len) +
                            (R == kRows ? kRows * hd : 0) + R * kM + kM) + 16;
}

}  // namespace mega

// Attention design of the layer-stack megakernel, per bank (session): decided
// at the bank's first megakernel step from its cache length -- the per-row
// design below kAutoChunkedKeys cached keys, the key-chunked design at or
// above (measured crossover ~700 keys) -- and fixed for the bank's
// lifetime, so every step of a session (lookahead or sequential) runs the same
// arithmetic.  SFG_ATTN=rows|chunked overrides the choice for every bank.
constexpr int kAutoChunkedKeys = 768;
int attn_env() {
    static const int v = [] {
        const char* e = getenv("SFG_ATTN");
        if (e && std::string(e) == "chunked") return 0;
        if (e && std::string(e) == "rows") return 1;
        return -1;
    }();
    return v;
}
bool bank_rows_attention(Bank& b) {
    if (b.attn_design < 0) {
        const int env = attn_env();
        b.attn_design = env >= 0 ? env : (b.len() < kAutoChunkedKeys ? 1 : 0);
    }
    return b.attn_design == 1;
}

using namespace mega;

// The megakernel covers decode batches (<= 16 rows) with frame-style masks
// (visible mask value 0); seam-2 additive masks and long prompts take the
// per-GEMM path.
// ring stages of a launch: the deepest even ring whose shared memory fits
int mega_stages(bool ra, int hd, int group, int max_len, int RS, int cap) {
    int stages = cap & ~1;  // the ring is walked in pairs of stages
    while (stages > 4 && smem_bytes(ra, stages, hd, group, max_len, RS) > dyn_smem_budget(ra)) stages -= 2;
    return stages;
}

bool mega_supported(const Engine& e, int rows, bool additive_mask, bool ra) {
    if (rows < 1 || rows > tc::kRows || additive_mask) return false;
    const ModelCfg& c = e.cfg();
    const int group = c.n_heads / c.n_kv_heads;
    if (group > kMaxGroup || !(c.head_dim == 32 || c.head_dim == 64 || c.head_dim == 128 || c.head_dim == 160)) return false;
    if (group > 4 && c.head_dim > 64) return false;  // register budget of the attention phase
    if (c.hidden_dim % tc::kKB || c.q_dim() % tc::kKB || c.ffn_dim % tc::kKB) return false;
    const size_t sm = smem_bytes(ra, 4, c.head_dim, c.n_heads / c.n_kv_heads, c.max_seq_len);
    if (sm > dyn_smem_budget(ra)) return false;
    if (!ra) {  // the chunked design stages a whole key chunk in the lent ring; at most 64 chunks merge
        const int kc = c.head_dim <= 128 ? attn_kc<128>() : attn_kc<160>();
        const int st = mega_stages(false, c.head_dim, group, c.max_seq_len, tc::kRows, kMaxStages);
        if (static_cast<size_t>(attn_lend_floats(c.head_dim, kc)) * 4 > static_cast<size_t>(st) * (tc::kABytes + 384 * tc::kRows))
            return false;
        if ((c.max_seq_len + kc - 1) / kc > 64) return false;
    }
    return true;
}

// Rows one cross-session weight pass can carry: 32 (two 16-row blocks, MMA
// N = 96) with the per-row attention design when its shared memory fits,
// else 16.
int mega_batch_rows(const Engine& e) {
    if (!mega_supported(e, 1, false, true) || e.tp_size() > 1) return tc::kRows;  // wide passes: per-row design
    const ModelCfg& c = e.cfg();
    const size_t sm = smem_bytes(true, 4, c.head_dim, c.n_heads / c.n_kv_heads, c.max_seq_len, kMaxRows);
    return sm <= dyn_smem_budget(true) ? kMaxRows : tc::kRows;
}

// per-phase CTA split (phase_ctas) and whole tiles (whole_tiles) of a launch,
// shared by the launch and by MegaState's partial-buffer sizing
// Default 85 %; 50 % under tensor parallelism, whose half-width phases have
// fewer tiles: every TP=2 NeMo-12B phase then runs tile-aligned (O and down on
// 80 CTAs, one 1/2 k piece each; step 4.87 -> 4.46 ms), while at TP=1 lower
// thresholds are slower (70 %: 5.04 -> 5.23 ms; tools/tp_knob_sweep.sh)
static int mega_align_pct(int tp, int p) {
    static const int v = [] {
        const char* e = getenv("SFG_MEGA_ALIGN");
        return e ? atoi(e) : -1;
    }();
    static const std::array<int, 4> vp = [] {  // dev knob: per phase "qkv,o,gu,down"
        std::array<int, 4> r{-1, -1, -1, -1};
        if (const char* e = getenv("SFG_MEGA_ALIGN4")) sscanf(e, "%d,%d,%d,%d", &r[0], &r[1], &r[2], &r[3]);
        return r;
    }();
    if (vp[p] >= 0) return vp[p];
    return v >= 0 ? v : (tp > 1 ? 50 : 85);
}
static bool mega_whole_on() {
    static const int v = [] {
        const char* e = getenv("SFG_MEGA_WHOLE");  // dev knob: 0 = plain stream-K everywhere
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}
static void mega_split(const Dims& dl, int nsm, int tp, int (&G)[4], int (&W)[4], int (&tiles)[4]) {
    const int tQ = (dl.qd + 2 * dl.kvd + tc::kM - 1) / tc::kM, tH = (dl.H + tc::kM - 1) / tc::kM;
    const int t_of[4] = {tQ, tH, dl.F / 64, tH};
    const int kb_of[4] = {dl.H / tc::kKB, dl.qd / tc::kKB, dl.H / tc::kKB, dl.F / tc::kKB};
    for (int p = 0; p < 4; ++p) {
        tiles[p] = t_of[p];
        G[p] = phase_ctas(t_of[p], kb_of[p], nsm, mega_align_pct(tp, p));
        W[p] = mega_whole_on() ? whole_tiles(t_of[p], kb_of[p], G[p]) : 0;
    }
}
static int mega_split_tiles_max(const Engine& e) {
    int G[4], W[4], t[4];
    mega_split(e.dims(), device_sm_count(), e.tp_size(), G, W, t);
    int m = 0;
    for (int p = 0; p < 4; ++p) m = std::max(m, t[p] - W[p] * G[p]);
    return m;
}

namespace {
struct MegaState {
    LayerDesc* d_layers = nullptr;
    int lb = -1, le = -1;
    unsigned* bar = nullptr;
    float* ss = nullptr;
    unsigned long long* trace = nullptr;
    uint8_t* xim = nullptr;  // the four phases' input images, back to back
    float* partials = nullptr;  // 2 parity buffers of stream-K partials
    int rcap = 0;               // row capacity the ss / image / partial buffers are sized for
    int* counters = nullptr;    // 2 parity arrays of per-tile arrival counters
    unsigned* flags = nullptr;  // dataflow completion flags
    float* apart = nullptr;     // attention chunk partials
    int32_t* rowinfo = nullptr;      // cross-session pass: per-row (bank, slot, prior)
    int32_t* rowinfo_pin = nullptr;
    unsigned* acnt = nullptr;
    size_t part_stride = 0;
    int cnt_stride = 0, nflags = 0;
    ~MegaState() {
        if (d_layers) cudaFree(d_layers);
        if (bar) cudaFree(bar);
        if (ss) cudaFree(ss);
        if (trace) cudaFree(trace);
        if (xim) cudaFree(xim);
        if (partials) cudaFree(partials);
        if (counters) cudaFree(counters);
        if (flags) cudaFree(flags);
        if (apart) cudaFree(apart);
        if (rowinfo) cudaFree(rowinfo);
        if (rowinfo_pin) cudaFreeHost(rowinfo_pin);
        if (acnt) cudaFree(acnt);
    }
};
}  // namespace

bool& mega_trace_enabled() {
    static bool on = false;
    return on;
}

// debugging: copy the bank's phase timeline ([G][256][8] globaltimer stamps)
int mega_trace_read(Bank& b, unsigned long long* out, size_t n) {
    MegaState* st = static_cast<MegaState*>(b.mega.get());
    if (!st || !st->trace) return 0;
    SFG_CUDA(cudaDeviceSynchronize());
    SFG_CUDA(cudaMemcpy(out, st->trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
    return 1;
}

// debugging: the bank's sum-of-squares partial buffers (0: ss_d, 1: ss_o)
float* mega_ss(Bank& b, int which, int tilesH) {
    MegaState* st = static_cast<MegaState*>(b.mega.get());
    if (!st) return nullptr;
    return st->ss + (which ? tilesH * st->rcap : 0);
}

int mega_forward(Engine& e, Bank& b, int lb, int le, int rows, Workspace& ws, cudaStream_t s,
                 const std::vector<Bank*>* banks, const int32_t* rowinfo) {
    const ModelCfg& c = e.cfg();
    // per-bank layer table (weights + this bank's KV slabs), grid barrier and
    // sum-of-squares buffers, owned by the bank
    MegaState* stp = static_cast<MegaState*>(b.mega.get());
    if (stp && (stp->lb != lb || stp->le != le)) {
        SFG_CUDA(cudaDeviceSynchronize());
        b.mega.reset();
        stp = nullptr;
    }
    if (!stp) {
        auto holder = std::make_shared<MegaState>();
        MegaState& st = *holder;
        st.lb = lb;
        st.le = le;
        std::vector<LayerDesc> host(le - lb);
        for (int l = lb; l < le; ++l) {
            const LayerWeights& L = e.layer(l);
            LayerDesc& d = host[l - lb];
            d.w[0] = static_cast<const uint8_t*>(L.f_qkv);
            d.w[1] = static_cast<const uint8_t*>(L.f_o);
            d.w[2] = static_cast<const uint8_t*>(L.f_gu);
            d.w[3] = static_cast<const uint8_t*>(L.f_down);
            d.attn_norm = L.attn_norm;
            d.ffn_norm = L.ffn_norm;
            d.next_attn_norm = l + 1 < le ? e.layer(l + 1).attn_norm : nullptr;
            d.kc = b.kslab(l);
            d.vc = b.vslab(l);
        }
        SFG_CUDA(cudaMalloc(&st.d_layers, sizeof(LayerDesc) * host.size()));
        SFG_CUDA(cudaMemcpy(st.d_layers, host.data(), sizeof(LayerDesc) * host.size(), cudaMemcpyHostToDevice));
        SFG_CUDA(cudaMalloc(&st.bar, sizeof(unsigned) * (kBarSlots + 1)));
        SFG_CUDA(cudaMemset(st.bar, 0, sizeof(unsigned) * (kBarSlots + 1)));
        const int tilesH = (c.hidden_dim + tc::kM - 1) / tc::kM;
        {
            const int tQ = (c.q_dim() + 2 * c.kv_dim() + tc::kM - 1) / tc::kM, tG = c.ffn_dim / 64;
            // stream-K partial slots only for the tiles a phase actually splits
            // (its whole tiles never store partials): 76 instead of 224 at 7B
            st.cnt_stride = std::max(1, mega_split_tiles_max(e));
            SFG_CUDA(cudaMalloc(&st.counters, sizeof(int) * 2 * st.cnt_stride));
            SFG_CUDA(cudaMemset(st.counters, 0, sizeof(int) * 2 * st.cnt_stride));
            // must match fptr(): stats tiles + counter, then per layer
            // (QKV, attention kv heads, O, gate|up, down) tiles + counter each
            const int lay = (tQ + 1) + (3 * c.n_kv_heads + 1) + (tilesH + 1) + (tG + 1) + (tilesH + 1);
            st.nflags = tilesH + 1 + (le - lb) * lay;
            SFG_CUDA(cudaMalloc(&st.flags, sizeof(unsigned) * st.nflags));
            // chunked attention partials (per kv head, chunk, query): only that design uses them
            const int kc = c.head_dim <= 128 ? attn_kc<128>() : attn_kc<160>();
            const size_t cpk = bank_rows_attention(b) ? 1 : (c.max_seq_len + kc - 1) / kc;
            SFG_CUDA(cudaMalloc(&st.apart, sizeof(float) * c.n_kv_heads * cpk * 128 * (c.head_dim + 2)));
            SFG_CUDA(cudaMalloc(&st.acnt, sizeof(unsigned) * c.n_kv_heads * 16));
            SFG_CUDA(cudaMemset(st.acnt, 0, sizeof(unsigned) * c.n_kv_heads * 16));
            SFG_CUDA(cudaMemset(st.flags, 0, sizeof(unsigned) * st.nflags));
        }
        SFG_CUDA(cudaDeviceSynchronize());
        b.mega = holder;
        stp = holder.get();
    }
    // row capacity of this launch: one 16-row block, or two for a
    // cross-session pass of more than 16 rows
    const int R = rows > tc::kRows ? kMaxRows : tc::kRows;
    const bool ra = bank_rows_attention(b);
    if (R > tc::kRows && (!ra || e.tp_size() > 1 || rows > kMaxRows))
        throw Error(Kind::internal, "a wide (> 16-row) pass needs <= 32 rows, the per-row attention and no tensor parallelism");
    if (stp->rcap < R) {  // (re)size the row-strided buffers
        SFG_CUDA(cudaDeviceSynchronize());
        if (stp->ss) cudaFree(stp->ss);
        if (stp->xim) cudaFree(stp->xim);
        if (stp->partials) cudaFree(stp->partials);
        const int tilesH = (c.hidden_dim + tc::kM - 1) / tc::kM;
        SFG_CUDA(cudaMalloc(&stp->ss, sizeof(float) * 2 * tilesH * R));
        SFG_CUDA(cudaMemset(stp->ss, 0, sizeof(float) * 2 * tilesH * R));
        const size_t xblocks = static_cast<size_t>(2 * c.hidden_dim + c.q_dim() + c.ffn_dim) / tc::kKB;
        SFG_CUDA(cudaMalloc(&stp->xim, xblocks * 384 * R));
        SFG_CUDA(cudaMemset(stp->xim, 0, xblocks * 384 * R));
        stp->part_stride = static_cast<size_t>(stp->cnt_stride) * kMaxPieces * R * tc::kM;
        SFG_CUDA(cudaMalloc(&stp->partials, sizeof(float) * 2 * stp->part_stride));
        stp->rcap = R;
        SFG_CUDA(cudaDeviceSynchronize());
    }
    const int nsm = device_sm_count();
    const int group = c.n_heads / c.n_kv_heads;
    static const int stages_cap = [] {
        const char* v = getenv("SFG_MEGA_STAGES");  // dev knob: ring depth sensitivity
        return v ? std::min(std::max(atoi(v), 2), kMaxStages) : kMaxStages;
    }();
    const int RS = stp->rcap;      // the buffers' row stride (>= R)
    const void* kfn = !ra ? reinterpret_cast<const void*>(mega_kernel<false, kRows>)
                      : RS == kRows ? reinterpret_cast<const void*>(mega_kernel<true, kRows>)
                                    : reinterpret_cast<const void*>(mega_kernel<true, kMaxRows>);
    const int stages = mega_stages(ra, c.head_dim, group, c.max_seq_len, RS, stages_cap);
    if (!ra) {
        const int kc = c.head_dim <= 128 ? attn_kc<128>() : attn_kc<160>();
        if (static_cast<size_t>(attn_lend_floats(c.head_dim, kc)) * 4 > static_cast<size_t>(stages) * (tc::kABytes + 384 * RS))
            throw Error(Kind::internal, "chunked attention: a key chunk does not fit the lent weight ring");
    }
    const size_t smem = smem_bytes(ra, stages, c.head_dim, group, c.max_seq_len, RS);
    {
        ensure_smem_attr(kfn, smem);
        int nb = 0;
        SFG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kfn, kThreads, smem));
        if (nb < 1) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kfn);
            throw Error(Kind::internal, "megakernel does not fit an SM: regs " + std::to_string(fa.numRegs) +
                                            " static smem " + std::to_string(fa.sharedSizeBytes) + " dyn smem " +
                                            std::to_string(smem) + " max threads " + std::to_string(fa.maxThreadsPerBlock));
        }
    }
    const int tilesH = (c.hidden_dim + tc::kM - 1) / tc::kM;
    MegaArgs a{};
    a.layers = stp->d_layers;
    a.nlayers = le - lb;
    a.rows = rows;
    a.stages = stages;
    a.R = RS;
    a.xbytes = 384 * RS;
    a.stage_bytes = tc::kABytes + a.xbytes;
    a.acc_cols = RS == tc::kRows ? kAccCols : 128;
    a.tmem_cols = 2 * a.acc_cols > kTmemCols ? 2 * a.acc_cols : kTmemCols;
    if (!ra) a.tmem_cols = 512;  // chunked attention: score pieces in columns [128, 512)
    a.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>((3 * RS) >> 3) << 17) |
              (static_cast<uint32_t>(tc::kM >> 4) << 24);
    const Dims dl = e.dims();  // this engine's shard (tensor parallelism: local heads / FFN columns)
    a.H = dl.H;
    a.qd = dl.qd;
    a.kvd = dl.kvd;
    a.F = dl.F;
    a.hd = dl.hd;
    a.n_heads = dl.n_heads;
    a.n_kv = dl.n_kv;
    a.tp = e.tp_size();
    a.tp_rank = e.tp_rank();
    if (a.tp > 1) {
        const TpPeer& tpp = e.tp_peer();
        if (!tpp.peer_inbox) throw Error(Kind::internal, "tensor-parallel peer inbox not mapped");
        a.inbox = tpp.inbox;
        a.inflag = tpp.inflag;
        a.peer_inbox = tpp.peer_inbox;
        a.peer_inflag = tpp.peer_inflag;
        a.epoch_ptr = tpp.epoch;
    }
    a.max_len = c.max_seq_len;
    a.eps = c.rms_eps;
    a.kbank[0] = b.kslab(lb);
    a.vbank[0] = b.vslab(lb);
    a.slab_stride = b.slab_elems();
    a.rowinfo = nullptr;
    if (banks && rowinfo) {  // cross-session pass
        if (banks->size() > static_cast<size_t>(kMaxBanks) || !ra)
            throw Error(Kind::internal, "cross-session pass needs <= 16 banks and the per-row attention");
        for (Bank* bi : *banks)
            if (!bank_rows_attention(*bi))
                throw Error(Kind::internal, "cross-session pass over a bank with the key-chunked attention");
        for (size_t i = 0; i < banks->size(); ++i) {
            Bank* bi = (*banks)[i];
            if (bi->layer_begin() != b.layer_begin() || bi->layer_end() != b.layer_end() ||
                bi->slab_elems() != b.slab_elems())
                throw Error(Kind::internal, "cross-session pass over banks with different layer ranges");
            a.kbank[i] = bi->kslab(lb);
            a.vbank[i] = bi->vslab(lb);
        }
        if (!stp->rowinfo) {
            SFG_CUDA(cudaMalloc(&stp->rowinfo, sizeof(int32_t) * 3 * kMaxRows));
            SFG_CUDA(cudaMallocHost(&stp->rowinfo_pin, sizeof(int32_t) * 3 * kMaxRows));
        }
        std::memcpy(stp->rowinfo_pin, rowinfo, sizeof(int32_t) * 3 * rows);
        SFG_CUDA(cudaMemcpyAsync(stp->rowinfo, stp->rowinfo_pin, sizeof(int32_t) * 3 * rows, cudaMemcpyHostToDevice, s));
        a.rowinfo = stp->rowinfo;
    }
    a.h = ws.h;
    a.q = ws.q;
    a.att = ws.att;
    a.act = ws.act;
    a.ss_d = stp->ss;
    a.ss_o = stp->ss + tilesH * RS;
    a.pos = ws.pos;
    a.rope_cos = e.rope_cos();
    a.rope_sin = e.rope_sin();
    a.prior = ws.meta;
    a.row_off = ws.row_off;
    a.runs = ws.runs;
    a.partials = stp->partials;
    a.counters = stp->counters;
    a.part_stride = stp->part_stride;
    a.cnt_stride = stp->cnt_stride;
    a.flags = stp->flags;
    a.apart = stp->apart;
    a.acnt = stp->acnt;
    a.nflags = stp->nflags;
    a.bar = stp->bar;
    a.status = ws.status;
    {
        static const int pf_env = [] {
            const char* v = getenv("SFG_MEGA_PF");
            return v ? atoi(v) : 0;
        }();
        a.pf = pf_env;
        static const int ef_env = [] {
            const char* v = getenv("SFG_MEGA_EVICT_FIRST");
            return v ? atoi(v) : 1;
        }();
        a.evict_first = ef_env;
        static const int spin_env = [] {
            const char* v = getenv("SFG_MEGA_SPIN");
            return v ? atoi(v) : 0;
        }();
        a.spin_mma = spin_env;
        static const int bpf_env = [] {
            const char* v = getenv("SFG_MEGA_BPF");
            return v ? atoi(v) : 0;
        }();
        static const long long bpfc_env = [] {
            const char* v = getenv("SFG_MEGA_BPF_CYC");
            return v ? atoll(v) : 2000LL;
        }();
        a.bpf = bpf_env;
        static const int noload_env = [] {
            const char* v = getenv("SFG_MEGA_NOLOAD");  // dev knob: latency floor without weight traffic
            return v ? atoi(v) : 0;
        }();
        a.noload = noload_env;
        int tiles_of[4];
        mega_split(dl, nsm, e.tp_size(), a.G, a.W, tiles_of);
        const int tQ = tiles_of[P_QKV], tH = tiles_of[P_O];
        // flag layout (must match kind_tiles): statistics tiles + counter, then
        // per layer QKV, attention kv heads, O, gate|up, down tiles + counter each
        // (K_ATT: per kv head published-query counts, then 2 chunk-arrival counters per head)
        const int kt[6] = {tH, tQ, 3 * dl.n_kv, tH, dl.F / 64, tH};
        a.fl_base = tH + 1;
        int off = 0;
        for (int k = mega::K_QKV; k <= mega::K_DOWN; ++k) {
            a.fl_off[k] = off;
            off += kt[k] + 1;
        }
        a.fl_off[mega::K_STATS] = 0;
        a.fl_lay = off;
        if (a.fl_base + (le - lb) * a.fl_lay > stp->nflags) throw Error(Kind::internal, "flag buffer too small");
        a.attn_rows = ra ? 1 : 0;
        a.bpf_cycles = bpfc_env;
    }
    {
        const size_t kbH = c.hidden_dim / tc::kKB, kbQ = c.q_dim() / tc::kKB;
        a.xim[P_QKV] = stp->xim;
        a.xim[P_O] = a.xim[P_QKV] + kbH * a.xbytes;
        a.xim[P_GU] = a.xim[P_O] + kbQ * a.xbytes;
        a.xim[P_DOWN] = a.xim[P_GU] + kbH * a.xbytes;
    }
    if (mega_trace_enabled() && !stp->trace) {
        const size_t bytes = sizeof(unsigned long long) * static_cast<size_t>(nsm) * kBarSlots * kTraceW;
        SFG_CUDA(cudaMalloc(&stp->trace, bytes));
        SFG_CUDA(cudaMemset(stp->trace, 0, bytes));
        SFG_CUDA(cudaDeviceSynchronize());
    }
    a.trace = mega_trace_enabled() ? stp->trace : nullptr;
    void* args[] = {&a};
    {
        const double H = c.hidden_dim, qd = c.q_dim(), kvd = c.kv_dim(), F = c.ffn_dim, L = le - lb, R = rows;
        const double bytes = L * 2.0 * (H * (qd + 2 * kvd) + qd * H + 2 * H * F + F * H) +
                             L * 2.0 * 4.0 * kvd * (b.len() + rows) + 4.0 * R * H * 2;
        const double flops = L * 2.0 * R * (H * (qd + 2 * kvd) + qd * H + 3 * H * F);
        ProfScope ps(K_LAYERS, s, bytes, flops);
        SFG_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(nsm), dim3(kThreads), args, smem, s));
    }
    return 1;
}

}  // namespace sfg
