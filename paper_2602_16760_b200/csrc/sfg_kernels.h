// Kernel launch interface shared by the host engine (sfg_engine.cpp) and the
// CUDA translation units.  Plain pointers only; every launcher takes the
// stream it must run on and returns the number of kernels it launched (so the
// engine can report gpu_launches exactly).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sfg {

// Device layout of one attention-visibility description: for batch row r the
// visible cache columns are the union of runs[row_off[r] .. row_off[r+1]),
// each run = [start, end) with an additive mask value (0 for every frame
// mask; seam 2 accepts any finite additive value like forward_layers does).
struct MaskRun {
    int32_t start;
    int32_t end;
    float mval;
    int32_t pad;
};

enum WeightType { W_BF16 = 0, W_F32 = 1 };

// Opt `fn` in to `smem` bytes of dynamic shared memory on the CURRENT device
// (function attributes are per device: one process may drive several GPUs).
// Remembers the largest size configured per (device, function); thread safe.
void ensure_smem_attr(const void* fn, size_t smem);
// SM count of the current device (cached per device).
int device_sm_count();

// status word bits written by kernels (checked by the host after the step)
enum : uint32_t {
    ST_EMPTY_ROW = 1u,      // mask row admits no attendable position (tinyformer.cpp:467)
    ST_NONFINITE = 2u,      // non-finite hidden state
    ST_ATTN_CAP = 4u,       // a row saw more keys than the attention launch was sized for
};

struct LayerPtrs {
    const float* attn_norm;  // [H] fp32
    const void* wq;          // [H x qd]
    const void* wk;          // [H x kvd]
    const void* wv;          // [H x kvd]
    const void* wo;          // [qd x H]
    const float* ffn_norm;   // [H]
    const void* w_gate;      // [H x F]
    const void* w_up;        // [H x F]
    const void* w_down;      // [F x H]
};

struct Dims {
    int H, qd, kvd, F, V, n_heads, n_kv, hd, max_len;
    float eps;
};

// ── exact mode (sfg_exact.cu, compiled with --fmad=false) ─────────────────
int launch_rmsnorm_exact(const float* h, const float* g, float* y, int rows, int H, float eps,
                         cudaStream_t s);
int launch_qkv_exact(const float* xn, int rows, const Dims& d, int wt, const void* wq,
                     const void* wk, const void* wv, const int32_t* pos, const float* rope_cos,
                     const float* rope_sin, float* q, float* kcache, float* vcache, const int32_t* prior,
                     cudaStream_t s);
int launch_attention_exact(const float* q, const float* kcache, const float* vcache,
                           const int32_t* row_off, const MaskRun* runs, int rows, int kv_len,
                           const Dims& d, float* att, uint32_t* status, cudaStream_t s);
int launch_matvec_residual_exact(const float* x, int rows, int K, int wt, const void* w, int N,
                                 float* h, cudaStream_t s);
int launch_gateup_exact(const float* xn, int rows, int H, int F, int wt, const void* wg,
                        const void* wu, float* act, cudaStream_t s);
int launch_matvec_store_exact(const float* x, int rows, int K, int wt, const void* w, int N,
                              float* out, cudaStream_t s);

// ── FAST-mode attention (sfg_attn.cu) ─────────────────────────────────────
int launch_attention_fast(const float* q, const float* kcache, const float* vcache,
                          const int32_t* row_off, const MaskRun* runs, int rows, const Dims& d,
                          float* att, uint32_t* status, cudaStream_t s, int kv_cap = 0);
// prompt passes whose mask follows the prefix law (every row one run [0, lim),
// value 0): K/V blocks staged once per 64 queries
bool attention_prompt_supported(const Dims& d);
// tensor-core causal prompt attention (sfg_attn_tc.cu): head_dim 128
bool attention_prompt_tc_supported(const Dims& d);
int launch_attention_prompt_tc(const float* q, const float* kcache, const float* vcache, const int32_t* row_off,
                               const MaskRun* runs, int rows, int keys, const Dims& d, float* att, uint32_t* status,
                               cudaStream_t s, void** scratch, size_t* scratch_bytes);
// keys: the cache length the prompt rows attend over (prior + rows); scratch:
// the workspace's buffer for the tensor-core path's pre-split operands
int launch_attention_prompt(const float* q, const float* kcache, const float* vcache, const int32_t* row_off,
                            const MaskRun* runs, int rows, int keys, const Dims& d, float* att, uint32_t* status,
                            cudaStream_t s, void** scratch, size_t* scratch_bytes);

// ── shared kernels (sfg_common.cu) ────────────────────────────────────────
int launch_embed(const void* table, int wt, const int32_t* ids, int rows, int H, float* out,
                 cudaStream_t s);
int launch_unpack_rows(const void* wire, int f32, int n, float* out, cudaStream_t s);
int launch_pack_rows(const float* in, int f32, int n, void* wire, unsigned long long* clamped,
                     cudaStream_t s);
int launch_wire_roundtrip(float* x, int f32, int n, unsigned long long* clamped, cudaStream_t s);
int launch_kv_compact(float* kcache, float* vcache, int layers, int n_kv, int max_len, int hd,
                      int committed, const int32_t* keep, int n_keep, cudaStream_t s);
int launch_kv_compact_meta(float* kcache, float* vcache, int layers, int n_kv, int max_len, int hd,
                           const int32_t* meta, int max_keep, cudaStream_t s);
int launch_argmax(const float* logits, int rows, int V, int32_t* out, cudaStream_t s);
int launch_link_delay(double ms, cudaStream_t s);
int launch_convert_weights(const float* src, void* dst, int wt, size_t n, cudaStream_t s);

}  // namespace sfg

namespace sfg {

// Lookahead verify / branch-selection tail (decoding.cpp:295-344), run on
// device right after the per-row argmax so the logits never leave HBM.
constexpr int kMaxWindow = 64;
constexpr int kMaxCand = 64;
constexpr int kMaxCont = 16;
struct VerifyIn {
    int32_t rows;          // B
    int32_t mode;          // 0 sequential, 2 lookahead
    int32_t active_w;
    int32_t ncand;
    int32_t cont;          // ngram_n - 1
    int32_t window[kMaxWindow];
    int32_t cand_begin[kMaxCand];
    int32_t cands[kMaxCand * kMaxCont];
};
struct VerifyOut {
    int32_t anchor;
    int32_t best;                       // accepted guesses of the winning branch
    int32_t committed[kMaxWindow + 1];  // anchor + accepted continuation
    int32_t best_rows[kMaxWindow];
    int32_t argmax[kMaxWindow + 1 + kMaxCand * kMaxCont];
};
int launch_verify(const int32_t* argmax, const VerifyIn* in, VerifyOut* out, cudaStream_t s);

}  // namespace sfg
