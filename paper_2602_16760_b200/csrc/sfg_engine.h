// Host-side engine (C++20): weights resident on one B200, KV-cache banks,
// the layer-executor orchestration, and the error taxonomy.  This is the
// B200 counterpart of tinyformer.{hpp,cpp}; the server (sfg_server.cpp) and
// the local client (sfg_client.cpp) are built on it, and sfg_capi.cpp
// exposes everything through include/sfg.h.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfg.h"
#include "sfg_kernels.h"

namespace sfg {

// splitf::ErrorKind (error.hpp:10-21); the numeric value is the C status.
enum class Kind : int32_t {
    config = 1, input, protocol, transport, capacity, session, numeric, training, decomposition,
    internal
};
const char* kind_name(Kind k);

// Mirrors splitf::SplitError: what() == "<category>: <msg>".
class Error : public std::runtime_error {
public:
    Error(Kind k, const std::string& msg) : std::runtime_error(std::string(kind_name(k)) + ": " + msg), kind_(k) {}
    Kind kind() const { return kind_; }

private:
    Kind kind_;
};

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define SFG_CUDA(x)                                                            \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) ::sfg::cuda_fail(e_, #x, __FILE__, __LINE__);   \
    } while (0)

struct ModelCfg {
    int vocab_size, n_layers, hidden_dim, n_heads, n_kv_heads, head_dim, ffn_dim, max_seq_len;
    float rope_base, rms_eps;
    uint64_t seed;
    int q_dim() const { return n_heads * head_dim; }
    int kv_dim() const { return n_kv_heads * head_dim; }
    // ModelConfig::validate, tinyformer.cpp:102-121; extended: q_dim may differ from hidden_dim
    void validate(bool extended = false) const;
    static ModelCfg from_c(const sfg_model_config& c);
};

// Device tensors of one decoder layer in the reference layout ([in x out]).
struct LayerWeights {
    float* attn_norm = nullptr;
    void* wq = nullptr;
    void* wk = nullptr;
    void* wv = nullptr;
    void* wo = nullptr;
    float* ffn_norm = nullptr;
    void* w_gate = nullptr;
    void* w_up = nullptr;
    void* w_down = nullptr;
    // FAST-mode operand layouts (sfg_fast.cu), built from the above at load.
    void* f_qkv = nullptr;    // [qd+2kvd x H] K-major bf16 (rows = output features)
    void* f_o = nullptr;      // [H x qd]
    void* f_gu = nullptr;     // [2F x H] gate/up interleaved by 64-row tiles
    void* f_down = nullptr;   // [H x F]
    bool hosted = false;
};

// Growable device workspace for one executor stream.
struct Workspace {
    int cap_rows = 0, cap_runs = 0, cap_logit_rows = 0;
    float *h = nullptr, *xn = nullptr, *q = nullptr, *att = nullptr, *act = nullptr;
    float* logits = nullptr;
    int32_t *pos = nullptr, *ids = nullptr, *argmax = nullptr, *keep = nullptr, *row_off = nullptr;
    MaskRun* runs = nullptr;
    uint32_t* status = nullptr;
    unsigned long long* clamped = nullptr;
    void* wire = nullptr;          // packed wire rows [cap_rows x H] (up to 4 B each)
    void* fast = nullptr;          // FAST-mode scratch (split operands, partials)
    size_t fast_bytes = 0;
    void* pimg = nullptr;          // FAST prompt passes: token-tiled split image [tiles][KB][3][128 x 64]
    size_t pimg_bytes = 0;
    void* apieces = nullptr;       // FAST prompt attention: pre-split Q / K / V^T tiles (sfg_attn_tc.cu)
    size_t apieces_bytes = 0;
    void* pinned = nullptr;        // host staging
    size_t pinned_bytes = 0;
    void* wire_pin = nullptr;      // pinned wire rows [cap_rows x H] (4 B each): frame tensors cross here
    // Per-step scalars read by kernels from device memory, so one captured
    // CUDA graph serves every step of a given batch size:
    //   meta[0] = cache length before the batch (QKV epilogue KV slot base)
    //   meta[1] = committed length before resolve, meta[2] = #kept rows,
    //   meta[3 .. 3+kMetaKeep) = keep list (in-place compaction).
    int32_t* meta = nullptr;       // device
    int32_t* meta_pin = nullptr;   // pinned mirror
    void* stage_pin = nullptr;     // pinned [ids | pos | row_off | runs] at cap-derived offsets
    size_t stage_bytes = 0;
    uint64_t generation = 0;       // bumped whenever a buffer is reallocated
    // the mask is outside the layer-stack megakernel's contract: some visible
    // column carries a non-zero (additive) value, or some row does not see the
    // whole cached prefix [0, prior) (see mega_mask_ok)
    bool additive_mask = false;
    // every row sees exactly [0, lim) with mask value 0 (the causal prefix law
    // of prompt passes): the tiled prompt attention applies
    bool prefix_mask = false;
    void release();
};

constexpr int kMetaKeep = 256;
struct StageLayout {
    size_t ids, pos, roff, runs, total;
};
inline StageLayout stage_layout(int cap_rows, int cap_runs) {
    StageLayout L{};
    size_t o = 0;
    L.ids = o;
    o += 4 * static_cast<size_t>(cap_rows);
    L.pos = o;
    o += 4 * static_cast<size_t>(cap_rows);
    L.roff = o;
    o += 4 * static_cast<size_t>(cap_rows + 1);
    o = (o + 15) & ~size_t(15);
    L.runs = o;
    o += sizeof(MaskRun) * static_cast<size_t>(cap_runs);
    L.total = o;
    return L;
}

class Engine;

// CacheBank (tinyformer.hpp:131-156) with device-resident fp32 K/V:
// K and V are each [layer][kv_head][max_len][head_dim].
class Bank {
public:
    Bank(Engine& eng, int layer_begin, int layer_end);
    ~Bank();
    Bank(const Bank&) = delete;
    Bank& operator=(const Bank&) = delete;

    int layer_begin() const { return lb_; }
    int layer_end() const { return le_; }
    int len() const { return lb_ == le_ ? 0 : len_; }
    int committed_len() const { return committed_; }
    int provisional() const { return len() - committed_; }
    void mark_committed(int c) { committed_ = c; }
    void set_len(int l) { len_ = l; }
    void reset() { len_ = 0; committed_ = 0; }
    void resolve(const int32_t* keep, int n, cudaStream_t s = nullptr);  // tinyformer.cpp:282-308
    // resolve() bookkeeping only (validation + committed/len); the caller
    // enqueues the meta-driven compaction itself (graph-captured steps).
    void resolve_meta(const int32_t* keep, int n);
    // device compaction of kept tail entries (the device half of resolve)
    void enqueue_compact(const int32_t* keep, int n, int committed, cudaStream_t st);
    void crop(int pos);                        // tinyformer.cpp:310-316
    float* kslab(int layer) const;
    size_t slab_elems() const { return slab_elems_; }
    float* vslab(int layer) const;
    void read_kv(int layer, int head, int pos, float* k, float* v);
    cudaStream_t stream() const { return stream_; }
    Workspace& ws() { return ws_; }
    Engine& engine() { return eng_; }
    // per-bank state of the FAST megakernel (layer table, grid barrier)
    std::shared_ptr<void> mega;
    // megakernel attention design: -1 undecided, 1 per-row, 0 key-chunked
    // (bank_rows_attention: chosen at the first megakernel step, then fixed)
    int attn_design = -1;
    // process-unique id (never reused, unlike the object's address): keys
    // the client's captured graphs that bake in this bank's device buffers
    uint64_t id() const { return id_; }

private:
    Engine& eng_;
    int lb_, le_;
    uint64_t id_;
    int len_ = 0, committed_ = 0;
    float* k_ = nullptr;
    float* v_ = nullptr;
    size_t slab_elems_ = 0;
    cudaStream_t stream_ = nullptr;
    int32_t* keep_pin_ = nullptr;
    int keep_pin_cap_ = 0;
    Workspace ws_;
};

// Visibility of the batch rows, as compacted runs (see MaskRun).
struct MaskRuns {
    std::vector<int32_t> row_off;  // rows + 1
    std::vector<MaskRun> runs;
    bool any_empty_row = false;
};
// Causal prefix law: row i sees committed + i + 1 columns (tinyformer.cpp:229-241).
MaskRuns causal_runs(int rows, int committed);
// Dense fp32 additive mask [rows x kv] with -inf = masked.
MaskRuns runs_from_dense(const float* mask, int rows, int kv);
// The megakernel's attention walks each row's visible keys in compacted order
// and shares the cached prefix between rows: every row must see all of
// [0, prior) with mask value 0 (causal, lookahead and branch masks do).
bool mega_mask_ok(const MaskRuns& mr, int prior);
// every row: one run [0, end) with value 0
bool prefix_law(const MaskRuns& mr);

// Tensor parallelism over NCCL (sfg_tp.cpp): a group of `size` engines, one
// per GPU, each holding 1/size of every layer's heads and FFN columns.
struct TpConfig {
    int size = 1, rank = 0;
    const uint8_t* unique_id = nullptr;  // ncclUniqueId bytes (same on every rank)
};
void tp_unique_id(uint8_t* out, size_t n);
void* tp_comm_init(int size, int rank, const uint8_t* uid);
void tp_comm_destroy(void* comm);
void tp_allreduce_sum(void* comm, float* buf, size_t n, cudaStream_t s);
void tp_allgather_bytes(void* comm, const void* src, void* dst, size_t n, cudaStream_t s);

// Peer-memory exchange for the layer-stack megakernel at TP=2: each rank owns
// an inbox (row-parallel partial tiles + epoch flags) that the peer writes
// over NVLink (CUDA IPC mapping), so the O / down all-reduce happens inside
// the producing tile's epilogue instead of as a separate collective.
struct TpPeer {
    float* inbox = nullptr;          // mine: [layers][2][tilesH][16][128] partial tiles, 64-bit {epoch, f32} words
    unsigned* inflag = nullptr;      // mine: [layers][2][tilesH] epoch flags
    float* peer_inbox = nullptr;     // the peer's, mapped
    unsigned* peer_inflag = nullptr;
    unsigned* epoch = nullptr;       // launch counter (device), bumped by each launch's last CTA
    void* base = nullptr;            // my allocation
    void* peer_base = nullptr;       // the peer's mapping
    size_t data_floats = 0;
};

class Engine {
public:
    Engine(const ModelCfg& cfg, const sfg_engine_options& opt, const float* params, const TpConfig& tp = TpConfig{});
    ~Engine();

    const ModelCfg& cfg() const { return cfg_; }
    const sfg_engine_options& opt() const { return opt_; }
    int device() const { return opt_.device; }
    bool fast() const { return opt_.math == SFG_MATH_FAST; }
    int wt() const { return opt_.weight_dtype == SFG_WEIGHTS_F32 ? W_F32 : W_BF16; }
    int64_t weight_bytes() const { return weight_bytes_; }
    // dims of THIS engine's shard: with tensor parallelism q/kv heads and the
    // FFN width are the local 1/tp slice (hidden_dim stays whole)
    Dims dims() const;
    int tp_size() const { return tp_size_; }
    int tp_rank() const { return tp_rank_; }
    const TpPeer& tp_peer() const { return tp_peer_; }
    // in-place sum over the tensor-parallel group (no-op at tp == 1)
    void tp_allreduce(float* buf, size_t n, cudaStream_t s);
    const LayerWeights& layer(int i) const { return layers_[i]; }

    // Ensure ws holds `rows` rows / `runs` runs / `logit_rows` logit rows.
    void ensure_ws(Workspace& ws, int rows, int runs, int logit_rows);
    // Eager paths: ws.meta[0] = prior (cache length) on stream s.
    void set_prior(Workspace& ws, int prior, cudaStream_t s);

    // Layer executor over device-resident rows (ws.h holds the input and
    // receives the output).  ws.pos / ws.row_off / ws.runs must be loaded.
    // Returns kernels launched.  Host-side checks are the caller's job.
    int forward_device(Bank& b, int lb, int le, int rows, Workspace& ws, cudaStream_t s);
    // finalize (tinyformer.cpp:510-526) + optional argmax on ws.h rows.
    int head_device(int rows, Workspace& ws, bool want_logits, bool want_argmax, cudaStream_t s);
    int embed_device(int rows, Workspace& ws, cudaStream_t s);  // ws.ids -> ws.h

    // Host-buffer entry points (seam 2).
    void forward_host(Bank& b, int lb, int le, int seq, const float* h, const int32_t* pos,
                      const float* mask, float* out);
    void embed_host(int seq, const int32_t* ids, const int32_t* pos, float* out);
    void finalize_host(int seq, const float* h, float* logits, int32_t* argmax);

    const float* rope_cos() const { return rope_cos_; }
    const float* rope_sin() const { return rope_sin_; }

    std::mutex& mutex() { return mu_; }
    Workspace& ws() { return ws_; }
    cudaStream_t stream() const { return stream_; }
    // take ownership of a device allocation holding weights
    void adopt(void* p, size_t bytes) {
        allocs_.push_back(p);
        weight_bytes_ += static_cast<int64_t>(bytes);
    }

private:
    void load(const float* params);
    void upload_tensor(const float* src, size_t n, void** dst, int wt);
    void build_fast_layouts();

    ModelCfg cfg_;
    sfg_engine_options opt_;
    std::vector<LayerWeights> layers_;
    void* embedding_ = nullptr;
    float* final_norm_ = nullptr;
    void* lm_head_ = nullptr;
    void* f_lm_head_ = nullptr;
    float* rope_cos_ = nullptr;
    float* rope_sin_ = nullptr;
    int64_t weight_bytes_ = 0;
    std::vector<void*> allocs_;
    float* staging_ = nullptr;
    size_t staging_elems_ = 0;
    cudaStream_t stream_ = nullptr;
    Workspace ws_;
    std::mutex mu_;
    int tp_size_ = 1, tp_rank_ = 0;
    void* tp_comm_ = nullptr;
    TpPeer tp_peer_;
    void tp_setup_peer();
};

// Process-wide switch: capture/replay the device part of decode steps as
// CUDA graphs (sfg_set_graphs).
bool& graphs_enabled();
// 1: FAST forward uses the layer-stack megakernel when it applies (default;
// env SFG_MEGA=0 or sfg_debug_set_mega(0) selects the per-GEMM kernels).
int& mega_mode();

// Host<->device bytes moved by the engine's copies (bench.py's e2e
// h2d/d2h_bytes_per_step are measured from these, sfg_copy_bytes).
struct CopyCounters {
    std::atomic<uint64_t> h2d{0}, d2h{0};
};
CopyCounters& copy_counters();
// cudaMemcpyAsync that also counts host<->device bytes
inline cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind k, cudaStream_t s) {
    if (k == cudaMemcpyHostToDevice) copy_counters().h2d.fetch_add(n, std::memory_order_relaxed);
    if (k == cudaMemcpyDeviceToHost) copy_counters().d2h.fetch_add(n, std::memory_order_relaxed);
    return cudaMemcpyAsync(dst, src, n, k, s);
}

// Scoped device selection.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

// FAST-mode layer executor (sfg_fast.cu).
int fast_forward_layer(Engine& e, Bank& b, int layer, int rows, Workspace& ws, int prior,
                       cudaStream_t s);
int fast_head(Engine& e, const void* f_lm_head, const float* final_norm, int rows, Workspace& ws,
              bool want_logits, cudaStream_t s);
size_t fast_workspace_bytes(const ModelCfg& c, int rows);
void fast_build_layer(Engine& e, LayerWeights& L, cudaStream_t s);
void* fast_build_head(Engine& e, const void* lm_head, cudaStream_t s);
float* fast_partials(const ModelCfg& c, Workspace& ws);
int* fast_counters(const ModelCfg& c, Workspace& ws);
// FAST layer-stack megakernel (sfg_mega.cu)
bool mega_supported(const Engine& e, int rows, bool additive_mask, bool rows_attention);
// rows of one cross-session layer-stack pass (32, or 16 where unsupported)
int mega_batch_rows(const Engine& e);
// banks/rowinfo (optional): rows of several sessions in one pass -- row r
// appends to (*banks)[rowinfo[3r]] at slot rowinfo[3r+1] and sees
// rowinfo[3r+2] cached keys; b supplies the launch state (same layer range)
int mega_forward(Engine& e, Bank& b, int lb, int le, int rows, Workspace& ws, cudaStream_t s,
                 const std::vector<Bank*>* banks = nullptr, const int32_t* rowinfo = nullptr);
// the bank's attention design (decided at its first megakernel step, see sfg_mega.cu)
bool bank_rows_attention(Bank& b);
float* mega_ss(Bank& b, int which, int tilesH);
bool& mega_trace_enabled();
int mega_trace_read(Bank& b, unsigned long long* out, size_t n);

}  // namespace sfg
