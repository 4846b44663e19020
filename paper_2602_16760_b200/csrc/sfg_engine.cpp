// Host engine: weights on device, KV banks, layer-executor orchestration.
// B200 counterpart of tinyformer.cpp (reference file:line cited per symbol).
#include "sfg_engine.h"

#include "sfg_prof.h"

#include <atomic>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <random>

namespace sfg {

const char* kind_name(Kind k) {
    switch (k) {
        case Kind::config: return "config";
        case Kind::input: return "input";
        case Kind::protocol: return "protocol";
        case Kind::transport: return "transport";
        case Kind::capacity: return "capacity";
        case Kind::session: return "session";
        case Kind::numeric: return "numeric";
        case Kind::training: return "training";
        case Kind::decomposition: return "decomposition";
        case Kind::internal: return "internal";
    }
    return "unknown";
}

void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    throw Error(Kind::internal, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what +
                                    " (" + file + ":" + std::to_string(line) + ")");
}

bool& graphs_enabled() {
    static bool on = true;
    return on;
}

DeviceGuard::DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) SFG_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

// ModelConfig::validate (tinyformer.cpp:102-121)
void ModelCfg::validate(bool extended) const {
    if (vocab_size < 2) throw Error(Kind::config, "vocab_size must be >= 2");
    if (n_layers < 4) throw Error(Kind::config, "n_layers must be >= 4");
    if (hidden_dim <= 0 || n_heads <= 0 || n_kv_heads <= 0 || head_dim <= 0 || ffn_dim <= 0 ||
        max_seq_len <= 0)
        throw Error(Kind::config, "all dimensions must be positive");
    if (n_heads * head_dim != hidden_dim && !extended)
        throw Error(Kind::config, "n_heads * head_dim must equal hidden_dim");
    if (n_heads % n_kv_heads != 0) throw Error(Kind::config, "n_kv_heads must divide n_heads");
    if (head_dim % 2 != 0) throw Error(Kind::config, "head_dim must be even for rotary pairs");
    if (!(rope_base > 0.0f) || !(rms_eps > 0.0f))
        throw Error(Kind::config, "rope_base and rms_eps must be positive");
}

ModelCfg ModelCfg::from_c(const sfg_model_config& c) {
    return ModelCfg{c.vocab_size, c.n_layers,  c.hidden_dim,  c.n_heads, c.n_kv_heads, c.head_dim,
                    c.ffn_dim,    c.max_seq_len, c.rope_base, c.rms_eps, c.seed};
}

// ── masks → runs ──────────────────────────────────────────────────────────
bool prefix_law(const MaskRuns& mr) {
    const int rows = static_cast<int>(mr.row_off.size()) - 1;
    for (int i = 0; i < rows; ++i) {
        if (mr.row_off[i + 1] - mr.row_off[i] != 1) return false;
        const MaskRun& r = mr.runs[mr.row_off[i]];
        if (r.start != 0 || r.end <= 0 || r.mval != 0.0f) return false;
    }
    return true;
}

bool mega_mask_ok(const MaskRuns& mr, int prior) {
    for (const MaskRun& r : mr.runs)
        if (r.mval != 0.0f) return false;
    const int rows = static_cast<int>(mr.row_off.size()) - 1;
    if (prior == 0) return true;
    for (int i = 0; i < rows; ++i) {
        if (mr.row_off[i] >= mr.row_off[i + 1]) return false;
        const MaskRun& first = mr.runs[mr.row_off[i]];
        if (first.start != 0 || first.end < prior) return false;
    }
    return true;
}

MaskRuns causal_runs(int rows, int committed) {
    MaskRuns m;
    m.row_off.resize(rows + 1);
    m.runs.resize(rows);
    for (int i = 0; i < rows; ++i) {
        m.row_off[i] = i;
        m.runs[i] = MaskRun{0, committed + i + 1, 0.0f, 0};
    }
    m.row_off[rows] = rows;
    return m;
}

MaskRuns runs_from_dense(const float* mask, int rows, int kv) {
    MaskRuns m;
    m.row_off.resize(rows + 1);
    for (int i = 0; i < rows; ++i) {
        m.row_off[i] = static_cast<int32_t>(m.runs.size());
        const float* r = mask + static_cast<size_t>(i) * kv;
        int j = 0;
        bool any = false;
        while (j < kv) {
            if (r[j] == -INFINITY) {
                ++j;
                continue;
            }
            uint32_t bits;
            std::memcpy(&bits, &r[j], 4);
            int e = j + 1;
            while (e < kv) {
                uint32_t b2;
                std::memcpy(&b2, &r[e], 4);
                if (b2 != bits) break;
                ++e;
            }
            m.runs.push_back(MaskRun{j, e, r[j], 0});
            any = true;
            j = e;
        }
        if (!any) m.any_empty_row = true;
    }
    m.row_off[rows] = static_cast<int32_t>(m.runs.size());
    return m;
}

// ── workspace ─────────────────────────────────────────────────────────────
void Workspace::release() {
    for (void* p : {(void*)h, (void*)xn, (void*)q, (void*)att, (void*)act, (void*)logits, (void*)pos,
                    (void*)ids, (void*)argmax, (void*)keep, (void*)row_off, (void*)runs, (void*)status,
                    (void*)clamped, wire, fast, pimg, apieces, (void*)meta})
        if (p) cudaFree(p);
    if (pinned) cudaFreeHost(pinned);
    if (meta_pin) cudaFreeHost(meta_pin);
    if (stage_pin) cudaFreeHost(stage_pin);
    if (wire_pin) cudaFreeHost(wire_pin);
    *this = Workspace{};
}

// cudaMemset runs on the legacy stream, which is NOT ordered with the
// engine's non-blocking streams: every zero-fill here is followed by a
// device sync before the buffer is handed to stream work (growth is rare).
static void grow(void** p, size_t bytes) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    SFG_CUDA(cudaMalloc(p, bytes ? bytes : 16));
    SFG_CUDA(cudaMemset(*p, 0, bytes ? bytes : 16));
}

void Engine::ensure_ws(Workspace& ws, int rows, int runs, int logit_rows) {
    const ModelCfg& c = cfg_;
    // A prompt pass grows the row-scaled buffers to the prompt length (~0.7 GB
    // for a 2048-token prompt at the 7B shape); the first decode step after it
    // gives them back, so 64 concurrent long-context sessions fit one GPU.
    const bool trim = rows <= 64 && ws.cap_rows > 256;
    if (trim) {
        SFG_CUDA(cudaDeviceSynchronize());
        for (void** p : {(void**)&ws.h, (void**)&ws.xn, (void**)&ws.q, (void**)&ws.att, (void**)&ws.act, (void**)&ws.pos,
                         (void**)&ws.ids, (void**)&ws.argmax, (void**)&ws.keep, (void**)&ws.row_off, &ws.wire, &ws.fast,
                         &ws.pimg, &ws.apieces}) {
            if (*p) cudaFree(*p);
            *p = nullptr;
        }
        ws.fast_bytes = ws.pimg_bytes = ws.apieces_bytes = 0;
        if (ws.wire_pin) cudaFreeHost(ws.wire_pin);
        ws.wire_pin = nullptr;
        if (ws.pinned) cudaFreeHost(ws.pinned);
        ws.pinned = nullptr;
        ws.pinned_bytes = 0;
        ws.cap_rows = 0;
    }
    const bool growing = rows > ws.cap_rows || runs > ws.cap_runs || logit_rows > ws.cap_logit_rows;
    if (!growing) return;
    // old buffers may still be read by queued work; new ones are zero-filled
    // on the legacy stream: fence on both sides.
    SFG_CUDA(cudaDeviceSynchronize());
    if (rows > ws.cap_rows) {
        const int r = std::max(rows, std::max(16, ws.cap_rows * 2));
        const size_t H = c.hidden_dim, qd = c.q_dim(), F = c.ffn_dim;
        grow((void**)&ws.h, sizeof(float) * r * H);
        grow((void**)&ws.xn, sizeof(float) * r * std::max(H, F));
        grow((void**)&ws.q, sizeof(float) * r * qd);
        grow((void**)&ws.att, sizeof(float) * r * qd);
        grow((void**)&ws.act, sizeof(float) * r * F);
        grow((void**)&ws.pos, sizeof(int32_t) * r);
        grow((void**)&ws.ids, sizeof(int32_t) * r);
        grow((void**)&ws.argmax, sizeof(int32_t) * r);
        grow((void**)&ws.keep, sizeof(int32_t) * r);
        grow((void**)&ws.row_off, sizeof(int32_t) * (r + 1));
        grow(&ws.wire, sizeof(float) * r * H);
        if (!ws.status) grow((void**)&ws.status, 64);
        if (!ws.clamped) grow((void**)&ws.clamped, 64);
        if (fast()) {
            ws.fast_bytes = fast_workspace_bytes(c, r);
            grow(&ws.fast, ws.fast_bytes);
        }
        if (ws.wire_pin) cudaFreeHost(ws.wire_pin);
        SFG_CUDA(cudaMallocHost(&ws.wire_pin, sizeof(float) * r * H));
        const size_t pin = sizeof(float) * r * std::max<size_t>(H, 64) * 2 + 4096 * 16;
        if (pin > ws.pinned_bytes) {
            if (ws.pinned) cudaFreeHost(ws.pinned);
            SFG_CUDA(cudaMallocHost(&ws.pinned, pin));
            ws.pinned_bytes = pin;
        }
        ws.cap_rows = r;
    }
    if (runs > ws.cap_runs) {
        const int r = std::max(runs, std::max(64, ws.cap_runs * 2));
        grow((void**)&ws.runs, sizeof(MaskRun) * r);
        ws.cap_runs = r;
    }
    if (logit_rows > ws.cap_logit_rows) {
        const int r = std::max(logit_rows, std::max(16, ws.cap_logit_rows * 2));
        grow((void**)&ws.logits, sizeof(float) * r * c.vocab_size);
        ws.cap_logit_rows = r;
    }
    if (!ws.meta) {
        grow((void**)&ws.meta, sizeof(int32_t) * (4 + kMetaKeep));
        SFG_CUDA(cudaMallocHost(&ws.meta_pin, sizeof(int32_t) * (4 + kMetaKeep)));
        std::memset(ws.meta_pin, 0, sizeof(int32_t) * (4 + kMetaKeep));
    }
    const StageLayout L = stage_layout(ws.cap_rows, ws.cap_runs);
    if (L.total > ws.stage_bytes) {
        if (ws.stage_pin) cudaFreeHost(ws.stage_pin);
        SFG_CUDA(cudaMallocHost(&ws.stage_pin, L.total));
        ws.stage_bytes = L.total;
    }
    ++ws.generation;
    SFG_CUDA(cudaDeviceSynchronize());
}

void Engine::set_prior(Workspace& ws, int prior, cudaStream_t s) {
    // eager paths sync at the end of every call, so the pinned slot is free
    ws.meta_pin[0] = prior;
    SFG_CUDA(cudaMemcpyAsync(ws.meta, ws.meta_pin, sizeof(int32_t), cudaMemcpyHostToDevice, s));
}

// ── banks ─────────────────────────────────────────────────────────────────
static std::atomic<uint64_t> g_bank_ids{1};

CopyCounters& copy_counters() {
    static CopyCounters c;
    return c;
}

Bank::Bank(Engine& eng, int lb, int le) : eng_(eng), lb_(lb), le_(le), id_(g_bank_ids.fetch_add(1)) {
    const ModelCfg& c = eng.cfg();
    if (lb < 0 || le > c.n_layers || lb > le) throw Error(Kind::config, "invalid layer range for cache bank");
    DeviceGuard g(eng.device());
    slab_elems_ = static_cast<size_t>(c.n_kv_heads) * c.max_seq_len * c.head_dim;
    const size_t n = slab_elems_ * std::max(1, le - lb);
    SFG_CUDA(cudaMalloc(&k_, n * sizeof(float)));
    SFG_CUDA(cudaMalloc(&v_, n * sizeof(float)));
    SFG_CUDA(cudaMemset(k_, 0, n * sizeof(float)));
    SFG_CUDA(cudaMemset(v_, 0, n * sizeof(float)));
    SFG_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    SFG_CUDA(cudaDeviceSynchronize());  // legacy-stream memsets vs non-blocking streams
}

Bank::~Bank() {
    DeviceGuard g(eng_.device());
    if (stream_) cudaStreamSynchronize(stream_);
    ws_.release();
    if (keep_pin_) cudaFreeHost(keep_pin_);
    cudaFree(k_);
    cudaFree(v_);
    if (stream_) cudaStreamDestroy(stream_);
}

float* Bank::kslab(int layer) const { return k_ + slab_elems_ * (layer - lb_); }
float* Bank::vslab(int layer) const { return v_ + slab_elems_ * (layer - lb_); }

// CacheBank::resolve (tinyformer.cpp:282-308): validate on the host, then
// enqueue the in-place compaction on `s` (the stream that runs the next
// forward, so no host sync is needed).  s == nullptr: the bank's own stream,
// synchronised (seam-2 callers).
void Bank::resolve(const int32_t* keep, int n, cudaStream_t s) {
    const int tail = provisional();
    int prev = -1;
    for (int i = 0; i < n; ++i) {
        if (keep[i] <= prev || keep[i] >= tail)
            throw Error(Kind::protocol,
                        "keep indices must be strictly increasing and within the provisional tail");
        prev = keep[i];
    }
    bool identity = true;
    for (int i = 0; i < n; ++i) identity = identity && keep[i] == i;
    if (!identity && le_ > lb_) {
        DeviceGuard g(eng_.device());
        const bool own = s == nullptr;
        cudaStream_t st = own ? stream_ : s;
        enqueue_compact(keep, n, committed_, st);
        if (own) SFG_CUDA(cudaStreamSynchronize(st));
    }
    committed_ += n;
    len_ = committed_;
}

// The device half of resolve: kept tail entries committed + keep[i] move to
// committed + i on stream st (any keep length: sfg_common.cu compacts in
// chunks).  The keep list crosses through this bank's pinned buffer; the
// previous resolve's copy has completed (every step ends in a sync).
void Bank::enqueue_compact(const int32_t* keep, int n, int committed, cudaStream_t st) {
    if (n <= 0 || le_ == lb_) return;
    DeviceGuard g(eng_.device());
    eng_.ensure_ws(ws_, std::max(n, 1), 1, 0);
    if (n > keep_pin_cap_) {
        if (keep_pin_) {
            SFG_CUDA(cudaDeviceSynchronize());
            cudaFreeHost(keep_pin_);
        }
        keep_pin_cap_ = std::max(n, 1024);
        SFG_CUDA(cudaMallocHost(&keep_pin_, sizeof(int32_t) * keep_pin_cap_));
    }
    std::memcpy(keep_pin_, keep, sizeof(int32_t) * n);
    SFG_CUDA(cudaMemcpyAsync(ws_.keep, keep_pin_, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    const ModelCfg& c = eng_.cfg();
    launch_kv_compact(k_, v_, le_ - lb_, c.n_kv_heads, c.max_seq_len, c.head_dim, committed, ws_.keep, n, st);
    SFG_CUDA(cudaGetLastError());
}

void Bank::resolve_meta(const int32_t* keep, int n) {
    const int tail = provisional();
    int prev = -1;
    for (int i = 0; i < n; ++i) {
        if (keep[i] <= prev || keep[i] >= tail)
            throw Error(Kind::protocol,
                        "keep indices must be strictly increasing and within the provisional tail");
        prev = keep[i];
    }
    committed_ += n;
    len_ = committed_;
}

// CacheBank::crop (tinyformer.cpp:310-316): metadata only.
void Bank::crop(int pos) {
    if (pos < 0 || pos > len()) throw Error(Kind::protocol, "crop position exceeds cache length");
    len_ = pos;
    committed_ = std::min(committed_, pos);
}

void Bank::read_kv(int layer, int head, int pos, float* k, float* v) {
    const ModelCfg& c = eng_.cfg();
    if (layer < lb_ || layer >= le_ || head < 0 || head >= c.n_kv_heads || pos < 0 || pos >= c.max_seq_len)
        throw Error(Kind::input, "kv index out of range");
    DeviceGuard g(eng_.device());
    SFG_CUDA(cudaStreamSynchronize(stream_));
    const size_t off = (static_cast<size_t>(head) * c.max_seq_len + pos) * c.head_dim;
    SFG_CUDA(cudaMemcpy(k, kslab(layer) + off, sizeof(float) * c.head_dim, cudaMemcpyDeviceToHost));
    SFG_CUDA(cudaMemcpy(v, vslab(layer) + off, sizeof(float) * c.head_dim, cudaMemcpyDeviceToHost));
}

// ── engine: weights ───────────────────────────────────────────────────────
Dims Engine::dims() const {
    const ModelCfg& c = cfg_;
    const int t = tp_size_;
    return Dims{c.hidden_dim, c.q_dim() / t, c.kv_dim() / t, c.ffn_dim / t, c.vocab_size, c.n_heads / t,
                c.n_kv_heads / t, c.head_dim, c.max_seq_len, c.rms_eps};
}

static float bf16_rne_host(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return v;
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&v, &u, 4);
    return v;
}

Engine::Engine(const ModelCfg& cfg, const sfg_engine_options& opt, const float* params, const TpConfig& tp)
    : cfg_(cfg), opt_(opt), tp_size_(tp.size), tp_rank_(tp.rank) {
    cfg_.validate(opt_.extended_shapes != 0);
    if (tp_size_ < 1 || tp_rank_ < 0 || tp_rank_ >= tp_size_) throw Error(Kind::config, "invalid tensor-parallel rank");
    if (tp_size_ > 1) {
        if (opt_.math != SFG_MATH_FAST) throw Error(Kind::config, "tensor parallelism runs FAST math");
        if (cfg_.n_kv_heads % tp_size_ || cfg_.ffn_dim % (64 * tp_size_) || (cfg_.q_dim() / tp_size_) % 64)
            throw Error(Kind::config, "kv heads, ffn_dim/64 and q_dim/64 must split evenly over the tensor-parallel group");
        if (!tp.unique_id) throw Error(Kind::input, "tensor parallelism needs the group's NCCL unique id");
    }
    if (opt_.layer_begin < 0 || opt_.layer_end > cfg_.n_layers || opt_.layer_begin > opt_.layer_end)
        throw Error(Kind::config, "hosted layer range must lie inside the model");
    if (opt_.math != SFG_MATH_EXACT && opt_.math != SFG_MATH_FAST)
        throw Error(Kind::config, "unknown math mode");
    if (opt_.math == SFG_MATH_FAST && opt_.weight_dtype != SFG_WEIGHTS_BF16)
        throw Error(Kind::config, "FAST math streams bf16 weights");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(Kind::internal, "no CUDA device: the B200 engine has no CPU fallback");
    if (opt_.device < 0 || opt_.device >= ndev) throw Error(Kind::config, "CUDA device ordinal out of range");
    DeviceGuard g(opt_.device);
    if (tp_size_ > 1) tp_comm_ = tp_comm_init(tp_size_, tp_rank_, tp.unique_id);
    cudaDeviceProp prop{};
    SFG_CUDA(cudaGetDeviceProperties(&prop, opt_.device));
    if (prop.major != 10) throw Error(Kind::internal, "libsfg is built for sm_100a (B200) only");
    SFG_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    layers_.resize(cfg_.n_layers);
    try {
        load(params);
        if (fast()) build_fast_layouts();
        SFG_CUDA(cudaStreamSynchronize(stream_));
    } catch (...) {
        for (void* p : allocs_) cudaFree(p);
        if (staging_) cudaFree(staging_);
        throw;
    }
    if (staging_) cudaFree(staging_);
    staging_ = nullptr;
    if (tp_size_ == 2 && fast()) tp_setup_peer();
}

// Allocate this rank's inbox, share its CUDA IPC handle over the NCCL group
// and map the peer's (TP = 2: one peer over NVLink).
void Engine::tp_setup_peer() {
    const ModelCfg& c = cfg_;
    const size_t tilesH = (c.hidden_dim + 127) / 128;
    // one 64-bit word {epoch, f32} per exchanged value (sfg_mega.cu epi_final)
    tp_peer_.data_floats = static_cast<size_t>(c.n_layers) * 2 * tilesH * 16 * 128 * 2;
    const size_t nflags = static_cast<size_t>(c.n_layers) * 2 * tilesH;
    const size_t bytes = tp_peer_.data_floats * sizeof(float) + nflags * sizeof(unsigned) + 256;
    SFG_CUDA(cudaMalloc(&tp_peer_.base, bytes));
    SFG_CUDA(cudaMemset(tp_peer_.base, 0, bytes));
    SFG_CUDA(cudaMalloc(&tp_peer_.epoch, sizeof(unsigned)));
    SFG_CUDA(cudaMemset(tp_peer_.epoch, 0, sizeof(unsigned)));
    tp_peer_.inbox = static_cast<float*>(tp_peer_.base);
    tp_peer_.inflag = reinterpret_cast<unsigned*>(tp_peer_.inbox + tp_peer_.data_floats);
    cudaIpcMemHandle_t mine{};
    SFG_CUDA(cudaIpcGetMemHandle(&mine, tp_peer_.base));
    void* dev = nullptr;
    SFG_CUDA(cudaMalloc(&dev, 2 * sizeof(cudaIpcMemHandle_t) + sizeof(cudaIpcMemHandle_t)));
    char* all = static_cast<char*>(dev) + sizeof(cudaIpcMemHandle_t);
    SFG_CUDA(cudaMemcpy(dev, &mine, sizeof(mine), cudaMemcpyHostToDevice));
    tp_allgather_bytes(tp_comm_, dev, all, sizeof(cudaIpcMemHandle_t), stream_);
    SFG_CUDA(cudaStreamSynchronize(stream_));
    cudaIpcMemHandle_t handles[2];
    SFG_CUDA(cudaMemcpy(handles, all, sizeof(handles), cudaMemcpyDeviceToHost));
    cudaFree(dev);
    SFG_CUDA(cudaIpcOpenMemHandle(&tp_peer_.peer_base, handles[1 - tp_rank_], cudaIpcMemLazyEnablePeerAccess));
    tp_peer_.peer_inbox = static_cast<float*>(tp_peer_.peer_base);
    tp_peer_.peer_inflag = reinterpret_cast<unsigned*>(tp_peer_.peer_inbox + tp_peer_.data_floats);
}

Engine::~Engine() {
    DeviceGuard g(opt_.device);
    cudaStreamSynchronize(stream_);
    ws_.release();
    for (void* p : allocs_) cudaFree(p);
    if (rope_cos_) cudaFree(rope_cos_);
    if (rope_sin_) cudaFree(rope_sin_);
    cudaStreamDestroy(stream_);
    if (tp_peer_.peer_base) cudaIpcCloseMemHandle(tp_peer_.peer_base);
    if (tp_peer_.base) cudaFree(tp_peer_.base);
    if (tp_peer_.epoch) cudaFree(tp_peer_.epoch);
    tp_comm_destroy(tp_comm_);
}

void Engine::tp_allreduce(float* buf, size_t n, cudaStream_t s) {
    if (tp_size_ > 1) tp_allreduce_sum(tp_comm_, buf, n, s);
}

// Upload n fp32 values (already on device staging) into storage dtype `wt`.
void Engine::upload_tensor(const float* dev_src, size_t n, void** dst, int wt) {
    const size_t bytes = n * (wt == W_BF16 ? 2 : 4);
    SFG_CUDA(cudaMalloc(dst, bytes));
    allocs_.push_back(*dst);
    weight_bytes_ += static_cast<int64_t>(bytes);
    launch_convert_weights(dev_src, *dst, wt, n, stream_);
    SFG_CUDA(cudaGetLastError());
}

// Weights: either the flat snapshot-order array, or the init_weights stream
// (tinyformer.cpp:123-152: one mt19937_64(seed) stream in declaration order,
// v = a * (float)(2 * ((rng() >> 11) * 2^-53) - 1), a = 1/sqrtf(hidden)).
// Tensors the engine does not host are skipped in the stream.  Values are
// rounded to the storage dtype (bf16 RNE) on device; norm gains are stored as
// fp32 holding the same rounded values.
void Engine::load(const float* params) {
    const ModelCfg& c = cfg_;
    const size_t H = c.hidden_dim, qd = c.q_dim(), kvd = c.kv_dim(), F = c.ffn_dim, V = c.vocab_size;
    const int wt_ = wt();
    std::mt19937_64 rng(c.seed);
    const float a = 1.0f / std::sqrt(static_cast<float>(c.hidden_dim));
    size_t cursor = 0;  // offset into params

    constexpr size_t kChunk = size_t{1} << 24;  // 16M floats per staging chunk
    staging_elems_ = kChunk;
    SFG_CUDA(cudaMalloc(&staging_, kChunk * sizeof(float) * 2));
    float* host[2] = {nullptr, nullptr};
    SFG_CUDA(cudaMallocHost(&host[0], kChunk * sizeof(float)));
    SFG_CUDA(cudaMallocHost(&host[1], kChunk * sizeof(float)));
    cudaEvent_t done[2];
    SFG_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    SFG_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    SFG_CUDA(cudaEventRecord(done[0], stream_));
    SFG_CUDA(cudaEventRecord(done[1], stream_));
    int slot = 0;

    auto next = [&](void) -> float {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        return a * static_cast<float>(2.0 * u - 1.0);
    };
    // Produce tensor of n values; keep=false skips it in the stream.
    auto tensor = [&](size_t n, bool keep, bool is_norm, void** dst) {
        if (!keep) {
            if (params) cursor += n;
            else rng.discard(n);
            return;
        }
        if (is_norm) {
            std::vector<float> tmp(n);
            for (size_t i = 0; i < n; ++i) {
                const float v = params ? params[cursor + i] : next();
                tmp[i] = wt_ == W_BF16 ? bf16_rne_host(v) : v;
            }
            if (params) cursor += n;
            SFG_CUDA(cudaMalloc(dst, n * sizeof(float)));
            allocs_.push_back(*dst);
            weight_bytes_ += static_cast<int64_t>(n * sizeof(float));
            SFG_CUDA(cudaMemcpy(*dst, tmp.data(), n * sizeof(float), cudaMemcpyHostToDevice));
            return;
        }
        const size_t bytes = n * (wt_ == W_BF16 ? 2 : 4);
        SFG_CUDA(cudaMalloc(dst, bytes));
        allocs_.push_back(*dst);
        weight_bytes_ += static_cast<int64_t>(bytes);
        for (size_t off = 0; off < n; off += kChunk) {
            const size_t m = std::min(kChunk, n - off);
            SFG_CUDA(cudaEventSynchronize(done[slot]));
            float* hb = host[slot];
            if (params) {
                for (size_t i = 0; i < m; ++i) {
                    const float v = params[cursor + off + i];
                    if (!std::isfinite(v)) throw Error(Kind::input, "non-finite parameter in weight snapshot");
                    hb[i] = v;
                }
            } else {
                for (size_t i = 0; i < m; ++i) hb[i] = next();
            }
            float* ds = staging_ + slot * kChunk;
            SFG_CUDA(cudaMemcpyAsync(ds, hb, m * sizeof(float), cudaMemcpyHostToDevice, stream_));
            char* d8 = static_cast<char*>(*dst) + off * (wt_ == W_BF16 ? 2 : 4);
            launch_convert_weights(ds, d8, wt_, m, stream_);
            SFG_CUDA(cudaGetLastError());
            SFG_CUDA(cudaEventRecord(done[slot], stream_));
            slot ^= 1;
        }
        if (params) cursor += n;
    };

    void* dummy = nullptr;
    tensor(V * H, opt_.with_embedding != 0, false, opt_.with_embedding ? &embedding_ : &dummy);
    for (int l = 0; l < c.n_layers; ++l) {
        LayerWeights& L = layers_[l];
        const bool k = l >= opt_.layer_begin && l < opt_.layer_end;
        L.hosted = k;
        tensor(H, k, true, (void**)&L.attn_norm);
        tensor(H * qd, k, false, &L.wq);
        tensor(H * kvd, k, false, &L.wk);
        tensor(H * kvd, k, false, &L.wv);
        tensor(qd * H, k, false, &L.wo);
        tensor(H, k, true, (void**)&L.ffn_norm);
        tensor(H * F, k, false, &L.w_gate);
        tensor(H * F, k, false, &L.w_up);
        tensor(F * H, k, false, &L.w_down);
    }
    tensor(H, opt_.with_head != 0, true, (void**)&final_norm_);
    tensor(H * V, opt_.with_head != 0, false, &lm_head_);
    SFG_CUDA(cudaStreamSynchronize(stream_));
    cudaFreeHost(host[0]);
    cudaFreeHost(host[1]);
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);

    // RoPE table: the reference recomputes, per call, freq = powf(base,
    // -2i/hd), angle = pos*freq, sincosf(angle) (tinyformer.cpp:52-63) with the
    // host libm; the same host expressions fill [max_seq][hd/2] once here.
    const int half = c.head_dim / 2;
    std::vector<float> cs(static_cast<size_t>(c.max_seq_len) * half), sn(cs.size());
    for (int i = 0; i < half; ++i) {
        const float freq = std::pow(c.rope_base, -2.0f * static_cast<float>(i) / static_cast<float>(c.head_dim));
        for (int p = 0; p < c.max_seq_len; ++p) {
            const float ang = static_cast<float>(p) * freq;
            float s, co;
            sincosf(ang, &s, &co);
            cs[static_cast<size_t>(p) * half + i] = co;
            sn[static_cast<size_t>(p) * half + i] = s;
        }
    }
    SFG_CUDA(cudaMalloc(&rope_cos_, cs.size() * sizeof(float)));
    SFG_CUDA(cudaMalloc(&rope_sin_, sn.size() * sizeof(float)));
    SFG_CUDA(cudaMemcpy(rope_cos_, cs.data(), cs.size() * sizeof(float), cudaMemcpyHostToDevice));
    SFG_CUDA(cudaMemcpy(rope_sin_, sn.data(), sn.size() * sizeof(float), cudaMemcpyHostToDevice));
}

// FAST math streams weights from a tiled, pre-swizzled W^T image (see
// sfg_fast.cu); the reference-layout copies are released afterwards.
void Engine::build_fast_layouts() {
    auto release = [&](void*& p) {
        if (!p) return;
        for (auto it = allocs_.begin(); it != allocs_.end(); ++it)
            if (*it == p) {
                allocs_.erase(it);
                break;
            }
        cudaFree(p);
        p = nullptr;
    };
    for (int l = 0; l < cfg_.n_layers; ++l) {
        LayerWeights& L = layers_[l];
        if (!L.hosted) continue;
        fast_build_layer(*this, L, stream_);
        SFG_CUDA(cudaStreamSynchronize(stream_));
        const size_t H = cfg_.hidden_dim, qd = cfg_.q_dim(), kvd = cfg_.kv_dim(), F = cfg_.ffn_dim;
        weight_bytes_ -= static_cast<int64_t>(2 * (H * qd + 2 * H * kvd + qd * H + 3 * H * F));  // full copies released
        release(L.wq);
        release(L.wk);
        release(L.wv);
        release(L.wo);
        release(L.w_gate);
        release(L.w_up);
        release(L.w_down);
    }
    if (lm_head_) {
        f_lm_head_ = fast_build_head(*this, lm_head_, stream_);
        SFG_CUDA(cudaStreamSynchronize(stream_));
        weight_bytes_ -= static_cast<int64_t>(2 * static_cast<size_t>(cfg_.hidden_dim) * cfg_.vocab_size);
        release(lm_head_);
    }
    SFG_CUDA(cudaStreamSynchronize(stream_));
}

// ── engine: execution ─────────────────────────────────────────────────────
int& mega_mode() {
    static int on = -1;
    if (on < 0) {
        const char* v = std::getenv("SFG_MEGA");
        on = (v && v[0] == '0') ? 0 : 1;
    }
    return on;
}
static bool mega_env_enabled() { return mega_mode() == 1; }

int Engine::forward_device(Bank& b, int lb, int le, int rows, Workspace& ws, cudaStream_t s) {
    const Dims d = dims();
    const int prior = b.len();
    int n = 0;
    if (lb >= le) return 0;
    // (the attention design is decided only for megakernel-sized steps, never at a prompt pass)
    if (fast() && (tp_size_ == 1 || tp_peer_.peer_inbox) && mega_env_enabled() && le - lb <= 50 &&
        rows <= 16 && !ws.additive_mask && mega_supported(*this, rows, false, bank_rows_attention(b))) {
        for (int layer = lb; layer < le; ++layer)
            if (!layers_[layer].hosted) throw Error(Kind::internal, "layer not hosted by this engine");
        return mega_forward(*this, b, lb, le, rows, ws, s);
    }
    for (int layer = lb; layer < le; ++layer) {
        const LayerWeights& L = layers_[layer];
        if (!L.hosted) throw Error(Kind::internal, "layer not hosted by this engine");
        if (fast()) {
            n += fast_forward_layer(*this, b, layer, rows, ws, prior, s);
            continue;
        }
        float* kc = b.kslab(layer);
        float* vc = b.vslab(layer);
        const double wb = wt() == W_BF16 ? 2.0 : 4.0, R = rows;
        const int qkv = d.qd + 2 * d.kvd;
        {
            ProfScope p(K_NORM, s, R * d.H * 8.0 + d.H * 4.0, 0);
            n += launch_rmsnorm_exact(ws.h, L.attn_norm, ws.xn, rows, d.H, d.eps, s);
        }
        {
            ProfScope p(K_QKV, s, wb * d.H * qkv + 4.0 * R * (d.H + qkv), 2.0 * R * d.H * qkv);
            n += launch_qkv_exact(ws.xn, rows, d, wt(), L.wq, L.wk, L.wv, ws.pos, rope_cos_, rope_sin_, ws.q, kc,
                                  vc, ws.meta, s);
        }
        {
            const double kvb = 2.0 * 4.0 * d.kvd * (prior + rows);
            ProfScope p(K_ATTN, s, kvb + 8.0 * R * d.qd, 4.0 * R * d.qd * (prior + rows));
            n += launch_attention_exact(ws.q, kc, vc, ws.row_off, ws.runs, rows, prior + rows, d, ws.att,
                                        ws.status, s);
        }
        {
            ProfScope p(K_OPROJ, s, wb * d.qd * d.H + 4.0 * R * (d.qd + 2.0 * d.H), 2.0 * R * d.qd * d.H);
            n += launch_matvec_residual_exact(ws.att, rows, d.qd, wt(), L.wo, d.H, ws.h, s);
        }
        {
            ProfScope p(K_NORM, s, R * d.H * 8.0 + d.H * 4.0, 0);
            n += launch_rmsnorm_exact(ws.h, L.ffn_norm, ws.xn, rows, d.H, d.eps, s);
        }
        {
            ProfScope p(K_GATEUP, s, 2.0 * wb * d.H * d.F + 4.0 * R * (d.H + d.F), 4.0 * R * d.H * d.F);
            n += launch_gateup_exact(ws.xn, rows, d.H, d.F, wt(), L.w_gate, L.w_up, ws.act, s);
        }
        {
            ProfScope p(K_DOWN, s, wb * d.F * d.H + 4.0 * R * (d.F + 2.0 * d.H), 2.0 * R * d.F * d.H);
            n += launch_matvec_residual_exact(ws.act, rows, d.F, wt(), L.w_down, d.H, ws.h, s);
        }
    }
    return n;
}

int Engine::head_device(int rows, Workspace& ws, bool want_logits, bool want_argmax, cudaStream_t s) {
    if (!final_norm_ || (!lm_head_ && !f_lm_head_)) throw Error(Kind::internal, "engine does not host the LM head");
    if (fast()) {
        (void)want_argmax;  // the FAST head always produces the argmax
        return fast_head(*this, f_lm_head_, final_norm_, rows, ws, want_logits, s);
    }
    const Dims d = dims();
    int n = 0;
    const double wb = wt() == W_BF16 ? 2.0 : 4.0, R = rows;
    n += launch_rmsnorm_exact(ws.h, final_norm_, ws.xn, rows, d.H, d.eps, s);
    {
        ProfScope p(K_HEAD, s, wb * d.H * d.V + 4.0 * R * (d.H + d.V), 2.0 * R * d.H * d.V);
        n += launch_matvec_store_exact(ws.xn, rows, d.H, wt(), lm_head_, d.V, ws.logits, s);
    }
    if (want_argmax) n += launch_argmax(ws.logits, rows, d.V, ws.argmax, s);
    (void)want_logits;
    return n;
}

int Engine::embed_device(int rows, Workspace& ws, cudaStream_t s) {
    if (!embedding_) throw Error(Kind::internal, "engine does not host the embedding");
    return launch_embed(embedding_, wt(), ws.ids, rows, cfg_.hidden_dim, ws.h, s);
}

static bool all_finite(const float* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) return false;
    return true;
}

// forward_layers (tinyformer.cpp:375-508) over host buffers, same checks in
// the same order.
void Engine::forward_host(Bank& b, int lb, int le, int seq, const float* h, const int32_t* pos,
                          const float* mask, float* out) {
    const ModelCfg& c = cfg_;
    const size_t H = c.hidden_dim;
    if (lb == le) {
        std::memcpy(out, h, sizeof(float) * seq * H);
        return;
    }
    if (lb < b.layer_begin() || le > b.layer_end()) throw Error(Kind::internal, "layer range outside cache bank");
    if (seq == 0) return;
    const int prior = b.len();
    if (prior + seq > c.max_seq_len) throw Error(Kind::capacity, "sequence exceeds max_seq_len");
    if (!all_finite(h, seq * H)) throw Error(Kind::numeric, "non-finite hidden state");
    for (int i = 0; i < seq; ++i)
        if (pos[i] < 0 || pos[i] >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
    MaskRuns mr = mask ? runs_from_dense(mask, seq, prior + seq) : causal_runs(seq, prior);
    if (mr.any_empty_row) throw Error(Kind::protocol, "mask row admits no attendable position");

    DeviceGuard g(device());
    Workspace& ws = b.ws();
    cudaStream_t s = b.stream();
    ensure_ws(ws, seq, static_cast<int>(mr.runs.size()), 0);
    ws.additive_mask = !mega_mask_ok(mr, prior);
    ws.prefix_mask = prefix_law(mr);
    SFG_CUDA(cudaMemcpyAsync(ws.h, h, sizeof(float) * seq * H, cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(ws.pos, pos, sizeof(int32_t) * seq, cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(ws.row_off, mr.row_off.data(), sizeof(int32_t) * (seq + 1), cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(ws.runs, mr.runs.data(), sizeof(MaskRun) * mr.runs.size(), cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemsetAsync(ws.status, 0, sizeof(uint32_t), s));
    set_prior(ws, prior, s);
    forward_device(b, lb, le, seq, ws, s);
    SFG_CUDA(cudaGetLastError());
    uint32_t st = 0;
    SFG_CUDA(cudaMemcpyAsync(out, ws.h, sizeof(float) * seq * H, cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaMemcpyAsync(&st, ws.status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    if (st & ST_ATTN_CAP) throw Error(Kind::internal, "attention launch sized below the visible key count");
    if (st & ST_EMPTY_ROW) throw Error(Kind::protocol, "mask row admits no attendable position");
    b.set_len(prior + seq);
}

// embed_at (tinyformer.cpp:348-373)
void Engine::embed_host(int seq, const int32_t* ids, const int32_t* pos, float* out) {
    const ModelCfg& c = cfg_;
    for (int i = 0; i < seq; ++i)
        if (pos[i] < 0 || pos[i] >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
    for (int i = 0; i < seq; ++i)
        if (ids[i] < 0 || ids[i] >= c.vocab_size) throw Error(Kind::input, "token id out of range");
    std::lock_guard<std::mutex> lk(mu_);
    DeviceGuard g(device());
    ensure_ws(ws_, seq, 1, 0);
    SFG_CUDA(cudaMemcpyAsync(ws_.ids, ids, sizeof(int32_t) * seq, cudaMemcpyHostToDevice, stream_));
    embed_device(seq, ws_, stream_);
    SFG_CUDA(cudaGetLastError());
    SFG_CUDA(cudaMemcpyAsync(out, ws_.h, sizeof(float) * seq * c.hidden_dim, cudaMemcpyDeviceToHost, stream_));
    SFG_CUDA(cudaStreamSynchronize(stream_));
}

// finalize (tinyformer.cpp:510-526) [+ argmax_row :329-340]
void Engine::finalize_host(int seq, const float* h, float* logits, int32_t* argmax) {
    const ModelCfg& c = cfg_;
    if (!all_finite(h, static_cast<size_t>(seq) * c.hidden_dim)) throw Error(Kind::numeric, "non-finite hidden state");
    if (seq == 0) return;
    std::lock_guard<std::mutex> lk(mu_);
    DeviceGuard g(device());
    ensure_ws(ws_, seq, 1, seq);
    SFG_CUDA(cudaMemcpyAsync(ws_.h, h, sizeof(float) * seq * c.hidden_dim, cudaMemcpyHostToDevice, stream_));
    head_device(seq, ws_, logits != nullptr, argmax != nullptr, stream_);
    SFG_CUDA(cudaGetLastError());
    if (logits)
        SFG_CUDA(cudaMemcpyAsync(logits, ws_.logits, sizeof(float) * seq * c.vocab_size, cudaMemcpyDeviceToHost, stream_));
    if (argmax)
        SFG_CUDA(cudaMemcpyAsync(argmax, ws_.argmax, sizeof(int32_t) * seq, cudaMemcpyDeviceToHost, stream_));
    SFG_CUDA(cudaStreamSynchronize(stream_));
}

}  // namespace sfg
