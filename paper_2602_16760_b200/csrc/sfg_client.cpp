// Trusted-side runtime: SplitClient::prefill/decode_step (client.cpp:120-228)
// and decode_sequential / decode_lookahead_with_pool (decoding.cpp:111-355)
// on the B200.
//
// A decode step splits into host work (protocol checks and cache
// bookkeeping, exactly as the reference orders them) and one device
// sequence: [inputs H2D] -> in-place KV compaction (prefix, suffix and, when
// device-linked, the server's bank) -> embed -> prefix layers -> wire round
// trip -> server layers -> wire round trip -> suffix layers -> final norm +
// LM head -> argmax -> verify/branch selection -> [summary D2H].  Every
// per-step scalar lives in device memory (Workspace::meta), so the device
// sequence of a device-linked step is captured once per batch size as a
// CUDA graph and replayed.
#include "sfg_client.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <cstdlib>
#include <thread>

#include "sfg_prof.h"

namespace sfg {

using Clock = std::chrono::steady_clock;

// ── NGramPool ─────────────────────────────────────────────────────────────
Pool::Pool(int n, size_t cap) : n_(n), cap_(cap) {
    if (n < 2) throw Error(Kind::config, "ngram_n must be >= 2");
    if (cap < 1) throw Error(Kind::config, "pool capacity must be >= 1");
}

Pool::~Pool() {
    for (Node* p = head_; p;) {
        Node* nx = p->gnext;
        delete p;
        p = nx;
    }
}

void Pool::link_front(Node* n) {
    n->gprev = nullptr;
    n->gnext = head_;
    if (head_) head_->gprev = n;
    head_ = n;
    if (!tail_) tail_ = n;
    KeyList& kl = keys_[n->key];
    n->kprev = nullptr;
    n->knext = kl.head;
    if (kl.head) kl.head->kprev = n;
    kl.head = n;
    if (!kl.tail) kl.tail = n;
}

void Pool::unlink(Node* n) {
    (n->gprev ? n->gprev->gnext : head_) = n->gnext;
    (n->gnext ? n->gnext->gprev : tail_) = n->gprev;
    KeyList& kl = keys_[n->key];
    (n->kprev ? n->kprev->knext : kl.head) = n->knext;
    (n->knext ? n->knext->kprev : kl.tail) = n->kprev;
}

// NGramPool::insert (decoding.cpp:66-75)
void Pool::insert(int32_t key, const int32_t* cont) {
    auto it = keys_.find(key);
    if (it != keys_.end())
        for (Node* p = it->second.head; p; p = p->knext)
            if (std::equal(p->cont.begin(), p->cont.end(), cont)) {  // refresh recency
                unlink(p);
                link_front(p);
                return;
            }
    Node* nd = new Node;
    nd->key = key;
    nd->cont.assign(cont, cont + (n_ - 1));
    link_front(nd);
    if (++size_ > cap_) {  // pop_back
        Node* old = tail_;
        unlink(old);
        delete old;
        --size_;
    }
}

// NGramPool::update (decoding.cpp:77-87)
void Pool::update(const int32_t* prev, const int32_t* cur, int w) {
    for (int i = 0; i + n_ - 1 <= w - 1; ++i) insert(prev[i], cur + i + 1);
}

// NGramPool::lookup (decoding.cpp:89-97): push, then stop at max_c, so
// lookup(key, 0) still yields one hit, as in the reference.
int Pool::lookup(int key, int max_c, std::vector<std::vector<int32_t>>& out) const {
    out.clear();
    auto it = keys_.find(key);
    if (it == keys_.end()) return 0;
    for (const Node* p = it->second.head; p; p = p->knext) {
        out.push_back(p->cont);
        if (static_cast<int>(out.size()) >= max_c) break;
    }
    return static_cast<int>(out.size());
}

// ── Client ────────────────────────────────────────────────────────────────
static Kind kind_from_message(const std::string& msg) {
    const size_t colon = msg.find(':');
    const std::string head = colon == std::string::npos ? msg : msg.substr(0, colon);
    for (int k = 1; k <= 10; ++k)
        if (head == kind_name(static_cast<Kind>(k))) return static_cast<Kind>(k);
    return Kind::protocol;
}

Client::Client(Engine& local, const ClientCfg& cfg, sfg_frame_handler handler, void* ctx, Server* linked,
               std::string sid)
    : eng_(local), cfg_(cfg), handler_(handler), ctx_(ctx), linked_(linked), sid_(std::move(sid)) {
    const ModelCfg& c = local.cfg();
    // SplitConfig::validate (client.cpp:39-46)
    if (cfg_.prefix_layers < 1 || cfg_.suffix_layers < 1)
        throw Error(Kind::config, "prefix and suffix must each host >= 1 layer");
    if (cfg_.prefix_layers + cfg_.suffix_layers >= c.n_layers)
        throw Error(Kind::config, "prefix + suffix must leave a non-empty middle range");
    if (!handler_ && !linked_) throw Error(Kind::config, "client needs a frame handler or a linked server");
    if (linked_) {
        const Engine& se = linked_->engine();
        const ModelCfg& sc = se.cfg();
        if (se.device() != local.device()) throw Error(Kind::config, "a linked server must live on the client's device");
        if (se.fast() != local.fast()) throw Error(Kind::config, "a linked server must use the client's math mode");
        if (sc.hidden_dim != c.hidden_dim || sc.ffn_dim != c.ffn_dim || sc.n_heads != c.n_heads ||
            sc.n_kv_heads != c.n_kv_heads || sc.head_dim != c.head_dim || sc.vocab_size != c.vocab_size ||
            sc.max_seq_len != c.max_seq_len || sc.n_layers != c.n_layers)
            throw Error(Kind::config, "a linked server must serve the client's model shape");
        if (linked_->config().layer_begin != cfg_.prefix_layers ||
            linked_->config().layer_end != c.n_layers - cfg_.suffix_layers)
            throw Error(Kind::config, "server layer range does not match the client split");
    }
    if (sid_.empty()) {  // random_session_id (client.cpp:16-23)
        static const char* hex = "0123456789abcdef";
        std::random_device rd;
        std::mt19937_64 rng((static_cast<uint64_t>(rd()) << 32) ^ rd());
        sid_ = "sess-";
        for (int i = 0; i < 16; ++i) sid_.push_back(hex[rng() & 0xf]);
    }
    prefix_ = std::make_unique<Bank>(local, 0, cfg_.prefix_layers);
    suffix_ = std::make_unique<Bank>(local, c.n_layers - cfg_.suffix_layers, c.n_layers);
    DeviceGuard g(local.device());
    for (auto& e : ev_) SFG_CUDA(cudaEventCreate(&e));
    SFG_CUDA(cudaMalloc(&d_vin_, sizeof(VerifyIn)));
    SFG_CUDA(cudaMalloc(&d_vout_, sizeof(VerifyOut)));
    SFG_CUDA(cudaMallocHost(&h_vin_, sizeof(VerifyIn)));
    SFG_CUDA(cudaMallocHost(&h_vout_, sizeof(VerifyOut)));
    std::memset(h_vin_, 0, sizeof(VerifyIn));
}

Client::~Client() {
    DeviceGuard g(eng_.device());
    cudaStreamSynchronize(prefix_->stream());
    for (auto& gr : graphs_) {
        if (gr.exec) cudaGraphExecDestroy(gr.exec);
        KernelProfiler::get().release_graph(gr.prof_slots);
    }
    for (auto& e : ev_) cudaEventDestroy(e);
    cudaFree(d_vin_);
    cudaFree(d_vout_);
    cudaFreeHost(h_vin_);
    cudaFreeHost(h_vout_);
    if (h_argmax_) cudaFreeHost(h_argmax_);
    if (h_logits_) cudaFreeHost(h_logits_);
}

uint64_t Client::clamped() {
    Workspace& ws = prefix_->ws();
    if (!ws.clamped) return 0;
    unsigned long long v = 0;
    DeviceGuard g(eng_.device());
    SFG_CUDA(cudaStreamSynchronize(prefix_->stream()));
    SFG_CUDA(cudaMemcpy(&v, ws.clamped, sizeof(v), cudaMemcpyDeviceToHost));
    return v;
}

// precise_sleep_ms (transport.cpp:36-46): coarse sleep then spin.
void Client::sleep_one_way() const {
    const double ms = cfg_.one_way_delay_ms;
    if (ms <= 0.0) return;
    const auto t0 = Clock::now();
    if (ms > 2.0) std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(ms - 2.0));
    while (std::chrono::duration<double, std::milli>(Clock::now() - t0).count() < ms) {
    }
}

void Client::ensure_out(int rows) {
    if (rows <= out_rows_) return;
    SFG_CUDA(cudaDeviceSynchronize());
    if (h_argmax_) cudaFreeHost(h_argmax_);
    if (h_logits_) cudaFreeHost(h_logits_);
    const int r = std::max(rows, 16);
    SFG_CUDA(cudaMallocHost(&h_argmax_, sizeof(int32_t) * r));
    SFG_CUDA(cudaMallocHost(&h_logits_, sizeof(float) * static_cast<size_t>(r) * eng_.cfg().vocab_size));
    out_rows_ = r;
    for (auto& gr : graphs_) gr.generation = ~0ull;  // outputs moved: recapture
}

// Host staging of the step inputs at cap-derived offsets (fixed addresses,
// so a captured graph's copy nodes stay valid).
void Client::stage_inputs(int seq, const int32_t* ids, const int32_t* pos, const MaskRuns& mr) {
    Workspace& ws = prefix_->ws();
    const StageLayout L = stage_layout(ws.cap_rows, ws.cap_runs);
    char* p = static_cast<char*>(ws.stage_pin);
    std::memcpy(p + L.ids, ids, sizeof(int32_t) * seq);
    std::memcpy(p + L.pos, pos, sizeof(int32_t) * seq);
    std::memcpy(p + L.roff, mr.row_off.data(), sizeof(int32_t) * mr.row_off.size());
    std::memcpy(p + L.runs, mr.runs.data(), sizeof(MaskRun) * mr.runs.size());
    ws.additive_mask = !mega_mask_ok(mr, prefix_->len());
    ws.prefix_mask = prefix_law(mr);
}

// [inputs H2D] -> compaction -> embed -> prefix layers
int Client::dev_pre(int rows, Bank* server_bank, bool verify, cudaStream_t s) {
    const ModelCfg& c = eng_.cfg();
    Workspace& ws = prefix_->ws();
    const StageLayout L = stage_layout(ws.cap_rows, ws.cap_runs);
    const char* p = static_cast<const char*>(ws.stage_pin);
    int n = 0;
    SFG_CUDA(copy_async(ws.meta, ws.meta_pin, sizeof(int32_t) * (4 + kMetaKeep), cudaMemcpyHostToDevice, s));
    SFG_CUDA(copy_async(ws.ids, p + L.ids, sizeof(int32_t) * ws.cap_rows, cudaMemcpyHostToDevice, s));
    SFG_CUDA(copy_async(ws.pos, p + L.pos, sizeof(int32_t) * ws.cap_rows, cudaMemcpyHostToDevice, s));
    SFG_CUDA(copy_async(ws.row_off, p + L.roff, sizeof(int32_t) * (ws.cap_rows + 1), cudaMemcpyHostToDevice, s));
    SFG_CUDA(copy_async(ws.runs, p + L.runs, sizeof(MaskRun) * ws.cap_runs, cudaMemcpyHostToDevice, s));
    if (verify) SFG_CUDA(copy_async(d_vin_, h_vin_, sizeof(VerifyIn), cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemsetAsync(ws.status, 0, sizeof(uint32_t), s));
    const int mk = std::min(kMetaKeep, ws.cap_rows);
    for (Bank* b : {prefix_.get(), suffix_.get(), server_bank}) {
        if (!b || b->layer_end() == b->layer_begin()) continue;
        n += launch_kv_compact_meta(b->kslab(b->layer_begin()), b->vslab(b->layer_begin()),
                                    b->layer_end() - b->layer_begin(), c.n_kv_heads, c.max_seq_len, c.head_dim,
                                    ws.meta, mk, s);
    }
    n += eng_.embed_device(rows, ws, s);
    n += eng_.forward_device(*prefix_, 0, cfg_.prefix_layers, rows, ws, s);
    return n;
}

// wire round trip -> server layers (device-linked) -> wire round trip
int Client::dev_server(int rows, Bank* server_bank, cudaStream_t s) {
    const ModelCfg& c = eng_.cfg();
    Workspace& ws = prefix_->ws();
    const int n = rows * c.hidden_dim;
    const int f32 = cfg_.wire_dtype == SFG_WIRE_F32;
    int k = launch_wire_roundtrip(ws.h, f32, n, ws.clamped, s);  // encode/decode_values
    k += launch_link_delay(cfg_.one_way_delay_ms, s);             // request leg
    // under stream capture the records are made External: they become
    // event-record nodes of the step's graph, so the server segment is timed
    // on every replay too (the flag is only legal while capturing)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    SFG_CUDA(cudaStreamIsCapturing(s, &cap));
    const unsigned evf = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    SFG_CUDA(cudaEventRecordWithFlags(ev_[1], s, evf));
    k += linked_->engine().forward_device(*server_bank, linked_->config().layer_begin, linked_->config().layer_end,
                                          rows, ws, s);
    SFG_CUDA(cudaEventRecordWithFlags(ev_[2], s, evf));
    const int rd = linked_->config().response_dtype;
    k += launch_wire_roundtrip(ws.h, rd < 0 ? f32 : rd == SFG_WIRE_F32, n, nullptr, s);
    k += launch_link_delay(cfg_.one_way_delay_ms, s);             // response leg
    return k;
}

// suffix layers -> head -> argmax -> verify -> [summary D2H]
int Client::dev_post(int rows, bool want_logits, bool verify, cudaStream_t s) {
    const ModelCfg& c = eng_.cfg();
    Workspace& ws = prefix_->ws();
    int n = eng_.forward_device(*suffix_, c.n_layers - cfg_.suffix_layers, c.n_layers, rows, ws, s);
    n += eng_.head_device(rows, ws, want_logits, true, s);
    if (verify) {
        n += launch_verify(ws.argmax, d_vin_, d_vout_, s);
        SFG_CUDA(copy_async(h_vout_, d_vout_, sizeof(VerifyOut), cudaMemcpyDeviceToHost, s));
    }
    SFG_CUDA(copy_async(h_argmax_, ws.argmax, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost, s));
    if (want_logits)
        SFG_CUDA(copy_async(h_logits_, ws.logits, sizeof(float) * rows * c.vocab_size, cudaMemcpyDeviceToHost, s));
    return n;
}

// Frame path: device pack -> host frame -> handler -> host frame -> device unpack
void Client::exchange_frames(bool prompt, int seq, const int32_t* pos, const MaskRuns* runs, int mask_kv,
                             const int32_t* keep, int n_keep, bool send_keep, std::optional<int> crop) {
    const ModelCfg& c = eng_.cfg();
    Workspace& ws = prefix_->ws();
    cudaStream_t s = prefix_->stream();
    const int n = seq * c.hidden_dim;
    const int f32 = cfg_.wire_dtype == SFG_WIRE_F32;
    const size_t wbytes = static_cast<size_t>(n) * (f32 ? 4 : 2);
    prof_.launches += launch_pack_rows(ws.h, f32, n, ws.wire, ws.clamped, s);
    // the wire rows cross through pinned staging (async DMA, no driver bounce)
    uint8_t* pin = static_cast<uint8_t*>(ws.wire_pin);
    SFG_CUDA(copy_async(pin, ws.wire, wbytes, cudaMemcpyDeviceToHost, s));
    wire::Header h;  // make_request (client.cpp:59-81)
    h.kind = prompt ? wire::FrameKind::prompt : (send_keep ? wire::FrameKind::accept_and_step : wire::FrameKind::step);
    h.session_id = sid_;
    h.shape = {seq, c.hidden_dim};
    h.dtype = f32 ? wire::Dtype::f32 : wire::Dtype::f16;
    h.pos.assign(pos, pos + seq);
    if (send_keep) h.keep = std::vector<int64_t>(keep, keep + n_keep);
    if (crop) h.crop = *crop;
    std::vector<uint16_t> mask;
    if (runs) {  // encode_values(mask, f16) of the dense mask (client.cpp:76-78)
        h.mask_shape = std::vector<int64_t>{1, 1, seq, mask_kv};
        mask.assign(static_cast<size_t>(seq) * mask_kv, 0xfc00u);  // -inf
        for (int i = 0; i < seq; ++i)
            for (int r = runs->row_off[i]; r < runs->row_off[i + 1]; ++r) {
                // the visible columns' real additive value: a non-zero one reaches
                // the server (which rejects it, server.cpp:165-169) as the
                // reference client would send it
                const uint16_t v = wire::f32_to_f16_bits(runs->runs[r].mval, nullptr);
                std::fill(mask.begin() + static_cast<size_t>(i) * mask_kv + runs->runs[r].start,
                          mask.begin() + static_cast<size_t>(i) * mask_kv + runs->runs[r].end, v);
            }
    }
    SFG_CUDA(cudaEventRecord(ev_[1], s));
    SFG_CUDA(cudaStreamSynchronize(s));
    wire::encode(h, pin, wbytes, reinterpret_cast<const uint8_t*>(mask.data()), mask.size() * 2, req_);
    sleep_one_way();
    const uint8_t* resp = nullptr;
    size_t rlen = 0;
    const int32_t rc = handler_(ctx_, req_.data(), req_.size(), &resp, &rlen);
    if (rc != 0) {
        dead_ = true;
        throw Error(Kind::transport, "frame handler failed");
    }
    sleep_one_way();
    wire::FrameView r;  // views into the handler's buffer (valid until its next call)
    try {
        r = wire::decode(resp, rlen);
    } catch (...) {
        dead_ = true;
        throw;
    }
    if (r.h.kind == wire::FrameKind::error) {  // exchange_hidden (client.cpp:93-97)
        dead_ = true;
        const std::string msg = r.h.err.value_or("unspecified server error");
        throw Error(kind_from_message(msg), "server: " + msg);
    }
    if (r.h.kind != wire::FrameKind::response) {
        dead_ = true;
        throw Error(Kind::protocol, "unexpected response kind");
    }
    prof_.server_ms = r.h.srv_ms.value_or(0.0);
    if (r.h.shape.size() != 2 || r.h.shape[0] != seq || r.h.shape[1] != c.hidden_dim) {
        dead_ = true;
        throw Error(Kind::protocol, "response tensor shape mismatch");
    }
    if (r.tensor_len > static_cast<size_t>(ws.cap_rows) * c.hidden_dim * 4) {
        dead_ = true;
        throw Error(Kind::protocol, "response tensor exceeds the workspace");
    }
    std::memcpy(pin, r.tensor, r.tensor_len);
    SFG_CUDA(copy_async(ws.wire, pin, r.tensor_len, cudaMemcpyHostToDevice, s));
    prof_.launches += launch_unpack_rows(ws.wire, r.h.dtype == wire::Dtype::f32, n, ws.h, s);
    SFG_CUDA(cudaEventRecord(ev_[2], s));
    SFG_CUDA(cudaStreamSynchronize(s));  // the staging buffer is reused next step
}

// SplitClient::prefill (client.cpp:120-167)
int Client::prefill(const int32_t* prompt, int n, float* logits_row) {
    const ModelCfg& c = eng_.cfg();
    if (n <= 0) throw Error(Kind::input, "prompt must be non-empty");
    if (dead_) throw Error(Kind::transport, "session is dead");
    if (n > c.max_seq_len) throw Error(Kind::capacity, "prompt exceeds max_seq_len");
    prefix_->reset();
    suffix_->reset();
    prefilled_ = false;
    first_step_done_ = false;
    std::vector<int32_t> pos(n);
    for (int i = 0; i < n; ++i) pos[i] = i;
    for (int i = 0; i < n; ++i)
        if (prompt[i] < 0 || prompt[i] >= c.vocab_size) throw Error(Kind::input, "token id out of range");
    DeviceGuard g(eng_.device());
    Workspace& ws = prefix_->ws();
    cudaStream_t s = prefix_->stream();
    const MaskRuns mr = causal_runs(n, 0);
    prof_ = StepProfile{};
    prof_.batch = n;
    eng_.ensure_ws(ws, n, static_cast<int>(mr.runs.size()), 1);
    ensure_out(1);
    stage_inputs(n, prompt, pos.data(), mr);
    std::memset(ws.meta_pin, 0, sizeof(int32_t) * 4);  // prior 0, no relocation
    prof_.launches += dev_pre(n, nullptr, false, s);
    prefix_->set_len(n);
    prefix_->mark_committed(n);
    if (linked_) {
        Server::LinkedStep st{&sid_, true, n, pos.data(), nullptr, std::nullopt, nullptr, n, n};
        Server::Lease lease;
        try {
            lease = linked_->linked_begin(st);
        } catch (const Error& e) {
            dead_ = true;
            throw Error(e.kind(), std::string("server: ") + e.what());
        }
        prof_.launches += dev_server(n, lease.bank, s);  // link delays run on the device timeline
        linked_->linked_end(lease, n);
    } else {
        exchange_frames(true, n, pos.data(), nullptr, n, nullptr, 0, false, std::nullopt);
    }
    prof_.launches += eng_.forward_device(*suffix_, c.n_layers - cfg_.suffix_layers, c.n_layers, n, ws, s);
    suffix_->set_len(n);
    suffix_->mark_committed(n);
    // finalize + argmax of the last row only (rows are independent)
    if (n > 1)
        SFG_CUDA(copy_async(ws.h, ws.h + static_cast<size_t>(n - 1) * c.hidden_dim,
                                 sizeof(float) * c.hidden_dim, cudaMemcpyDeviceToDevice, s));
    prof_.launches += eng_.head_device(1, ws, logits_row != nullptr, true, s);
    SFG_CUDA(copy_async(h_argmax_, ws.argmax, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (logits_row)
        SFG_CUDA(copy_async(h_logits_, ws.logits, sizeof(float) * c.vocab_size, cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    SFG_CUDA(cudaGetLastError());
    if (logits_row) std::memcpy(logits_row, h_logits_, sizeof(float) * c.vocab_size);
    prompt_len_ = n;
    prefilled_ = true;
    return h_argmax_[0];
}

Client::Graph* Client::find_graph(int rows, bool logits, bool verify, bool additive, const Bank* server_bank) {
    const uint64_t gen = prefix_->ws().generation;
    const uint64_t bid = server_bank ? server_bank->id() : 0;
    for (auto& g : graphs_)
        if (g.rows == rows && g.logits == logits && g.verify == verify && g.additive == additive &&
            g.server_bank == bid && g.generation == gen)
            return &g;
    // drop stale entries (workspace reallocated or server session replaced)
    for (auto it = graphs_.begin(); it != graphs_.end();) {
        if (it->generation != gen || graphs_.size() > 16) {
            if (it->exec) cudaGraphExecDestroy(it->exec);
            KernelProfiler::get().release_graph(it->prof_slots);
            it = graphs_.erase(it);
        } else {
            ++it;
        }
    }
    Graph g;
    g.rows = rows;
    g.logits = logits;
    g.verify = verify;
    g.additive = additive;
    g.server_bank = bid;
    g.generation = gen;
    graphs_.push_back(g);
    return &graphs_.back();
}

// SplitClient::decode_step (client.cpp:169-228)
void Client::decode_step(int seq, const int32_t* tokens, const int32_t* positions, const MaskRuns* runs,
                         const int32_t* keep, int n_keep, std::optional<int> crop, float* logits_out,
                         int32_t* argmax_out, const VerifyIn* vin, VerifyOut* vout) {
    const ModelCfg& c = eng_.cfg();
    if (!prefilled_) throw Error(Kind::input, "decode_step before prefill");
    if (dead_) throw Error(Kind::transport, "session is dead");
    if (seq <= 0) throw Error(Kind::input, "empty decode batch");
    DeviceGuard g(eng_.device());
    Workspace& ws = prefix_->ws();
    cudaStream_t s = prefix_->stream();
    prof_ = StepProfile{};
    prof_.batch = seq;
    int kv = 0;
    MaskRuns causal;
    const MaskRuns* mr = runs;
    const int committed_before = prefix_->committed_len();
    bool relocate = false;
    // a keep list longer than the step meta block holds is compacted by
    // eager kernels ahead of the (graph-captured) step instead
    const bool big_keep = n_keep > kMetaKeep;
    try {
        if (n_keep > 0 || prefix_->provisional() > 0) {
            prefix_->resolve_meta(keep, n_keep);
            suffix_->resolve_meta(keep, n_keep);
            relocate = n_keep > 0 && !big_keep;
        }
        if (crop) {
            prefix_->crop(*crop);
            suffix_->crop(*crop);
        }
        if (prefix_->len() != suffix_->len()) throw Error(Kind::internal, "local cache banks desynced");
        kv = prefix_->len() + seq;
        if (runs && static_cast<int>(runs->row_off.size()) != seq + 1)
            throw Error(Kind::protocol, "mask shape does not match local cache state");
        for (int i = 0; i < seq; ++i)
            if (positions[i] < 0 || positions[i] >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
        for (int i = 0; i < seq; ++i)
            if (tokens[i] < 0 || tokens[i] >= c.vocab_size) throw Error(Kind::input, "token id out of range");
        if (kv > c.max_seq_len) throw Error(Kind::capacity, "sequence exceeds max_seq_len");
        if (!mr) {
            causal = causal_runs(seq, prefix_->len());
            mr = &causal;
        }
        if (mr->any_empty_row) throw Error(Kind::protocol, "mask row admits no attendable position");
    } catch (...) {
        dead_ = true;
        throw;
    }
    const bool want_logits = logits_out != nullptr;
    eng_.ensure_ws(ws, seq, static_cast<int>(mr->runs.size()), seq);
    ensure_out(seq);
    stage_inputs(seq, tokens, positions, *mr);
    ws.meta_pin[0] = prefix_->len();
    ws.meta_pin[1] = committed_before;
    ws.meta_pin[2] = relocate ? n_keep : 0;
    if (relocate) std::memcpy(ws.meta_pin + 3, keep, sizeof(int32_t) * n_keep);
    if (big_keep) {
        prefix_->enqueue_compact(keep, n_keep, committed_before, s);
        suffix_->enqueue_compact(keep, n_keep, committed_before, s);
    }
    if (vin) std::memcpy(h_vin_, vin, sizeof(VerifyIn));
    const bool send_keep = first_step_done_;

    if (linked_) {
        std::vector<int64_t> kv64;
        if (send_keep) kv64.assign(keep, keep + n_keep);
        Server::LinkedStep st{&sid_, false, seq, positions, send_keep ? &kv64 : nullptr,
                              crop ? std::optional<int64_t>(*crop) : std::nullopt, runs, seq, kv};
        Server::Lease lease;
        try {
            lease = linked_->linked_begin(st);
        } catch (const Error& e) {
            dead_ = true;
            throw Error(e.kind(), std::string("server: ") + e.what());
        }
        if (lease.committed_before != committed_before || lease.prior != prefix_->len() ||
            lease.n_keep != (relocate || big_keep ? n_keep : lease.n_keep)) {
            dead_ = true;
            throw Error(Kind::internal, "client and server caches out of lockstep");
        }
        if (big_keep) lease.bank->enqueue_compact(keep, n_keep, lease.committed_before, s);
        SFG_CUDA(cudaEventRecord(ev_[0], s));
        Graph* gr = nullptr;
        static const bool debug_eager = std::getenv("SFG_DEBUG") != nullptr;
        if (graphs_enabled() && !debug_eager) {
            gr = find_graph(seq, want_logits, vin != nullptr, ws.additive_mask, lease.bank);
            ++gr->seen;
        }
        if (gr && gr->exec) {
            SFG_CUDA(cudaGraphLaunch(gr->exec, s));
            prof_.launches = gr->launches;
            prof_.graph = true;
        } else if (gr && gr->seen >= 2) {  // first replay-eligible occurrence: capture
            KernelProfiler::get().begin_capture(&gr->prof_slots);
            SFG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            int k = 0;
            try {
                k += dev_pre(seq, lease.bank, vin != nullptr, s);
                k += dev_server(seq, lease.bank, s);
                k += dev_post(seq, want_logits, vin != nullptr, s);
            } catch (...) {
                cudaGraph_t dead = nullptr;
                cudaStreamEndCapture(s, &dead);
                if (dead) cudaGraphDestroy(dead);
                KernelProfiler::get().end_capture();
                throw;
            }
            cudaGraph_t graph = nullptr;
            SFG_CUDA(cudaStreamEndCapture(s, &graph));
            KernelProfiler::get().end_capture();
            SFG_CUDA(cudaGraphInstantiate(&gr->exec, graph, 0));
            cudaGraphDestroy(graph);
            gr->launches = k;
            SFG_CUDA(cudaGraphLaunch(gr->exec, s));
            prof_.launches = k;
            prof_.graph = true;
        } else {
            static const bool dbg = std::getenv("SFG_DEBUG") != nullptr;
            auto check = [&](const char* where) {
                if (!dbg) return;
                const cudaError_t e1 = cudaStreamSynchronize(s);
                const cudaError_t e2 = cudaGetLastError();
                if (e1 != cudaSuccess || e2 != cudaSuccess)
                    throw Error(Kind::internal, std::string("debug: CUDA error after ") + where + ": " +
                                                    cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
            };
            check("entry");
            prof_.launches += dev_pre(seq, lease.bank, vin != nullptr, s);
            check("dev_pre");
            prof_.launches += dev_server(seq, lease.bank, s);
            check("dev_server");
            prof_.launches += dev_post(seq, want_logits, vin != nullptr, s);
            check("dev_post");
        }
        SFG_CUDA(cudaEventRecord(ev_[3], s));
        linked_->linked_end(lease, seq);
        SFG_CUDA(cudaEventSynchronize(ev_[3]));
        if (gr && gr->exec && KernelProfiler::get().on()) KernelProfiler::get().collect_graph(gr->prof_slots);
    } else {
        SFG_CUDA(cudaEventRecord(ev_[0], s));
        prof_.launches += dev_pre(seq, nullptr, vin != nullptr, s);
        exchange_frames(false, seq, positions, runs, kv, keep, n_keep, send_keep, crop);
        prof_.launches += dev_post(seq, want_logits, vin != nullptr, s);
        SFG_CUDA(cudaEventRecord(ev_[3], s));
        SFG_CUDA(cudaEventSynchronize(ev_[3]));
    }
    SFG_CUDA(cudaGetLastError());
    prefix_->set_len(kv);
    suffix_->set_len(kv);
    first_step_done_ = true;
    if (vout) std::memcpy(vout, h_vout_, sizeof(VerifyOut));
    if (argmax_out) std::memcpy(argmax_out, h_argmax_, sizeof(int32_t) * seq);
    if (logits_out) std::memcpy(logits_out, h_logits_, sizeof(float) * seq * c.vocab_size);
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev_[0], ev_[3]);
    if (linked_) SFG_CUDA(cudaEventElapsedTime(&b, ev_[1], ev_[2]));
    prof_.step_ms = a;
    if (linked_) prof_.server_ms = b;
    prof_.local_ms = a - b;
}

// ── decode loops ──────────────────────────────────────────────────────────
Decoder::Decoder(Client& c, const Cfg& dc, Pool* pool, const int32_t* prompt, int n, int max_new, bool want_logits)
    : c_(c), cfg_(dc), pool_(pool), max_new_(max_new), want_logits_(want_logits) {
    if (dc.mode == 2) {
        if (dc.ngram_n < 2) throw Error(Kind::config, "ngram_n must be >= 2");
        if (dc.window_w < dc.ngram_n) throw Error(Kind::config, "window_w must be >= ngram_n");
        if (dc.max_candidates_g < 0) throw Error(Kind::config, "max_candidates_g must be >= 0");
        if (dc.window_w > kMaxWindow || dc.max_candidates_g > kMaxCand - 1 || dc.ngram_n - 1 > kMaxCont)
            throw Error(Kind::config, "lookahead shape exceeds the device verify tail limits");
        if (pool && pool->ngram_n() != dc.ngram_n) throw Error(Kind::config, "pool n-gram size does not match the config");
        if (!pool_) {
            own_ = std::make_unique<Pool>(dc.ngram_n, dc.pool_capacity);
            pool_ = own_.get();
        }
    } else if (dc.mode != 0) {
        throw Error(Kind::config, "decode mode must be sequential (0) or lookahead (2)");
    }
    if (max_new == 0) return;
    const int V = c.engine().cfg().vocab_size;
    std::vector<float> row(want_logits ? V : 0);
    tokens.push_back(c.prefill(prompt, n, want_logits ? row.data() : nullptr));
    if (want_logits) logits.insert(logits.end(), row.begin(), row.end());
    total_ = n + 1;
    window_.assign(std::max(dc.window_w, 1), tokens.back());
}

int Decoder::step() {
    const auto w0 = Clock::now();
    const ModelCfg& mc = c_.engine().cfg();
    const int V = mc.vocab_size;
    const int ctx = total_ - 1;
    const int W = cfg_.window_w, cl = cfg_.ngram_n - 1;
    MaskRuns mr;
    int B = 1, active_w = 0;
    std::vector<int> cand_begin;
    batch_.clear();
    pos_.clear();
    cands_.clear();
    if (cfg_.mode == 0) {  // decode_sequential (decoding.cpp:120-136)
        batch_.push_back(tokens.back());
        pos_.push_back(ctx);
        mr = causal_runs(1, ctx);
    } else {  // decode_lookahead_with_pool (decoding.cpp:236-293)
        pool_->lookup(tokens.back(), cfg_.max_candidates_g, cands_);
        active_w = W;
        auto bsize = [&] {
            int b = 1 + active_w;
            for (auto& cc : cands_) b += static_cast<int>(cc.size());
            return b;
        };
        while (!cands_.empty() && ctx + bsize() > mc.max_seq_len) cands_.pop_back();
        while (active_w > 1 && ctx + bsize() > mc.max_seq_len) --active_w;
        hits += cands_.empty() ? 0 : 1;
        B = bsize();
        batch_.push_back(tokens.back());
        pos_.push_back(ctx);
        for (int i = 0; i < active_w; ++i) {
            batch_.push_back(window_[i]);
            pos_.push_back(total_ + i);
        }
        int row = 1 + active_w;
        for (auto& cc : cands_) {
            cand_begin.push_back(row);
            for (size_t j = 0; j < cc.size(); ++j) {
                batch_.push_back(cc[j]);
                pos_.push_back(total_ + static_cast<int>(j));
            }
            row += static_cast<int>(cc.size());
        }
        // branch mask (decoding.cpp:277-293) as visibility runs
        mr.row_off.resize(B + 1);
        for (int i = 0; i <= active_w; ++i) {
            mr.row_off[i] = static_cast<int32_t>(mr.runs.size());
            mr.runs.push_back(MaskRun{0, ctx + i + 1, 0.0f, 0});
        }
        for (size_t b = 0; b < cands_.size(); ++b)
            for (size_t j = 0; j < cands_[b].size(); ++j) {
                const int r = cand_begin[b] + static_cast<int>(j);
                mr.row_off[r] = static_cast<int32_t>(mr.runs.size());
                mr.runs.push_back(MaskRun{0, ctx + 1, 0.0f, 0});
                mr.runs.push_back(MaskRun{ctx + cand_begin[b], ctx + cand_begin[b] + static_cast<int>(j) + 1, 0.0f, 0});
            }
        mr.row_off[B] = static_cast<int32_t>(mr.runs.size());
    }
    vin_.rows = B;
    vin_.mode = cfg_.mode;
    vin_.active_w = active_w;
    vin_.ncand = static_cast<int>(cands_.size());
    vin_.cont = cl;
    for (int i = 0; i < active_w; ++i) vin_.window[i] = window_[i];
    for (size_t b = 0; b < cands_.size(); ++b) {
        vin_.cand_begin[b] = cand_begin[b];
        for (int j = 0; j < cl; ++j) vin_.cands[b * cl + j] = cands_[b][j];
    }
    if (want_logits_) lbuf_.resize(static_cast<size_t>(B) * V);
    c_.decode_step(B, batch_.data(), pos_.data(), &mr, keep_.data(), static_cast<int>(keep_.size()), std::nullopt,
                   want_logits_ ? lbuf_.data() : nullptr, nullptr, &vin_, &vout_);
    const VerifyOut& vo = vout_;
    step_batch.push_back(B);
    int commit_n;
    if (cfg_.mode == 0) {
        tokens.push_back(vo.anchor);
        if (want_logits_) logits.insert(logits.end(), lbuf_.begin(), lbuf_.begin() + V);
        commit_n = 1;
        total_ += 1;
        keep_.assign(1, 0);
    } else {  // decoding.cpp:296-344
        const int best = vo.best;
        const int room = max_new_ - static_cast<int>(tokens.size());
        commit_n = std::min(best + 1, room);
        for (int i = 0; i < commit_n; ++i) tokens.push_back(vo.committed[i]);
        if (want_logits_) {
            logits.insert(logits.end(), lbuf_.begin(), lbuf_.begin() + V);
            for (int i = 1; i < commit_n; ++i) {
                const size_t r = static_cast<size_t>(vo.best_rows[i - 1]);
                logits.insert(logits.end(), lbuf_.begin() + r * V, lbuf_.begin() + (r + 1) * V);
            }
        }
        total_ += commit_n;
        keep_.assign(1, 0);
        for (int i = 0; i < best; ++i) keep_.push_back(vo.best_rows[i]);
        std::vector<int32_t> current(active_w);
        current[0] = vo.anchor;
        for (int i = 1; i < active_w; ++i) current[i] = vo.argmax[i];
        pool_->update(window_.data(), current.data(), active_w);
        std::vector<int32_t> preds(active_w + 1);
        preds[0] = vo.anchor;
        for (int i = 0; i < active_w; ++i) preds[i + 1] = vo.argmax[1 + i];
        const int adv = best + 1;
        for (int i = 0; i < W; ++i) window_[i] = preds[std::min(adv + i, active_w)];
    }
    step_accepted.push_back(commit_n);
    committed += commit_n;
    ++steps;
    wall_s += std::chrono::duration<double>(Clock::now() - w0).count();
    return commit_n;
}

}  // namespace sfg
