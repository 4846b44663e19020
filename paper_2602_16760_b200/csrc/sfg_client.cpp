// Trusted-side runtime: SplitClient::prefill/decode_step (client.cpp:120-228)
// and decode_sequential / decode_lookahead_with_pool (decoding.cpp:111-355)
// on the B200.  Per step the device runs embed -> prefix layers -> [wire] ->
// suffix layers -> final norm + LM head -> argmax -> verify/branch selection;
// only the committed-token summary returns to the host.
#include "sfg_client.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <thread>

namespace sfg {

using Clock = std::chrono::steady_clock;

// ── NGramPool ─────────────────────────────────────────────────────────────
Pool::Pool(int n, size_t cap) : n_(n), cap_(cap) {
    if (n < 2) throw Error(Kind::config, "ngram_n must be >= 2");
    if (cap < 1) throw Error(Kind::config, "pool capacity must be >= 1");
}

void Pool::insert(int32_t key, std::vector<int32_t> cont) {
    for (auto it = entries_.begin(); it != entries_.end(); ++it)
        if (it->key == key && it->cont == cont) {
            entries_.splice(entries_.begin(), entries_, it);
            return;
        }
    entries_.push_front(Entry{key, std::move(cont)});
    if (entries_.size() > cap_) entries_.pop_back();
}

void Pool::update(const int32_t* prev, const int32_t* cur, int w) {
    for (int i = 0; i + n_ - 1 <= w - 1; ++i) insert(prev[i], std::vector<int32_t>(cur + i + 1, cur + i + n_));
}

int Pool::lookup(int key, int max_c, std::vector<std::vector<int32_t>>& out) const {
    out.clear();
    // push, then stop at max_c: lookup(key, 0) yields one hit (decoding.cpp:91-95)
    for (const auto& e : entries_) {
        if (e.key != key) continue;
        out.push_back(e.cont);
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
    if (linked_ && linked_->engine().device() != local.device())
        throw Error(Kind::config, "a linked server must live on the client's device");
    if (sid_.empty()) {
        static const char* hex = "0123456789abcdef";
        std::mt19937_64 rng(std::random_device{}() ^ (uint64_t(std::random_device{}()) << 32));
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
}

Client::~Client() {
    DeviceGuard g(eng_.device());
    cudaStreamSynchronize(prefix_->stream());
    for (auto& e : ev_) cudaEventDestroy(e);
    cudaFree(d_vin_);
    cudaFree(d_vout_);
    cudaFreeHost(h_vin_);
    cudaFreeHost(h_vout_);
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

// One request/response exchange of the hidden rows currently in ws.h.
void Client::exchange(bool prompt, int seq, const int32_t* pos, const MaskRuns* runs, int mask_kv,
                      const int32_t* keep, int n_keep, bool send_keep, std::optional<int> crop) {
    const ModelCfg& c = eng_.cfg();
    Workspace& ws = prefix_->ws();
    cudaStream_t s = prefix_->stream();
    const int n = seq * c.hidden_dim;
    const int f32 = cfg_.wire_dtype == SFG_WIRE_F32;
    if (linked_) {
        // encode_values/decode_values round trip on device (same values the
        // frame would carry), then the server's middle layers in place.
        prof_.launches += launch_wire_roundtrip(ws.h, f32, n, ws.clamped, s);
        sleep_one_way();
        std::vector<int64_t> kv;
        if (send_keep) kv.assign(keep, keep + n_keep);
        Server::LinkedStep st{&sid_, prompt, seq, pos, send_keep ? &kv : nullptr,
                              crop ? std::optional<int64_t>(*crop) : std::nullopt,
                              runs, seq, mask_kv, ws.h, s};
        SFG_CUDA(cudaEventRecord(ev_[1], s));
        try {
            prof_.launches += linked_->linked_step(st);
        } catch (const Error& e) {
            dead_ = true;
            throw Error(e.kind(), std::string("server: ") + e.what());
        }
        SFG_CUDA(cudaEventRecord(ev_[2], s));
        const int rf = linked_->config().response_dtype < 0 ? f32 : linked_->config().response_dtype == SFG_WIRE_F32;
        prof_.launches += launch_wire_roundtrip(ws.h, rf, n, nullptr, s);
        sleep_one_way();
        return;
    }
    // frame path: device pack -> host frame -> handler -> host frame -> device unpack
    const size_t wbytes = static_cast<size_t>(n) * (f32 ? 4 : 2);
    prof_.launches += launch_pack_rows(ws.h, f32, n, ws.wire, ws.clamped, s);
    std::vector<uint8_t>& payload = maskbuf_;
    payload.resize(wbytes);
    SFG_CUDA(cudaMemcpyAsync(payload.data(), ws.wire, wbytes, cudaMemcpyDeviceToHost, s));
    wire::Header h;
    h.kind = prompt ? wire::FrameKind::prompt : (send_keep ? wire::FrameKind::accept_and_step : wire::FrameKind::step);
    h.session_id = sid_;
    h.shape = {seq, c.hidden_dim};
    h.dtype = f32 ? wire::Dtype::f32 : wire::Dtype::f16;
    h.pos.assign(pos, pos + seq);
    if (send_keep) h.keep = std::vector<int64_t>(keep, keep + n_keep);
    if (crop) h.crop = *crop;
    std::vector<uint16_t> mask;
    if (runs) {  // encode_values(mask, f16) of the dense {0,-inf} mask
        h.mask_shape = std::vector<int64_t>{1, 1, seq, mask_kv};
        mask.assign(static_cast<size_t>(seq) * mask_kv, 0xfc00u);
        for (int i = 0; i < seq; ++i)
            for (int r = runs->row_off[i]; r < runs->row_off[i + 1]; ++r)
                std::fill(mask.begin() + static_cast<size_t>(i) * mask_kv + runs->runs[r].start,
                          mask.begin() + static_cast<size_t>(i) * mask_kv + runs->runs[r].end, uint16_t(0));
    }
    SFG_CUDA(cudaStreamSynchronize(s));
    wire::encode(h, payload.data(), wbytes, reinterpret_cast<const uint8_t*>(mask.data()), mask.size() * 2, req_);
    sleep_one_way();
    const uint8_t* resp = nullptr;
    size_t rlen = 0;
    const int32_t rc = handler_(ctx_, req_.data(), req_.size(), &resp, &rlen);
    if (rc != 0) {
        dead_ = true;
        throw Error(Kind::transport, "frame handler failed");
    }
    std::vector<uint8_t> rcopy(resp, resp + rlen);
    sleep_one_way();
    wire::FrameView r;
    try {
        r = wire::decode(rcopy.data(), rcopy.size());
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
    SFG_CUDA(cudaMemcpyAsync(ws.wire, r.tensor, r.tensor_len, cudaMemcpyHostToDevice, s));
    prof_.launches += launch_unpack_rows(ws.wire, r.h.dtype == wire::Dtype::f32, n, ws.h, s);
    SFG_CUDA(cudaStreamSynchronize(s));  // rcopy must outlive the copy
}

// final norm + LM head + argmax (+ verify tail) on the rows in ws.h.
void Client::run_head(int rows, bool want_logits, VerifyIn* vin) {
    Workspace& ws = prefix_->ws();
    cudaStream_t s = prefix_->stream();
    prof_.launches += eng_.head_device(rows, ws, want_logits, true, s);
    if (vin) {
        std::memcpy(h_vin_, vin, sizeof(VerifyIn));
        SFG_CUDA(cudaMemcpyAsync(d_vin_, h_vin_, sizeof(VerifyIn), cudaMemcpyHostToDevice, s));
        prof_.launches += launch_verify(ws.argmax, d_vin_, d_vout_, s);
        SFG_CUDA(cudaMemcpyAsync(h_vout_, d_vout_, sizeof(VerifyOut), cudaMemcpyDeviceToHost, s));
    }
}

static void upload_local_meta(Engine& e, Workspace& ws, int seq, const int32_t* ids, const int32_t* pos,
                              const MaskRuns& mr, cudaStream_t s) {
    e.ensure_ws(ws, seq, static_cast<int>(mr.runs.size()), seq);
    char* pin = static_cast<char*>(ws.pinned);
    const size_t ib = sizeof(int32_t) * seq, rb = sizeof(int32_t) * mr.row_off.size(),
                 ub = sizeof(MaskRun) * mr.runs.size();
    if (2 * ib + rb + ub + 4096 > ws.pinned_bytes) {
        SFG_CUDA(cudaMemcpyAsync(ws.ids, ids, ib, cudaMemcpyHostToDevice, s));
        SFG_CUDA(cudaMemcpyAsync(ws.pos, pos, ib, cudaMemcpyHostToDevice, s));
        SFG_CUDA(cudaMemcpyAsync(ws.row_off, mr.row_off.data(), rb, cudaMemcpyHostToDevice, s));
        SFG_CUDA(cudaMemcpyAsync(ws.runs, mr.runs.data(), ub, cudaMemcpyHostToDevice, s));
        SFG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    SFG_CUDA(cudaStreamSynchronize(s));  // staging reuse
    std::memcpy(pin, ids, ib);
    std::memcpy(pin + ib, pos, ib);
    std::memcpy(pin + 2 * ib, mr.row_off.data(), rb);
    std::memcpy(pin + 2 * ib + rb, mr.runs.data(), ub);
    SFG_CUDA(cudaMemcpyAsync(ws.ids, pin, ib, cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(ws.pos, pin + ib, ib, cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(ws.row_off, pin + 2 * ib, rb, cudaMemcpyHostToDevice, s));
    SFG_CUDA(cudaMemcpyAsync(ws.runs, pin + 2 * ib + rb, ub, cudaMemcpyHostToDevice, s));
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
    upload_local_meta(eng_, ws, n, prompt, pos.data(), mr, s);
    prof_.launches += eng_.embed_device(n, ws, s);
    prof_.launches += eng_.forward_device(*prefix_, 0, cfg_.prefix_layers, n, ws, s);
    prefix_->set_len(n);
    prefix_->mark_committed(n);
    exchange(true, n, pos.data(), nullptr, n, nullptr, 0, false, std::nullopt);
    // the linked server may have re-uploaded its own metadata on this stream;
    // the client's ws.pos/runs are untouched (separate workspaces).
    prof_.launches += eng_.forward_device(*suffix_, c.n_layers - cfg_.suffix_layers, c.n_layers, n, ws, s);
    suffix_->set_len(n);
    suffix_->mark_committed(n);
    // finalize + argmax of the last row only (rows are independent).
    if (n > 1)
        SFG_CUDA(cudaMemcpyAsync(ws.h, ws.h + static_cast<size_t>(n - 1) * c.hidden_dim,
                                 sizeof(float) * c.hidden_dim, cudaMemcpyDeviceToDevice, s));
    run_head(1, logits_row != nullptr, nullptr);
    int32_t first = 0;
    SFG_CUDA(cudaMemcpyAsync(&first, ws.argmax, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (logits_row)
        SFG_CUDA(cudaMemcpyAsync(logits_row, ws.logits, sizeof(float) * c.vocab_size, cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    SFG_CUDA(cudaGetLastError());
    prompt_len_ = n;
    prefilled_ = true;
    return first;
}

// SplitClient::decode_step (client.cpp:169-228); outputs stay on device.
void Client::decode_step(int seq, const int32_t* tokens, const int32_t* positions, const MaskRuns* runs,
                         const int32_t* keep, int n_keep, std::optional<int> crop, bool want_logits) {
    const ModelCfg& c = eng_.cfg();
    if (!prefilled_) throw Error(Kind::input, "decode_step before prefill");
    if (dead_) throw Error(Kind::transport, "session is dead");
    if (seq <= 0) throw Error(Kind::input, "empty decode batch");
    const auto t0 = Clock::now();
    DeviceGuard g(eng_.device());
    Workspace& ws = prefix_->ws();
    cudaStream_t s = prefix_->stream();
    prof_ = StepProfile{};
    prof_.batch = seq;
    int kv = 0;
    try {
        if (n_keep > 0 || prefix_->provisional() > 0) {
            prefix_->resolve(keep, n_keep);
            suffix_->resolve(keep, n_keep);
        }
        if (crop) {
            prefix_->crop(*crop);
            suffix_->crop(*crop);
        }
        if (prefix_->len() != suffix_->len()) throw Error(Kind::internal, "local cache banks desynced");
        kv = prefix_->len() + seq;
        if (runs && (static_cast<int>(runs->row_off.size()) != seq + 1))
            throw Error(Kind::protocol, "mask shape does not match local cache state");
        for (int i = 0; i < seq; ++i)
            if (positions[i] < 0 || positions[i] >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
        for (int i = 0; i < seq; ++i)
            if (tokens[i] < 0 || tokens[i] >= c.vocab_size) throw Error(Kind::input, "token id out of range");
        if (prefix_->len() + seq > c.max_seq_len) throw Error(Kind::capacity, "sequence exceeds max_seq_len");
        MaskRuns causal;
        const MaskRuns* mr = runs;
        if (!mr) {
            causal = causal_runs(seq, prefix_->len());
            mr = &causal;
        }
        if (mr->any_empty_row) throw Error(Kind::protocol, "mask row admits no attendable position");
        upload_local_meta(eng_, ws, seq, tokens, positions, *mr, s);
        SFG_CUDA(cudaEventRecord(ev_[0], s));
        prof_.launches += eng_.embed_device(seq, ws, s);
        prof_.launches += eng_.forward_device(*prefix_, 0, cfg_.prefix_layers, seq, ws, s);
        prefix_->set_len(kv);
    } catch (...) {
        dead_ = true;
        throw;
    }
    const bool send_keep = first_step_done_;
    // client sends the mask it built (decode loops always do); a null runs
    // pointer means "no mask" on the wire and causal on both sides.
    SFG_CUDA(cudaEventRecord(ev_[1], s));
    exchange(false, seq, positions, runs, kv, keep, n_keep, send_keep, crop);
    if (!linked_) SFG_CUDA(cudaEventRecord(ev_[2], s));
    MaskRuns causal2;
    const MaskRuns* mr = runs;
    if (!mr) {
        causal2 = causal_runs(seq, suffix_->len());
        mr = &causal2;
    }
    // suffix uses the same visibility; client metadata is still in ws.
    prof_.launches += eng_.forward_device(*suffix_, c.n_layers - cfg_.suffix_layers, c.n_layers, seq, ws, s);
    suffix_->set_len(kv);
    run_head(seq, want_logits, nullptr);
    SFG_CUDA(cudaEventRecord(ev_[3], s));
    first_step_done_ = true;
    SFG_CUDA(cudaEventSynchronize(ev_[3]));
    SFG_CUDA(cudaGetLastError());
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, ev_[0], ev_[3]);
    cudaEventElapsedTime(&b, ev_[1], ev_[2]);
    cudaEventElapsedTime(&d, ev_[0], ev_[1]);
    prof_.step_ms = a;
    if (linked_) prof_.server_ms = b;
    prof_.local_ms = linked_ ? a - b : d;
    (void)t0;
}

void Client::fetch_logits(int rows, float* out) {
    DeviceGuard g(eng_.device());
    SFG_CUDA(cudaMemcpyAsync(out, prefix_->ws().logits, sizeof(float) * rows * eng_.cfg().vocab_size,
                             cudaMemcpyDeviceToHost, prefix_->stream()));
    SFG_CUDA(cudaStreamSynchronize(prefix_->stream()));
}

void Client::fetch_argmax(int rows, int32_t* out) {
    DeviceGuard g(eng_.device());
    SFG_CUDA(cudaMemcpyAsync(out, prefix_->ws().argmax, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost,
                             prefix_->stream()));
    SFG_CUDA(cudaStreamSynchronize(prefix_->stream()));
}

// decode_sequential / decode_lookahead_with_pool (decoding.cpp:111-139, 209-355)
void Client::decode(const DecodeCfg& dc, Pool* pool_in, const int32_t* prompt, int n, int max_new,
                    bool want_logits, DecodeOut& out) {
    const ModelCfg& c = eng_.cfg();
    const int V = c.vocab_size;
    if (dc.mode == 2) {
        if (dc.ngram_n < 2) throw Error(Kind::config, "ngram_n must be >= 2");
        if (dc.window_w < dc.ngram_n) throw Error(Kind::config, "window_w must be >= ngram_n");
        if (dc.max_candidates_g < 0) throw Error(Kind::config, "max_candidates_g must be >= 0");
        if (dc.window_w > kMaxWindow || dc.max_candidates_g > kMaxCand || dc.ngram_n - 1 > kMaxCont)
            throw Error(Kind::config, "lookahead shape exceeds the device verify tail limits");
        if (pool_in && pool_in->ngram_n() != dc.ngram_n)
            throw Error(Kind::config, "pool n-gram size does not match the config");
    } else if (dc.mode != 0) {
        throw Error(Kind::config, "decode mode must be sequential (0) or lookahead (2)");
    }
    out = DecodeOut{};
    if (max_new == 0) return;
    std::unique_ptr<Pool> own;
    Pool* pool = pool_in;
    if (!pool && dc.mode == 2) {
        own = std::make_unique<Pool>(dc.ngram_n, dc.pool_capacity);
        pool = own.get();
    }
    std::vector<float> row(want_logits ? V : 0);
    out.tokens.push_back(prefill(prompt, n, want_logits ? row.data() : nullptr));
    if (want_logits) out.logits.insert(out.logits.end(), row.begin(), row.end());

    int total = n + 1;
    const int W = dc.window_w, cl = dc.ngram_n - 1;
    std::vector<int32_t> window(std::max(W, 1), out.tokens.back());
    std::vector<int32_t> keep;
    int hits = 0;
    std::vector<std::vector<int32_t>> cands;
    std::vector<int32_t> batch, pos;
    std::vector<float> logits_buf;
    VerifyIn vin{};
    while (static_cast<int>(out.tokens.size()) < max_new) {
        const auto w0 = Clock::now();
        const int ctx = total - 1;
        MaskRuns mr;
        int B = 1, active_w = 0;
        std::vector<int> cand_begin;
        batch.clear();
        pos.clear();
        if (dc.mode == 0) {
            batch.push_back(out.tokens.back());
            pos.push_back(ctx);
            mr = causal_runs(1, ctx);
        } else {
            pool->lookup(out.tokens.back(), dc.max_candidates_g, cands);
            active_w = W;
            auto bsize = [&] {
                int b = 1 + active_w;
                for (auto& cc : cands) b += static_cast<int>(cc.size());
                return b;
            };
            while (!cands.empty() && ctx + bsize() > c.max_seq_len) cands.pop_back();
            while (active_w > 1 && ctx + bsize() > c.max_seq_len) --active_w;
            hits += cands.empty() ? 0 : 1;
            B = bsize();
            batch.push_back(out.tokens.back());
            pos.push_back(ctx);
            for (int i = 0; i < active_w; ++i) {
                batch.push_back(window[i]);
                pos.push_back(total + i);
            }
            int rrow = 1 + active_w;
            for (auto& cc : cands) {
                cand_begin.push_back(rrow);
                for (size_t j = 0; j < cc.size(); ++j) {
                    batch.push_back(cc[j]);
                    pos.push_back(total + static_cast<int>(j));
                }
                rrow += static_cast<int>(cc.size());
            }
            // branch mask (decoding.cpp:277-293) as runs
            mr.row_off.resize(B + 1);
            mr.runs.clear();
            for (int i = 0; i <= active_w; ++i) {
                mr.row_off[i] = static_cast<int32_t>(mr.runs.size());
                mr.runs.push_back(MaskRun{0, ctx + i + 1, 0.0f, 0});
            }
            for (size_t b = 0; b < cands.size(); ++b)
                for (size_t j = 0; j < cands[b].size(); ++j) {
                    const int r = cand_begin[b] + static_cast<int>(j);
                    mr.row_off[r] = static_cast<int32_t>(mr.runs.size());
                    mr.runs.push_back(MaskRun{0, ctx + 1, 0.0f, 0});
                    mr.runs.push_back(MaskRun{ctx + cand_begin[b], ctx + cand_begin[b] + static_cast<int>(j) + 1, 0.0f, 0});
                }
            mr.row_off[B] = static_cast<int32_t>(mr.runs.size());
        }
        decode_step(B, batch.data(), pos.data(), &mr, keep.data(), static_cast<int>(keep.size()), std::nullopt,
                    want_logits);
        // device verify tail
        vin.rows = B;
        vin.mode = dc.mode;
        vin.active_w = active_w;
        vin.ncand = static_cast<int>(cands.size());
        vin.cont = cl;
        for (int i = 0; i < active_w; ++i) vin.window[i] = window[i];
        for (size_t b = 0; b < cands.size(); ++b) {
            vin.cand_begin[b] = cand_begin[b];
            for (int j = 0; j < cl; ++j) vin.cands[b * cl + j] = cands[b][j];
        }
        {
            DeviceGuard g(eng_.device());
            std::memcpy(h_vin_, &vin, sizeof(VerifyIn));
            cudaStream_t s = prefix_->stream();
            SFG_CUDA(cudaMemcpyAsync(d_vin_, h_vin_, sizeof(VerifyIn), cudaMemcpyHostToDevice, s));
            prof_.launches += launch_verify(prefix_->ws().argmax, d_vin_, d_vout_, s);
            SFG_CUDA(cudaMemcpyAsync(h_vout_, d_vout_, sizeof(VerifyOut), cudaMemcpyDeviceToHost, s));
            if (want_logits) {
                logits_buf.resize(static_cast<size_t>(B) * V);
                SFG_CUDA(cudaMemcpyAsync(logits_buf.data(), prefix_->ws().logits, sizeof(float) * B * V,
                                         cudaMemcpyDeviceToHost, s));
            }
            SFG_CUDA(cudaStreamSynchronize(s));
        }
        const VerifyOut& vo = *h_vout_;
        out.step_batch.push_back(B);
        int commit_n;
        if (dc.mode == 0) {
            out.tokens.push_back(vo.anchor);
            if (want_logits) out.logits.insert(out.logits.end(), logits_buf.begin(), logits_buf.begin() + V);
            commit_n = 1;
            total += 1;
            keep.assign(1, 0);
        } else {
            const int best = vo.best;
            const int room = max_new - static_cast<int>(out.tokens.size());
            commit_n = std::min(best + 1, room);
            for (int i = 0; i < commit_n; ++i) out.tokens.push_back(vo.committed[i]);
            if (want_logits) {
                out.logits.insert(out.logits.end(), logits_buf.begin(), logits_buf.begin() + V);
                for (int i = 1; i < commit_n; ++i) {
                    const size_t r = static_cast<size_t>(vo.best_rows[i - 1]);
                    out.logits.insert(out.logits.end(), logits_buf.begin() + r * V, logits_buf.begin() + (r + 1) * V);
                }
            }
            total += commit_n;
            keep.assign(1, 0);
            for (int i = 0; i < best; ++i) keep.push_back(vo.best_rows[i]);
            std::vector<int32_t> current(active_w);
            current[0] = vo.anchor;
            for (int i = 1; i < active_w; ++i) current[i] = vo.argmax[i];
            pool->update(window.data(), current.data(), active_w);
            std::vector<int32_t> preds(active_w + 1);
            preds[0] = vo.anchor;
            for (int i = 0; i < active_w; ++i) preds[i + 1] = vo.argmax[1 + i];
            const int adv = best + 1;
            for (int i = 0; i < W; ++i) window[i] = preds[std::min(adv + i, active_w)];
        }
        out.step_accepted.push_back(commit_n);
        out.committed += commit_n;
        ++out.steps;
        out.wall_s += std::chrono::duration<double>(Clock::now() - w0).count();
    }
    out.match_rate = out.steps > 0 ? static_cast<double>(hits) / out.steps : 0.0;
}

}  // namespace sfg
