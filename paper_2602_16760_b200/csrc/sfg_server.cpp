// GPU ServerEngine — state machine of server.cpp:173-265 / PROTOCOL.md with
// the forward on device.  Host work is limited to framing, protocol
// validation and bookkeeping; hidden rows are unpacked, transformed and
// packed on the B200.
#include "sfg_server.h"

#include <chrono>
#include <cmath>
#include <cstring>

namespace sfg {

static double steady_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Server::Server(Engine& eng, const ServerCfg& cfg) : eng_(eng), cfg_(cfg), now_s_(steady_seconds) {
    const ModelCfg& m = eng.cfg();
    // ServerEngine ctor checks (server.cpp:26-39)
    if (cfg_.layer_begin <= 0 || cfg_.layer_end >= m.n_layers || cfg_.layer_begin >= cfg_.layer_end)
        throw Error(Kind::config, "hosted layer range must be non-empty and strictly inside the model");
    if (cfg_.session_expiry_s <= 0) throw Error(Kind::config, "session expiry must be positive");
    if (cfg_.max_sessions < 1) throw Error(Kind::config, "max_sessions must be >= 1");
    for (int l = cfg_.layer_begin; l < cfg_.layer_end; ++l)
        if (!eng.layer(l).hosted) throw Error(Kind::config, "engine does not host the server's layer range");
}

size_t Server::expire_sessions() {
    const double now = now_s_();
    std::lock_guard<std::mutex> lk(table_mutex_);
    size_t removed = 0;
    for (auto it = sessions_.begin(); it != sessions_.end();) {
        if (now - it->second->last_active > cfg_.session_expiry_s) {
            it = sessions_.erase(it);
            ++removed;
        } else {
            ++it;
        }
    }
    return removed;
}

size_t Server::session_count() const {
    std::lock_guard<std::mutex> lk(table_mutex_);
    return sessions_.size();
}

bool Server::session_view(const std::string& id, int* len, int* committed, int* prov) const {
    std::lock_guard<std::mutex> lk(table_mutex_);
    auto it = sessions_.find(id);
    if (it == sessions_.end()) return false;
    *len = it->second->bank->len();
    *committed = it->second->bank->committed_len();
    *prov = it->second->bank->provisional();
    return true;
}

// find_session with lazy expiry (server.cpp:75-85)
std::shared_ptr<Server::Session> Server::find_session(const std::string& id) {
    const double now = now_s_();
    std::lock_guard<std::mutex> lk(table_mutex_);
    auto it = sessions_.find(id);
    if (it == sessions_.end()) return nullptr;
    if (now - it->second->last_active > cfg_.session_expiry_s) {
        sessions_.erase(it);
        return nullptr;
    }
    return it->second;
}

// create_or_reset_session (server.cpp:87-99)
std::shared_ptr<Server::Session> Server::create_or_reset_session(const std::string& id) {
    std::lock_guard<std::mutex> lk(table_mutex_);
    auto it = sessions_.find(id);
    if (it != sessions_.end()) return it->second;
    if (static_cast<int>(sessions_.size()) >= cfg_.max_sessions) throw Error(Kind::capacity, "session table full");
    auto s = std::make_shared<Session>();
    s->bank = std::make_unique<Bank>(eng_, cfg_.layer_begin, cfg_.layer_end);
    sessions_[id] = s;
    return s;
}

MaskRuns runs_from_f16_mask(const uint16_t* m, int q, int kv) {
    // mask_from_frame entry validation (server.cpp:165-169): only 0 (either
    // sign) and -inf are legal.  Scanned four f16 entries (one 64-bit word) at
    // a time: an all-visible or all-masked word extends / closes the current
    // run without per-entry work (a 16 x 2064 long-context mask is ~99 % such
    // words); mixed words fall back to entry-wise checks.
    constexpr uint64_t kNegInf4 = 0xfc00fc00fc00fc00ull;
    MaskRuns r;
    r.row_off.resize(q + 1);
    bool bad = false;
    for (int i = 0; i < q; ++i) {
        r.row_off[i] = static_cast<int32_t>(r.runs.size());
        const uint16_t* row = m + static_cast<size_t>(i) * kv;
        int j = 0, start = -1;
        auto close = [&](int end) {
            if (start >= 0) r.runs.push_back(MaskRun{start, end, 0.0f, 0});
            start = -1;
        };
        auto entry = [&](int c) {
            const uint16_t b = row[c];
            if (b == 0xfc00u) {
                close(c);
            } else {
                bad |= (b != 0x0000u) & (b != 0x8000u);
                if (start < 0) start = c;
            }
        };
        for (; j + 4 <= kv; j += 4) {
            uint64_t w;
            std::memcpy(&w, row + j, sizeof(w));
            if (w == 0) {
                if (start < 0) start = j;
            } else if (w == kNegInf4) {
                close(j);
            } else {
                for (int c = j; c < j + 4; ++c) entry(c);
            }
        }
        for (; j < kv; ++j) entry(j);
        close(kv);
        if (static_cast<int32_t>(r.runs.size()) == r.row_off[i]) r.any_empty_row = true;
    }
    if (bad) throw Error(Kind::protocol, "mask entries must be 0 or -inf");
    r.row_off[q] = static_cast<int32_t>(r.runs.size());
    return r;
}

void Server::error_frame(const std::string& sid, const std::string& msg, std::vector<uint8_t>& resp) {
    wire::Header h;
    h.kind = wire::FrameKind::error;
    h.session_id = sid;
    h.shape = {0};
    h.err = msg;
    wire::encode(h, nullptr, 0, nullptr, 0, resp);
}

void Server::handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp) {
    wire::FrameView f;
    try {
        f = wire::decode(req, n);
    } catch (const Error& e) {
        error_frame("", e.what(), resp);
        return;
    }
    const std::string sid = f.h.session_id;
    try {
        handle_frame(f, resp);
    } catch (const Error& e) {
        error_frame(sid, e.what(), resp);
    } catch (const std::exception& e) {
        error_frame(sid, std::string("internal: ") + e.what(), resp);
    }
}

namespace {

struct HiddenCheck {
    int seq = 0;
    std::vector<int32_t> pos;
};

// frame_to_hidden (server.cpp:101-133), validation only: the rows are
// decoded on device.  Non-finite detection reads the raw binary16/32
// exponent fields, which is exactly isfinite() of the decoded value.
HiddenCheck frame_to_hidden(const wire::FrameView& f, const ModelCfg& c) {
    const auto& h = f.h;
    if (h.shape.size() != 2) throw Error(Kind::protocol, "hidden tensor must be rank 2 [seq, hidden]");
    const int seq = static_cast<int>(h.shape[0]);
    const int dim = static_cast<int>(h.shape[1]);
    if (dim != c.hidden_dim) throw Error(Kind::protocol, "hidden dim mismatch");
    if (seq < 1) throw Error(Kind::protocol, "empty batch");
    if (static_cast<int>(h.pos.size()) != seq) throw Error(Kind::protocol, "positions must match the batch seq dim");
    HiddenCheck hc;
    hc.seq = seq;
    hc.pos.reserve(seq);
    for (int64_t p : h.pos) {
        if (p < 0 || p >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
        hc.pos.push_back(static_cast<int32_t>(p));
    }
    const size_t n = static_cast<size_t>(seq) * dim;
    bool finite = true;
    if (h.dtype == wire::Dtype::f16) {
        const uint16_t* v = reinterpret_cast<const uint16_t*>(f.tensor);
        for (size_t i = 0; i < n; ++i) finite &= (v[i] & 0x7c00u) != 0x7c00u;
    } else {
        const uint32_t* v = reinterpret_cast<const uint32_t*>(f.tensor);
        for (size_t i = 0; i < n; ++i) finite &= (v[i] & 0x7f800000u) != 0x7f800000u;
    }
    if (!finite) throw Error(Kind::numeric, "non-finite hidden payload");
    return hc;
}

// mask_from_frame (server.cpp:148-171)
MaskRuns mask_from_frame(const wire::FrameView& f, int cache_len, int seq) {
    const auto& h = f.h;
    if (!h.mask_shape) return causal_runs(seq, cache_len);
    const auto& ms = *h.mask_shape;
    if (ms.size() != 4 || ms[0] != 1 || ms[1] != 1) throw Error(Kind::protocol, "mask_shape must be [1, 1, q, kv]");
    const int q = static_cast<int>(ms[2]), kv = static_cast<int>(ms[3]);
    if (q != seq || kv != cache_len + seq)
        throw Error(Kind::protocol, "mask shape does not match cache length plus batch");
    return runs_from_f16_mask(reinterpret_cast<const uint16_t*>(f.mask), q, kv);
}

// forward_layers pre-compute checks that can fire after the mask
// (tinyformer.cpp:390-392, 467-469).
void forward_checks(const Bank& b, int seq, const MaskRuns& mr, int max_seq) {
    if (b.len() + seq > max_seq) throw Error(Kind::capacity, "sequence exceeds max_seq_len");
    if (mr.any_empty_row) throw Error(Kind::protocol, "mask row admits no attendable position");
}

// H2D of the launch metadata (positions + visibility runs) for one step.
void upload_meta(Engine& e, Workspace& ws, const std::vector<int32_t>& pos, const MaskRuns& mr,
                 cudaStream_t s) {
    e.ensure_ws(ws, static_cast<int>(pos.size()), static_cast<int>(mr.runs.size()), 0);
    char* pin = static_cast<char*>(ws.pinned);
    // pinned layout: [pos | row_off | runs]; the copies complete before the
    // host touches the staging buffer again (each step ends with a sync).
    const size_t pb = sizeof(int32_t) * pos.size(), rb = sizeof(int32_t) * mr.row_off.size(),
                 ub = sizeof(MaskRun) * mr.runs.size();
    if (pb + rb + ub > ws.pinned_bytes) {
        SFG_CUDA(copy_async(ws.pos, pos.data(), pb, cudaMemcpyHostToDevice, s));
        SFG_CUDA(copy_async(ws.row_off, mr.row_off.data(), rb, cudaMemcpyHostToDevice, s));
        SFG_CUDA(copy_async(ws.runs, mr.runs.data(), ub, cudaMemcpyHostToDevice, s));
        SFG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    std::memcpy(pin, pos.data(), pb);
    std::memcpy(pin + pb, mr.row_off.data(), rb);
    std::memcpy(pin + pb + rb, mr.runs.data(), ub);
    SFG_CUDA(copy_async(ws.pos, pin, pb, cudaMemcpyHostToDevice, s));
    SFG_CUDA(copy_async(ws.row_off, pin + pb, rb, cudaMemcpyHostToDevice, s));
    SFG_CUDA(copy_async(ws.runs, pin + pb + rb, ub, cudaMemcpyHostToDevice, s));
}

}  // namespace

// handle_prompt / handle_step (server.cpp:203-265), host part: session state
// machine, validation, keep/crop, mask -> runs.  Leaves the session locked.
// With try_lock, a session whose mutex is held elsewhere is not waited for:
// returns false before touching any state (handle_batch already holds other
// sessions' locks, and waiting there could deadlock against another batch).
bool Server::prepare(const wire::FrameView& f, StepState& st, bool try_lock) {
    const ModelCfg& c = eng_.cfg();
    const auto kind = f.h.kind;
    if (kind == wire::FrameKind::response || kind == wire::FrameKind::error)
        throw Error(Kind::protocol, "response/error frames are not requests");
    st.f = f;
    st.prompt = kind == wire::FrameKind::prompt;
    if (st.prompt) {  // handle_prompt (server.cpp:203-224)
        if (f.h.session_id.empty()) throw Error(Kind::protocol, "prompt frame requires a session_id");
        { auto hc = frame_to_hidden(f, c); st.hc.seq = hc.seq; st.hc.pos = std::move(hc.pos); }
        if (st.hc.seq > c.max_seq_len) throw Error(Kind::capacity, "prompt exceeds max_seq_len");
        st.sess = create_or_reset_session(f.h.session_id);
    } else {  // handle_step (server.cpp:226-265)
        st.sess = find_session(f.h.session_id);
        if (!st.sess) throw Error(Kind::session, "unknown or expired session: " + f.h.session_id);
    }
    if (try_lock) {
        st.lock = std::unique_lock<std::mutex>(st.sess->mutex, std::try_to_lock);
        if (!st.lock.owns_lock()) return false;
    } else {
        st.lock = std::unique_lock<std::mutex>(st.sess->mutex);
    }
    Bank& bank = *st.sess->bank;
    if (st.prompt) {
        bank.reset();
    } else {
        { auto hc = frame_to_hidden(f, c); st.hc.seq = hc.seq; st.hc.pos = std::move(hc.pos); }
    }
    st.t0 = steady_seconds();
    if (!st.prompt) {
        std::vector<int32_t> keep;
        if (f.h.keep) {
            keep.reserve(f.h.keep->size());
            for (int64_t k : *f.h.keep) keep.push_back(static_cast<int32_t>(k));
        }
        if (!keep.empty() || bank.provisional() > 0)
            bank.resolve(keep.data(), static_cast<int>(keep.size()), bank.stream());
        if (f.h.crop) {
            const int64_t p = *f.h.crop;
            if (p < 0 || p > bank.len()) throw Error(Kind::protocol, "crop position exceeds session length");
            bank.crop(static_cast<int>(p));
        }
    }
    st.mr = mask_from_frame(f, bank.len(), st.hc.seq);
    forward_checks(bank, st.hc.seq, st.mr, c.max_seq_len);
    st.out_dt = cfg_.response_dtype < 0 ? f.h.dtype
                                        : (cfg_.response_dtype == SFG_WIRE_F32 ? wire::Dtype::f32 : wire::Dtype::f16);
    return true;
}

// Device part for one step or for several sessions' steps in ONE weight
// pass (cross-session batching): rows are concatenated, each row appends to
// and attends over its own session's cache (mega_forward's per-row banks).
// Every kernel is batch invariant, so each response is bitwise the one the
// step gets alone.
void Server::run(std::vector<StepState*>& group) {
    const ModelCfg& c = eng_.cfg();
    DeviceGuard g(eng_.device());
    StepState& s0 = *group.front();
    Bank& bank0 = *s0.sess->bank;
    Workspace& ws = bank0.ws();
    cudaStream_t s = bank0.stream();
    const int k = static_cast<int>(group.size());
    std::vector<int32_t> pos;
    MaskRuns mr;
    std::vector<int> row0(k);
    int rows = 0;
    for (int i = 0; i < k; ++i) {
        StepState& st = *group[i];
        row0[i] = rows;
        pos.insert(pos.end(), st.hc.pos.begin(), st.hc.pos.end());
        const int base = static_cast<int>(mr.runs.size());
        for (int r = 0; r < st.hc.seq; ++r) mr.row_off.push_back(base + st.mr.row_off[r]);
        mr.runs.insert(mr.runs.end(), st.mr.runs.begin(), st.mr.runs.end());
        rows += st.hc.seq;
        if (i > 0) SFG_CUDA(cudaStreamSynchronize(st.sess->bank->stream()));  // its keep/crop kernels
    }
    mr.row_off.push_back(static_cast<int32_t>(mr.runs.size()));
    upload_meta(eng_, ws, pos, mr, s);
    ws.additive_mask = k > 1 ? false : !mega_mask_ok(s0.mr, bank0.len());
    ws.prefix_mask = k == 1 && prefix_law(s0.mr);
    char* wire = static_cast<char*>(ws.wire);
    for (int i = 0; i < k; ++i) {
        StepState& st = *group[i];
        const int in_f32 = st.f.h.dtype == wire::Dtype::f32;
        const size_t off = static_cast<size_t>(row0[i]) * c.hidden_dim * 4;
        char* pin = static_cast<char*>(ws.wire_pin) + off;  // pinned: an async DMA, no driver staging
        std::memcpy(pin, st.f.tensor, st.f.tensor_len);
        SFG_CUDA(copy_async(wire + off, pin, st.f.tensor_len, cudaMemcpyHostToDevice, s));
        launch_unpack_rows(wire + off, in_f32, st.hc.seq * c.hidden_dim, ws.h + static_cast<size_t>(row0[i]) * c.hidden_dim, s);
    }
    SFG_CUDA(cudaMemsetAsync(ws.status, 0, sizeof(uint32_t), s));
    eng_.set_prior(ws, bank0.len(), s);
    if (k == 1) {
        eng_.forward_device(bank0, cfg_.layer_begin, cfg_.layer_end, rows, ws, s);
    } else {
        std::vector<Bank*> banks(k);
        std::vector<int32_t> info(3 * rows);
        for (int i = 0; i < k; ++i) {
            Bank* b = group[i]->sess->bank.get();
            banks[i] = b;
            for (int r = 0; r < group[i]->hc.seq; ++r) {
                const int row = row0[i] + r;
                info[3 * row] = i;
                info[3 * row + 1] = b->len() + r;
                info[3 * row + 2] = b->len();
            }
        }
        mega_forward(eng_, bank0, cfg_.layer_begin, cfg_.layer_end, rows, ws, s, &banks, info.data());
        shared_passes_.fetch_add(1);
    }
    std::vector<size_t> out_bytes(k);
    for (int i = 0; i < k; ++i) {
        StepState& st = *group[i];
        const int n = st.hc.seq * c.hidden_dim;
        const size_t off = static_cast<size_t>(row0[i]) * c.hidden_dim * 4;
        launch_pack_rows(ws.h + static_cast<size_t>(row0[i]) * c.hidden_dim, st.out_dt == wire::Dtype::f32, n,
                         wire + off, nullptr, s);
        out_bytes[i] = static_cast<size_t>(n) * wire::width(st.out_dt);
        SFG_CUDA(copy_async(static_cast<char*>(ws.wire_pin) + off, wire + off, out_bytes[i],
                                 cudaMemcpyDeviceToHost, s));
    }
    SFG_CUDA(cudaGetLastError());
    uint32_t* stw = reinterpret_cast<uint32_t*>(static_cast<char*>(ws.pinned) + ws.pinned_bytes - 64);
    SFG_CUDA(copy_async(stw, ws.status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SFG_CUDA(cudaStreamSynchronize(s));
    if (*stw & ST_ATTN_CAP) throw Error(Kind::internal, "attention launch sized below the visible key count");
    if (*stw & ST_EMPTY_ROW) throw Error(Kind::protocol, "mask row admits no attendable position");
    for (int i = 0; i < k; ++i) {
        StepState& st = *group[i];
        Bank& bank = *st.sess->bank;
        bank.set_len(bank.len() + st.hc.seq);
        if (st.prompt) bank.mark_committed(bank.len());
        st.sess->last_active = now_s_();
        wire::Header h;  // hidden_to_response (server.cpp:135-146)
        h.kind = wire::FrameKind::response;
        h.session_id = st.f.h.session_id;
        h.shape = {st.hc.seq, c.hidden_dim};
        h.dtype = st.out_dt;
        h.srv_ms = (steady_seconds() - st.t0) * 1000.0;
        wire::encode(h, static_cast<const uint8_t*>(ws.wire_pin) + static_cast<size_t>(row0[i]) * c.hidden_dim * 4,
                     out_bytes[i], nullptr, 0, *st.resp);
    }
}

void Server::handle_frame(const wire::FrameView& f, std::vector<uint8_t>& resp) {
    if (f.h.kind == wire::FrameKind::ping) {  // handle_ping (server.cpp:193-201)
        wire::Header h;
        h.kind = wire::FrameKind::response;
        h.session_id = f.h.session_id;
        h.shape = {0};
        h.dtype = f.h.dtype;
        h.srv_ms = 0.0;
        wire::encode(h, nullptr, 0, nullptr, 0, resp);
        return;
    }
    StepState st;
    st.resp = &resp;
    prepare(f, st);
    std::vector<StepState*> one{&st};
    run(one);
}

// handle() over several frames: step frames of distinct sessions whose rows
// fit one pass (<= 32 rows, each session <= 16, masks inside the layer-stack
// contract) share ONE weight pass; everything else is handled frame by frame.  Responses (and
// error frames) are exactly what handle() returns for each frame.
void Server::handle_batch(int n, const uint8_t* const* reqs, const size_t* lens,
                          std::vector<std::vector<uint8_t>>& resps) {
    resps.assign(static_cast<size_t>(n), {});
    // the shared pass is the layer-stack megakernel; one-by-one steps take it
    // too for these shapes, so responses stay bitwise those of handle()
    const bool batchable = eng_.fast() && eng_.tp_size() == 1 && mega_mode() == 1 &&
                           mega_supported(eng_, 1, false, true) && cfg_.layer_end - cfg_.layer_begin <= 50;
    // rows one shared weight pass carries: two sessions' 16-row lookahead
    // batches (32) when the layer stack supports it
    const int pass_rows = batchable ? mega_batch_rows(eng_) : tc_rows();
    std::vector<std::unique_ptr<StepState>> pending;
    std::vector<StepState*> group;
    int group_rows = 0;
    auto flush = [&]() {
        if (group.empty()) return;
        try {
            run(group);
        } catch (const Error& e) {  // a failed shared pass: report it on each of its frames
            for (StepState* st : group) error_frame(st->f.h.session_id, e.what(), *st->resp);
        }
        group.clear();
        group_rows = 0;
        pending.clear();
    };
    for (int i = 0; i < n; ++i) {
        wire::FrameView f;
        try {
            f = wire::decode(reqs[i], lens[i]);
        } catch (const Error& e) {
            error_frame("", e.what(), resps[i]);
            continue;
        }
        bool shared = false;
        if (batchable && (f.h.kind == wire::FrameKind::step || f.h.kind == wire::FrameKind::accept_and_step)) {
            auto sess = find_session(f.h.session_id);
            bool dup = false;
            for (StepState* st : group) dup = dup || st->sess == sess;
            // only per-row-attention sessions share a weight pass
            shared = sess && !dup && bank_rows_attention(*sess->bank);
        }
        if (!shared) {
            flush();
            handle(reqs[i], lens[i], resps[i]);
            continue;
        }
        auto st = std::make_unique<StepState>();
        st->resp = &resps[i];
        try {
            // never block on a session lock while the group holds others
            if (!prepare(f, *st, !group.empty())) {
                flush();
                prepare(f, *st, false);
            }
        } catch (const Error& e) {
            error_frame(f.h.session_id, e.what(), resps[i]);
            continue;
        } catch (const std::exception& e) {
            error_frame(f.h.session_id, std::string("internal: ") + e.what(), resps[i]);
            continue;
        }
        Bank& b = *st->sess->bank;
        const bool fits = mega_mask_ok(st->mr, b.len()) && st->hc.seq <= tc_rows();
        if (!fits) {  // run it alone (its keep/crop already applied)
            flush();
            std::vector<StepState*> one{st.get()};
            try {
                run(one);
            } catch (const Error& e) {
                error_frame(f.h.session_id, e.what(), resps[i]);
            }
            continue;
        }
        if (group_rows + st->hc.seq > pass_rows || static_cast<int>(group.size()) >= 16) flush();
        group_rows += st->hc.seq;
        group.push_back(st.get());
        pending.push_back(std::move(st));
    }
    flush();
}

// handle_prompt / handle_step (server.cpp:203-265) for a device-linked
// client: identical checks and state transitions, no device work.
Server::Lease Server::linked_begin(const LinkedStep& st) {
    const ModelCfg& c = eng_.cfg();
    Lease l;
    l.is_prompt = st.is_prompt;
    if (st.is_prompt) {
        if (st.session_id->empty()) throw Error(Kind::protocol, "prompt frame requires a session_id");
        for (int i = 0; i < st.seq; ++i)
            if (st.pos[i] < 0 || st.pos[i] >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
        if (st.seq > c.max_seq_len) throw Error(Kind::capacity, "prompt exceeds max_seq_len");
        l.sess = create_or_reset_session(*st.session_id);
    } else {
        l.sess = find_session(*st.session_id);
        if (!l.sess) throw Error(Kind::session, "unknown or expired session: " + *st.session_id);
    }
    l.lock = std::unique_lock<std::mutex>(l.sess->mutex);
    Bank& bank = *l.sess->bank;
    l.bank = &bank;
    l.committed_before = bank.committed_len();
    if (st.is_prompt) {
        bank.reset();
        l.committed_before = 0;
    } else {
        for (int i = 0; i < st.seq; ++i)
            if (st.pos[i] < 0 || st.pos[i] >= c.max_seq_len) throw Error(Kind::capacity, "position exceeds max_seq_len");
        std::vector<int32_t> keep;
        if (st.keep)
            for (int64_t k : *st.keep) keep.push_back(static_cast<int32_t>(k));
        if (!keep.empty() || bank.provisional() > 0) {
            bank.resolve_meta(keep.data(), static_cast<int>(keep.size()));
            l.n_keep = static_cast<int>(keep.size());
        }
        if (st.crop) {
            if (*st.crop < 0 || *st.crop > bank.len()) throw Error(Kind::protocol, "crop position exceeds session length");
            bank.crop(static_cast<int>(*st.crop));
        }
    }
    MaskRuns causal;
    const MaskRuns* mr = st.runs;
    if (!mr) {
        causal = causal_runs(st.seq, bank.len());
        mr = &causal;
    } else if (st.mask_q != st.seq || st.mask_kv != bank.len() + st.seq) {
        throw Error(Kind::protocol, "mask shape does not match cache length plus batch");
    }
    forward_checks(bank, st.seq, *mr, c.max_seq_len);
    l.prior = bank.len();
    return l;
}

void Server::linked_end(Lease& l, int seq) {
    l.bank->set_len(l.bank->len() + seq);
    if (l.is_prompt) l.bank->mark_committed(l.bank->len());
    l.sess->last_active = now_s_();
    l.lock.unlock();
}

}  // namespace sfg
