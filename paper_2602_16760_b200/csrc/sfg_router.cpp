// Multi-device router and cross-session batching queue (see sfg_router.h).
#include "sfg_router.h"

#include <algorithm>
#include <chrono>

#include "sfg_wire.h"

namespace sfg {

namespace {
double steady_now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void error_frame(const std::string& sid, const std::string& msg, std::vector<uint8_t>& resp) {
    wire::Header h;  // server.cpp:186-190
    h.kind = wire::FrameKind::error;
    h.session_id = sid;
    h.shape = {0};
    h.err = msg;
    wire::encode(h, nullptr, 0, nullptr, 0, resp);
}
}  // namespace

void Backend::handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp) {
    if (server) {
        server->handle(req, n, resp);
        return;
    }
    const uint8_t* rp = nullptr;
    size_t rn = 0;
    if (fn(ctx, req, n, &rp, &rn) != 0) {
        error_frame("", "transport: frame handler failed", resp);
        return;
    }
    resp.assign(rp, rp + rn);
}

void Backend::handle_batch(int n, const uint8_t* const* reqs, const size_t* lens,
                           std::vector<std::vector<uint8_t>>& resps) {
    if (server) {
        server->handle_batch(n, reqs, lens, resps);
        return;
    }
    resps.assign(static_cast<size_t>(n), {});
    for (int i = 0; i < n; ++i) handle(reqs[i], lens[i], resps[i]);
}

// ── Router ──────────────────────────────────────────────────────────────
Router::Router(std::vector<Backend> backends, double session_expiry_s)
    : backends_(std::move(backends)), expiry_s_(session_expiry_s), now_s_(steady_now) {
    if (backends_.empty()) throw Error(Kind::config, "router needs at least one backend");
    if (!(session_expiry_s > 0.0)) throw Error(Kind::config, "session expiry must be positive");
    for (const Backend& b : backends_)
        if (!b.server && !b.fn) throw Error(Kind::config, "router backend has neither a server nor a handler");
}

void Router::expire_locked(double now) {
    for (auto it = placed_.begin(); it != placed_.end();) {
        if (now - it->second.last_active > expiry_s_) it = placed_.erase(it);
        else ++it;
    }
}

int Router::route(const uint8_t* req, size_t n, std::vector<uint8_t>& resp, std::string* sid_out) {
    wire::FrameView f;
    try {
        f = wire::decode(req, n);
    } catch (const Error& e) {
        error_frame("", e.what(), resp);
        return -1;
    }
    if (sid_out) *sid_out = f.h.session_id;
    const auto kind = f.h.kind;
    // pings, sessionless prompts and non-request kinds carry no placement: any
    // backend answers them exactly as the reference server would
    if (kind == wire::FrameKind::ping || kind == wire::FrameKind::response || kind == wire::FrameKind::error ||
        (kind == wire::FrameKind::prompt && f.h.session_id.empty()))
        return 0;
    std::lock_guard<std::mutex> g(mu_);
    const double now = now_s_();
    auto it = placed_.find(f.h.session_id);
    if (it != placed_.end()) {
        it->second.last_active = now;
        return it->second.backend;  // sticky (a re-prompt resets the session where it lives)
    }
    if (kind != wire::FrameKind::prompt) {  // handle_step's lookup (server.cpp:226-232)
        error_frame(f.h.session_id, std::string(kind_name(Kind::session)) + ": unknown or expired session: " +
                                        f.h.session_id,
                    resp);
        return -1;
    }
    expire_locked(now);
    std::vector<int> cnt(backends_.size(), 0);
    for (const auto& kv : placed_) ++cnt[kv.second.backend];
    const int b = static_cast<int>(std::min_element(cnt.begin(), cnt.end()) - cnt.begin());
    placed_[f.h.session_id] = Placement{b, now};
    return b;
}

void Router::observe_response(int backend, const std::string& sid, const std::vector<uint8_t>& resp) {
    if (sid.empty()) return;
    wire::FrameView r;
    try {
        r = wire::decode(resp.data(), resp.size());
    } catch (...) {
        return;
    }
    if (r.h.kind != wire::FrameKind::error || !r.h.err) return;
    // the backend no longer holds the session (expired, or a failed prompt)
    const std::string pfx = std::string(kind_name(Kind::session)) + ":";
    const std::string cap = std::string(kind_name(Kind::capacity)) + ":";
    if (r.h.err->compare(0, pfx.size(), pfx) != 0 && r.h.err->compare(0, cap.size(), cap) != 0) return;
    std::lock_guard<std::mutex> g(mu_);
    auto it = placed_.find(sid);
    if (it != placed_.end() && it->second.backend == backend) placed_.erase(it);
}

void Router::handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp) {
    std::string sid;
    const int b = route(req, n, resp, &sid);
    if (b < 0) return;
    backends_[b].handle(req, n, resp);
    observe_response(b, sid, resp);
}

int Router::device_of(const std::string& sid) const {
    std::lock_guard<std::mutex> g(mu_);
    auto it = placed_.find(sid);
    return it == placed_.end() ? -1 : it->second.backend;
}

std::vector<int> Router::load() const {
    std::lock_guard<std::mutex> g(mu_);
    std::vector<int> cnt(backends_.size(), 0);
    for (const auto& kv : placed_) ++cnt[kv.second.backend];
    return cnt;
}

// ── Batcher ─────────────────────────────────────────────────────────────
Batcher::Batcher(Router& r, int max_frames) : r_(r), max_frames_(max_frames) {
    for (int b = 0; b < r_.size(); ++b) q_.push_back(std::make_unique<Queue>());
    for (int b = 0; b < r_.size(); ++b) q_[b]->worker = std::thread([this, b] { run(b); });
}

Batcher::~Batcher() {
    for (auto& q : q_) {
        std::lock_guard<std::mutex> g(q->mu);
        stop_ = true;
        q->cv.notify_all();
    }
    for (auto& q : q_)
        if (q->worker.joinable()) q->worker.join();
}

void Batcher::handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp) {
    Item it{req, n, &resp, {}};
    const int b = r_.route(req, n, resp, &it.sid);
    if (b < 0) return;
    Queue& q = *q_[b];
    {
        std::lock_guard<std::mutex> g(q.mu);
        q.items.push_back(&it);
    }
    q.cv.notify_one();
    std::unique_lock<std::mutex> lk(done_mu_);
    done_cv_.wait(lk, [&] { return it.done; });
}

void Batcher::run(int b) {
    Queue& q = *q_[b];
    std::vector<Item*> batch;
    std::vector<const uint8_t*> reqs;
    std::vector<size_t> lens;
    std::vector<std::vector<uint8_t>> resps;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(q.mu);
            q.cv.wait(lk, [&] { return stop_ || !q.items.empty(); });
            if (q.items.empty()) return;  // stopping
            batch.clear();
            // whatever is queued now forms the batch: no waiting for it to fill
            while (!q.items.empty() && (max_frames_ <= 0 || static_cast<int>(batch.size()) < max_frames_)) {
                batch.push_back(q.items.front());
                q.items.pop_front();
            }
        }
        reqs.clear();
        lens.clear();
        for (Item* it : batch) {
            reqs.push_back(it->req);
            lens.push_back(it->n);
        }
        try {
            r_.backend(b).handle_batch(static_cast<int>(batch.size()), reqs.data(), lens.data(), resps);
        } catch (const std::exception& e) {  // handle_batch never throws; belt and braces
            resps.assign(batch.size(), {});
            for (size_t i = 0; i < batch.size(); ++i)
                error_frame(batch[i]->sid, std::string("internal: ") + e.what(), resps[i]);
        }
        for (size_t i = 0; i < batch.size(); ++i) {
            *batch[i]->resp = std::move(resps[i]);
            r_.observe_response(b, batch[i]->sid, *batch[i]->resp);
        }
        batches_.fetch_add(1);
        frames_.fetch_add(batch.size());
        uint64_t m = max_batch_.load();
        while (batch.size() > m && !max_batch_.compare_exchange_weak(m, batch.size())) {
        }
        {
            std::lock_guard<std::mutex> g(done_mu_);
            for (Item* it : batch) it->done = true;
        }
        done_cv_.notify_all();
    }
}

}  // namespace sfg
