// GPU ServerEngine (server.hpp:28-77): session table + per-session device
// KV banks + the request state machine of PROTOCOL.md, with the middle-layer
// forward on the B200.  handle() is the FrameHandler-compatible entry point.
#pragma once
#include <atomic>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "sfg_engine.h"
#include "sfg_wire.h"

namespace sfg {

struct ServerCfg {
    int layer_begin = 2;
    int layer_end = 6;
    double session_expiry_s = 300.0;
    int max_sessions = 64;
    int response_dtype = -1;  // -1 mirror
};

class Server {
public:
    Server(Engine& eng, const ServerCfg& cfg);

    // ServerEngine::handle over encoded frames; never throws.
    void handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp);
    // handle() over several frames; step frames of distinct sessions share one
    // weight pass when their rows fit (cross-session batching); never throws.
    void handle_batch(int n, const uint8_t* const* reqs, const size_t* lens,
                      std::vector<std::vector<uint8_t>>& resps);
    // Weight passes handle_batch shared between >= 2 sessions' steps.
    uint64_t shared_passes() const { return shared_passes_.load(); }

    size_t expire_sessions();
    size_t session_count() const;
    bool session_view(const std::string& id, int* len, int* committed, int* prov) const;
    void set_clock(std::function<double()> now) { now_s_ = std::move(now); }
    const ServerCfg& config() const { return cfg_; }
    Engine& engine() { return eng_; }

    struct Session {
        std::unique_ptr<Bank> bank;
        double last_active = 0.0;
        std::mutex mutex;
    };

    // Device-linked steps for an in-process client on the same device.
    // linked_begin runs the handle_prompt / handle_step state machine and all
    // host-side checks (session, positions, keep, crop, mask shape, capacity)
    // and applies the bookkeeping; it does NOT touch the device.  The client
    // then runs the server's layers over its own device rows against
    // lease.bank (KV compaction driven by the client's step meta), and calls
    // linked_end once the step's work is enqueued.
    struct LinkedStep {
        const std::string* session_id;
        bool is_prompt;
        int seq;
        const int32_t* pos;               // host
        const std::vector<int64_t>* keep; // nullptr = absent
        std::optional<int64_t> crop;
        const MaskRuns* runs;             // nullptr = causal
        int mask_q, mask_kv;              // declared mask shape (when runs != nullptr)
    };
    struct Lease {
        std::shared_ptr<Session> sess;
        std::unique_lock<std::mutex> lock;
        Bank* bank = nullptr;
        int prior = 0;                    // cache length the forward appends at
        int committed_before = 0;         // committed length before resolve
        int n_keep = 0;                   // rows relocated by resolve (0: none)
        bool is_prompt = false;
    };
    Lease linked_begin(const LinkedStep& st);
    void linked_end(Lease& l, int seq);

private:
    struct StepState {
        wire::FrameView f;
        std::shared_ptr<Session> sess;
        std::unique_lock<std::mutex> lock;
        struct {
            int seq = 0;
            std::vector<int32_t> pos;
        } hc;
        MaskRuns mr;
        bool prompt = false;
        double t0 = 0.0;
        wire::Dtype out_dt = wire::Dtype::f16;
        std::vector<uint8_t>* resp = nullptr;
    };
    bool prepare(const wire::FrameView& f, StepState& st, bool try_lock = false);
    void run(std::vector<StepState*>& group);
    static int tc_rows() { return 16; }
    std::atomic<uint64_t> shared_passes_{0};
    std::shared_ptr<Session> find_session(const std::string& id);
    std::shared_ptr<Session> create_or_reset_session(const std::string& id);
    void handle_frame(const wire::FrameView& f, std::vector<uint8_t>& resp);
    void error_frame(const std::string& sid, const std::string& msg, std::vector<uint8_t>& resp);

    Engine& eng_;
    ServerCfg cfg_;
    std::function<double()> now_s_;
    mutable std::mutex table_mutex_;
    std::map<std::string, std::shared_ptr<Session>> sessions_;
};

// Validates a binary16 mask payload ({0,-0,-inf} only) and compacts it into
// runs; throws protocol errors with the reference messages (server.cpp:148-171).
MaskRuns runs_from_f16_mask(const uint16_t* m, int q, int kv);

}  // namespace sfg
