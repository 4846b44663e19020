// GPU ServerEngine (server.hpp:28-77): session table + per-session device
// KV banks + the request state machine of PROTOCOL.md, with the middle-layer
// forward on the B200.  handle() is the FrameHandler-compatible entry point.
#pragma once
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

    // Device-linked step for an in-process client on the same device: rows
    // are device fp32 already carrying the wire quantisation; they are
    // transformed in place on stream s.  Same state machine and checks as
    // handle_step; returns kernels launched.
    struct LinkedStep {
        const std::string* session_id;
        bool is_prompt;
        int seq;
        const int32_t* pos;               // host
        const std::vector<int64_t>* keep; // nullptr = absent
        std::optional<int64_t> crop;
        const MaskRuns* runs;             // nullptr = causal
        int mask_q, mask_kv;              // declared mask shape (when runs != nullptr)
        float* rows;                      // device [seq x H], in/out
        cudaStream_t stream;
    };
    int linked_step(const LinkedStep& st);

private:
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
