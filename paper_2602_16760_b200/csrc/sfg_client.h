// Trusted-side runtime on the B200: SplitClient (client.hpp:41-100) and the
// decode loops of decoding.cpp with a host NGramPool.  The exchange is either
// frame-level through a FrameHandler-like C callback (drop-in against any
// splitf server) or device-linked to an in-process sfg::Server on the same
// device (no host copies; wire quantisation applied on device).
#pragma once
#include <chrono>
#include <list>
#include <optional>
#include <string>
#include <vector>

#include "sfg_engine.h"
#include "sfg_server.h"

namespace sfg {

// NGramPool (decoding.hpp:35-60, decoding.cpp:61-97): recency-ordered list,
// dedup on (key, continuation), capacity eviction from the back.
class Pool {
public:
    Pool(int ngram_n, size_t capacity);
    void update(const int32_t* prev, const int32_t* cur, int w);
    int lookup(int key, int max_c, std::vector<std::vector<int32_t>>& out) const;
    size_t size() const { return entries_.size(); }
    int ngram_n() const { return n_; }

private:
    struct Entry {
        int32_t key;
        std::vector<int32_t> cont;
    };
    void insert(int32_t key, std::vector<int32_t> cont);
    int n_;
    size_t cap_;
    std::list<Entry> entries_;
};

struct ClientCfg {
    int prefix_layers = 2;
    int suffix_layers = 2;
    int wire_dtype = SFG_WIRE_F16;
    double one_way_delay_ms = 0.0;
};

struct StepProfile {
    double step_ms = 0, server_ms = 0, local_ms = 0;
    int launches = 0, batch = 0;
};

class Client {
public:
    Client(Engine& local, const ClientCfg& cfg, sfg_frame_handler handler, void* ctx, Server* linked,
           std::string session_id);
    ~Client();

    int prefill(const int32_t* prompt, int n, float* logits_row);
    // One exchange; results stay on device (ws.logits if want_logits, ws.argmax).
    void decode_step(int seq, const int32_t* tokens, const int32_t* positions, const MaskRuns* runs,
                     const int32_t* keep, int n_keep, std::optional<int> crop, bool want_logits);
    // Host copies of the last step's outputs.
    void fetch_logits(int rows, float* out);
    void fetch_argmax(int rows, int32_t* out);

    struct DecodeCfg {
        int mode = 2, window_w = 8, ngram_n = 3, max_candidates_g = 2;
        size_t pool_capacity = 4096;
    };
    struct DecodeOut {
        std::vector<int32_t> tokens, step_batch, step_accepted;
        std::vector<float> logits;  // committed rows (optional)
        int steps = 0, committed = 0;
        double wall_s = 0, match_rate = 0;
    };
    void decode(const DecodeCfg& cfg, Pool* pool, const int32_t* prompt, int n, int max_new,
                bool want_logits, DecodeOut& out);

    const StepProfile& last_profile() const { return prof_; }
    uint64_t clamped();
    Bank& prefix() { return *prefix_; }
    Bank& suffix() { return *suffix_; }
    int committed_len() const { return prefix_->committed_len(); }

private:
    void exchange(bool prompt, int seq, const int32_t* pos, const MaskRuns* runs, int mask_kv,
                  const int32_t* keep, int n_keep, bool send_keep, std::optional<int> crop);
    void sleep_one_way() const;
    void run_head(int rows, bool want_logits, VerifyIn* vin);

    Engine& eng_;
    ClientCfg cfg_;
    sfg_frame_handler handler_;
    void* ctx_;
    Server* linked_;
    std::string sid_;
    std::unique_ptr<Bank> prefix_, suffix_;
    bool prefilled_ = false, dead_ = false, first_step_done_ = false;
    int prompt_len_ = 0;
    StepProfile prof_;
    cudaEvent_t ev_[6] = {};
    VerifyIn* d_vin_ = nullptr;
    VerifyOut* d_vout_ = nullptr;
    VerifyIn* h_vin_ = nullptr;
    VerifyOut* h_vout_ = nullptr;
    std::vector<uint8_t> req_, maskbuf_;
};

}  // namespace sfg
