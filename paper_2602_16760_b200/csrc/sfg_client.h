// Trusted-side runtime on the B200: SplitClient (client.hpp:41-100) and the
// decode loops of decoding.cpp with a host NGramPool.  The exchange is either
// frame-level through a FrameHandler-like C callback (drop-in against any
// splitf server) or device-linked to an in-process sfg::Server on the same
// device (no host copies; wire quantisation applied on device).  Linked
// steps are captured once per batch size as a CUDA graph and replayed.
#pragma once
#include <chrono>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

#include "sfg_engine.h"
#include "sfg_server.h"

namespace sfg {

// NGramPool (decoding.hpp:35-60, decoding.cpp:61-97): one recency list,
// dedup on (key, continuation), eviction from the back, lookup returns a
// key's entries most-recent-first.  Same observable behaviour as the
// reference's std::list scan, but entries are also threaded on a per-key
// list so insert/lookup cost O(entries of that key) instead of O(pool):
// the forced-B=16 benchmark pool holds G continuations for every token.
class Pool {
public:
    Pool(int ngram_n, size_t capacity);
    ~Pool();
    Pool(const Pool&) = delete;
    Pool& operator=(const Pool&) = delete;
    void update(const int32_t* prev, const int32_t* cur, int w);
    int lookup(int key, int max_c, std::vector<std::vector<int32_t>>& out) const;
    size_t size() const { return size_; }
    int ngram_n() const { return n_; }

private:
    struct Node {
        int32_t key;
        std::vector<int32_t> cont;
        Node *gprev = nullptr, *gnext = nullptr;  // global recency list
        Node *kprev = nullptr, *knext = nullptr;  // per-key recency list
    };
    struct KeyList {
        Node *head = nullptr, *tail = nullptr;
    };
    void insert(int32_t key, const int32_t* cont);
    void link_front(Node* n);
    void unlink(Node* n);
    int n_;
    size_t cap_, size_ = 0;
    Node *head_ = nullptr, *tail_ = nullptr;
    std::unordered_map<int32_t, KeyList> keys_;
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
    bool graph = false;
};

class Client {
public:
    Client(Engine& local, const ClientCfg& cfg, sfg_frame_handler handler, void* ctx, Server* linked,
           std::string session_id);
    ~Client();

    int prefill(const int32_t* prompt, int n, float* logits_row);
    // One exchange (client.cpp:169-228).  Outputs: logits rows (host), row
    // argmaxes (host), verify tail (VerifyOut) when vin is given.
    void decode_step(int seq, const int32_t* tokens, const int32_t* positions, const MaskRuns* runs,
                     const int32_t* keep, int n_keep, std::optional<int> crop, float* logits_out,
                     int32_t* argmax_out, const VerifyIn* vin, VerifyOut* vout);

    const StepProfile& last_profile() const { return prof_; }
    uint64_t clamped();
    Bank& prefix() { return *prefix_; }
    Bank& suffix() { return *suffix_; }
    Engine& engine() { return eng_; }

private:
    struct Graph {
        int rows;
        bool logits, verify;
        // the mask class fixes the kernel choice baked into the graph
        // (megakernel vs per-GEMM path, Engine::forward_device)
        bool additive;
        uint64_t server_bank;  // Bank::id(), never an address (banks are freed and reallocated)
        uint64_t generation;
        cudaGraphExec_t exec = nullptr;
        std::vector<int> prof_slots;
        int launches = 0;
        int seen = 0;
    };
    // device step pieces (graph-capturable: no host syncs, fixed sizes)
    int dev_pre(int rows, Bank* server_bank, bool verify, cudaStream_t s);
    int dev_server(int rows, Bank* server_bank, cudaStream_t s);
    int dev_post(int rows, bool want_logits, bool verify, cudaStream_t s);
    void exchange_frames(bool prompt, int seq, const int32_t* pos, const MaskRuns* runs, int mask_kv,
                         const int32_t* keep, int n_keep, bool send_keep, std::optional<int> crop);
    void sleep_one_way() const;
    void stage_inputs(int seq, const int32_t* ids, const int32_t* pos, const MaskRuns& mr);
    void ensure_out(int rows);
    Graph* find_graph(int rows, bool logits, bool verify, bool additive, const Bank* server_bank);

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
    cudaEvent_t ev_[4] = {};
    VerifyIn* d_vin_ = nullptr;
    VerifyOut* d_vout_ = nullptr;
    VerifyIn* h_vin_ = nullptr;
    VerifyOut* h_vout_ = nullptr;
    int32_t* h_argmax_ = nullptr;   // pinned [out_rows_]
    float* h_logits_ = nullptr;     // pinned [out_rows_ x vocab]
    int out_rows_ = 0;
    std::vector<Graph> graphs_;
    std::vector<uint8_t> req_;
};

// decode_sequential / decode_lookahead_with_pool (decoding.cpp:111-355) as a
// resumable loop: the constructor runs prefill, step() runs one iteration.
class Decoder {
public:
    struct Cfg {
        int mode = 2, window_w = 8, ngram_n = 3, max_candidates_g = 2;
        size_t pool_capacity = 4096;
    };
    Decoder(Client& c, const Cfg& cfg, Pool* pool, const int32_t* prompt, int n, int max_new, bool want_logits);
    bool done() const { return static_cast<int>(tokens.size()) >= max_new_; }
    int step();  // committed tokens this step

    std::vector<int32_t> tokens, step_batch, step_accepted;
    std::vector<float> logits;  // committed rows (want_logits)
    int steps = 0, committed = 0, hits = 0;
    double wall_s = 0;

private:
    Client& c_;
    Cfg cfg_;
    Pool* pool_;
    std::unique_ptr<Pool> own_;
    int max_new_, total_;
    bool want_logits_;
    std::vector<int32_t> window_, keep_, batch_, pos_;
    std::vector<std::vector<int32_t>> cands_;
    std::vector<float> lbuf_;
    VerifyIn vin_{};
    VerifyOut vout_{};
};

}  // namespace sfg
