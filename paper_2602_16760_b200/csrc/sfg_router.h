// Multi-device serving front end.
//
// The reference serves every session through ONE ServerEngine behind a
// FrameServer that runs one thread per connection (transport.cpp:531,
// :565-581).  On an 8-GPU box the B200 equivalent is one server (engine
// replica) per device plus:
//
//   Router  — a FrameHandler over N backends: a session is placed on the
//             least-loaded backend when its prompt frame arrives and every
//             later frame of that session goes to the same backend (sticky;
//             sessions are independent, so there is no cross-device state
//             and no collective on the data path);
//   Batcher — a FrameHandler for many concurrent connection threads: frames
//             queue per backend and one worker thread per backend drains the
//             queue through Server::handle_batch, so the steps of concurrent
//             sessions share one weight pass (responses are bitwise those of
//             handle(): every FAST kernel is batch invariant).  Nothing waits
//             for a batch to fill: a worker takes whatever is queued when it
//             becomes free, so a lone session pays no added latency.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sfg.h"
#include "sfg_server.h"

namespace sfg {

// One device's server (batching capable) or any frame handler (tests,
// remote hops).
struct Backend {
    Server* server = nullptr;
    sfg_frame_handler fn = nullptr;
    void* ctx = nullptr;
    void handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp);
    void handle_batch(int n, const uint8_t* const* reqs, const size_t* lens, std::vector<std::vector<uint8_t>>& resps);
};

class Router {
public:
    Router(std::vector<Backend> backends, double session_expiry_s);
    // FrameHandler: route by session id, then the backend's handle(); never throws.
    void handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp);
    // Backend index for this frame (placing a new session on a prompt), or -1
    // with `resp` holding the error frame the reference server would send.
    int route(const uint8_t* req, size_t n, std::vector<uint8_t>& resp, std::string* sid = nullptr);
    // A backend answered a frame of `sid` with an error frame: a session the
    // backend no longer knows (expired / evicted) is dropped from the map.
    void observe_response(int backend, const std::string& sid, const std::vector<uint8_t>& resp);
    int device_of(const std::string& sid) const;
    std::vector<int> load() const;
    int size() const { return static_cast<int>(backends_.size()); }
    Backend& backend(int i) { return backends_[i]; }
    void set_clock(std::function<double()> now) { now_s_ = std::move(now); }

private:
    struct Placement {
        int backend;
        double last_active;
    };
    void expire_locked(double now);
    std::vector<Backend> backends_;
    double expiry_s_;
    std::function<double()> now_s_;
    mutable std::mutex mu_;
    std::map<std::string, Placement> placed_;
};

class Batcher {
public:
    // max_frames: frames per handle_batch call (0: unlimited)
    Batcher(Router& r, int max_frames);
    ~Batcher();
    // FrameHandler for concurrent connection threads: blocks until this
    // frame's response is ready; never throws.
    void handle(const uint8_t* req, size_t n, std::vector<uint8_t>& resp);
    uint64_t batches() const { return batches_; }
    uint64_t frames() const { return frames_; }
    uint64_t max_batch() const { return max_batch_; }

private:
    struct Item {
        const uint8_t* req;
        size_t n;
        std::vector<uint8_t>* resp;
        std::string sid;
        bool done = false;
    };
    struct Queue {
        std::mutex mu;
        std::condition_variable cv;
        std::deque<Item*> items;
        std::thread worker;
    };
    void run(int b);
    Router& r_;
    int max_frames_;
    bool stop_ = false;
    std::vector<std::unique_ptr<Queue>> q_;
    std::mutex done_mu_;
    std::condition_variable done_cv_;
    std::atomic<uint64_t> batches_{0}, frames_{0}, max_batch_{0};
};

}  // namespace sfg
