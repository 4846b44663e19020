// Per-kernel-class device timing for bench.py's roofline line: when enabled,
// launch sites bracket their kernel with CUDA events on the launching
// stream; collect() (called after the step's stream sync) accumulates the
// elapsed times.  Disabled (the default) it costs one branch per launch.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

namespace sfg {

enum KClass : int {
    K_QKV = 0, K_ATTN, K_OPROJ, K_GATEUP, K_DOWN, K_NORM, K_HEAD, K_OTHER, K_LAYERS, K_NCLASS
};

class KernelProfiler {
public:
    static KernelProfiler& get();
    bool on() const { return on_; }
    void enable(bool v);
    // returns a slot index, or -1 when disabled
    int begin(int cls, cudaStream_t s);
    void end(int slot, cudaStream_t s, double bytes, double flops);
    void collect();  // after the work has completed
    void reset();
    void stats(int cls, int64_t* count, double* ms, double* bytes, double* flops);

    // Graph capture: slots recorded while capturing belong to the graph (its
    // event-record nodes fire on every replay); collect_graph() accumulates
    // them after each replay, release_graph() frees them with the graph.
    void begin_capture(std::vector<int>* list);
    void end_capture();
    void collect_graph(const std::vector<int>& list);
    void release_graph(const std::vector<int>& list);

private:
    struct Slot {
        int cls;
        cudaEvent_t a, b;
        double bytes, flops;
        bool used;
    };
    bool on_ = false;
    bool warned_ = false;
    std::vector<int>* capture_ = nullptr;
    std::mutex mu_;
    std::vector<Slot> slots_;
    std::vector<int> pending_;
    int64_t count_[K_NCLASS] = {};
    double ms_[K_NCLASS] = {}, bytes_[K_NCLASS] = {}, flops_[K_NCLASS] = {};
};

struct ProfScope {
    int slot;
    cudaStream_t s;
    double bytes, flops;
    ProfScope(int cls, cudaStream_t st, double by, double fl) : s(st), bytes(by), flops(fl) {
        slot = KernelProfiler::get().begin(cls, st);
    }
    ~ProfScope() {
        if (slot >= 0) KernelProfiler::get().end(slot, s, bytes, flops);
    }
};

}  // namespace sfg
