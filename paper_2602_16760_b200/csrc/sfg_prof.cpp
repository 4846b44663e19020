#include "sfg_prof.h"

#include <cstdio>

namespace sfg {

KernelProfiler& KernelProfiler::get() {
    static KernelProfiler p;
    return p;
}

void KernelProfiler::enable(bool v) {
    std::lock_guard<std::mutex> lk(mu_);
    on_ = v;
}

int KernelProfiler::begin(int cls, cudaStream_t s) {
    // while capturing, always record: the graph's event nodes must exist for
    // later replays that run with the profiler on
    if (!on_ && !capture_) return -1;
    std::lock_guard<std::mutex> lk(mu_);
    int idx = -1;
    for (size_t i = 0; i < slots_.size(); ++i)
        if (!slots_[i].used) {
            idx = static_cast<int>(i);
            break;
        }
    if (idx < 0) {
        Slot sl{};
        cudaEventCreate(&sl.a);
        cudaEventCreate(&sl.b);
        slots_.push_back(sl);
        idx = static_cast<int>(slots_.size()) - 1;
    }
    Slot& sl = slots_[idx];
    sl.used = true;
    sl.cls = cls;
    // inside stream capture an event record only becomes a graph node (and
    // so timeable after replay) when recorded as an external event
    cudaEventRecordWithFlags(sl.a, s, capture_ ? cudaEventRecordExternal : cudaEventRecordDefault);
    return idx;
}

void KernelProfiler::end(int slot, cudaStream_t s, double bytes, double flops) {
    std::lock_guard<std::mutex> lk(mu_);
    Slot& sl = slots_[slot];
    sl.bytes = bytes;
    sl.flops = flops;
    cudaEventRecordWithFlags(sl.b, s, capture_ ? cudaEventRecordExternal : cudaEventRecordDefault);
    if (capture_)
        capture_->push_back(slot);
    else
        pending_.push_back(slot);
}

void KernelProfiler::begin_capture(std::vector<int>* list) {
    std::lock_guard<std::mutex> lk(mu_);
    capture_ = list;
}

void KernelProfiler::end_capture() {
    std::lock_guard<std::mutex> lk(mu_);
    capture_ = nullptr;
}

void KernelProfiler::collect_graph(const std::vector<int>& list) {
    std::lock_guard<std::mutex> lk(mu_);
    for (int i : list) {
        Slot& sl = slots_[i];
        float ms = 0;
        const cudaError_t e = cudaEventElapsedTime(&ms, sl.a, sl.b);
        if (e != cudaSuccess) {
            // a failed query must not leak into the caller's cudaGetLastError()
            cudaGetLastError();
            if (!warned_) {
                warned_ = true;
                fprintf(stderr, "sfg profiler: graph event timing unavailable (%s)\n", cudaGetErrorString(e));
            }
            continue;
        }
        count_[sl.cls] += 1;
        ms_[sl.cls] += ms;
        bytes_[sl.cls] += sl.bytes;
        flops_[sl.cls] += sl.flops;
    }
}

void KernelProfiler::release_graph(const std::vector<int>& list) {
    std::lock_guard<std::mutex> lk(mu_);
    for (int i : list) slots_[i].used = false;
}

void KernelProfiler::collect() {
    std::lock_guard<std::mutex> lk(mu_);
    std::vector<int> keep;
    for (int i : pending_) {
        Slot& sl = slots_[i];
        if (cudaEventQuery(sl.b) != cudaSuccess) {
            keep.push_back(i);
            continue;
        }
        float ms = 0;
        if (cudaEventElapsedTime(&ms, sl.a, sl.b) != cudaSuccess) {
            cudaGetLastError();
            sl.used = false;
            continue;
        }
        count_[sl.cls] += 1;
        ms_[sl.cls] += ms;
        bytes_[sl.cls] += sl.bytes;
        flops_[sl.cls] += sl.flops;
        sl.used = false;
    }
    pending_.swap(keep);
}

void KernelProfiler::reset() {
    collect();
    std::lock_guard<std::mutex> lk(mu_);
    for (int c = 0; c < K_NCLASS; ++c) count_[c] = 0, ms_[c] = bytes_[c] = flops_[c] = 0;
}

void KernelProfiler::stats(int cls, int64_t* count, double* ms, double* bytes, double* flops) {
    collect();
    std::lock_guard<std::mutex> lk(mu_);
    if (cls < 0 || cls >= K_NCLASS) return;
    *count = count_[cls];
    *ms = ms_[cls];
    *bytes = bytes_[cls];
    *flops = flops_[cls];
}

}  // namespace sfg
