// record.cuh — on-device record_and_check (engine.cpp:47-57) shared by the block, tile and
// bit-sliced kernels.
#pragma once
#include <cstdint>

#include "launch.h"

namespace escgd {
namespace {

constexpr int kStatusRunning = -1;
constexpr int kCompleted = 0, kStasis = 1, kStopped = 2;
constexpr uint32_t kStopTracked = 1u, kStopStasis = 2u;

__host__ __device__ __forceinline__ int align16(int x) { return (x + 15) & ~15; }

// record_and_check (engine.cpp:47-57) for one replica, executed by a single thread.
__device__ int record_decide(const uint64_t* counts, int S1, int64_t mcs, int r, const RunArgs& run) {
    const int64_t k = run.n_rec[r];
    if (run.trace_steps != nullptr && k < run.trace_cap) {
        run.trace_steps[r * run.trace_cap + k] = mcs;
        for (int v = 0; v < S1; ++v) run.trace_counts[(r * run.trace_cap + k) * S1 + v] = counts[v];
    }
    run.n_rec[r] = k + 1;
    int alive = 0;
    for (int v = 0; v < S1; ++v) {
        run.last_counts[r * S1 + v] = counts[v];
        if (v >= 1 && counts[v] > 0) ++alive;
    }
    run.mcs[r] = mcs;
    int st = kStatusRunning;
    if ((run.stop_flags & kStopTracked) && run.tracked >= 1 && run.tracked < S1 && counts[run.tracked] == 0)
        st = kStopped;
    else if (mcs >= run.mcs_limit)
        st = kCompleted;
    else if ((run.stop_flags & kStopStasis) && alive <= 1)
        st = kStasis;
    run.status[r] = st;
    return st;
}

}  // namespace
}  // namespace escgd
