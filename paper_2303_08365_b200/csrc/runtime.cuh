// runtime.cuh — host runtime pieces shared by the single-grid driver (abi.cu)
// and the multi-slab driver (multi.cu): validation, engine planning, the
// sweep dispatch and host<->device staging of BasicGrid<T> buffers.
#pragma once

#include <functional>
#include <string>

#include "common.cuh"

namespace tsr {

// Records the status message for tsr_last_error() and returns its code.
int report(const Status& s);

// check_applicable (proj/include/tessera/naive.hpp:26-34): dims match and
// every halo covers the kernel radius.
Status check_applicable(const Geo& g, const TapSet& t);

struct Plan {
    const Engine* engine = nullptr;  // nullptr = generic one-thread-per-point sweep
    int k = 1;                       // fused steps per HBM pass
};
Status plan_for(const Geo& g, const TapSet& t, const tsr_opts& o, Plan& p);

// One fused pass of k steps from `in` to `out` over the ctx's plane range.
Status sweep(const LaunchCtx& c, const Plan& p, const void* in, void* out, int k);

tsr_opts opts_or_default(const tsr_opts* o);

// Host layout <-> pitched device layout, as pitched 3-D copies.
Status upload(const Geo& g, const void* host, void* dev, cudaStream_t s);
Status download(const Geo& g, const void* dev, void* host, bool interior_only, cudaStream_t s);

// True when the halo shells of the two host buffers are bitwise equal.
bool halos_equal(const Geo& g, const void* b0, const void* b1);

// `steps` time steps on device buffers d0/d1 (*cur = the read buffer, flipped
// per launch); keep_prev leaves step T-1 in the other buffer (abi.cu).
Status advance_grid(const Geo& g, const TapSet& t, const tsr_opts& o, void* d0, void* d1,
                    int* cur, int64_t steps, bool keep_prev, cudaStream_t s, tsr_stats* st);

// tsr_run on one device (the naive_run drop-in over host buffers), and the
// release of the buffers it caches per device (roundtrip.cu).
Status run_host_single(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int parity,
                       int64_t steps, const tsr_opts* o, tsr_stats* st);
void release_run_cache();
// The chunked round trip for the interior planes [r_lo, r_hi) of the
// outermost axis only (one device's share of tsr_run_multi's short runs):
// the planes its windows read beyond the range go up first, then
// `after_margins` runs (the split round trip's barrier across devices),
// then the pipeline.  TSR_EUNSUPPORTED when that path does not apply.
bool range_chunkable(const Geo& g, const TapSet& t, int64_t steps, int64_t r_lo, int64_t r_hi);
Status run_host_range(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int parity,
                      int64_t steps, const tsr_opts* o, tsr_stats* st, int64_t r_lo,
                      int64_t r_hi, const std::function<void()>& after_margins,
                      int cache_sub = 0);

// Sets the calling thread's device for a scope (and checks one exists).
struct DeviceGuard {
    int prev = -1;
    bool set = false;
    Status enter(int want);
    ~DeviceGuard();
};

// fill_random (proj/include/tessera/random.hpp:20-24) on host buffers.
void fill_random_host(const Geo& g, void* b0, void* b1, uint64_t seed, double lo, double hi,
                      uint64_t skip = 0);

}  // namespace tsr
