// tma.cu — host helpers behind tma.cuh.
#include <mutex>
#include <vector>

#include "tma.cuh"

namespace tsr {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }();
    return fn;
}

int pick_chunk(int64_t n0, int64_t tiles, int64_t slots, int overlap, int min_chunk) {
    // Grids that cannot fill the GPU with min_chunk-plane chunks (a few
    // tiles of a small grid) split down to single planes: latency, not the
    // per-chunk overlap, bounds them.
    if (tiles * ((n0 + min_chunk - 1) / min_chunk) < slots) min_chunk = 1;
    int64_t best_chunk = n0;
    double best = 1e300;
    for (int64_t nz = 1; nz <= 256; ++nz) {
        const int64_t chunk = (n0 + nz - 1) / nz;
        if (chunk < min_chunk && nz > 1) break;
        const int64_t ctas = tiles * ((n0 + chunk - 1) / chunk);
        const int64_t waves = (ctas + slots - 1) / slots;
        const double cost = (double)waves * (double)(chunk + overlap);
        if (cost < best) {
            best = cost;
            best_chunk = chunk;
        }
    }
    return (int)best_chunk;
}

namespace {
struct OccEntry {
    const void* fn;
    int dev, threads, smem, per_sm, nsm;
};
std::mutex g_occ_mu;
std::vector<OccEntry> g_occ;
}  // namespace

bool occupancy_cached(const void* fn, int dev, int threads, int smem, int* per_sm, int* nsm) {
    std::lock_guard<std::mutex> lock(g_occ_mu);
    for (const OccEntry& e : g_occ)
        if (e.fn == fn && e.dev == dev && e.threads == threads && e.smem == smem) {
            *per_sm = e.per_sm;
            *nsm = e.nsm;
            return true;
        }
    return false;
}

void occupancy_store(const void* fn, int dev, int threads, int smem, int per_sm, int nsm) {
    std::lock_guard<std::mutex> lock(g_occ_mu);
    g_occ.push_back(OccEntry{fn, dev, threads, smem, per_sm, nsm});
}

}  // namespace tsr
