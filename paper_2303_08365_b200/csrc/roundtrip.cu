// roundtrip.cu — tsr_run, the naive_run drop-in over host buffers
// (proj/include/tessera/naive.hpp:96-100): one contiguous upload of the read
// buffer, the sweeps, and both buffers back, with the device buffers cached
// per device between calls; short runs of large grids take the chunked
// round trip (windows widened by T*r planes, uploads, sweeps and downloads
// overlapped), from pinned host memory directly or staged through pinned
// slots by host threads from pageable memory.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "runtime.cuh"

namespace tsr {

namespace {

// Device buffers cached by tsr_run between calls, one set per device.
struct DeviceCache {
    void* d[2] = {nullptr, nullptr};
    int64_t bytes = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // host-layout staging buffer for contiguous device->host copies (lazily
    // allocated; without it the downloads are pitched 3-D copies)
    void* stage = nullptr;
    int64_t stage_bytes = 0;
    // chunked round trip (run_chunked): compute and device->host streams,
    // an event pool and the two window sets
    cudaStream_t s_comp = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> pool;
    void* pipe = nullptr;
    int64_t pipe_bytes = 0;
    void* hstage = nullptr;  // pinned host slots of the staged (pageable) round trip
    int64_t hstage_bytes = 0;
    std::mutex mu;  // held by the call using this device's cache
    int device = 0;
};
std::mutex g_cache_mu;  // guards g_cache itself
std::vector<std::unique_ptr<DeviceCache>> g_cache;

// Cache `sub` of device `dev` (sub > 0: a second range of tsr_run_multi's
// split round trip on the same device, which needs buffers of its own).
constexpr int kSubs = 16;
DeviceCache* cache_slot(int dev, int sub = 0) {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    const size_t key = static_cast<size_t>(dev) * kSubs + sub % kSubs;
    if (g_cache.size() <= key) g_cache.resize(key + 1);
    if (!g_cache[key]) {
        g_cache[key] = std::make_unique<DeviceCache>();
        g_cache[key]->device = dev;
    }
    return g_cache[key].get();
}

// Streams, events and the two work buffers of device `dev`'s cache (the
// caller holds its mutex).
Status cache_for(DeviceCache* slot, int64_t bytes, DeviceCache** out) {
    DeviceCache& c = *slot;
    if (!c.stream) {
        TSR_CUDA_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        TSR_CUDA_TRY(cudaEventCreate(&c.ev[0]));
        TSR_CUDA_TRY(cudaEventCreate(&c.ev[1]));
    }
    if (c.bytes < bytes) {
        for (void*& p : c.d)
            if (p) {
                cudaFree(p);
                p = nullptr;
            }
        c.bytes = 0;
        for (void*& p : c.d) {
            if (cudaMalloc(&p, bytes) != cudaSuccess) {
                cudaGetLastError();
                for (void*& q : c.d)
                    if (q) {
                        cudaFree(q);
                        q = nullptr;
                    }
                return Status::Err(TSR_ENOMEM, "device allocation failed");
            }
        }
        c.bytes = bytes;
    }
    *out = &c;
    return Status::Ok();
}

// ---- chunked host round trip ------------------------------------------
// A short run's tsr_run is PCIe-bound: one buffer up, two down.  Step T at a
// plane of the outermost axis depends only on the planes within T*r of it, so
// for T*r small against that axis the grid is cut into chunks of planes, each
// advanced T steps on its own window (the chunk widened by T*r planes per side:
// the window's edge planes act as a frozen halo whose error moves inward r
// planes per step and never reaches the chunk).  Window j computes once the
// planes it reads are uploaded, and its chunk of steps T and T-1 goes down
// while later windows compute and later pieces go up: host->device and
// device->host copies run concurrently (PCIe is full duplex) instead of one
// after the other.  Each point runs the same per-point arithmetic as the
// whole-grid run (same engine, same fused depth), so the result is identical.
struct Chunks {
    int ax = 0;           // normalised outermost axis (3 - dims)
    int64_t n0 = 0, h0 = 0, margin = 0, size = 0;
    int nchunks = 0;
    int64_t piece = 0;    // host planes per upload piece
    int npieces = 0;
    int64_t hplane = 0;   // host elements per plane
    int64_t win_elems = 0, out_elems = 0;  // per buffer of one window set
    int64_t r_lo = 0, r_hi = 0;            // the planes this call returns
    int piece_lo = 0, piece_hi = 0;        // the pieces its windows read
    // split round trip (tsr_run_multi): the pieces holding planes outside
    // [r_lo, r_hi) go up first, before any device writes its planes back
    bool margins_first = false;
    bool pre(int i) const {
        const int64_t a = i * piece, b = a + piece;
        return margins_first && !(a >= r_lo + h0 && b <= r_hi + h0);
    }
};

// Chunks over the interior planes [r_lo, r_hi) of the outermost axis (the
// whole axis for tsr_run; one device's share for tsr_run_multi's short runs).
bool plan_chunks(const Geo& g, const TapSet& t, int64_t steps, int64_t r_lo, int64_t r_hi,
                 Chunks* ch) {
    if (g.dims < 2) return false;
    // TSR_RUN_CHUNKED: 0 = never, 1 = whenever there are >= 3 chunks, unset =
    // where the time model below predicts a gain, for grids of >= 64 MiB per
    // buffer (TSR_CHUNK_MIN_MB; below that the copies
    // take a few ms and the extra launches cancel the overlap).  At most 16
    // chunks below 1 GiB per buffer, 32 above (TSR_CHUNKS_MAX), from a sweep
    // at T = 20 (tools/probe/chunk_sweep.py): 4096^2 fp64 7.8 -> 5.9 ms with
    // 16 (7.1 with 32), 16384^2 121.6 -> 84.2 ms with 32 (85.8 with 16).
    const int64_t n_all = g.n[3 - g.dims];
    const int64_t bytes = g.host_elements * g.esize * (r_hi - r_lo) / std::max<int64_t>(1, n_all);
    const char* env = std::getenv("TSR_RUN_CHUNKED");
    if (env && *env == '0') return false;
    const char* min_mb = std::getenv("TSR_CHUNK_MIN_MB");
    const int64_t min_bytes = (min_mb ? std::atoll(min_mb) : 64) << 20;
    if (!(env && *env == '1') && bytes < min_bytes) return false;
    const char* mx = std::getenv("TSR_CHUNKS_MAX");
    const int64_t max_chunks =
        mx ? std::max(3, std::atoi(mx)) : (bytes < (int64_t(1) << 30) ? 16 : 32);
    Chunks c;
    c.ax = 3 - g.dims;
    c.n0 = g.n[c.ax];
    c.h0 = g.h[c.ax];
    c.r_lo = r_lo;
    c.r_hi = r_hi;
    const int64_t n = r_hi - r_lo;
    if (steps > n) return false;  // the cone spans the range (and T*r cannot overflow)
    c.margin = steps * std::max(1, t.radius);
    // chunks of 2*T*r planes (windows twice the chunk): the first download
    // starts after a small share of the upload; at most max_chunks of them
    c.size = std::max<int64_t>(
        {16, 2 * c.margin, (n + max_chunks - 1) / max_chunks, 2 * c.h0 + 1});
    // n / size chunks of equal size (+-1 plane): no wide last chunk whose
    // download would trail the others
    c.nchunks = static_cast<int>(n / c.size);
    if (c.nchunks < 3) return false;
    c.hplane = g.hpitch[c.ax];
    c.piece = c.size;
    c.npieces = static_cast<int>((c.n0 + 2 * c.h0 + c.piece - 1) / c.piece);
    // host planes [max(0, r_lo - margin), min(n0, r_hi + margin) + 2 h0)
    c.piece_lo = static_cast<int>(std::max<int64_t>(0, r_lo - c.margin) / c.piece);
    c.piece_hi = static_cast<int>((std::min(c.n0, r_hi + c.margin) + 2 * c.h0 - 1) / c.piece);
    if (!(env && *env == '1')) {
        // Time model (seconds): copies at ~50 GB/s per direction, ~1.4x that
        // with both directions busy; sweeps at a conservative 800 GS/s for
        // fp64 (x 8/esize, x 9/taps beyond 9 taps); the windows sweep
        // (size + 2 margin) / size times the points, and the first window
        // waits for its planes.  Chunked only where it wins by >= 5%
        // (measured crossover, tools/probe/chunk_T.py: 10000^2 Heat-2D
        // T = 200 1.19x faster chunked, T = 400 0.86x).
        const double up = double(bytes) / 50e9, down = (steps >= 2 ? 2 : 1) * up;
        const double rate = 800e9 * (8.0 / g.esize) * std::min(1.0, 9.0 / std::max(1, t.ntaps));
        const double sweep = double(g.interior()) * double(n) / double(c.n0) * double(steps) / rate;
        const double avg = double(n) / c.nchunks;
        const double f = (avg + 2.0 * double(c.margin)) / avg;
        const double ramp = up * (avg + c.margin) / n + sweep * (avg + 2.0 * c.margin) / n;
        const double whole = up + sweep + down;
        const double chunked = std::max((up + down) / 1.4, f * sweep) + ramp;
        if (chunked > 0.95 * whole) return false;
    }
    *ch = c;
    return true;
}

tsr_grid window_grid(const tsr_grid& gg, int64_t planes) {
    tsr_grid w = gg;
    w.extent[0] = planes;
    return w;
}

Status chunk_resources(const Geo& g, Chunks& ch, DeviceCache* c) {
    if (!c->s_comp) {
        TSR_CUDA_TRY(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
        TSR_CUDA_TRY(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
    }
    const size_t need = static_cast<size_t>(ch.npieces + 4 * ch.nchunks);
    while (c->pool.size() < need) {
        cudaEvent_t e;
        TSR_CUDA_TRY(cudaEventCreate(&e));
        c->pool.push_back(e);
    }
    // window device buffers: the widest window's pitched layout (same row
    // pitch as the whole grid: only the plane count differs)
    const int64_t last = (ch.r_hi - ch.r_lo + ch.nchunks - 1) / ch.nchunks;  // the widest chunk
    const int64_t wplanes = std::min(ch.n0, last + 2 * ch.margin);
    ch.win_elems = (wplanes + 2 * ch.h0) * g.pitch[ch.ax];
    ch.out_elems = last * ch.hplane;
    const int64_t bytes = 2 * (2 * ch.win_elems + 2 * ch.out_elems) * g.esize;
    if (c->pipe_bytes < bytes) {
        if (c->pipe) cudaFree(c->pipe);
        c->pipe = nullptr;
        c->pipe_bytes = 0;
        if (cudaMalloc(&c->pipe, bytes) != cudaSuccess) {
            cudaGetLastError();  // no room: the unchunked round trip
            return Status::Ok();
        }
        c->pipe_bytes = bytes;
    }
    return Status::Ok();
}

Status run_chunked_impl(const tsr_grid& gg, const Geo& g, const TapSet& t, const tsr_opts& o,
                        DeviceCache* c, void* const host[2], int parity, int64_t steps,
                        const Chunks& ch, tsr_stats* st, bool staged);

Status run_chunked(const tsr_grid& gg, const Geo& g, const TapSet& t, const tsr_opts& o,
                   DeviceCache* c, void* const host[2], int parity, int64_t steps,
                   const Chunks& ch, tsr_stats* st, bool staged) {
    Status r = run_chunked_impl(gg, g, t, o, c, host, parity, steps, ch, st, staged);
    if (!r.ok()) {
        // nothing queued may still write the caller's host buffers
        cudaStreamSynchronize(c->s_out);
        cudaStreamSynchronize(c->s_comp);
        cudaStreamSynchronize(c->stream);
    }
    return r;
}

// memcpy over up to 8 host threads (pageable <-> pinned staging: one thread
// copies ~10 GB/s, the driver's own pageable staging ~15 GB/s)
void par_memcpy(void* dst, const void* src, int64_t n) {
    const int nt = static_cast<int>(std::min<int64_t>(8, n / (4 << 20) + 1));
    if (nt == 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t part = (n / nt + 63) / 64 * 64;
    for (int i = 1; i < nt; ++i) {
        const int64_t o = i * part;
        if (o >= n) break;
        th.emplace_back([=] {
            std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                        std::min(part, n - o));
        });
    }
    std::memcpy(dst, src, std::min(part, n));
    for (auto& x : th) x.join();
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// pinned host staging of the staged (pageable) round trip: NIN upload slots
// of one piece, two sets of two download slots of the widest chunk
constexpr int kInSlots = 3;
Status host_stage_for(DeviceCache* c, int64_t bytes) {
    if (c->hstage_bytes >= bytes) return Status::Ok();
    if (c->hstage) cudaFreeHost(c->hstage);
    c->hstage = nullptr;
    c->hstage_bytes = 0;
    TSR_CUDA_TRY(cudaHostAlloc(&c->hstage, bytes, cudaHostAllocDefault));
    c->hstage_bytes = bytes;
    return Status::Ok();
}

// The chunk loop of the chunked round trip.  Pinned host buffers: the upload
// pieces are already queued (run_host) and every copy is a DMA straight
// to/from the caller's buffers.  Pageable host buffers (STAGED): this thread
// drives the pipeline — each piece is copied by host threads into a pinned
// slot and DMA'd up, windows are queued as soon as their pieces are up, and
// each finished chunk is DMA'd into a pinned slot and copied out by host
// threads while later pieces go up.
Status run_chunked_impl(const tsr_grid& gg, const Geo& g, const TapSet& t, const tsr_opts& o,
                        DeviceCache* c, void* const host[2], int parity, int64_t steps,
                        const Chunks& ch, tsr_stats* st, bool staged) {
    // the whole grid's plan (engine, fused depth) for every window
    Plan p;
    Status r = plan_for(g, t, o, p);
    if (!r.ok()) return r;
    tsr_opts wo = o;
    wo.fused_steps = p.k;
    const int64_t es = g.esize;
    cudaEvent_t* ev_in = c->pool.data();
    cudaEvent_t* ev_c0 = ev_in + ch.npieces;
    cudaEvent_t* ev_c1 = ev_c0 + ch.nchunks;
    cudaEvent_t* ev_rel = ev_c1 + ch.nchunks;
    cudaEvent_t* ev_out = ev_rel + ch.nchunks;
    const int pfinal = parity ^ static_cast<int>(steps & 1);
    const int nout = steps >= 2 ? 2 : 1;
    const int64_t hbytes = g.host_elements * es;
    const int64_t pb = ch.piece * ch.hplane * es;   // bytes per upload piece
    const int64_t ob = ch.out_elems * es;           // bytes per download slot
    char* in_slot[kInSlots] = {};
    char* out_slot[2][2] = {};
    if (staged) {
        r = host_stage_for(c, kInSlots * pb + 4 * ob);
        if (!r.ok()) return r;
        char* h = static_cast<char*>(c->hstage);
        for (int i = 0; i < kInSlots; ++i) in_slot[i] = h + i * pb;
        for (int s2 = 0; s2 < 2; ++s2)
            for (int q = 0; q < 2; ++q) out_slot[s2][q] = h + kInSlots * pb + (2 * s2 + q) * ob;
    }
    auto chunk_span = [&](int j, int64_t* a, int64_t* b) {
        const int64_t n = ch.r_hi - ch.r_lo;
        *a = ch.r_lo + j * n / ch.nchunks;
        *b = ch.r_lo + (j + 1) * n / ch.nchunks;
    };
    auto last_piece = [&](int j) {  // host planes [wa, wb + 2 h0) of window j
        int64_t a, b;
        chunk_span(j, &a, &b);
        const int64_t wb = std::min(ch.n0, b + ch.margin);
        return static_cast<int>((wb + 2 * ch.h0 - 1) / ch.piece);
    };
    tsr_stats local{};
    int64_t d2h = 0;
    // STAGED: a drainer thread copies each finished chunk out of its pinned
    // slots while this thread copies pieces in and queues windows; `queued`
    // (ev_out[j] recorded) and `drained` (slots of chunk j free) hand over.
    std::mutex mu;
    std::condition_variable cv;
    int queued = 0, drained = 0;
    bool stop = false;
    Status drain_err;
    int dev = 0;
    cudaGetDevice(&dev);
    auto drainer = [&] {
        cudaSetDevice(dev);
        for (int j = 0; j < ch.nchunks; ++j) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return queued > j || stop; });
                if (queued <= j) break;  // stopped
            }
            int64_t a, b;
            chunk_span(j, &a, &b);
            const cudaError_t e = cudaEventSynchronize(ev_out[j]);
            if (e == cudaSuccess) {
                const int64_t n = (b - a) * ch.hplane * es, dst = (a + ch.h0) * ch.hplane * es;
                for (int q = 0; q < nout; ++q)
                    par_memcpy(static_cast<char*>(host[q == 0 ? pfinal : 1 - pfinal]) + dst,
                               out_slot[j & 1][q], n);
            }
            std::lock_guard<std::mutex> lk(mu);
            if (e != cudaSuccess) {
                drain_err = Status::Err(TSR_ECUDA, cudaGetErrorString(e));
                drained = ch.nchunks;  // unblock the queueing thread
            } else {
                drained = j + 1;
            }
            cv.notify_all();
            if (e != cudaSuccess) break;
        }
    };
    auto queue_chunk = [&](int j) -> Status {
        char* set = static_cast<char*>(c->pipe) + (j & 1) * (2 * ch.win_elems + 2 * ch.out_elems) * es;
        void* wbuf[2] = {set, set + ch.win_elems * es};
        char* ostage[2] = {set + 2 * ch.win_elems * es, set + (2 * ch.win_elems + ch.out_elems) * es};
        int64_t a, b;
        chunk_span(j, &a, &b);
        const int64_t wa = std::max<int64_t>(0, a - ch.margin);
        const int64_t wb = std::min(ch.n0, b + ch.margin);
        Geo gw;
        Status q0 = make_geo(window_grid(gg, wb - wa), gw);
        if (!q0.ok()) return q0;
        // pieces go up in index order on one stream, so the event of the
        // window's last piece covers the ones before it; pieces that went up
        // before the margins barrier have arrived already
        int lp = last_piece(j);
        while (lp >= ch.piece_lo && ch.pre(lp)) --lp;
        if (lp >= ch.piece_lo) TSR_CUDA_TRY(cudaStreamWaitEvent(c->s_comp, ev_in[lp], 0));
        if (j >= 2) TSR_CUDA_TRY(cudaStreamWaitEvent(c->s_comp, ev_out[j - 2], 0));
        TSR_CUDA_TRY(cudaEventRecord(ev_c0[j], c->s_comp));
        q0 = relayout(gw, static_cast<const char*>(c->d[1]) + wa * ch.hplane * es, wbuf[0], true,
                      c->s_comp);
        if (!q0.ok()) return q0;
        q0 = halo_copy(gw, wbuf[0], wbuf[1], c->s_comp);
        if (!q0.ok()) return q0;
        int cur = 0;
        tsr_stats ws{};
        q0 = advance_grid(gw, t, wo, wbuf[0], wbuf[1], &cur, steps, true, c->s_comp, &ws);
        if (!q0.ok()) return q0;
        TSR_CUDA_TRY(cudaEventRecord(ev_c1[j], c->s_comp));
        if (j == 0) {
            local.rounds = ws.rounds;
            local.trailing_steps = ws.trailing_steps;
            local.fused_steps = ws.fused_steps;
            local.engine = ws.engine;
        }
        local.kernel_launches += ws.kernel_launches;
        // the window's planes beyond the chunk are swept and thrown away
        local.ghost_recompute_points += ((wb - wa) - (b - a)) * (g.interior() / ch.n0) * steps;
        // planes [a, b) of steps T and T-1 into host layout
        Geo go = gw;
        go.n[ch.ax] = b - a;
        go.h[ch.ax] = 0;
        const int64_t src_off = (a - wa + ch.h0) * gw.pitch[ch.ax] * es;
        for (int q = 0; q < nout; ++q) {
            q0 = relayout(go, static_cast<const char*>(wbuf[q == 0 ? cur : 1 - cur]) + src_off,
                          ostage[q], false, c->s_comp);
            if (!q0.ok()) return q0;
        }
        TSR_CUDA_TRY(cudaEventRecord(ev_rel[j], c->s_comp));
        TSR_CUDA_TRY(cudaStreamWaitEvent(c->s_out, ev_rel[j], 0));
        const int64_t n = (b - a) * ch.hplane * es, dst = (a + ch.h0) * ch.hplane * es;
        if (staged && j >= 2) {  // chunk j-2's pinned slots are this chunk's
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return drained >= j - 1; });
            if (!drain_err.ok()) return drain_err;
        }
        for (int q = 0; q < nout; ++q) {
            void* to = staged ? static_cast<void*>(out_slot[j & 1][q])
                              : static_cast<void*>(static_cast<char*>(
                                    host[q == 0 ? pfinal : 1 - pfinal]) + dst);
            TSR_CUDA_TRY(cudaMemcpyAsync(to, ostage[q], n, cudaMemcpyDeviceToHost, c->s_out));
            d2h += n;
        }
        TSR_CUDA_TRY(cudaEventRecord(ev_out[j], c->s_out));
        {
            std::lock_guard<std::mutex> lk(mu);
            queued = j + 1;
        }
        cv.notify_all();
        return Status::Ok();
    };
    if (!staged) {
        for (int j = 0; j < ch.nchunks; ++j) {
            r = queue_chunk(j);
            if (!r.ok()) return r;
        }
    } else {
        std::thread th(drainer);
        int slot_owner[kInSlots];
        for (int& x : slot_owner) x = -1;
        auto upload_and_queue = [&]() -> Status {
            for (int i = ch.piece_lo; i <= ch.piece_hi; ++i) {
                if (ch.pre(i)) {  // uploaded before the margins barrier
                    while (queued < ch.nchunks && last_piece(queued) <= i) {
                        Status q = queue_chunk(queued);
                        if (!q.ok()) return q;
                    }
                    continue;
                }
                // a slot is free once the piece last copied through it is up
                const int si = (i - ch.piece_lo) % kInSlots;
                if (slot_owner[si] >= 0) TSR_CUDA_TRY(cudaEventSynchronize(ev_in[slot_owner[si]]));
                slot_owner[si] = i;
                const int64_t off = i * pb, n = std::min(pb, hbytes - off);
                char* sl = in_slot[si];
                par_memcpy(sl, static_cast<const char*>(host[parity]) + off, n);
                TSR_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(c->d[1]) + off, sl, n,
                                             cudaMemcpyHostToDevice, c->stream));
                TSR_CUDA_TRY(cudaEventRecord(ev_in[i], c->stream));
                while (queued < ch.nchunks && last_piece(queued) <= i) {
                    Status q = queue_chunk(queued);
                    if (!q.ok()) return q;
                }
            }
            while (queued < ch.nchunks) {
                Status q = queue_chunk(queued);
                if (!q.ok()) return q;
            }
            return Status::Ok();
        };
        r = upload_and_queue();
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;  // the drainer finishes the chunks queued so far
        }
        cv.notify_all();
        th.join();
        if (!r.ok()) return r;
        if (!drain_err.ok()) return drain_err;
    }
    const auto t_enq = std::chrono::steady_clock::now();
    TSR_CUDA_TRY(cudaStreamSynchronize(c->s_out));
    TSR_CUDA_TRY(cudaStreamSynchronize(c->s_comp));
    TSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const double wait_ms = std::chrono::duration<double, std::milli>(
                               std::chrono::steady_clock::now() - t_enq).count();
    double ms = 0;
    for (int j = 0; j < ch.nchunks; ++j) {
        float m = 0.f;
        TSR_CUDA_TRY(cudaEventElapsedTime(&m, ev_c0[j], ev_c1[j]));
        ms += m;
    }
    if (const char* tr = std::getenv("TSR_CHUNK_TRACE"); tr && *tr == '1') {
        // per-window timeline (ms from the first upload piece's completion)
        for (int j = 0; j < ch.nchunks; ++j) {
            float tt[4] = {0, 0, 0, 0};
            cudaEventElapsedTime(&tt[0], ev_in[ch.piece_lo], ev_c0[j]);
            cudaEventElapsedTime(&tt[1], ev_in[ch.piece_lo], ev_c1[j]);
            cudaEventElapsedTime(&tt[2], ev_in[ch.piece_lo], ev_rel[j]);
            cudaEventElapsedTime(&tt[3], ev_in[ch.piece_lo], ev_out[j]);
            std::fprintf(stderr, "chunk %d: start %.2f swept %.2f relaid %.2f downloaded %.2f\n", j,
                         tt[0], tt[1], tt[2], tt[3]);
        }
        float tl = 0;
        cudaEventElapsedTime(&tl, ev_in[ch.piece_lo], ev_in[ch.piece_hi]);
        std::fprintf(stderr, "pieces %d, last piece uploaded %.2f; host waited %.2f ms (staged=%d)\n",
                     ch.npieces, tl, wait_ms, int(staged));
    }
    local.point_updates = g.interior() / ch.n0 * (ch.r_hi - ch.r_lo) * steps;
    local.device_ms = ms;
    local.h2d_bytes = std::min(hbytes, (int64_t(ch.piece_hi) + 1) * pb) - int64_t(ch.piece_lo) * pb;
    local.d2h_bytes = d2h;
    if (st) *st = local;
    return Status::Ok();
}

// With a plane range [r_lo, r_hi) of the outermost axis (r_hi >= 0), only
// those planes of the two buffers are computed and returned, through the
// chunked round trip (TSR_EUNSUPPORTED when it does not apply); the windows
// read the planes they need beyond the range from the host buffers.
Status run_host(const tsr_kernel* kk, const tsr_grid* gg, void* b0, void* b1, int parity,
                int64_t steps, const tsr_opts* oo, tsr_stats* st, int64_t r_lo = 0,
                int64_t r_hi = -1, const std::function<void()>* after_margins = nullptr,
                int cache_sub = 0) {
    if (!kk || !gg || !b0 || !b1) return Status::Err(TSR_EINVAL, "null argument");
    if (parity != 0 && parity != 1) return Status::Err(TSR_EINVAL, "parity must be 0 or 1");
    if (steps < 0) return Status::Err(TSR_EINVAL, "negative step count");
    Geo g;
    Status r = make_geo(*gg, g);
    if (!r.ok()) return r;
    TapSet t;
    r = make_taps(*kk, t);
    if (!r.ok()) return r;
    r = check_applicable(g, t);
    if (!r.ok()) return r;
    const tsr_opts o = opts_or_default(oo);
    if (st) *st = tsr_stats{};
    if (steps == 0) return Status::Ok();
    DeviceGuard guard;
    r = guard.enter(o.device);
    if (!r.ok()) return r;
    int dev = 0;
    TSR_CUDA_TRY(cudaGetDevice(&dev));
    DeviceCache* slot = cache_slot(dev, cache_sub);
    std::lock_guard<std::mutex> lock(slot->mu);
    DeviceCache* c = nullptr;
    r = cache_for(slot, g.elements * g.esize, &c);
    if (!r.ok()) return r;
    void* host[2] = {b0, b1};
    // PCIe moves one contiguous block per buffer; the pitched device layout
    // is produced / undone on the device (relayout, ~0.3 ms per GB), which
    // is 1.4x faster than pitched 3-D copies of 4 KB rows.
    const int64_t hbytes = g.host_elements * g.esize;
    const bool staged_up = c->bytes >= hbytes;  // d[1] can hold the host layout
    Chunks ch;
    const int64_t n_all = g.n[3 - g.dims];
    const bool partial = r_hi >= 0 && !(r_lo == 0 && r_hi == n_all);
    if (r_hi < 0) r_hi = n_all;
    if (r_lo < 0 || r_hi > n_all || r_lo >= r_hi)
        return Status::Err(TSR_EINVAL, "plane range outside the grid");
    bool chunked = staged_up && plan_chunks(g, t, steps, r_lo, r_hi, &ch);
    if (chunked) {
        r = chunk_resources(g, ch, c);
        if (!r.ok()) return r;
        chunked = c->pipe != nullptr;
    }
    if (partial && !chunked)
        return Status::Err(TSR_EUNSUPPORTED, "plane range without the chunked round trip");
    if (chunked && after_margins) {
        // Split round trip: every other device writes its planes of steps T
        // and T-1 back into these host buffers, the read buffer included, so
        // the planes this range's windows read beyond it go up (and arrive)
        // before any device downloads; then the pipeline as usual.
        ch.margins_first = true;
        const int64_t pb = ch.piece * ch.hplane * g.esize;
        for (int i = ch.piece_lo; i <= ch.piece_hi; ++i) {
            if (!ch.pre(i)) continue;
            const int64_t off = i * pb, n = std::min(pb, hbytes - off);
            TSR_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(c->d[1]) + off,
                                         static_cast<const char*>(host[parity]) + off, n,
                                         cudaMemcpyHostToDevice, c->stream));
            TSR_CUDA_TRY(cudaEventRecord(c->pool[i], c->stream));
        }
        TSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
        (*after_margins)();
    }
    // Pageable caller buffers: the chunked round trip stages its copies
    // through pinned slots itself (run_chunked_impl) after the halo check.
    const bool staged = chunked && !(is_pinned(b0) && is_pinned(b1));
    if (chunked && !staged) {
        // the read buffer goes up in pieces, an event after each, so window
        // j computes as soon as the planes it reads have arrived
        const int64_t pb = ch.piece * ch.hplane * g.esize;
        for (int i = ch.piece_lo; i <= ch.piece_hi; ++i) {
            if (ch.pre(i)) continue;  // already up
            const int64_t off = i * pb, n = std::min(pb, hbytes - off);
            TSR_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(c->d[1]) + off,
                                         static_cast<const char*>(host[parity]) + off, n,
                                         cudaMemcpyHostToDevice, c->stream));
            TSR_CUDA_TRY(cudaEventRecord(c->pool[i], c->stream));
        }
    } else if (staged) {
        // uploaded piece by piece in run_chunked_impl
    } else if (staged_up) {
        TSR_CUDA_TRY(cudaMemcpyAsync(c->d[1], host[parity], hbytes, cudaMemcpyHostToDevice,
                                     c->stream));
    } else {
        r = upload(g, host[parity], c->d[0], c->stream);
        if (!r.ok()) return r;
    }
    // The host-side halo comparison (it touches every page of both buffers:
    // ~10-20 ms at 512^3) runs while the upload is in flight.
    const auto t_enq = std::chrono::steady_clock::now();
    const bool same_halo = halos_equal(g, b0, b1);
    if (const char* tr = std::getenv("TSR_CHUNK_TRACE"); tr && *tr == '1')
        std::fprintf(stderr, "run_host: chunked=%d halo check %.2f ms\n", int(chunked),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                               t_enq).count());
    if (chunked && same_halo)
        return run_chunked(*gg, g, t, o, c, host, parity, steps, ch, st, staged);
    if (partial) {
        cudaStreamSynchronize(c->stream);
        return Status::Err(TSR_EUNSUPPORTED, "plane range with differing halos");
    }
    if (staged) {  // differing halos: the whole read buffer after all
        TSR_CUDA_TRY(cudaMemcpyAsync(c->d[1], host[parity], hbytes, cudaMemcpyHostToDevice,
                                     c->stream));
    }
    if (staged_up) {
        r = relayout(g, c->d[1], c->d[0], true, c->stream);
        if (!r.ok()) return r;
    }
    int64_t h2d = hbytes;
    tsr_opts run_o = o;
    if (same_halo) {
        // one upload + a device-side halo copy is exact
        r = halo_copy(g, c->d[0], c->d[1], c->stream);
    } else {
        // naive_run (naive.hpp:96-100) reads every step's halo from that
        // step's read buffer: with two different halos the write buffer is
        // uploaded too (its halo is what the odd steps read) and every step
        // is its own sweep, which reads the halo of its input buffer.
        r = upload(g, host[1 - parity], c->d[1], c->stream);
        h2d += hbytes;
        run_o.fused_steps = 1;
    }
    if (!r.ok()) return r;
    int cur = 0;
    tsr_stats local{};
    TSR_CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
    r = advance_grid(g, t, run_o, c->d[0], c->d[1], &cur, steps, true, c->stream, &local);
    if (!r.ok()) return r;
    TSR_CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
    const int pfinal = parity ^ static_cast<int>(steps & 1);
    if (c->stage_bytes < hbytes) {
        if (c->stage) cudaFree(c->stage);
        c->stage = nullptr;
        c->stage_bytes = 0;
        if (cudaMalloc(&c->stage, hbytes) == cudaSuccess)
            c->stage_bytes = hbytes;
        else
            cudaGetLastError();  // no room: pitched copies below
    }
    // The staged path copies the whole host layout back: each device
    // buffer's halo cells are its own host buffer's (uploaded, or copied
    // from the other buffer when the two halos are equal), so the host halo
    // is rewritten with its own bytes.
    auto fetch = [&](int which, int into, int64_t* bytes) -> Status {
        if (c->stage) {
            Status q = relayout(g, c->d[which], c->stage, false, c->stream);
            if (!q.ok()) return q;
            TSR_CUDA_TRY(cudaMemcpyAsync(host[into], c->stage, hbytes, cudaMemcpyDeviceToHost,
                                         c->stream));
            *bytes += hbytes;
            return Status::Ok();
        }
        *bytes += g.interior() * g.esize;
        return download(g, c->d[which], host[into], true, c->stream);
    };
    int64_t d2h = 0;
    r = fetch(cur, pfinal, &d2h);
    if (!r.ok()) return r;
    if (steps >= 2) {
        r = fetch(1 - cur, 1 - pfinal, &d2h);
        if (!r.ok()) return r;
    }
    TSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    TSR_CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
    local.device_ms = ms;
    local.h2d_bytes = h2d;
    local.d2h_bytes = d2h;
    if (st) *st = local;
    return Status::Ok();
}

}  // namespace

Status run_host_single(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int parity,
                       int64_t steps, const tsr_opts* o, tsr_stats* st) {
    return run_host(k, g, b0, b1, parity, steps, o, st);
}

bool range_chunkable(const Geo& g, const TapSet& t, int64_t steps, int64_t r_lo, int64_t r_hi) {
    Chunks ch;
    return plan_chunks(g, t, steps, r_lo, r_hi, &ch);
}

Status run_host_range(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int parity,
                      int64_t steps, const tsr_opts* o, tsr_stats* st, int64_t r_lo,
                      int64_t r_hi, const std::function<void()>& after_margins, int cache_sub) {
    return run_host(k, g, b0, b1, parity, steps, o, st, r_lo, r_hi, &after_margins, cache_sub);
}

// Frees what tsr_run caches per device (tsr_release_cache).
void release_run_cache() {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    int prev = 0;
    cudaGetDevice(&prev);
    for (size_t dev = 0; dev < g_cache.size(); ++dev) {
        if (!g_cache[dev]) continue;
        DeviceCache& c = *g_cache[dev];
        std::lock_guard<std::mutex> held(c.mu);
        if (!c.stream && !c.stage && !c.d[0]) continue;
        cudaSetDevice(c.device);
        for (void*& p : c.d)
            if (p) {
                cudaFree(p);
                p = nullptr;
            }
        c.bytes = 0;
        if (c.stage) cudaFree(c.stage);
        c.stage = nullptr;
        c.stage_bytes = 0;
        for (cudaEvent_t& e : c.ev)
            if (e) cudaEventDestroy(e), e = nullptr;
        if (c.stream) cudaStreamDestroy(c.stream), c.stream = nullptr;
        if (c.pipe) cudaFree(c.pipe);
        c.pipe = nullptr;
        c.pipe_bytes = 0;
        if (c.hstage) cudaFreeHost(c.hstage);
        c.hstage = nullptr;
        c.hstage_bytes = 0;
        for (cudaEvent_t e : c.pool) cudaEventDestroy(e);
        c.pool.clear();
        if (c.s_comp) cudaStreamDestroy(c.s_comp), c.s_comp = nullptr;
        if (c.s_out) cudaStreamDestroy(c.s_out), c.s_out = nullptr;
    }
    cudaSetDevice(prev);
}

}  // namespace tsr
