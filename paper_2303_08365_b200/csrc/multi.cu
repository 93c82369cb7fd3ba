// multi.cu — memory-level tetrominoes: one host thread driving a slab
// decomposition of axis 0 over the GPUs of one box (tsr_multi_* and
// tsr_run_multi in include/tessera_b200.h).
//
// The reference's run_heterogeneous (proj/src/scheduler.cpp:441-563) splits
// axis 0 between two workers, each holding its rows plus a ghost slab of
// r*tb rows, and per tb-step round sends one slab per direction through a
// mutex-guarded SlabChannel (:142-194), computes the interior of step 0
// while the message is in flight, installs it, finishes the seam, then runs
// the remaining steps on a shrinking range (HaloWorker::run_round,
// :371-406).  Here:
//   * P slabs (one per GPU; several may share a device for tests), each
//     with r*k ghost planes per seam, k = the engine's fused step count;
//   * a round is ONE fused pass per range: the seam passes compute the r*k
//     boundary planes and store every output row both locally and into the
//     neighbour's next-buffer ghost planes through peer memory (NVLink), so
//     the "message" is the kernel's own store stream (TSR_XPORT_MIRROR); the
//     interior pass runs concurrently on a second stream and never waits;
//   * ordering is by CUDA events, no host round trip: a slab's seam pass of
//     round n waits for its neighbours' seam passes of round n-1 (which both
//     filled its ghosts and finished reading the planes it overwrites) and
//     for its own interior pass of round n-1; its interior pass of round n
//     waits for its own seam pass of round n-1.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <random>
#include <string>
#include <vector>

#include "runtime.cuh"

namespace tsr {
namespace {

struct Slab {
    int device = 0;
    int64_t own_lo = 0, own_hi = 0;      // owned global interior planes
    int64_t ghost_lo = 0, ghost_hi = 0;  // ghost planes below / above
    int64_t plane0 = 0;                  // global padded plane of local padded plane 0
    tsr_grid desc{};
    Geo geo;
    void* d[2] = {nullptr, nullptr};
    void* stage = nullptr;  // local grid in the host layout (staged copies)
    cudaStream_t s_seam = nullptr, s_int = nullptr;
    cudaEvent_t ev_seam[2] = {nullptr, nullptr};
    cudaEvent_t ev_int = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    int nb[2] = {-1, -1};          // lo / hi neighbour slab
    int64_t shift[2] = {0, 0};     // plane shift of my seam rows in the neighbour
    int64_t own() const { return own_hi - own_lo; }
};

struct LogEntry {
    int64_t round;
    int slab;
    cudaEvent_t a, b;  // seam passes (seam stream)
    cudaEvent_t c, d;  // interior pass (second stream)
};

}  // namespace
}  // namespace tsr

struct tsr_multi {
    tsr::Geo g;  // global geometry
    tsr::TapSet taps;
    tsr_opts opts{};
    tsr::Plan plan;
    int axis = 0;        // normalised slab axis (3 - dims)
    int64_t depth = 0;   // ghost planes per seam: r * k
    int64_t cross = 1;   // interior cells per plane
    int transport = TSR_XPORT_MIRROR;
    std::vector<tsr::Slab> s;
    int cur = 0;
    bool prev_valid = false;
    int64_t round = 0;
    bool logging = false;
    std::vector<tsr::LogEntry> log;
    bool poison = false;  // TSR_PART_POISON
    // cache key (tsr_run_multi)
    std::vector<int32_t> key_devices;
    std::vector<int64_t> key_bounds;
    int key_transport = 0;
    int key_flags = 0;
};

namespace tsr {
namespace {

using Multi = tsr_multi;

// Element offset and length of local interior plane p (slab axis) in the
// pitched device layout: whole padded planes for 2-D/3-D grids (axis-0
// planes / axis-0 rows are contiguous), single elements for 1-D.
int64_t plane_start(const Geo& g, int axis, int64_t p) {
    return axis == 2 ? g.off2 + p : (p + g.h[axis]) * g.pitch[axis];
}

Status each_device(Multi& m, const std::function<Status(Slab&)>& f) {
    for (Slab& sl : m.s) {
        TSR_CUDA_TRY(cudaSetDevice(sl.device));
        Status r = f(sl);
        if (!r.ok()) return r;
    }
    return Status::Ok();
}

Status sync_all(Multi& m) {
    return each_device(m, [](Slab& sl) -> Status {
        TSR_CUDA_TRY(cudaStreamSynchronize(sl.s_seam));
        TSR_CUDA_TRY(cudaStreamSynchronize(sl.s_int));
        return Status::Ok();
    });
}

void free_slab(Slab& sl) {
    cudaSetDevice(sl.device);
    for (void*& p : sl.d)
        if (p) cudaFree(p), p = nullptr;
    if (sl.stage) cudaFree(sl.stage), sl.stage = nullptr;
    for (cudaEvent_t* e : {&sl.ev_seam[0], &sl.ev_seam[1], &sl.ev_int, &sl.ev_t0, &sl.ev_t1})
        if (*e) cudaEventDestroy(*e), *e = nullptr;
    for (cudaStream_t* st : {&sl.s_seam, &sl.s_int})
        if (*st) cudaStreamDestroy(*st), *st = nullptr;
}

void drop_log(Multi& m) {
    int prev = 0;
    cudaGetDevice(&prev);
    for (LogEntry& e : m.log) {
        cudaSetDevice(m.s[e.slab].device);
        for (cudaEvent_t ev : {e.a, e.b, e.c, e.d})
            if (ev) cudaEventDestroy(ev);
    }
    m.log.clear();
    cudaSetDevice(prev);
}

void destroy(Multi* m) {
    if (!m) return;
    int prev = 0;
    cudaGetDevice(&prev);
    drop_log(*m);
    for (Slab& sl : m->s) free_slab(sl);
    cudaSetDevice(prev);
    delete m;
}

Status create(const tsr_kernel* kk, const tsr_grid* gg, const tsr_partition* part,
              const tsr_opts* oo, Multi** out) {
    if (!kk || !gg || !out) return Status::Err(TSR_EINVAL, "null argument");
    auto m = std::make_unique<Multi>();
    Status r = make_geo(*gg, m->g);
    if (!r.ok()) return r;
    r = make_taps(*kk, m->taps);
    if (!r.ok()) return r;
    r = check_applicable(m->g, m->taps);
    if (!r.ok()) return r;
    m->opts = opts_or_default(oo);
    const int P = part ? part->ngpus : std::max(1, m->opts.ngpus);
    const int split = part ? part->split_axis : m->opts.split_axis;
    if (P < 1) return Status::Err(TSR_EINVAL, "ngpus must be >= 1");
    if (split != 0)
        return Status::Err(TSR_EUNSUPPORTED, "only split_axis 0 is supported (PartitionPlan)");
    m->axis = 3 - m->g.dims;
    const int a = m->axis;
    const int64_t n = m->g.n[a];
    for (int b = a + 1; b < 3; ++b) m->cross *= m->g.n[b];

    // slab boundaries: equal split (the first n % P slabs one plane larger)
    // or the caller's (PartitionPlan::boundary for two workers)
    std::vector<int64_t> lo(P), hi(P);
    if (part && part->boundaries && P > 1) {
        for (int i = 0; i < P; ++i) {
            lo[i] = i == 0 ? 0 : part->boundaries[i - 1];
            hi[i] = i == P - 1 ? n : part->boundaries[i];
            if (lo[i] >= hi[i] || lo[i] < 0 || hi[i] > n)
                return Status::Err(TSR_EINVAL, "partition boundary outside the grid");
        }
    } else {
        const int64_t base = n / P, extra = n % P;
        for (int i = 0; i < P; ++i) {
            lo[i] = i * base + std::min<int64_t>(i, extra);
            hi[i] = lo[i] + base + (i < extra ? 1 : 0);
            if (hi[i] <= lo[i])
                return Status::Err(TSR_EINVAL, "more slabs than planes along the split axis");
        }
    }

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return Status::Err(TSR_ECUDA, "no CUDA device available to the B200 sweep engine");
    }

    // Engine plan: the fused depth k is fixed before the ghost depth (r*k)
    // and the local extents follow from it; every slab must accept the same k.
    Plan p;
    r = plan_for(m->g, m->taps, m->opts, p);
    if (!r.ok()) return r;
    int k = p.k;
    for (;;) {
        const int64_t depth = int64_t(m->taps.radius) * k;
        int kmin = k;
        m->s.assign(P, Slab{});
        for (int i = 0; i < P; ++i) {
            Slab& sl = m->s[i];
            sl.own_lo = lo[i];
            sl.own_hi = hi[i];
            if (P > 1 && sl.own() < depth)
                return Status::Err(TSR_EINVAL, "subdomain smaller than the halo depth");
            sl.ghost_lo = i > 0 ? depth : 0;
            sl.ghost_hi = i < P - 1 ? depth : 0;
            sl.plane0 = sl.own_lo - sl.ghost_lo;
            sl.desc = *gg;
            sl.desc.extent[0] = sl.ghost_lo + sl.own() + sl.ghost_hi;
            r = make_geo(sl.desc, sl.geo);
            if (!r.ok()) return r;
            tsr_opts o = m->opts;
            o.fused_steps = k;
            Plan q;
            r = plan_for(sl.geo, m->taps, o, q);
            if (!r.ok()) return r;
            if (q.engine != p.engine)
                return Status::Err(TSR_EUNSUPPORTED, "slabs would run different engines");
            kmin = std::min(kmin, q.k);
        }
        if (kmin == k) break;
        k = kmin;  // re-plan with the smaller depth (k strictly decreases)
    }
    m->plan = p;
    m->plan.k = k;
    m->depth = int64_t(m->taps.radius) * k;

    for (int i = 0; i < P; ++i) {
        Slab& sl = m->s[i];
        sl.device = part && part->devices ? part->devices[i] : i % ndev;
        if (sl.device < 0 || sl.device >= ndev)
            return Status::Err(TSR_EINVAL, "device ordinal out of range");
        sl.nb[0] = i > 0 ? i - 1 : -1;
        sl.nb[1] = i < P - 1 ? i + 1 : -1;
    }
    for (int i = 0; i < P; ++i) {
        Slab& sl = m->s[i];
        // my boundary own plane at local row j lands on the neighbour's ghost
        // plane j + shift (its ghost_hi planes for the lo side, its ghost_lo
        // planes for the hi side)
        if (sl.nb[0] >= 0) {
            const Slab& nb = m->s[sl.nb[0]];
            sl.shift[0] = (nb.ghost_lo + nb.own()) - sl.ghost_lo;
        }
        if (sl.nb[1] >= 0) sl.shift[1] = -(sl.ghost_lo + sl.own() - m->depth);
    }

    // transport: peer stores need peer access between every neighbour pair
    // on different devices
    const int want = part ? part->transport : TSR_XPORT_AUTO;
    if (want < TSR_XPORT_AUTO || want > TSR_XPORT_COPY)
        return Status::Err(TSR_EINVAL, "unknown transport");
    bool peer_ok = true;
    for (const Slab& sl : m->s)
        for (int side = 0; side < 2; ++side) {
            if (sl.nb[side] < 0) continue;
            const int od = m->s[sl.nb[side]].device;
            if (od == sl.device) continue;
            int can = 0;
            TSR_CUDA_TRY(cudaDeviceCanAccessPeer(&can, sl.device, od));
            peer_ok &= can != 0;
        }
    if (want == TSR_XPORT_MIRROR && !peer_ok)
        return Status::Err(TSR_EUNSUPPORTED, "peer access between neighbour GPUs unavailable");
    m->poison = part && (part->flags & TSR_PART_POISON);
    m->transport = want == TSR_XPORT_COPY ? TSR_XPORT_COPY
                   : peer_ok              ? TSR_XPORT_MIRROR
                                          : TSR_XPORT_COPY;

    Multi* raw = m.release();
    auto fail = [&](Status s) {
        destroy(raw);
        return s;
    };
    for (Slab& sl : raw->s) {
        if (cudaSetDevice(sl.device) != cudaSuccess) {
            cudaGetLastError();
            return fail(Status::Err(TSR_ECUDA, "cudaSetDevice failed"));
        }
        if (raw->transport == TSR_XPORT_MIRROR)
            for (int side = 0; side < 2; ++side) {
                if (sl.nb[side] < 0) continue;
                const int od = raw->s[sl.nb[side]].device;
                if (od == sl.device) continue;
                const cudaError_t e = cudaDeviceEnablePeerAccess(od, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) {
                    cudaGetLastError();
                } else if (e != cudaSuccess) {
                    cudaGetLastError();
                    return fail(Status::Err(TSR_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") +
                                                           cudaGetErrorString(e)));
                }
            }
        const int64_t bytes = sl.geo.elements * sl.geo.esize;
        const int64_t sbytes = sl.geo.host_elements * sl.geo.esize;
        for (void** ptr : {&sl.d[0], &sl.d[1], &sl.stage}) {
            if (cudaMalloc(ptr, ptr == &sl.stage ? sbytes : bytes) != cudaSuccess) {
                cudaGetLastError();
                return fail(Status::Err(TSR_ENOMEM, "device allocation failed for a slab"));
            }
        }
        bool ok = cudaStreamCreateWithFlags(&sl.s_seam, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&sl.s_int, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaEventCreateWithFlags(&sl.ev_seam[0], cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&sl.ev_seam[1], cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreateWithFlags(&sl.ev_int, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventCreate(&sl.ev_t0) == cudaSuccess &&
                  cudaEventCreate(&sl.ev_t1) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            return fail(Status::Err(TSR_ECUDA, "stream/event creation failed"));
        }
    }
    *out = raw;
    return Status::Ok();
}

// ---- data in / out -------------------------------------------------------

Status finish_upload(Multi& m) {
    Status r = each_device(m, [&](Slab& sl) -> Status {
        Status q = relayout(sl.geo, sl.stage, sl.d[0], true, sl.s_int);
        if (!q.ok()) return q;
        q = halo_copy(sl.geo, sl.d[0], sl.d[1], sl.s_int);
        if (!q.ok() || !m.poison) return q;
        // all-ones bytes are a NaN in fp64 and fp32
        const int a = m.axis;
        const int64_t h = sl.geo.h[a], plen = a == 2 ? 1 : sl.geo.pitch[a];
        for (int side = 0; side < 2; ++side) {
            if (sl.nb[side] < 0 || h == 0) continue;
            const int64_t p0 = side == 0 ? -h : sl.geo.n[a];
            for (void* d : sl.d)
                TSR_CUDA_TRY(cudaMemsetAsync(
                    static_cast<char*>(d) + plane_start(sl.geo, a, p0) * sl.geo.esize, 0xFF,
                    h * plen * sl.geo.esize, sl.s_int));
        }
        return Status::Ok();
    });
    if (!r.ok()) return r;
    r = sync_all(m);
    m.cur = 0;
    m.prev_valid = false;
    return r;
}

Status upload_host(Multi& m, const void* host) {
    const int64_t plane = m.g.hpitch[m.axis] * m.g.esize;
    Status r = each_device(m, [&](Slab& sl) -> Status {
        const char* src = static_cast<const char*>(host) + sl.plane0 * plane;
        TSR_CUDA_TRY(cudaMemcpyAsync(sl.stage, src, sl.geo.host_elements * sl.geo.esize,
                                     cudaMemcpyHostToDevice, sl.s_int));
        return Status::Ok();
    });
    if (!r.ok()) return r;
    return finish_upload(m);
}

// fill_random of the global grid streamed into the slabs: global padded
// planes are generated in order (the reference's i -> j -> k draw order,
// random.hpp:20-24) into a pinned chunk and copied to every slab whose
// local range (ghosts and halo planes included) covers them.
template <typename T>
Status fill_stream(Multi& m, uint64_t seed, double lo, double hi) {
    const Geo& g = m.g;
    const int a = m.axis;
    const int64_t plane_el = g.hpitch[a];
    const int64_t nplanes = g.n[a] + 2 * g.h[a];
    const int64_t chunk =
        std::max<int64_t>(1, std::min<int64_t>(nplanes, (128ll << 20) / (plane_el * sizeof(T))));
    T* buf[2] = {nullptr, nullptr};
    for (T*& b : buf)
        if (cudaMallocHost(&b, chunk * plane_el * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            for (T* q : buf)
                if (q) cudaFreeHost(q);
            return Status::Err(TSR_ENOMEM, "pinned staging allocation failed");
        }
    std::vector<cudaEvent_t> done(2 * m.s.size(), nullptr);
    Status r = Status::Ok();
    for (size_t i = 0; i < m.s.size() && r.ok(); ++i) {
        cudaSetDevice(m.s[i].device);
        for (int b = 0; b < 2; ++b)
            if (cudaEventCreateWithFlags(&done[2 * i + b], cudaEventDisableTiming) != cudaSuccess)
                r = Status::Err(TSR_ECUDA, "event creation failed");
    }
    std::mt19937_64 rng(seed);
    int64_t issued = 0;
    for (int64_t q0 = 0; q0 < nplanes && r.ok(); q0 += chunk, ++issued) {
        const int64_t q1 = std::min(nplanes, q0 + chunk);
        const int b = issued & 1;
        for (size_t i = 0; i < m.s.size(); ++i)  // copies out of this buffer are done
            if (issued >= 2) cudaEventSynchronize(done[2 * i + b]);
        T* pb = buf[b];
        std::memset(pb, 0, (q1 - q0) * plane_el * sizeof(T));
        for (int64_t q = q0; q < q1; ++q) {
            const int64_t p = q - g.h[a];
            if (p < 0 || p >= g.n[a]) continue;  // halo plane: zero
            T* row0 = pb + (q - q0) * plane_el;
            const int64_t nj = a == 0 ? g.n[1] : 1, nk = a <= 1 ? g.n[2] : 1;
            for (int64_t j = 0; j < nj; ++j) {
                T* row = row0 + (a == 0 ? (j + g.h[1]) * g.hpitch[1] : 0) + (a <= 1 ? g.h[2] : 0);
                for (int64_t kk = 0; kk < nk; ++kk) {
                    const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
                    row[kk] = static_cast<T>(lo + (hi - lo) * u);
                }
            }
        }
        for (size_t i = 0; i < m.s.size() && r.ok(); ++i) {
            Slab& sl = m.s[i];
            const int64_t s0 = std::max(q0, sl.plane0);
            const int64_t s1 = std::min(q1, sl.plane0 + sl.geo.n[a] + 2 * sl.geo.h[a]);
            cudaSetDevice(sl.device);
            if (s1 > s0 &&
                cudaMemcpyAsync(static_cast<T*>(sl.stage) + (s0 - sl.plane0) * plane_el,
                                pb + (s0 - q0) * plane_el, (s1 - s0) * plane_el * sizeof(T),
                                cudaMemcpyHostToDevice, sl.s_int) != cudaSuccess)
                r = Status::Err(TSR_ECUDA, "staging copy failed");
            cudaEventRecord(done[2 * i + b], sl.s_int);
        }
    }
    for (size_t i = 0; i < m.s.size(); ++i) {
        cudaSetDevice(m.s[i].device);
        cudaStreamSynchronize(m.s[i].s_int);
        for (int b = 0; b < 2; ++b)
            if (done[2 * i + b]) cudaEventDestroy(done[2 * i + b]);
    }
    for (T* q : buf) cudaFreeHost(q);
    if (!r.ok()) return r;
    return finish_upload(m);
}

// Owned planes of device buffer `which` -> the global host buffer.  Whole
// padded planes through the staging buffer (contiguous over PCIe) when
// `whole_planes`, else interior cells only (pitched copy).
Status fetch_slab(Multi& m, Slab& sl, int which, void* host, bool whole_planes) {
    const Geo& lg = sl.geo;
    const int a = m.axis;
    char* base = static_cast<char*>(host);
    if (whole_planes) {
        Status q = relayout(lg, sl.d[which], sl.stage, false, sl.s_int);
        if (!q.ok()) return q;
        const int64_t plane = lg.hpitch[a] * lg.esize;
        const int64_t lplane = lg.h[a] + sl.ghost_lo;  // local padded plane of own_lo
        const int64_t src_off = a == 2 ? (lg.h[2] + sl.ghost_lo) * lg.esize : lplane * plane;
        const int64_t dst_off = a == 2 ? (m.g.h[2] + sl.own_lo) * lg.esize
                                       : (m.g.h[a] + sl.own_lo) * plane;
        const int64_t bytes = sl.own() * (a == 2 ? lg.esize : plane);
        TSR_CUDA_TRY(cudaMemcpyAsync(base + dst_off, static_cast<char*>(sl.stage) + src_off, bytes,
                                     cudaMemcpyDeviceToHost, sl.s_int));
        return Status::Ok();
    }
    // interior cells of the owned planes: a 3-D copy (w = a2 interior, h =
    // a1 interior rows, d = planes), axes normalised like the grids
    int64_t ext[3] = {lg.n[0], lg.n[1], lg.n[2]};
    int64_t dpos[3] = {lg.h[0], lg.h[1], 0}, hpos[3] = {m.g.h[0], m.g.h[1], m.g.h[2]};
    ext[a] = sl.own();
    dpos[a] += a == 2 ? 0 : sl.ghost_lo;
    hpos[a] += sl.own_lo;
    cudaMemcpy3DParms p{};
    const int64_t rows_d = lg.n[1] + 2 * lg.h[1], rows_h = m.g.n[1] + 2 * m.g.h[1];
    p.srcPtr = make_cudaPitchedPtr(sl.d[which], lg.pitch[1] * lg.esize, lg.pitch[1] * lg.esize,
                                   rows_d);
    p.dstPtr = make_cudaPitchedPtr(host, m.g.hpitch[1] * lg.esize, m.g.hpitch[1] * lg.esize, rows_h);
    p.srcPos = make_cudaPos((lg.off2 + (a == 2 ? sl.ghost_lo : 0)) * lg.esize, dpos[1], dpos[0]);
    p.dstPos = make_cudaPos(hpos[2] * lg.esize, hpos[1], hpos[0]);
    p.extent = make_cudaExtent(ext[2] * lg.esize, ext[1], ext[0]);
    p.kind = cudaMemcpyDeviceToHost;
    TSR_CUDA_TRY(cudaMemcpy3DAsync(&p, sl.s_int));
    return Status::Ok();
}

Status download_to(Multi& m, void* host_cur, void* host_prev, bool whole_planes) {
    if (host_prev && !m.prev_valid)
        return Status::Err(TSR_EINVAL, "the other buffers do not hold step T-1 (advance with "
                                       "keep_previous)");
    Status r = each_device(m, [&](Slab& sl) -> Status {
        Status q = fetch_slab(m, sl, m.cur, host_cur, whole_planes);
        if (q.ok() && host_prev) q = fetch_slab(m, sl, 1 - m.cur, host_prev, whole_planes);
        return q;
    });
    if (!r.ok()) return r;
    return sync_all(m);
}

// ---- rounds ----------------------------------------------------------------

Status sweep_range(Multi& m, Slab& sl, cudaStream_t s, int64_t lo, int64_t hi, int n,
                   void* mirror, int64_t mirror_planes) {
    if (hi <= lo) return Status::Ok();
    LaunchCtx c{&sl.geo, &m.taps, m.opts.mode != TSR_FAST, s};
    c.lo0 = lo;
    c.hi0 = hi;
    if (mirror) {
        c.mirror = mirror;
        c.mirror_shift = mirror_planes * sl.geo.pitch[m.axis];
    }
    return sweep(c, m.plan, sl.d[m.cur], sl.d[1 - m.cur], n);
}

Status run_round(Multi& m, int n, tsr_stats& st) {
    const int c = m.cur;
    const int64_t rnd = m.round;
    const int64_t msg_bytes = m.depth * m.cross * m.g.esize;
    for (size_t i = 0; i < m.s.size(); ++i) {
        Slab& sl = m.s[i];
        TSR_CUDA_TRY(cudaSetDevice(sl.device));
        // ---- seam stream: wait for the neighbours' previous round and my own
        // previous interior pass, then the boundary planes, mirrored
        if (rnd > 0) {
            TSR_CUDA_TRY(cudaStreamWaitEvent(sl.s_seam, sl.ev_int, 0));
            for (int side = 0; side < 2; ++side)
                if (sl.nb[side] >= 0)
                    TSR_CUDA_TRY(cudaStreamWaitEvent(sl.s_seam,
                                                     m.s[sl.nb[side]].ev_seam[(rnd - 1) & 1], 0));
        }
        LogEntry le{rnd, static_cast<int>(i), nullptr, nullptr, nullptr, nullptr};
        if (m.logging) {
            for (cudaEvent_t* ev : {&le.a, &le.b, &le.c, &le.d})
                TSR_CUDA_TRY(cudaEventCreate(ev));
            TSR_CUDA_TRY(cudaEventRecord(le.a, sl.s_seam));
        }
        const int64_t first = sl.ghost_lo, last = sl.ghost_lo + sl.own();
        const int64_t rng[2][2] = {{first, std::min(last, first + m.depth)},
                                   {std::max(first, last - m.depth), last}};
        for (int side = 0; side < 2; ++side) {
            if (sl.nb[side] < 0) continue;
            Slab& nb = m.s[sl.nb[side]];
            const bool mirror = m.transport == TSR_XPORT_MIRROR;
            Status r = sweep_range(m, sl, sl.s_seam, rng[side][0], rng[side][1], n,
                                   mirror ? nb.d[1 - c] : nullptr, sl.shift[side]);
            if (!r.ok()) return r;
            ++st.kernel_launches;
            if (!mirror) {  // local store, then the planes move as one peer copy
                const int a = m.axis;
                const int64_t plen = a == 2 ? 1 : sl.geo.pitch[a];
                const int64_t cnt = (rng[side][1] - rng[side][0]) * plen * sl.geo.esize;
                const char* src = static_cast<const char*>(sl.d[1 - c]) +
                                  plane_start(sl.geo, a, rng[side][0]) * sl.geo.esize;
                char* dst = static_cast<char*>(nb.d[1 - c]) +
                            plane_start(nb.geo, a, rng[side][0] + sl.shift[side]) * sl.geo.esize;
                TSR_CUDA_TRY(
                    cudaMemcpyPeerAsync(dst, nb.device, src, sl.device, cnt, sl.s_seam));
            }
            st.messages += 1;
            st.bytes_exchanged += msg_bytes;
            // HaloWorker::tally_ghost (scheduler.cpp:358-366): step s of a
            // round computes depth - r(s+1) ghost planes per seam
            const int64_t rad = m.taps.radius, kk = m.plan.k;
            st.ghost_recompute_points += rad * (kk * n - int64_t(n) * (n + 1) / 2) * m.cross;
        }
        TSR_CUDA_TRY(cudaEventRecord(sl.ev_seam[rnd & 1], sl.s_seam));
        if (m.logging) TSR_CUDA_TRY(cudaEventRecord(le.b, sl.s_seam));
        // ---- interior stream: planes whose n-step cone stays inside the
        // owned planes; concurrent with the seam passes
        if (rnd > 0)
            TSR_CUDA_TRY(cudaStreamWaitEvent(sl.s_int, sl.ev_seam[(rnd - 1) & 1], 0));
        const int64_t ilo = first + (sl.nb[0] >= 0 ? m.depth : 0);
        const int64_t ihi = last - (sl.nb[1] >= 0 ? m.depth : 0);
        if (m.logging) TSR_CUDA_TRY(cudaEventRecord(le.c, sl.s_int));
        if (ihi > ilo) {
            Status r = sweep_range(m, sl, sl.s_int, ilo, ihi, n, nullptr, 0);
            if (!r.ok()) return r;
            ++st.kernel_launches;
        }
        if (m.logging) {
            TSR_CUDA_TRY(cudaEventRecord(le.d, sl.s_int));
            m.log.push_back(le);
        }
        TSR_CUDA_TRY(cudaEventRecord(sl.ev_int, sl.s_int));
    }
    m.cur ^= 1;
    ++m.round;
    return Status::Ok();
}

Status advance(Multi& m, int64_t steps, bool keep_prev, tsr_stats* out) {
    if (steps < 0) return Status::Err(TSR_EINVAL, "negative step count");
    tsr_stats st{};
    st.fused_steps = m.plan.k;
    st.engine = m.plan.engine ? TSR_ENGINE_TUNED : TSR_ENGINE_GENERIC;
    st.ngpus = static_cast<int32_t>(m.s.size());
    st.transport = m.transport;
    if (steps > 0) {
        Status r = sync_all(m);  // common start: every device idle
        if (!r.ok()) return r;
        r = each_device(m, [](Slab& sl) -> Status {
            TSR_CUDA_TRY(cudaEventRecord(sl.ev_t0, sl.s_int));
            TSR_CUDA_TRY(cudaStreamWaitEvent(sl.s_seam, sl.ev_t0, 0));
            return Status::Ok();
        });
        if (!r.ok()) return r;
        int64_t body = keep_prev ? steps - 1 : steps;
        int last = 0;
        while (body > 0) {
            const int n = static_cast<int>(std::min<int64_t>(m.plan.k, body));
            r = run_round(m, n, st);
            if (!r.ok()) return r;
            body -= n;
            last = n;
            if (n == m.plan.k) ++st.rounds; else st.trailing_steps += n;
        }
        if (keep_prev) {
            r = run_round(m, 1, st);
            if (!r.ok()) return r;
            last = 1;
            if (m.plan.k == 1) ++st.rounds; else st.trailing_steps += 1;
        }
        const int64_t rnd = m.round;
        r = each_device(m, [&](Slab& sl) -> Status {
            TSR_CUDA_TRY(cudaStreamWaitEvent(sl.s_int, sl.ev_seam[(rnd - 1) & 1], 0));
            TSR_CUDA_TRY(cudaEventRecord(sl.ev_t1, sl.s_int));
            return Status::Ok();
        });
        if (!r.ok()) return r;
        r = sync_all(m);
        if (!r.ok()) return r;
        float worst = 0.f;
        for (Slab& sl : m.s) {
            float ms = 0.f;
            TSR_CUDA_TRY(cudaEventElapsedTime(&ms, sl.ev_t0, sl.ev_t1));
            worst = std::max(worst, ms);
        }
        st.device_ms = worst;
        m.prev_valid = last == 1;
    }
    st.point_updates = m.g.interior() * steps;
    if (out) *out = st;
    return Status::Ok();
}

// ---- plane checksums ---------------------------------------------------------

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// out[p - lo] = sum over the interior cells (j, k) of plane p of
// mix(bits(x) + (pos + 1) * golden): order-independent, position-sensitive.
template <typename T>
__global__ void plane_checksum_kernel(const T* __restrict__ buf, int64_t lo, int64_t nj,
                                      int64_t nk, int64_t pitch_p, int64_t pitch_j,
                                      int64_t origin, unsigned long long* out) {
    const int64_t p = lo + blockIdx.y;
    const int64_t cells = nj * nk;
    unsigned long long acc = 0;
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cells;
         c += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = c / nk, kk = c - j * nk;
        const T v = buf[origin + p * pitch_p + j * pitch_j + kk];
        unsigned long long bits;
        if constexpr (sizeof(T) == 8) bits = __double_as_longlong(v);
        else bits = static_cast<unsigned>(__float_as_int(v));
        acc += mix64(bits + (static_cast<unsigned long long>(c) + 1) * 0x9E3779B97F4A7C15ull);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out + blockIdx.y, acc);
}

Status plane_checksums(const Geo& g, const void* dev, int64_t lo, int64_t hi, uint64_t* out,
                       cudaStream_t s) {
    if (hi <= lo) return Status::Ok();
    const int a = 3 - g.dims;
    const int64_t np = hi - lo;
    int64_t nj = 1, nk = 1, pitch_j = 0;
    if (a == 0) nj = g.n[1], nk = g.n[2], pitch_j = g.pitch[1];
    if (a == 1) nk = g.n[2];
    const int64_t pitch_p = g.pitch[a];
    unsigned long long* d = nullptr;
    TSR_CUDA_TRY(cudaMallocAsync(&d, np * sizeof(unsigned long long), s));
    TSR_CUDA_TRY(cudaMemsetAsync(d, 0, np * sizeof(unsigned long long), s));
    const int64_t cells = nj * nk;
    const unsigned bx = static_cast<unsigned>(std::min<int64_t>((cells + 255) / 256, 64));
    for (int64_t p0 = 0; p0 < np; p0 += 65535) {
        const unsigned by = static_cast<unsigned>(std::min<int64_t>(65535, np - p0));
        dim3 grid(bx, by);
        if (g.dtype == TSR_F64)
            plane_checksum_kernel<double><<<grid, 256, 0, s>>>(
                static_cast<const double*>(dev), lo + p0, nj, nk, pitch_p, pitch_j, g.origin,
                d + p0);
        else
            plane_checksum_kernel<float><<<grid, 256, 0, s>>>(
                static_cast<const float*>(dev), lo + p0, nj, nk, pitch_p, pitch_j, g.origin,
                d + p0);
        TSR_CUDA_TRY(cudaGetLastError());
    }
    TSR_CUDA_TRY(cudaMemcpyAsync(out, d, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    TSR_CUDA_TRY(cudaFreeAsync(d, s));
    TSR_CUDA_TRY(cudaStreamSynchronize(s));
    return Status::Ok();
}

// ---- tsr_run_multi's cached slab set ---------------------------------------

std::mutex g_multi_mu;
Multi* g_multi = nullptr;

bool same_taps(const TapSet& a, const TapSet& b) {
    if (a.dims != b.dims || a.shape != b.shape || a.radius != b.radius || a.ntaps != b.ntaps)
        return false;
    for (int i = 0; i < a.ntaps; ++i)
        if (a.w[i] != b.w[i] || std::memcmp(a.off[i], b.off[i], sizeof(a.off[i])) != 0)
            return false;
    return true;
}

bool cache_matches(const Multi* m, const Geo& g, const TapSet& t, const tsr_opts& o,
                   const std::vector<int32_t>& devs, const std::vector<int64_t>& bounds,
                   int transport, int flags) {
    if (!m) return false;
    for (int a = 0; a < 3; ++a)
        if (m->g.n[a] != g.n[a] || m->g.h[a] != g.h[a]) return false;
    return m->g.dims == g.dims && m->g.dtype == g.dtype && same_taps(m->taps, t) &&
           m->opts.fused_steps == o.fused_steps && m->opts.mode == o.mode &&
           m->opts.engine == o.engine && m->key_devices == devs && m->key_bounds == bounds &&
           m->key_transport == transport && m->key_flags == flags;
}

// Short runs (T*r small against each slab) need no exchange at all: each
// device computes its slab's planes of steps T and T-1 through the chunked
// round trip (run_host_range), its windows reading the T*r planes beyond the
// slab from the host buffers — replicated ghost zones, the seam work done
// twice instead of exchanged.  One host thread per device (slabs sharing a
// device run one after the other); TSR_EUNSUPPORTED when a slab is too
// short for the chunked round trip, and the slab runtime runs instead.
Status run_split(const tsr_kernel* kk, const tsr_grid* gg, const Geo& g, void* b0, void* b1,
                 int parity, int64_t steps, const tsr_partition* part, const tsr_opts& o, int P,
                 tsr_stats* st) {
    if (g.dims < 2) return Status::Err(TSR_EUNSUPPORTED, "1-D grid");
    if ((part ? part->split_axis : o.split_axis) != 0)
        return Status::Err(TSR_EUNSUPPORTED, "split axis");
    if (const char* e = std::getenv("TSR_MULTI_SPLIT"); e && *e == '0')
        return Status::Err(TSR_EUNSUPPORTED, "disabled");
    const int64_t n = g.n[3 - g.dims];
    if (P > n) return Status::Err(TSR_EUNSUPPORTED, "more slabs than planes");
    std::vector<int64_t> lo(P), hi(P);
    for (int i = 0; i < P; ++i) {
        if (part && part->boundaries) {
            lo[i] = i == 0 ? 0 : part->boundaries[i - 1];
            hi[i] = i == P - 1 ? n : part->boundaries[i];
        } else {
            const int64_t base = n / P, extra = n % P;
            lo[i] = i * base + std::min<int64_t>(i, extra);
            hi[i] = lo[i] + base + (i < extra ? 1 : 0);
        }
        if (lo[i] >= hi[i]) return Status::Err(TSR_EUNSUPPORTED, "empty slab");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return Status::Err(TSR_ECUDA, "no CUDA device available to the B200 sweep engine");
    }
    std::vector<int> dev(P);
    for (int i = 0; i < P; ++i) dev[i] = part && part->devices ? part->devices[i] : i % ndev;
    // One plane range per device: its slabs must be consecutive (round-robin
    // placement on fewer devices than slabs is not), merged into one range.
    // (TSR_SPLIT_PER_SLAB=1 keeps one range per slab, each with buffers of
    // its own: the barrier across ranges can then run on a single device.)
    const char* per = std::getenv("TSR_SPLIT_PER_SLAB");
    const bool per_slab = per && *per == '1';
    std::vector<int> rdev, rsub;
    std::vector<int64_t> rlo, rhi;
    for (int i = 0; i < P; ++i) {
        if (!per_slab && !rdev.empty() && rdev.back() == dev[i]) {
            rhi.back() = hi[i];
            continue;
        }
        const int prior = static_cast<int>(std::count(rdev.begin(), rdev.end(), dev[i]));
        if (prior > 0 && !per_slab)
            return Status::Err(TSR_EUNSUPPORTED, "a device's slabs are not consecutive");
        rdev.push_back(dev[i]);
        rsub.push_back(prior);
        rlo.push_back(lo[i]);
        rhi.push_back(hi[i]);
    }
    const int D = static_cast<int>(rdev.size());
    // every range must take the chunked round trip (checked before any
    // buffer is written; else the slab runtime runs the whole call)
    TapSet t;
    Status r = make_taps(*kk, t);
    if (!r.ok()) return r;
    for (int i = 0; i < D; ++i)
        if (!range_chunkable(g, t, steps, rlo[i], rhi[i]))
            return Status::Err(TSR_EUNSUPPORTED, "slab too short for the chunked round trip");
    // Barrier: every device has its margin planes up before any device
    // writes planes back into the host buffers.  A device that fails before
    // the barrier still arrives, so the others do not wait forever.
    std::mutex bm;
    std::condition_variable bcv;
    int arrived = 0;
    auto arrive = [&](bool wait) {
        std::unique_lock<std::mutex> lk(bm);
        ++arrived;
        bcv.notify_all();
        if (wait) bcv.wait(lk, [&] { return arrived >= D; });
    };
    std::vector<Status> res(D);
    std::vector<tsr_stats> sts(D);
    std::vector<std::thread> th;
    for (int i = 0; i < D; ++i)
        th.emplace_back([&, i] {
            bool did = false;
            const std::function<void()> cb = [&] {
                did = true;
                arrive(true);
            };
            tsr_opts od = o;
            od.ngpus = 1;
            od.device = rdev[i];
            res[i] = run_host_range(kk, gg, b0, b1, parity, steps, &od, &sts[i], rlo[i], rhi[i], cb,
                                    rsub[i]);
            if (!did) arrive(false);
        });
    for (auto& x : th) x.join();
    for (int i = 0; i < D; ++i)
        if (!res[i].ok())
            return res[i].code == TSR_EUNSUPPORTED ? Status::Err(TSR_ECUDA, res[i].msg) : res[i];
    tsr_stats out{};
    for (int i = 0; i < D; ++i) {
        out.point_updates += sts[i].point_updates;
        out.kernel_launches += sts[i].kernel_launches;
        out.h2d_bytes += sts[i].h2d_bytes;
        out.d2h_bytes += sts[i].d2h_bytes;
        out.device_ms = std::max(out.device_ms, sts[i].device_ms);
        out.ghost_recompute_points += sts[i].ghost_recompute_points;
    }
    out.rounds = sts[0].rounds;
    out.trailing_steps = sts[0].trailing_steps;
    out.fused_steps = sts[0].fused_steps;
    out.engine = sts[0].engine;
    out.ngpus = P;
    if (st) *st = out;
    return Status::Ok();
}

Status run_multi(const tsr_kernel* kk, const tsr_grid* gg, void* b0, void* b1, int parity,
                 int64_t steps, const tsr_partition* part, bool keep_prev, const tsr_opts* oo,
                 tsr_stats* st) {
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
    void* host[2] = {b0, b1};
    const bool equal_halos = halos_equal(g, b0, b1);
    if (steps == 0) return Status::Ok();
    if (keep_prev && !equal_halos) {
        // naive_run semantics with two different halos (every step reads its
        // read buffer's halo): one device, one sweep per step (run_host)
        tsr_opts o1 = o;
        o1.ngpus = 1;
        o1.device = part && part->devices ? part->devices[0] : -1;
        return run_host_single(kk, gg, b0, b1, parity, steps, &o1, st);
    }
    DeviceGuard guard;
    r = guard.enter(-1);
    if (!r.ok()) return r;

    const int P = part ? part->ngpus : std::max(1, o.ngpus);
    if (keep_prev && P > 1) {
        r = run_split(kk, gg, g, b0, b1, parity, steps, part, o, P, st);
        if (r.code != TSR_EUNSUPPORTED) return r;
        cudaGetLastError();
    }
    std::vector<int32_t> devs;
    std::vector<int64_t> bounds;
    if (part && part->devices) devs.assign(part->devices, part->devices + P);
    if (part && part->boundaries && P > 1) bounds.assign(part->boundaries, part->boundaries + P - 1);
    tsr_partition dflt{P, o.split_axis, nullptr, nullptr, TSR_XPORT_AUTO, 0};
    const tsr_partition* pp = part ? part : &dflt;

    std::lock_guard<std::mutex> lock(g_multi_mu);
    if (!cache_matches(g_multi, g, t, o, devs, bounds, pp->transport, pp->flags)) {
        destroy(g_multi);
        g_multi = nullptr;
        r = create(kk, gg, pp, &o, &g_multi);
        if (!r.ok()) return r;
        g_multi->key_devices = devs;
        g_multi->key_bounds = bounds;
        g_multi->key_transport = pp->transport;
        g_multi->key_flags = pp->flags;
    }
    Multi& m = *g_multi;
    drop_log(m);
    m.logging = false;
    r = upload_host(m, host[parity]);
    if (!r.ok()) return r;
    tsr_stats local{};
    r = advance(m, steps, keep_prev, &local);
    if (!r.ok()) return r;
    const int pfinal = parity ^ static_cast<int>(steps & 1);
    r = download_to(m, host[pfinal], keep_prev && steps >= 2 ? host[1 - pfinal] : nullptr,
                    equal_halos);
    if (!r.ok()) return r;
    int64_t own_bytes = 0;
    for (const Slab& sl : m.s)
        own_bytes += sl.own() * (m.axis == 2 ? g.esize : g.hpitch[m.axis] * g.esize);
    local.h2d_bytes = 0;
    for (const Slab& sl : m.s) local.h2d_bytes += sl.geo.host_elements * g.esize;
    local.d2h_bytes = (keep_prev && steps >= 2 ? 2 : 1) *
                      (equal_halos ? own_bytes : g.interior() * g.esize);
    if (st) *st = local;
    return Status::Ok();
}

}  // namespace

void release_multi_cache() {
    std::lock_guard<std::mutex> lock(g_multi_mu);
    destroy(g_multi);
    g_multi = nullptr;
}

Status run_multi_opts(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int parity,
                      int64_t steps, const tsr_opts* o, tsr_stats* st) {
    return run_multi(k, g, b0, b1, parity, steps, nullptr, true, o, st);
}

}  // namespace tsr

using namespace tsr;

extern "C" {

int tsr_multi_create(const tsr_kernel* k, const tsr_grid* g, const tsr_partition* part,
                     const tsr_opts* opts, tsr_multi** out) {
    if (!out) return report(Status::Err(TSR_EINVAL, "null argument"));
    *out = nullptr;
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (!r.ok()) return report(r);
    return report(create(k, g, part, opts, out));
}

int tsr_multi_destroy(tsr_multi* m) {
    destroy(m);
    return TSR_OK;
}

int tsr_multi_upload(tsr_multi* m, const void* host) {
    if (!m || !host) return report(Status::Err(TSR_EINVAL, "null argument"));
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (r.ok()) r = upload_host(*m, host);
    return report(r);
}

int tsr_multi_fill_random(tsr_multi* m, uint64_t seed, double lo, double hi) {
    if (!m) return report(Status::Err(TSR_EINVAL, "null argument"));
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (r.ok())
        r = m->g.dtype == TSR_F64 ? fill_stream<double>(*m, seed, lo, hi)
                                  : fill_stream<float>(*m, seed, lo, hi);
    return report(r);
}

int tsr_multi_advance(tsr_multi* m, int64_t steps, int32_t keep_previous, tsr_stats* stats) {
    if (!m) return report(Status::Err(TSR_EINVAL, "null argument"));
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (r.ok()) r = advance(*m, steps, keep_previous != 0, stats);
    return report(r);
}

int tsr_multi_download(tsr_multi* m, void* host_cur, void* host_prev) {
    if (!m || !host_cur) return report(Status::Err(TSR_EINVAL, "null argument"));
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (r.ok()) r = download_to(*m, host_cur, host_prev, true);
    return report(r);
}

int tsr_multi_slab_info(const tsr_multi* m, int32_t slab, tsr_slab_info* out) {
    if (!m || !out) return report(Status::Err(TSR_EINVAL, "null argument"));
    if (slab < 0 || slab >= static_cast<int32_t>(m->s.size()))
        return report(Status::Err(TSR_EINVAL, "slab index out of range"));
    const Slab& sl = m->s[slab];
    out->device = sl.device;
    out->cur = m->cur;
    out->own_lo = sl.own_lo;
    out->own_hi = sl.own_hi;
    out->ghost_lo = sl.ghost_lo;
    out->ghost_hi = sl.ghost_hi;
    out->grid = sl.desc;
    const int shift = 3 - sl.geo.dims;
    for (int a = 0; a < 3; ++a) out->layout.pitch[a] = a < sl.geo.dims ? sl.geo.pitch[a + shift] : 0;
    out->layout.origin = sl.geo.origin;
    out->layout.elements = sl.geo.elements;
    out->buf[0] = sl.d[0];
    out->buf[1] = sl.d[1];
    return TSR_OK;
}

int tsr_multi_set_logging(tsr_multi* m, int32_t on) {
    if (!m) return report(Status::Err(TSR_EINVAL, "null argument"));
    m->logging = on != 0;
    if (!m->logging) drop_log(*m);
    return TSR_OK;
}

int tsr_multi_comm_log(tsr_multi* m, tsr_comm_record* out, int64_t cap, int64_t* count) {
    if (!m || !count) return report(Status::Err(TSR_EINVAL, "null argument"));
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (r.ok()) r = sync_all(*m);
    if (!r.ok()) return report(r);
    int64_t n = 0;
    const int64_t bytes = m->depth * m->cross * m->g.esize;
    std::vector<cudaEvent_t> epoch(m->s.size(), nullptr);  // per slab: its first logged round
    for (const LogEntry& e : m->log)
        if (!epoch[e.slab]) epoch[e.slab] = e.a;
    for (const LogEntry& e : m->log) {
        cudaSetDevice(m->s[e.slab].device);
        float ms = 0.f, s0 = 0.f, s1 = 0.f, i0 = 0.f, i1 = 0.f;
        cudaEventElapsedTime(&ms, e.a, e.b);
        cudaEventElapsedTime(&s0, epoch[e.slab], e.a);
        cudaEventElapsedTime(&s1, epoch[e.slab], e.b);
        cudaEventElapsedTime(&i0, epoch[e.slab], e.c);
        cudaEventElapsedTime(&i1, epoch[e.slab], e.d);
        const Slab& sl = m->s[e.slab];
        for (int side = 0; side < 2; ++side) {
            if (sl.nb[side] < 0) continue;
            if (out && n < cap)
                out[n] = tsr_comm_record{e.round, e.slab, sl.nb[side], bytes, ms, s0, s1, i0, i1};
            ++n;
        }
    }
    *count = n;
    if (out && n <= cap) drop_log(*m);
    return TSR_OK;
}

int tsr_multi_plane_checksums(tsr_multi* m, int32_t which, uint64_t* out) {
    if (!m || !out) return report(Status::Err(TSR_EINVAL, "null argument"));
    if (which == 1 && !m->prev_valid)
        return report(Status::Err(TSR_EINVAL, "the other buffers do not hold step T-1"));
    DeviceGuard guard;
    Status r = guard.enter(-1);
    if (r.ok())
        r = each_device(*m, [&](Slab& sl) -> Status {
            const int buf = which ? 1 - m->cur : m->cur;
            return plane_checksums(sl.geo, sl.d[buf], sl.ghost_lo, sl.ghost_lo + sl.own(),
                                   out + sl.own_lo, sl.s_int);
        });
    return report(r);
}

int tsr_plane_checksums(const tsr_grid* g, const tsr_layout* l, const void* dev, int64_t lo,
                        int64_t hi, uint64_t* out, void* stream) {
    if (!g || !dev || !out) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    if (s.ok() && (lo < 0 || hi > geo.n[3 - geo.dims] || lo > hi))
        s = Status::Err(TSR_EINVAL, "plane range outside the grid's axis 0");
    if (s.ok()) s = plane_checksums(geo, dev, lo, hi, out, static_cast<cudaStream_t>(stream));
    return report(s);
}

int tsr_run_multi(const tsr_kernel* k, const tsr_grid* g, void* buf0, void* buf1,
                  int32_t parity, int64_t steps, const tsr_partition* part,
                  int32_t keep_previous, const tsr_opts* opts, tsr_stats* stats) {
    return report(run_multi(k, g, buf0, buf1, parity, steps, part, keep_previous != 0, opts,
                            stats));
}

}  // extern "C"
