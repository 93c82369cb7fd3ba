// abi.cu — the extern "C" boundary (include/tessera_b200.h) and the host
// runtime behind it: validation with the reference's error semantics, the
// pitched device layout, H2D/D2H of BasicGrid<T> buffers, the fused-round
// driver and engine dispatch (tsr_run's host round trip: roundtrip.cu).
#include <algorithm>
#include <array>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <sstream>
#include <thread>
#include <vector>

#include "runtime.cuh"

namespace tsr {

extern const Engine kStream2dEngine;
extern const Engine kTb3dEngine;
extern const Engine kBox3dEngine;
extern const Engine kStream1dEngine;

thread_local std::string g_last_error;

int report(const Status& s) {
    if (!s.ok()) g_last_error = s.msg;
    return s.code;
}

namespace {

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

bool offset_less(const int* a, const int* b) {
    return std::lexicographical_compare(a, a + 3, b, b + 3);
}

// The exact lattice for (dims, shape, radius) in lexicographic order
// (proj/src/kernel.cpp:19-43).
std::vector<std::array<int, 3>> lattice(int dims, int shape, int radius) {
    std::vector<std::array<int, 3>> out;
    std::array<int, 3> cur{0, 0, 0};
    std::function<void(int)> rec = [&](int axis) {
        if (axis == dims) {
            int nonzero = 0;
            for (int a = 0; a < dims; ++a) nonzero += cur[a] != 0;
            if (shape == TSR_BOX || nonzero <= 1) out.push_back(cur);
            return;
        }
        for (int v = -radius; v <= radius; ++v) {
            cur[axis] = v;
            rec(axis + 1);
        }
        cur[axis] = 0;
    };
    rec(0);
    std::sort(out.begin(), out.end(),
              [](const auto& a, const auto& b) { return offset_less(a.data(), b.data()); });
    return out;
}

}  // namespace

Status make_taps(const tsr_kernel& k, TapSet& t) {
    if (k.dims < 1 || k.dims > 3) return Status::Err(TSR_EINVAL, "kernel dims must be 1, 2 or 3");
    if (k.radius < 1) return Status::Err(TSR_EINVAL, "kernel radius must be positive");
    if (k.shape != TSR_STAR && k.shape != TSR_BOX)
        return Status::Err(TSR_EINVAL, "kernel shape must be 'star' or 'box'");
    if (!k.offsets || !k.weights) return Status::Err(TSR_EINVAL, "null kernel tap arrays");
    const auto lat = lattice(k.dims, k.shape, k.radius);
    if (static_cast<int64_t>(lat.size()) != k.ntaps) {
        std::ostringstream os;
        os << "kernel offset count mismatch: expected " << lat.size() << " offsets for "
           << (k.shape == TSR_STAR ? "star" : "box") << " radius " << k.radius << " in "
           << k.dims << "D, got " << k.ntaps;
        return Status::Err(TSR_EINVAL, os.str());
    }
    if (k.ntaps > kMaxTaps) return Status::Err(TSR_EUNSUPPORTED, "more than 1024 taps");
    t.dims = k.dims;
    t.shape = k.shape;
    t.radius = k.radius;
    t.ntaps = k.ntaps;
    const int shift = 3 - k.dims;
    for (int i = 0; i < k.ntaps; ++i) {
        const int32_t* o = k.offsets + 3 * i;
        for (int a = k.dims; a < 3; ++a)
            if (o[a] != 0)
                return Status::Err(TSR_EINVAL, "offset uses components beyond kernel dims");
        if (!std::isfinite(k.weights[i]))
            return Status::Err(TSR_EINVAL, "non-finite kernel weight");
        for (int a = 0; a < 3; ++a)
            if (o[a] != lat[i][a])
                return Status::Err(TSR_EINVAL,
                                   "taps are not the canonical lexicographic lattice of the "
                                   "kernel shape (make_kernel order)");
        for (int a = 0; a < 3; ++a) t.off[i][a] = 0;
        for (int a = 0; a < k.dims; ++a) t.off[i][a + shift] = o[a];
        t.w[i] = k.weights[i];
    }
    return Status::Ok();
}

Status make_geo(const tsr_grid& g, Geo& o) {
    if (g.dims < 1 || g.dims > 3) return Status::Err(TSR_EINVAL, "grid dims must be 1, 2 or 3");
    if (g.dtype != TSR_F64 && g.dtype != TSR_F32)
        return Status::Err(TSR_EINVAL, "grid dtype must be f64 or f32");
    o = Geo{};
    o.dims = g.dims;
    o.dtype = g.dtype;
    o.esize = g.dtype == TSR_F64 ? 8 : 4;
    const int shift = 3 - g.dims;
    for (int a = 0; a < 3; ++a) {
        o.n[a] = 1;
        o.h[a] = 0;
    }
    for (int a = 0; a < g.dims; ++a) {
        if (g.halo[a] < 0) return Status::Err(TSR_EINVAL, "negative halo width");
        if (g.extent[a] < 2 * g.halo[a] + 1) {
            std::ostringstream os;
            os << "degenerate extent " << g.extent[a] << " on axis " << a << ": need at least "
               << 2 * g.halo[a] + 1 << " interior points";
            return Status::Err(TSR_EINVAL, os.str());
        }
        o.n[a + shift] = g.extent[a];
        o.h[a + shift] = g.halo[a];
    }
    // Device layout: the interior of every row starts on a 128-byte boundary
    // and rows are padded to a multiple of 128 bytes (TMA / vector alignment).
    const int64_t align = 128 / o.esize;
    o.off2 = round_up(std::max<int64_t>(o.h[2], 1), align);
    o.pitch[2] = 1;
    o.pitch[1] = round_up(o.off2 + o.n[2] + o.h[2], align);
    o.pitch[0] = o.pitch[1] * (o.n[1] + 2 * o.h[1]);
    o.origin = o.h[0] * o.pitch[0] + o.h[1] * o.pitch[1] + o.off2;
    o.elements = (o.n[0] + 2 * o.h[0]) * o.pitch[0];
    // Reference host layout.
    o.hpitch[2] = 1;
    o.hpitch[1] = o.n[2] + 2 * o.h[2];
    o.hpitch[0] = o.hpitch[1] * (o.n[1] + 2 * o.h[1]);
    o.horigin = o.h[0] * o.hpitch[0] + o.h[1] * o.hpitch[1] + o.h[2];
    o.host_elements = (o.n[0] + 2 * o.h[0]) * o.hpitch[0];
    return Status::Ok();
}

Status check_layout(const Geo& g, const tsr_layout* l) {
    if (!l) return Status::Ok();
    const int shift = 3 - g.dims;
    bool same = l->origin == g.origin && l->elements == g.elements;
    for (int a = 0; a < g.dims; ++a) same &= l->pitch[a] == g.pitch[a + shift];
    if (!same) return Status::Err(TSR_EINVAL, "layout does not match tsr_layout_of(grid)");
    return Status::Ok();
}

// Tuned engines in preference order.  TSR_ENGINE=<name> (environment) pins
// one by name for A/B measurements; it never falls back to the CPU.
const Engine* find_engine(const Geo& g, const TapSet& t, int* max_fused, int* default_fused) {
    static const Engine* const engines[] = {&kTb3dEngine, &kBox3dEngine, &kStream2dEngine,
                                            &kStream1dEngine};
    const char* pin = std::getenv("TSR_ENGINE");
    for (const Engine* e : engines) {
        if (pin && *pin && std::strcmp(pin, e->name) != 0) continue;
        if (e->supports(g, t, max_fused, default_fused)) return e;
    }
    return nullptr;
}

Status check_applicable(const Geo& g, const TapSet& t) {
    if (t.dims != g.dims) return Status::Err(TSR_EINVAL, "kernel/grid dimensionality mismatch");
    for (int a = 3 - g.dims; a < 3; ++a)
        if (g.h[a] < t.radius)
            return Status::Err(TSR_EINVAL, "grid halo too small for kernel radius");
    return Status::Ok();
}

namespace {

cudaMemcpy3DParms copy_parms(void* dst, int64_t dpitch_el, int64_t dx, int64_t dy, int64_t dz,
                             const void* src, int64_t spitch_el, int64_t sx, int64_t sy,
                             int64_t sz, int64_t w_el, int64_t h, int64_t d, int64_t ysize,
                             int esize, cudaMemcpyKind kind) {
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), spitch_el * esize, spitch_el * esize,
                                   ysize);
    p.dstPtr = make_cudaPitchedPtr(dst, dpitch_el * esize, dpitch_el * esize, ysize);
    p.srcPos = make_cudaPos(sx * esize, sy, sz);
    p.dstPos = make_cudaPos(dx * esize, dy, dz);
    p.extent = make_cudaExtent(w_el * esize, h, d);
    p.kind = kind;
    return p;
}

}  // namespace

Status upload(const Geo& g, const void* host, void* dev, cudaStream_t s) {
    const int64_t ysize = g.n[1] + 2 * g.h[1];
    auto p = copy_parms(dev, g.pitch[1], g.off2 - g.h[2], 0, 0, host, g.hpitch[1], 0, 0, 0,
                        g.n[2] + 2 * g.h[2], ysize, g.n[0] + 2 * g.h[0], ysize, g.esize,
                        cudaMemcpyHostToDevice);
    TSR_CUDA_TRY(cudaMemcpy3DAsync(&p, s));
    return Status::Ok();
}

Status download(const Geo& g, const void* dev, void* host, bool interior_only, cudaStream_t s) {
    const int64_t ysize = g.n[1] + 2 * g.h[1];
    cudaMemcpy3DParms p;
    if (interior_only)
        p = copy_parms(host, g.hpitch[1], g.h[2], g.h[1], g.h[0], dev, g.pitch[1], g.off2,
                       g.h[1], g.h[0], g.n[2], g.n[1], g.n[0], ysize, g.esize,
                       cudaMemcpyDeviceToHost);
    else
        p = copy_parms(host, g.hpitch[1], 0, 0, 0, dev, g.pitch[1], g.off2 - g.h[2], 0, 0,
                       g.n[2] + 2 * g.h[2], ysize, g.n[0] + 2 * g.h[0], ysize, g.esize,
                       cudaMemcpyDeviceToHost);
    TSR_CUDA_TRY(cudaMemcpy3DAsync(&p, s));
    return Status::Ok();
}

// True when the halo shells of the two host buffers are bitwise equal.
static bool halos_equal_rows(const Geo& g, const void* b0, const void* b1, int64_t r_lo, int64_t r_hi) {
    const char* a = static_cast<const char*>(b0);
    const char* b = static_cast<const char*>(b1);
    const int64_t rows1 = g.n[1] + 2 * g.h[1];
    const int64_t rowlen = g.hpitch[1] * g.esize;
    for (int64_t r = r_lo; r < r_hi; ++r) {
        const int64_t r0 = r / rows1, r1 = r % rows1;
        const int64_t off = (r0 * g.hpitch[0] + r1 * g.hpitch[1]) * g.esize;
        const bool halo_row = r0 < g.h[0] || r0 >= g.n[0] + g.h[0] || r1 < g.h[1] ||
                              r1 >= g.n[1] + g.h[1];
        if (halo_row) {
            if (std::memcmp(a + off, b + off, rowlen) != 0) return false;
        } else if (g.h[2] > 0) {
            const int64_t hb = g.h[2] * g.esize;
            if (std::memcmp(a + off, b + off, hb) != 0) return false;
            const int64_t tail = off + (g.h[2] + g.n[2]) * g.esize;
            if (std::memcmp(a + tail, b + tail, hb) != 0) return false;
        }
    }
    return true;
}

// The comparison touches a few bytes of every row of both buffers (page- and
// TLB-bound: ~8 ms for two 1 GB buffers on one thread); rows are split over
// up to 8 host threads, so it ends before the first upload pieces do.
bool halos_equal(const Geo& g, const void* b0, const void* b1) {
    const int64_t rows = (g.n[0] + 2 * g.h[0]) * (g.n[1] + 2 * g.h[1]);
    const int nt = static_cast<int>(std::min<int64_t>(
        std::max(1u, std::min(8u, std::thread::hardware_concurrency())), rows / 4096 + 1));
    if (nt == 1) return halos_equal_rows(g, b0, b1, 0, rows);
    std::vector<std::thread> th;
    std::vector<char> ok(nt, 1);
    for (int i = 0; i < nt; ++i)
        th.emplace_back([&, i] {
            ok[i] = halos_equal_rows(g, b0, b1, rows * i / nt, rows * (i + 1) / nt);
        });
    for (auto& x : th) x.join();
    for (char v : ok)
        if (!v) return false;
    return true;
}

Status plan_for(const Geo& g, const TapSet& t, const tsr_opts& o, Plan& p) {
    int maxk = 1, defk = 1;
    const Engine* e = nullptr;
    if (o.engine != TSR_ENGINE_GENERIC) e = find_engine(g, t, &maxk, &defk);
    if (o.engine == TSR_ENGINE_TUNED && !e)
        return Status::Err(TSR_EUNSUPPORTED, "no tuned engine for this kernel/grid");
    if (o.fused_steps < 0) return Status::Err(TSR_EINVAL, "fused_steps must be >= 0");
    p.engine = e;
    if (!e) {
        p.k = 1;
    } else {
        if (o.mode == TSR_FAST && e->fast_max) maxk = e->fast_max(g, t);
        if (o.mode == TSR_FAST && e->fast_default) defk = std::min(e->fast_default(g, t), maxk);
        p.k = o.fused_steps > 0 ? std::min(o.fused_steps, maxk) : defk;
    }
    return Status::Ok();
}

Status sweep(const LaunchCtx& c, const Plan& p, const void* in, void* out, int k) {
    if (p.engine) return p.engine->run(c, in, out, k);
    int64_t lo[3] = {0, 0, 0};
    int64_t hi[3] = {c.g->n[0], c.g->n[1], c.g->n[2]};
    const int s = 3 - c.g->dims;
    lo[s] = c.range_lo();
    hi[s] = c.range_hi();
    if (hi[s] <= lo[s]) return Status::Ok();
    return generic_sweep(c, in, out, lo, hi);
}

Status advance_grid(const Geo& g, const TapSet& t, const tsr_opts& o, void* d0, void* d1,
                    int* cur, int64_t steps, bool keep_prev, cudaStream_t s, tsr_stats* st) {
    if (steps < 0) return Status::Err(TSR_EINVAL, "negative step count");
    Status r = check_applicable(g, t);
    if (!r.ok()) return r;
    Plan p;
    r = plan_for(g, t, o, p);
    if (!r.ok()) return r;
    LaunchCtx c{&g, &t, o.mode != TSR_FAST, s};
    void* d[2] = {d0, d1};
    int64_t body = keep_prev && steps > 0 ? steps - 1 : steps;
    int64_t rounds = 0, trailing = 0, launches = 0;
    while (body > 0) {
        const int kk = static_cast<int>(std::min<int64_t>(p.k, body));
        r = sweep(c, p, d[*cur], d[1 - *cur], kk);
        if (!r.ok()) return r;
        *cur ^= 1;
        body -= kk;
        ++launches;
        if (kk == p.k) ++rounds; else trailing += kk;
    }
    if (keep_prev && steps > 0) {
        r = sweep(c, p, d[*cur], d[1 - *cur], 1);
        if (!r.ok()) return r;
        *cur ^= 1;
        ++launches;
        if (p.k == 1) ++rounds; else trailing += 1;
    }
    if (st) {
        st->point_updates += g.interior() * steps;
        st->rounds += rounds;
        st->trailing_steps += trailing;
        st->kernel_launches += launches;
        st->fused_steps = p.k;
        st->engine = p.engine ? TSR_ENGINE_TUNED : TSR_ENGINE_GENERIC;
    }
    return Status::Ok();
}

Status DeviceGuard::enter(int want) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return Status::Err(TSR_ECUDA, "no CUDA device available to the B200 sweep engine");
    }
    TSR_CUDA_TRY(cudaGetDevice(&prev));
    if (want >= 0 && want != prev) {
        TSR_CUDA_TRY(cudaSetDevice(want));
        set = true;
    }
    return Status::Ok();
}

DeviceGuard::~DeviceGuard() {
    if (set) cudaSetDevice(prev);
}

tsr_opts opts_or_default(const tsr_opts* o) {
    if (o) return *o;
    tsr_opts d{};
    d.fused_steps = 0;
    d.mode = TSR_EXACT;
    d.engine = TSR_ENGINE_AUTO;
    d.device = -1;
    d.ngpus = 1;
    d.split_axis = 0;
    return d;
}


template <typename T>
void fill_random_t(const Geo& g, T* b0, T* b1, uint64_t seed, double lo, double hi,
                   uint64_t skip) {
    std::mt19937_64 rng(seed);
    rng.discard(skip);
    for (int64_t i = 0; i < g.n[0]; ++i)
        for (int64_t j = 0; j < g.n[1]; ++j) {
            const int64_t row = g.horigin + i * g.hpitch[0] + j * g.hpitch[1];
            for (int64_t k = 0; k < g.n[2]; ++k) {
                const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
                const T v = static_cast<T>(lo + (hi - lo) * u);
                b0[row + k] = v;
                b1[row + k] = v;
            }
        }
}

void fill_random_host(const Geo& g, void* b0, void* b1, uint64_t seed, double lo, double hi,
                      uint64_t skip) {
    if (g.dtype == TSR_F64)
        fill_random_t(g, static_cast<double*>(b0), static_cast<double*>(b1), seed, lo, hi, skip);
    else
        fill_random_t(g, static_cast<float*>(b0), static_cast<float*>(b1), seed, lo, hi, skip);
}

// The case study's plate (proj/src/case_study.cpp:193-207): every cell of
// both buffers is the ambient temperature except the interior, which holds
// ambient + (peak - ambient) * exp(-(di^2 + dj^2) / (2 sigma^2)) around the
// plate centre c0 = (n - 1) / 2, evaluated in double with std::exp and then
// cast to T, exactly as the reference's init_temp / initialize do.  (Host
// code: x86-64 without -mfma, so nothing is contracted into an FMA.)
template <typename T>
void fill_plate_t(const Geo& g, T* b0, T* b1, double ambient, double peak, double sigma) {
    const int64_t rows = g.n[1] + 2 * g.h[1], cols = g.n[2] + 2 * g.h[2];
    const double ci = static_cast<double>(g.n[1] - 1) / 2.0;
    const double cj = static_cast<double>(g.n[2] - 1) / 2.0;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            const int64_t i = r - g.h[1], j = c - g.h[2];
            double v = ambient;
            if (i >= 0 && i < g.n[1] && j >= 0 && j < g.n[2]) {
                const double di = static_cast<double>(i) - ci, dj = static_cast<double>(j) - cj;
                v = ambient + (peak - ambient) * std::exp(-(di * di + dj * dj) / (2.0 * sigma * sigma));
            }
            b0[r * g.hpitch[1] + c] = static_cast<T>(v);
            b1[r * g.hpitch[1] + c] = static_cast<T>(v);
        }
}

}  // namespace tsr

using namespace tsr;

namespace tsr {
Status peer_signal(void* flag, unsigned value, cudaStream_t s);
Status peer_wait(const void* flag, unsigned value, cudaStream_t s);
Status peer_round_wait(const void* flag_lo, const void* flag_hi, const void* counter,
                       cudaStream_t s);
Status peer_round_signal(void* peer_lo, void* peer_hi, void* counter, cudaStream_t s);
Status ipc_export(const void* ptr, unsigned char* handle, int64_t* offset);
Status ipc_open(const unsigned char* handle, void** base);
Status ipc_close(void* base);
void release_multi_cache();
Status run_multi_opts(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int parity,
                      int64_t steps, const tsr_opts* o, tsr_stats* st);
}  // namespace tsr

extern "C" {

int tsr_abi_version(void) { return TSR_ABI_VERSION; }

const char* tsr_last_error(void) { return g_last_error.c_str(); }

int tsr_release_cache(void) {
    release_multi_cache();
    release_run_cache();
    return TSR_OK;
}

int tsr_check_kernel(const tsr_kernel* k) {
    if (!k) return report(Status::Err(TSR_EINVAL, "null kernel"));
    static thread_local TapSet t;
    return report(make_taps(*k, t));
}

int tsr_layout_of(const tsr_grid* g, tsr_layout* out) {
    if (!g || !out) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (!s.ok()) return report(s);
    const int shift = 3 - geo.dims;
    for (int a = 0; a < 3; ++a) out->pitch[a] = a < geo.dims ? geo.pitch[a + shift] : 0;
    out->origin = geo.origin;
    out->elements = geo.elements;
    return TSR_OK;
}

int tsr_fill_random(const tsr_grid* g, void* b0, void* b1, uint64_t seed, double lo, double hi) {
    return tsr_fill_random_at(g, b0, b1, seed, lo, hi, 0);
}

int tsr_fill_random_at(const tsr_grid* g, void* b0, void* b1, uint64_t seed, double lo,
                       double hi, uint64_t skip) {
    if (!g || !b0 || !b1) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (!s.ok()) return report(s);
    fill_random_host(geo, b0, b1, seed, lo, hi, skip);
    return TSR_OK;
}

int tsr_fill_plate(const tsr_grid* g, void* b0, void* b1, double ambient, double peak,
                   double sigma) {
    if (!g || !b0 || !b1) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (!s.ok()) return report(s);
    if (geo.dims != 2) return report(Status::Err(TSR_EINVAL, "the plate is a 2-D grid"));
    if (!(sigma > 0.0)) return report(Status::Err(TSR_EINVAL, "sigma must be positive"));
    if (geo.dtype == TSR_F64)
        fill_plate_t(geo, static_cast<double*>(b0), static_cast<double*>(b1), ambient, peak, sigma);
    else
        fill_plate_t(geo, static_cast<float*>(b0), static_cast<float*>(b1), ambient, peak, sigma);
    return TSR_OK;
}

int tsr_run(const tsr_kernel* k, const tsr_grid* g, void* b0, void* b1, int32_t parity,
            int64_t steps, const tsr_opts* opts, tsr_stats* stats) {
    if (opts && opts->ngpus > 1)
        return report(run_multi_opts(k, g, b0, b1, parity, steps, opts, stats));
    return report(run_host_single(k, g, b0, b1, parity, steps, opts, stats));
}

int tsr_upload(const tsr_grid* g, const tsr_layout* l, const void* host, void* dev,
               void* stream) {
    if (!g || !host || !dev) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    if (s.ok()) s = upload(geo, host, dev, static_cast<cudaStream_t>(stream));
    return report(s);
}

int tsr_download(const tsr_grid* g, const tsr_layout* l, const void* dev, void* host,
                 int32_t interior_only, void* stream) {
    if (!g || !host || !dev) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    if (s.ok()) s = download(geo, dev, host, interior_only != 0, static_cast<cudaStream_t>(stream));
    return report(s);
}

int tsr_copy_halo(const tsr_grid* g, const tsr_layout* l, const void* src, void* dst,
                  void* stream) {
    if (!g || !src || !dst) return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    if (s.ok()) s = halo_copy(geo, src, dst, static_cast<cudaStream_t>(stream));
    return report(s);
}

int tsr_advance(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l, void* dev0,
                void* dev1, int32_t* cur, int64_t steps, int32_t keep_previous,
                const tsr_opts* opts, void* stream, tsr_stats* stats) {
    if (!k || !g || !dev0 || !dev1 || !cur)
        return report(Status::Err(TSR_EINVAL, "null argument"));
    if (*cur != 0 && *cur != 1) return report(Status::Err(TSR_EINVAL, "cur must be 0 or 1"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    TapSet t;
    if (s.ok()) s = make_taps(*k, t);
    if (!s.ok()) return report(s);
    const tsr_opts o = opts_or_default(opts);
    int c = *cur;
    s = advance_grid(geo, t, o, dev0, dev1, &c, steps, keep_previous != 0,
                static_cast<cudaStream_t>(stream), stats);
    if (s.ok()) *cur = c;
    return report(s);
}

int tsr_sweep_range(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l, const void* in,
                    void* out, int64_t lo, int64_t hi, int32_t steps, const tsr_opts* opts,
                    void* stream) {
    return tsr_sweep_range_mirror(k, g, l, in, out, lo, hi, steps, opts, nullptr, 0, stream);
}

int tsr_sweep_range_mirror(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l,
                           const void* in, void* out, int64_t lo, int64_t hi, int32_t steps,
                           const tsr_opts* opts, void* mirror, int64_t mirror_planes,
                           void* stream) {
    if (!k || !g || !in || !out) return report(Status::Err(TSR_EINVAL, "null argument"));
    if (in == out) return report(Status::Err(TSR_EINVAL, "in and out must be distinct buffers"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    TapSet t;
    if (s.ok()) s = make_taps(*k, t);
    if (s.ok()) s = check_applicable(geo, t);
    if (!s.ok()) return report(s);
    const int64_t n = geo.n[3 - geo.dims];
    if (lo < 0 || hi > n || lo > hi)
        return report(Status::Err(TSR_EINVAL, "plane range outside the grid's axis 0"));
    const tsr_opts o = opts_or_default(opts);
    Plan p;
    s = plan_for(geo, t, o, p);
    if (!s.ok()) return report(s);
    if (steps < 1 || steps > p.k)
        return report(Status::Err(TSR_EINVAL, "steps must be 1..k of the engine plan"));
    LaunchCtx c{&geo, &t, o.mode != TSR_FAST, static_cast<cudaStream_t>(stream)};
    c.lo0 = lo;
    c.hi0 = hi;
    if (mirror) {
        if (mirror == out) return report(Status::Err(TSR_EINVAL, "mirror aliases out"));
        c.mirror = mirror;
        c.mirror_shift = mirror_planes * geo.pitch[3 - geo.dims];  // axis-0 planes -> elements
    }
    return report(sweep(c, p, in, out, steps));
}

int tsr_peer_signal(void* flag, uint32_t value, void* stream) {
    if (!flag) return report(Status::Err(TSR_EINVAL, "null flag"));
    return report(peer_signal(flag, value, static_cast<cudaStream_t>(stream)));
}

int tsr_peer_wait(const void* flag, uint32_t value, void* stream) {
    if (!flag) return report(Status::Err(TSR_EINVAL, "null flag"));
    return report(peer_wait(flag, value, static_cast<cudaStream_t>(stream)));
}

int tsr_peer_round_wait(const void* flag_lo, const void* flag_hi, const void* counter,
                        void* stream) {
    if (!counter) return report(Status::Err(TSR_EINVAL, "null counter"));
    return report(peer_round_wait(flag_lo, flag_hi, counter, static_cast<cudaStream_t>(stream)));
}

int tsr_peer_round_signal(void* peer_lo, void* peer_hi, void* counter, void* stream) {
    if (!counter) return report(Status::Err(TSR_EINVAL, "null counter"));
    return report(peer_round_signal(peer_lo, peer_hi, counter, static_cast<cudaStream_t>(stream)));
}

int tsr_ipc_export(const void* ptr, tsr_ipc_handle* handle, int64_t* offset) {
    if (!ptr || !handle || !offset) return report(Status::Err(TSR_EINVAL, "null argument"));
    return report(ipc_export(ptr, handle->bytes, offset));
}

int tsr_ipc_open(const tsr_ipc_handle* handle, void** base) {
    if (!handle || !base) return report(Status::Err(TSR_EINVAL, "null argument"));
    return report(ipc_open(handle->bytes, base));
}

int tsr_ipc_close(void* base) {
    if (!base) return report(Status::Err(TSR_EINVAL, "null argument"));
    return report(ipc_close(base));
}

int tsr_query_plan(const tsr_kernel* k, const tsr_grid* g, const tsr_opts* opts,
                   int32_t* engine, int32_t* fused_steps) {
    if (!k || !g || !engine || !fused_steps)
        return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    TapSet t;
    if (s.ok()) s = make_taps(*k, t);
    if (s.ok()) s = check_applicable(geo, t);
    Plan p;
    if (s.ok()) s = plan_for(geo, t, opts_or_default(opts), p);
    if (!s.ok()) return report(s);
    *engine = p.engine ? TSR_ENGINE_TUNED : TSR_ENGINE_GENERIC;
    *fused_steps = p.k;
    return TSR_OK;
}

int tsr_apply_box(const tsr_kernel* k, const tsr_grid* g, const tsr_layout* l, const void* in,
                  void* out, const int64_t* lo, const int64_t* hi, const tsr_opts* opts,
                  void* stream) {
    if (!k || !g || !in || !out || !lo || !hi)
        return report(Status::Err(TSR_EINVAL, "null argument"));
    Geo geo;
    Status s = make_geo(*g, geo);
    if (s.ok()) s = check_layout(geo, l);
    TapSet t;
    if (s.ok()) s = make_taps(*k, t);
    if (s.ok()) s = check_applicable(geo, t);
    if (!s.ok()) return report(s);
    const tsr_opts o = opts_or_default(opts);
    int64_t blo[3] = {0, 0, 0}, bhi[3] = {1, 1, 1};
    const int shift = 3 - geo.dims;
    for (int a = 0; a < geo.dims; ++a) {
        blo[a + shift] = std::max<int64_t>(lo[a], 0);
        bhi[a + shift] = std::min<int64_t>(hi[a], geo.n[a + shift]);
        if (blo[a + shift] >= bhi[a + shift]) return TSR_OK;
    }
    LaunchCtx c{&geo, &t, o.mode != TSR_FAST, static_cast<cudaStream_t>(stream)};
    return report(generic_sweep(c, in, out, blo, bhi));
}

}  // extern "C"
