// tessera_b200.hpp — header-only C++ adapter: the reference's run API over the
// C-ABI (tessera_b200.h), for the reference's own types.
//
// A maintainer of the reference (namespace tessera) includes this header and
// calls tessera_b200::naive_run / run_tessellated with an unmodified
// tessera::BasicGrid<T> and tessera::StencilKernel; the signatures mirror
//   naive_run        proj/include/tessera/naive.hpp:96-100
//   naive_step       proj/include/tessera/naive.hpp:89-94
//   run_tessellated  proj/include/tessera/tiling.hpp:82-83
//   run_heterogeneous proj/include/tessera/scheduler.hpp:109-113 (two GPU
//                    slabs, the reference's PartitionPlan / WorkerSpec /
//                    CommLog / HeteroMode / CommCostModel)
// plus run_multi (P slabs on P GPUs from this thread, tsr_run_multi),
// and errors surface as the same std exceptions (std::invalid_argument for
// bad arguments, std::runtime_error for device failures).  The grid is left
// exactly as the reference leaves it: parity flipped `steps` times, both
// buffers holding steps T and T-1, halo untouched.
//
// The templates only use the public accessors of BasicGrid (dims, extent,
// halo, parity, flip_parity, buffer) and StencilKernel (dims, shape, radius,
// taps), so this header does not include the reference's headers.
#pragma once

#include <algorithm>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "tessera_b200.h"

namespace tessera_b200 {

struct GpuOptions {
    int fused_steps = 0;           // k time steps per HBM pass (0 = engine default)
    bool exact = true;             // bitwise naive_run; false = FMA (within 1e-12 / 1e-5)
    int engine = TSR_ENGINE_AUTO;  // TSR_ENGINE_GENERIC forces the one-thread-per-point kernel
    int device = -1;               // CUDA ordinal, -1 = current
};

using GpuStats = tsr_stats;

inline void throw_status(int code) {
    switch (code) {
        case TSR_OK: return;
        case TSR_EINVAL: throw std::invalid_argument(tsr_last_error());
        case TSR_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(std::string("tessera_b200: ") + tsr_last_error());
    }
}

// tsr_kernel view of a StencilKernel (canonical tap order is the kernel's own).
class KernelView {
public:
    template <class Kernel>
    explicit KernelView(const Kernel& k) {
        for (const auto& tap : k.taps()) {
            for (int a = 0; a < 3; ++a) offsets_.push_back(static_cast<int32_t>(tap.offset[a]));
            weights_.push_back(tap.weight);
        }
        view_.dims = k.dims();
        view_.shape = static_cast<int32_t>(k.shape());  // KernelShape{star, box} == {0, 1}
        view_.radius = k.radius();
        view_.ntaps = static_cast<int32_t>(weights_.size());
        view_.offsets = offsets_.data();
        view_.weights = weights_.data();
    }
    const tsr_kernel* get() const { return &view_; }

private:
    std::vector<int32_t> offsets_;
    std::vector<double> weights_;
    tsr_kernel view_{};
};

template <class Grid>
using value_type_of = std::remove_cv_t<std::remove_pointer_t<decltype(std::declval<Grid&>().buffer(0))>>;

template <class Grid>
tsr_grid grid_desc(const Grid& g) {
    using T = value_type_of<Grid>;
    static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>,
                  "tessera_b200 serves BasicGrid<double> and BasicGrid<float>");
    tsr_grid d{};
    d.dims = g.dims();
    d.dtype = std::is_same_v<T, double> ? TSR_F64 : TSR_F32;
    for (int a = 0; a < 3; ++a) {
        d.extent[a] = a < g.dims() ? g.extent(a) : 1;
        d.halo[a] = a < g.dims() ? g.halo(a) : 0;
    }
    return d;
}

// Advances `steps` time steps on the GPU; the grid ends as naive_run leaves it.
template <class Grid, class Kernel>
GpuStats run_gpu(Grid& g, const Kernel& k, std::int64_t steps, const GpuOptions& o = {}) {
    if (steps < 0) throw std::invalid_argument("negative step count");  // naive.hpp:98
    const KernelView kv(k);
    const tsr_grid gd = grid_desc(g);
    tsr_opts opts{};
    opts.fused_steps = o.fused_steps;
    opts.mode = o.exact ? TSR_EXACT : TSR_FAST;
    opts.engine = o.engine;
    opts.device = o.device;
    GpuStats st{};
    throw_status(tsr_run(kv.get(), &gd, g.buffer(0), g.buffer(1), g.parity(), steps, &opts, &st));
    if (steps & 1) g.flip_parity();
    return st;
}

template <class Grid, class Kernel>
void naive_run(Grid& g, const Kernel& k, std::int64_t steps) {
    run_gpu(g, k, steps);
}

template <class Grid, class Kernel>
void naive_step(Grid& g, const Kernel& k) {
    run_gpu(g, k, 1);
}

// run_tessellated (tiling.cpp:137-184): the plan's tb becomes the number of
// fused steps per HBM pass; stats mirror TessellateStats.
template <class Grid, class Kernel, class Plan, class Stats = void>
void run_tessellated(Grid& g, const Kernel& k, std::int64_t steps, const Plan& plan,
                     int /*threads*/ = 1, Stats* stats = nullptr) {
    if (k.radius() != plan.radius)
        throw std::invalid_argument("plan radius differs from kernel radius");
    if (plan.dims != g.dims()) throw std::invalid_argument("plan dimensionality differs from grid");
    for (int a = 0; a < g.dims(); ++a)
        if (plan.extent[a] != g.extent(a))
            throw std::invalid_argument("plan extent differs from grid extent");
    GpuOptions o;
    o.fused_steps = plan.tb;
    run_gpu(g, k, steps, o);
    if constexpr (!std::is_void_v<Stats>) {
        if (stats) {
            std::int64_t pts = 1;
            for (int a = 0; a < g.dims(); ++a) pts *= g.extent(a);
            stats->point_updates = pts * steps;
            stats->rounds = steps / plan.tb;
            stats->trailing_steps = steps % plan.tb;
        }
    }
}

// ---- slabs on several GPUs (tsr_run_multi / tsr_multi_*) ----------------

struct MultiOptions : GpuOptions {
    std::vector<int32_t> devices;          // slab i on devices[i]; empty = i mod device count
    std::vector<std::int64_t> boundaries;  // ngpus-1 ascending axis-0 boundaries; empty = equal
    int transport = TSR_XPORT_AUTO;
    bool keep_previous = true;  // both buffers as naive_run leaves them; false: only the final
                                // read buffer is written (run_heterogeneous's post-condition)
};

inline tsr_partition partition_of(int ngpus, const MultiOptions& o, int flags = 0) {
    tsr_partition p{};
    p.ngpus = ngpus;
    p.split_axis = 0;
    p.devices = o.devices.empty() ? nullptr : o.devices.data();
    p.boundaries = o.boundaries.empty() ? nullptr : o.boundaries.data();
    p.transport = o.transport;
    p.flags = flags;
    return p;
}

// naive_run over `ngpus` slabs of axis 0 in one call: host buffers in, host
// buffers out, the grid left as naive_run leaves it (keep_previous).
template <class Grid, class Kernel>
GpuStats run_multi(Grid& g, const Kernel& k, std::int64_t steps, int ngpus,
                   const MultiOptions& o = {}) {
    if (steps < 0) throw std::invalid_argument("negative step count");
    if (ngpus < 1) throw std::invalid_argument("ngpus must be >= 1");
    const KernelView kv(k);
    const tsr_grid gd = grid_desc(g);
    tsr_opts opts{};
    opts.fused_steps = o.fused_steps;
    opts.mode = o.exact ? TSR_EXACT : TSR_FAST;
    opts.engine = o.engine;
    opts.device = -1;
    opts.ngpus = ngpus;
    const tsr_partition part = partition_of(ngpus, o);
    GpuStats st{};
    throw_status(tsr_run_multi(kv.get(), &gd, g.buffer(0), g.buffer(1), g.parity(), steps, &part,
                               o.keep_previous ? 1 : 0, &opts, &st));
    if (steps & 1) g.flip_parity();
    return st;
}

namespace detail {
template <class M, class = void>
struct has_alpha_beta : std::false_type {};
template <class M>
struct has_alpha_beta<M, std::void_t<decltype(std::declval<const M&>().alpha),
                                     decltype(std::declval<const M&>().beta)>> : std::true_type {};

// The reference's run_heterogeneous_impl (scheduler.cpp:441-563) on two GPU
// slabs split at plan.boundary, rounds of plan.tb steps (clamped to the
// engine's fused depth), deep halo r*k; the CommLog gets one record per
// seam delivery (round, "w0_to_w1" / "w1_to_w0", bytes, alpha-beta cost,
// the sender's seam-pass device time) and the ghost recompute tally.
template <class Grid, class Kernel, class Plan, class Log>
void hetero(Grid& g, const Kernel& k, std::int64_t steps, const Plan& plan, Log* log,
            double alpha, double beta, bool poison) {
    // the reference's checks, in its order
    if (g.dims() != k.dims()) throw std::invalid_argument("kernel/grid dimensionality mismatch");
    for (int a = 0; a < g.dims(); ++a)
        if (g.halo(a) < k.radius()) throw std::invalid_argument("grid halo too small for kernel radius");
    if (steps < 0) throw std::invalid_argument("negative step count");
    if (k.radius() != plan.radius)
        throw std::invalid_argument("partition plan radius differs from kernel radius");
    if (plan.halo_depth != static_cast<std::int64_t>(plan.radius) * plan.tb)
        throw std::invalid_argument("partition plan halo depth must be radius*tb");
    const std::int64_t n = g.extent(0), b = plan.boundary;
    if (b <= 0 || b >= n) throw std::invalid_argument("partition boundary outside the grid");
    if (b < plan.halo_depth || n - b < plan.halo_depth)
        throw std::invalid_argument("subdomain smaller than the halo depth");
    if (log) *log = Log{};
    if (steps == 0) return;

    const KernelView kv(k);
    const tsr_grid gd = grid_desc(g);
    tsr_opts opts{};
    opts.fused_steps = plan.tb;
    opts.mode = TSR_EXACT;
    opts.engine = TSR_ENGINE_AUTO;
    opts.device = -1;
    opts.ngpus = 2;
    MultiOptions mo;
    mo.boundaries = {b};
    const tsr_partition part = partition_of(2, mo, poison ? TSR_PART_POISON : 0);
    tsr_multi* m = nullptr;
    throw_status(tsr_multi_create(kv.get(), &gd, &part, &opts, &m));
    struct Guard {
        tsr_multi* m;
        ~Guard() { tsr_multi_destroy(m); }
    } guard{m};
    throw_status(tsr_multi_upload(m, g.buffer(g.parity())));
    throw_status(tsr_multi_set_logging(m, log ? 1 : 0));
    GpuStats st{};
    throw_status(tsr_multi_advance(m, steps, 0, &st));
    if (steps & 1) g.flip_parity();
    // run_heterogeneous scatters the workers' rows into the final read
    // buffer only (scheduler.cpp:555-557)
    throw_status(tsr_multi_download(m, g.buffer(g.parity()), nullptr));
    if (log) {
        std::int64_t count = 0;
        throw_status(tsr_multi_comm_log(m, nullptr, 0, &count));
        std::vector<tsr_comm_record> recs(static_cast<size_t>(count));
        throw_status(tsr_multi_comm_log(m, recs.data(), count, &count));
        for (const tsr_comm_record& r : recs) {
            typename std::decay_t<decltype(log->records)>::value_type c{};
            c.round = r.round;
            c.direction = "w" + std::to_string(r.from_slab) + "_to_w" + std::to_string(r.to_slab);
            c.bytes = r.bytes;
            c.modeled_cost_alpha_beta = alpha + static_cast<double>(r.bytes) * beta;
            c.wall_seconds = r.seam_ms / 1e3;
            log->records.push_back(c);
        }
        std::sort(log->records.begin(), log->records.end(), [](const auto& x, const auto& y) {
            return x.round != y.round ? x.round < y.round : x.direction < y.direction;
        });
        log->ghost_recompute_points = st.ghost_recompute_points;
    }
}
}  // namespace detail

// run_heterogeneous (scheduler.hpp:109-113): the same call, the two workers
// become two GPU slabs (the worker specs and the drive mode only select the
// reference's CPU engines and threads; every GPU slab runs the tuned engine
// from one host thread, which gives the same bits as both of its drives).
template <class Grid, class Kernel, class Plan, class Worker, class Log = void, class Mode = int,
          class Model = int>
void run_heterogeneous(Grid& g, const Kernel& k, std::int64_t steps, const Plan& plan,
                       const Worker& /*first*/, const Worker& /*second*/, Log* log = nullptr,
                       Mode /*mode*/ = Mode{}, const Model& model = Model{}) {
    double alpha = 1e-5, beta = 1e-9;  // CommCostModel defaults (scheduler.hpp:66-73)
    if constexpr (detail::has_alpha_beta<Model>::value) {
        alpha = model.alpha;
        beta = model.beta;
    }
    if constexpr (std::is_void_v<Log>) {
        struct NoRec {
            std::int64_t round;
            std::string direction;
            std::int64_t bytes;
            double modeled_cost_alpha_beta, wall_seconds;
        };
        struct NoLog {
            std::vector<NoRec> records;
            std::int64_t ghost_recompute_points = 0;
        };
        detail::hetero(g, k, steps, plan, static_cast<NoLog*>(nullptr), alpha, beta, false);
    } else {
        detail::hetero(g, k, steps, plan, log, alpha, beta, false);
    }
}

}  // namespace tessera_b200
