// tessera_b200.hpp — header-only C++ adapter: the reference's run API over the
// C-ABI (tessera_b200.h), for the reference's own types.
//
// A maintainer of the reference (namespace tessera) includes this header and
// calls tessera_b200::naive_run / run_tessellated with an unmodified
// tessera::BasicGrid<T> and tessera::StencilKernel; the signatures mirror
//   naive_run        proj/include/tessera/naive.hpp:96-100
//   naive_step       proj/include/tessera/naive.hpp:89-94
//   run_tessellated  proj/include/tessera/tiling.hpp:82-83
// and errors surface as the same std exceptions (std::invalid_argument for
// bad arguments, std::runtime_error for device failures).  The grid is left
// exactly as the reference leaves it: parity flipped `steps` times, both
// buffers holding steps T and T-1, halo untouched.
//
// The templates only use the public accessors of BasicGrid (dims, extent,
// halo, parity, flip_parity, buffer) and StencilKernel (dims, shape, radius,
// taps), so this header does not include the reference's headers.
#pragma once

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

}  // namespace tessera_b200
