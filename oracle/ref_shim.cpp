// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources (/root/reference/proj/src/*.cpp,
// never copied into this repo) into oracle/_ref/libtessera_ref.so.  It lets
// the tests pin oracle/oracle.c against the real reference and lets
// `bench.py --impl reference` time the reference's own CPU path.
//
// Buffers cross this boundary in the reference's own host layout
// (proj/include/tessera/grid.hpp:46-49), so they are memcpy'd in and out of
// a tessera::BasicGrid<T> verbatim.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "tessera/bench.hpp"
#include "tessera/grid_io.hpp"
#include "tessera/kernel.hpp"
#include "tessera/metrics.hpp"
#include "tessera/naive.hpp"
#include "tessera/parallel.hpp"
#include "tessera/random.hpp"
#include "tessera/scheduler.hpp"
#include "tessera/tiling.hpp"

using namespace tessera;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

Coords coords(int dims, const int64_t* v, Index fill) {
    Coords c{fill, fill, fill};
    for (int a = 0; a < dims; ++a) c[a] = v[a];
    return c;
}

StencilKernel kernel_from(int dims, int shape, int radius, int ntaps, const int32_t* offsets,
                          const double* weights) {
    std::vector<std::pair<Offset, double>> w;
    for (int t = 0; t < ntaps; ++t) {
        Offset o{};
        for (int a = 0; a < 3; ++a) o[a] = offsets[3 * t + a];
        w.push_back({o, weights[t]});
    }
    return make_kernel(dims, shape == 0 ? KernelShape::star : KernelShape::box, radius, w);
}

template <typename T>
BasicGrid<T> grid_in(int dims, const int64_t* ext, const int64_t* halo, const T* b0, const T* b1,
                     int parity) {
    BasicGrid<T> g(dims, coords(dims, ext, 1), coords(dims, halo, 0));
    std::memcpy(g.buffer(0), b0, g.buffer_size() * sizeof(T));
    std::memcpy(g.buffer(1), b1, g.buffer_size() * sizeof(T));
    if (parity) g.flip_parity();
    return g;
}

template <typename T>
void grid_out(const BasicGrid<T>& g, T* b0, T* b1) {
    std::memcpy(b0, g.buffer(0), g.buffer_size() * sizeof(T));
    std::memcpy(b1, g.buffer(1), g.buffer_size() * sizeof(T));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_default_threads() { return default_threads(); }

// Validates a tap list with the reference's make_kernel and writes back the
// canonical tap order (offsets[ntaps*3], weights[ntaps]).  0 ok, -1 invalid.
int ref_make_kernel(int dims, int shape, int radius, int ntaps, int32_t* offsets,
                    double* weights) {
    try {
        const StencilKernel k = kernel_from(dims, shape, radius, ntaps, offsets, weights);
        for (size_t t = 0; t < k.taps().size(); ++t) {
            for (int a = 0; a < 3; ++a) offsets[3 * t + a] = k.taps()[t].offset[a];
            weights[t] = k.taps()[t].weight;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_heat_coefficients(double mu, int32_t* offsets, double* weights) {
    try {
        const StencilKernel k = heat_coefficients(mu);
        for (size_t t = 0; t < k.taps().size(); ++t) {
            for (int a = 0; a < 3; ++a) offsets[3 * t + a] = k.taps()[t].offset[a];
            weights[t] = k.taps()[t].weight;
        }
        return static_cast<int>(k.taps().size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Writes the Table-1 kernel of benchmark `name` (bench.cpp:63-85).  Returns
// ntaps and fills dims/shape/radius plus the tap arrays (capacity 125).
int ref_benchmark_kernel(const char* name, int* dims, int* shape, int* radius, int32_t* offsets,
                         double* weights) {
    try {
        const BenchmarkSpec& s = find_benchmark(name);
        *dims = s.kernel.dims();
        *shape = s.kernel.shape() == KernelShape::star ? 0 : 1;
        *radius = s.kernel.radius();
        for (size_t t = 0; t < s.kernel.taps().size(); ++t) {
            for (int a = 0; a < 3; ++a) offsets[3 * t + a] = s.kernel.taps()[t].offset[a];
            weights[t] = s.kernel.taps()[t].weight;
        }
        return static_cast<int>(s.kernel.taps().size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_fill_random_f64(int dims, const int64_t* ext, const int64_t* halo, uint64_t seed,
                        double lo, double hi, double* b0, double* b1) {
    try {
        Grid g = grid_in<double>(dims, ext, halo, b0, b1, 0);
        fill_random(g, seed, lo, hi);
        grid_out(g, b0, b1);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_fill_random_f32(int dims, const int64_t* ext, const int64_t* halo, uint64_t seed,
                        double lo, double hi, float* b0, float* b1) {
    try {
        GridF g = grid_in<float>(dims, ext, halo, b0, b1, 0);
        fill_random(g, seed, lo, hi);
        grid_out(g, b0, b1);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// naive_run on a grid given by its two buffers and read parity.  Returns the
// final parity, or -1 on error (message in ref_last_error).
int ref_naive_run_f64(int dims, const int64_t* ext, const int64_t* halo, int shape, int radius,
                      int ntaps, const int32_t* offsets, const double* weights, double* b0,
                      double* b1, int parity, int64_t steps) {
    try {
        const StencilKernel k = kernel_from(dims, shape, radius, ntaps, offsets, weights);
        Grid g = grid_in<double>(dims, ext, halo, b0, b1, parity);
        naive_run(g, k, steps);
        grid_out(g, b0, b1);
        return g.parity();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_naive_run_f32(int dims, const int64_t* ext, const int64_t* halo, int shape, int radius,
                      int ntaps, const int32_t* offsets, const double* weights, float* b0,
                      float* b1, int parity, int64_t steps) {
    try {
        const StencilKernel k = kernel_from(dims, shape, radius, ntaps, offsets, weights);
        GridF g = grid_in<float>(dims, ext, halo, b0, b1, parity);
        naive_run(g, k, steps);
        grid_out(g, b0, b1);
        return g.parity();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// run_tessellated (tiling.cpp:137-184), fp64 only like the reference.
// stats_out = {point_updates, rounds, trailing_steps}; *seconds = wall time of
// the run_tessellated call alone.
int ref_run_tessellated(int dims, const int64_t* ext, const int64_t* halo, int shape, int radius,
                        int ntaps, const int32_t* offsets, const double* weights, double* b0,
                        double* b1, int parity, int64_t steps, const int64_t* tile, int tb,
                        int threads, int64_t* stats_out, double* seconds) {
    try {
        const StencilKernel k = kernel_from(dims, shape, radius, ntaps, offsets, weights);
        Grid g = grid_in<double>(dims, ext, halo, b0, b1, parity);
        std::vector<Index> e(ext, ext + dims), t(tile, tile + dims);
        const TilePlan plan = plan_tiles(e, t, tb, radius);
        TessellateStats st;
        const auto t0 = std::chrono::steady_clock::now();
        run_tessellated(g, k, steps, plan, threads, &st);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        grid_out(g, b0, b1);
        if (stats_out) {
            stats_out[0] = st.point_updates;
            stats_out[1] = st.rounds;
            stats_out[2] = st.trailing_steps;
        }
        return g.parity();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Timed naive_run for the fp32 CPU baseline (the reference has no threaded
// fp32 path).  Same contract as ref_naive_run_f32 plus the wall time.
int ref_time_naive_f32(int dims, const int64_t* ext, const int64_t* halo, int shape, int radius,
                       int ntaps, const int32_t* offsets, const double* weights, float* b0,
                       float* b1, int parity, int64_t steps, double* seconds) {
    try {
        const StencilKernel k = kernel_from(dims, shape, radius, ntaps, offsets, weights);
        GridF g = grid_in<float>(dims, ext, halo, b0, b1, parity);
        const auto t0 = std::chrono::steady_clock::now();
        naive_run(g, k, steps);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        grid_out(g, b0, b1);
        return g.parity();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// run_heterogeneous (scheduler.cpp:441-563) with two simulated equal-rate
// workers on the naive engine: the reference's deep-halo two-way partition.
// log_out = {messages, ghost_recompute_points, bytes_of_first_message}.
int ref_run_heterogeneous(int dims, const int64_t* ext, const int64_t* halo, int shape,
                          int radius, int ntaps, const int32_t* offsets, const double* weights,
                          double* b0, double* b1, int parity, int64_t steps, int64_t tile_width,
                          int tb, int threaded, int64_t* log_out, int64_t* boundary_out) {
    try {
        const StencilKernel k = kernel_from(dims, shape, radius, ntaps, offsets, weights);
        Grid g = grid_in<double>(dims, ext, halo, b0, b1, parity);
        WorkerSpec a{WorkerKind::cpu_like, StepEngine::naive, 1.0};
        WorkerSpec b{WorkerKind::accel_like, StepEngine::naive, 1.0};
        std::vector<Index> e(ext, ext + dims);
        auto [pa, pb] = profile_workers(a, b, k, e, 1);
        const PartitionPlan plan = plan_partition(pa, pb, e, tile_width, tb, radius);
        CommLog log;
        run_heterogeneous(g, k, steps, plan, a, b, &log,
                          threaded ? HeteroMode::threaded : HeteroMode::sequential);
        grid_out(g, b0, b1);
        if (log_out) {
            log_out[0] = static_cast<int64_t>(log.records.size());
            log_out[1] = log.ghost_recompute_points;
            log_out[2] = log.records.empty() ? 0 : log.records.front().bytes;
        }
        if (boundary_out) *boundary_out = plan.boundary;
        return g.parity();
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// TTRS dump of the read buffer (grid_io.cpp:34-45).
int ref_dump_grid(const char* path, int dims, const int64_t* ext, const int64_t* halo,
                  const double* b0, const double* b1, int parity) {
    try {
        Grid g = grid_in<double>(dims, ext, halo, b0, b1, parity);
        dump_grid(path, g);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// plan_tiles + count_coverage (tiling.cpp:48-135): out5 = {phase_a size,
// phase_b size, all_ones, min_count, max_count}; tiles_out (capacity cap
// tiles, 7 ints each: kind[3], index[3], wave) lists phase A then phase B.
int ref_plan_tiles(int dims, const int64_t* ext, const int64_t* tile, int tb, int radius,
                   int64_t* out5, int32_t* tiles_out, int64_t cap) {
    try {
        std::vector<Index> e(ext, ext + dims), t(tile, tile + dims);
        const TilePlan p = plan_tiles(e, t, tb, radius);
        const CoverageCount c = count_coverage(p);
        out5[0] = static_cast<int64_t>(p.phase_a.size());
        out5[1] = static_cast<int64_t>(p.phase_b.size());
        out5[2] = c.all_ones();
        out5[3] = c.min_count();
        out5[4] = c.max_count();
        int64_t n = 0;
        for (const auto* ph : {&p.phase_a, &p.phase_b})
            for (const Tile& x : *ph) {
                if (n >= cap) break;
                for (int a = 0; a < 3; ++a) {
                    tiles_out[7 * n + a] = static_cast<int32_t>(x.kind[a]);
                    tiles_out[7 * n + 3 + a] = static_cast<int32_t>(x.index[a]);
                }
                tiles_out[7 * n + 6] = x.wave;
                ++n;
            }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
