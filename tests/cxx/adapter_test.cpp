// The C++ drop-in (include/tessera_b200.hpp) driven with the reference's own
// types, compiled against the unmodified reference headers and library.
// Without a GPU it checks the error paths; with one it checks that
// tessera_b200::naive_run / run_tessellated leave a tessera::BasicGrid<T>
// bitwise as tessera::naive_run does.
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "tessera/bench.hpp"
#include "tessera/kernel.hpp"
#include "tessera/naive.hpp"
#include "tessera/random.hpp"
#include "tessera/scheduler.hpp"
#include "tessera/tiling.hpp"
#include "tessera_b200.hpp"

using namespace tessera;

static int failures = 0;
#define CHECK(c)                                                     \
    do {                                                             \
        if (!(c)) {                                                  \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                              \
        }                                                            \
    } while (0)

template <typename T>
static bool same(const BasicGrid<T>& a, const BasicGrid<T>& b) {
    return a.parity() == b.parity() &&
           std::memcmp(a.buffer(0), b.buffer(0), a.buffer_size() * sizeof(T)) == 0 &&
           std::memcmp(a.buffer(1), b.buffer(1), a.buffer_size() * sizeof(T)) == 0;
}

int main() {
    // Error paths: identical exception classes to the reference.
    {
        Grid g(2, {8, 8, 1}, {1, 1, 0});
        bool threw = false;
        try {
            tessera_b200::naive_run(g, find_benchmark("Heat-3D").kernel, 1);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            tessera_b200::naive_run(g, heat_coefficients(0.2), -1);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    bool gpu = true;
    try {
        Grid g(2, {8, 8, 1}, {1, 1, 0});
        tessera_b200::naive_run(g, heat_coefficients(0.2), 1);
    } catch (const std::runtime_error& e) {
        gpu = false;
        std::printf("no GPU: %s\n", e.what());
    }
    if (gpu) {
        for (const char* name : {"Heat-2D", "Box-2D9P", "Star-2D9P", "Heat-3D", "Box-3D27P",
                                 "Heat-1D", "Box-2D25P"}) {
            const StencilKernel& k = find_benchmark(name).kernel;
            Coords ext{1, 1, 1}, halo{0, 0, 0};
            for (int a = 0; a < k.dims(); ++a) {
                ext[a] = k.dims() == 3 ? 21 + 3 * a : 70 + 9 * a;
                halo[a] = k.radius();
            }
            Grid a(k.dims(), ext, halo), b(k.dims(), ext, halo);
            fill_random(a, 7);
            fill_random(b, 7);
            tessera_b200::naive_run(a, k, 9);
            naive_run(b, k, 9);
            CHECK(same(a, b));
            GridF fa(k.dims(), ext, halo), fb(k.dims(), ext, halo);
            fill_random(fa, 8);
            fill_random(fb, 8);
            tessera_b200::naive_run(fa, k, 5);
            naive_run(fb, k, 5);
            CHECK(same(fa, fb));
            std::printf("%s: %s\n", name, failures ? "mismatch" : "bitwise equal");
        }
        // run_tessellated drop-in incl. TessellateStats (test_tiling.cpp:118-133)
        const StencilKernel k = heat_coefficients(0.24);
        Grid a(2, {64, 64, 1}, {1, 1, 0}), b(2, {64, 64, 1}, {1, 1, 0});
        fill_random(a, 9);
        fill_random(b, 9);
        TessellateStats st;
        tessera_b200::run_tessellated(a, k, 12, plan_tiles({64, 64}, {16, 16}, 3, 1), 1, &st);
        naive_run(b, k, 12);
        CHECK(same(a, b));
        CHECK(st.point_updates == 64 * 64 * 12 && st.rounds == 4 && st.trailing_steps == 0);

        // run_multi: P slabs (sharing the visible devices) == naive_run, both buffers
        for (int P = 1; P <= 4; ++P)
            for (const char* name : {"Heat-3D", "Box-2D9P", "Box-3D27P"}) {
                const StencilKernel& kk = find_benchmark(name).kernel;
                Coords ext{1, 1, 1}, hl{0, 0, 0};
                for (int ax = 0; ax < kk.dims(); ++ax) {
                    ext[ax] = ax == 0 ? 48 : 20 + 5 * ax;
                    hl[ax] = kk.radius();
                }
                Grid x(kk.dims(), ext, hl), y(kk.dims(), ext, hl);
                fill_random(x, 11);
                fill_random(y, 11);
                tessera_b200::MultiOptions mo;
                mo.fused_steps = 2;
                const tsr_stats ms = tessera_b200::run_multi(x, kk, 7, P, mo);
                naive_run(y, kk, 7);
                CHECK(same(x, y));
                CHECK(ms.ngpus == P && (P == 1 || ms.messages > 0));
            }

        // run_heterogeneous with the reference's own plan and CommLog:
        // test_scheduler.cpp:137-158's case, against the reference's run
        {
            const StencilKernel hk = heat_coefficients(0.23);
            WorkerSpec cpu{WorkerKind::cpu_like, StepEngine::naive, 1.0};
            WorkerSpec acc{WorkerKind::accel_like, StepEngine::naive, 1.0};
            auto [pc, pa] = profile_workers(cpu, acc, hk, {16, 16}, 1);
            const PartitionPlan plan = plan_partition(pc, pa, {128, 64}, 16, 3, 1);
            CHECK(plan.boundary == 64);
            Grid x(2, {128, 64, 1}, {1, 1, 0}), y(2, {128, 64, 1}, {1, 1, 0});
            fill_random(x, 500);
            fill_random(y, 500);
            CommLog lx, ly;
            tessera_b200::run_heterogeneous(x, hk, 6, plan, cpu, acc, &lx, HeteroMode::threaded);
            run_heterogeneous(y, hk, 6, plan, cpu, acc, &ly, HeteroMode::sequential);
            CHECK(same(x, y));
            CHECK(lx.records.size() == ly.records.size() && lx.records.size() == 4);
            for (size_t r = 0; r < lx.records.size() && r < ly.records.size(); ++r) {
                CHECK(lx.records[r].round == ly.records[r].round);
                CHECK(lx.records[r].direction == ly.records[r].direction);
                CHECK(lx.records[r].bytes == ly.records[r].bytes);
                CHECK(lx.records[r].modeled_cost_alpha_beta == ly.records[r].modeled_cost_alpha_beta);
            }
            CHECK(lx.ghost_recompute_points == ly.ghost_recompute_points);
            // T = 0 sends nothing; the reference's argument errors
            CommLog l0;
            tessera_b200::run_heterogeneous(x, hk, 0, plan, cpu, acc, &l0);
            CHECK(l0.records.empty());
            bool threw = false;
            try {
                PartitionPlan bad = plan;
                bad.boundary = 1;
                tessera_b200::run_heterogeneous(x, hk, 4, bad, cpu, acc);
            } catch (const std::invalid_argument&) {
                threw = true;
            }
            CHECK(threw);
            std::printf("run_heterogeneous: %zu records, ghost %lld\n", lx.records.size(),
                        static_cast<long long>(lx.ghost_recompute_points));
        }
    }
    std::printf("%s (%s)\n", failures ? "FAILED" : "PASSED", gpu ? "gpu" : "no-gpu");
    return failures ? 1 : 0;
}
