"""Pins the CPU oracle (oracle/oracle.c) before anything is checked against it:
known answers, the reference library itself, and the golden fixtures."""
import os
import zlib

import numpy as np
import pytest

from conftest import GOLDEN, bitwise_equal_interior, golden_index, load_golden, random_grid


def test_mt19937_64_known_answer(orc):
    # C++11 [rand.predef]: the 10000th output of a default-constructed
    # std::mt19937_64 (seed 5489) is 9981545732273789042.
    assert int(orc.mt64(5489, 10000)[-1]) == 9981545732273789042


def test_fill_random_matches_reference(ts, orc, ref):
    for extent, halo, dt in [([7], [2], "f64"), ([6, 9], [1, 2], "f64"), ([5, 4, 6], [1, 1, 1],
                                                                            "f64"),
                             ([5, 4, 6], [1, 1, 1], "f32"), ([3, 8], [1, 1], "f32")]:
        cls = ts.Grid if dt == "f64" else ts.GridF
        a, b, c = cls(extent, halo), cls(extent, halo), cls(extent, halo)
        orc.fill_random(a, 42, -0.5, 2.0)
        ref.fill_random(b, 42, -0.5, 2.0)
        ts.fill_random(c, 42, -0.5, 2.0)  # the product's host-side generator
        for w in (0, 1):
            assert a.buffer(w).tobytes() == b.buffer(w).tobytes()
            assert c.buffer(w).tobytes() == b.buffer(w).tobytes()
        # halo untouched
        mask = np.ones(a.padded(0).shape, bool)
        mask[tuple(slice(h, h + e) for e, h in zip(extent, halo))] = False
        assert not a.padded(0)[mask].any() and not a.padded(1)[mask].any()


@pytest.mark.parametrize("name", ["Heat-1D", "Star-1D5P", "Heat-2D", "Star-2D9P", "Box-2D9P",
                                  "Box-2D25P", "Heat-3D", "Box-3D27P"])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_oracle_naive_run_bitwise_equals_reference(ts, orc, ref, name, dt):
    k = ts.find_benchmark(name).kernel
    rng = np.random.default_rng(zlib.crc32(f"{name}{dt}".encode()))
    for rep in range(2):
        halo = [k.radius + int(rng.integers(0, 2)) for _ in range(k.dims)]
        extent = [int(rng.integers(2 * h + 1, 15 if k.dims == 3 else 40)) for h in halo]
        steps = int(rng.integers(0, 9))
        a = random_grid(ts, orc, extent, halo, 100 + rep, dt)
        b = a.copy()
        orc.naive_run(a, k, steps)
        ref.naive_run(b, k, steps)
        assert a.parity == b.parity == steps % 2
        for w in (0, 1):
            assert a.buffer(w).tobytes() == b.buffer(w).tobytes()


def test_reference_kernels_match_product_definitions(ts, ref):
    """The product's Table-1 kernels carry the reference's exact fp64 weights."""
    for spec in ts.benchmark_table():
        dims, shape, radius, taps = ref.benchmark_kernel(spec.name)
        assert (dims, shape, radius) == (spec.kernel.dims, spec.kernel.shape,
                                         spec.kernel.radius)
        assert [(tuple(o), w) for o, w in taps] == spec.kernel.tap_list()


def test_golden_star2d9p_ttrs(ts, orc):
    """test_stencil_core.cpp:254-270: Star-2D9P 64x64 halo 2 seed 42 T=12, bitwise."""
    golden = ts.load_grid(os.path.join(GOLDEN, "star2d9p_64x64_t12.ttrs"))
    k = ts.find_benchmark("Star-2D9P").kernel
    g = random_grid(ts, orc, [64, 64], [2, 2], 42)
    orc.naive_run(g, k, 12)
    assert golden.extent == [64, 64] and golden.halo == [2, 2]
    assert bitwise_equal_interior(g, golden)


@pytest.mark.parametrize("name", sorted(golden_index()))
def test_oracle_matches_golden_fixtures(ts, orc, name):
    meta = golden_index()[name]
    cur, prev = load_golden(name)
    k = ts.find_benchmark(meta["benchmark"]).kernel
    g = random_grid(ts, orc, meta["extent"], meta["halo"], meta["seed"], meta["dtype"])
    orc.naive_run(g, k, meta["steps"])
    assert g.parity == meta["final_parity"]
    assert g.interior_view(g.parity).tobytes() == cur.tobytes()
    assert g.interior_view(1 - g.parity).tobytes() == prev.tobytes()


def test_known_answers(ts, orc):
    """test_stencil_core.cpp:104-122: convex fixed point and impulse response."""
    k = ts.heat_coefficients(0.25)
    g = ts.Grid([9, 9], [1, 1])
    g.fill(7.5)
    orc.naive_run(g, k, 1)
    assert np.allclose(g.to_numpy(), 7.5, rtol=1e-15)
    imp = ts.Grid([9, 9], [1, 1])
    imp.set_both(4, 4, 0, 1.0)
    orc.naive_run(imp, k, 1)
    assert imp.at(4, 4) == 0.0
    for i, j in [(3, 4), (5, 4), (4, 3), (4, 5)]:
        assert imp.at(i, j) == 0.25
    assert imp.at(3, 3) == 0.0


def test_linearity(ts, orc):
    """test_stencil_core.cpp:199-218."""
    k = ts.find_benchmark("Box-2D9P").kernel
    a, b = 1.7, -0.6
    u = random_grid(ts, orc, [14, 14], [1, 1], 21)
    v = random_grid(ts, orc, [14, 14], [1, 1], 22)
    combo = ts.grid_from_numpy(a * u.to_numpy() + b * v.to_numpy(), [1, 1])
    for g in (u, v, combo):
        orc.naive_run(g, k, 4)
    expect = a * u.to_numpy() + b * v.to_numpy()
    dev = np.max(np.abs(combo.to_numpy() - expect)) / max(np.max(np.abs(expect)), 1.0)
    assert dev < 1e-12


def test_reference_tessellate_equals_oracle(ts, orc, ref):
    """The reference's temporal tiling is bitwise the oracle (survey §0.3)."""
    k = ts.heat_coefficients(0.22)
    a = random_grid(ts, orc, [32, 32], [1, 1], 7)
    b = a.copy()
    (upd, rounds, trailing), _ = ref.run_tessellated(a, k, 7, [8, 8], 3, threads=2)
    orc.naive_run(b, k, 7)
    assert (upd, rounds, trailing) == (32 * 32 * 7, 2, 1)
    assert bitwise_equal_interior(a, b)


def test_reference_heterogeneous_equals_oracle(ts, orc, ref):
    """test_scheduler.cpp:137-158: 2 rounds x 2 messages of 3*64*8 bytes,
    ghost recompute 2*2*3*64, result equal to the oracle."""
    k = ts.heat_coefficients(0.23)
    a = random_grid(ts, orc, [128, 64], [1, 1], 500)
    b = a.copy()
    msgs, ghost, nbytes, boundary = ref.run_heterogeneous(a, k, 6, 16, 3)
    orc.naive_run(b, k, 6)
    assert boundary == 64
    assert (msgs, nbytes, ghost) == (4, 3 * 64 * 8, 2 * 2 * 3 * 64)
    assert bitwise_equal_interior(a, b)


def test_oracle_apply_box_matches_full_sweep(ts, orc):
    """apply_box over a partition of the interior == one full sweep."""
    k = ts.find_benchmark("Heat-3D").kernel
    a = random_grid(ts, orc, [9, 7, 8], [1, 1, 1], 3)
    b = a.copy()
    n = 0
    for lo0, hi0 in [(0, 4), (4, 9)]:
        for lo1, hi1 in [(0, 3), (3, 7)]:
            n += orc.apply_box(a, k, [lo0, lo1, -5], [hi0, hi1, 50], 0)
    a.flip_parity()
    orc.naive_run(b, k, 1)
    assert n == 9 * 7 * 8
    assert bitwise_equal_interior(a, b)


def test_deviation_metric(ts, orc):
    a = random_grid(ts, orc, [6, 6], [1, 1], 1)
    b = a.copy()
    b.buffer(0)[b.flat(2, 3)] += 0.5
    d = orc.deviation(b, a)
    assert d["max_abs_err"] == pytest.approx(0.5)
    assert d["max_rel_deviation"] == pytest.approx(0.5)
    assert d == pytest.approx({k: v for k, v in ts.deviation(b, a).items()
                               if k != "bitwise_equal"})


@pytest.mark.parametrize("name,extent,dt", [("Heat-3D", [120, 100, 96], "f64"),
                                            ("Box-3D27P", [100, 110, 97], "f32"),
                                            ("Box-2D9P", [1200, 1100], "f64")])
def test_threaded_oracle_matches_reference(ts, orc, ref, name, extent, dt):
    """Boxes above 2^20 points run the oracle's row-split host threads; the
    result stays bitwise the reference's serial naive_run."""
    k = ts.find_benchmark(name).kernel
    a = random_grid(ts, orc, extent, [1] * len(extent), 9, dt)
    b = a.copy()
    orc.naive_run(a, k, 3)
    ref.naive_run(b, k, 3)
    assert a.parity == b.parity
    for w in (0, 1):
        assert a.interior_view(w).tobytes() == b.interior_view(w).tobytes()
