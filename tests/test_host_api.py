"""Host-side API of the drop-in (no GPU): kernel definition, grids, plans,
metrics and TTRS I/O behave like the reference's (error classes included)."""
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN


def test_heat_kernel(ts):
    """tests/python/test_smoke.py:7-16 and test_stencil_core.cpp:33-47."""
    k = ts.heat_coefficients(0.23)
    assert (k.dims, k.radius, len(k.taps())) == (2, 1, 5)
    taps = {tuple(off): w for off, w in k.taps()}
    assert taps[(0, 0)] == pytest.approx(0.08, abs=1e-14)
    assert taps[(1, 0)] == 0.23
    k25 = ts.heat_coefficients(0.25)
    assert k25.weight_at([0, 0]) == 0.0 and k25.weight_at([0, -1]) == 0.25
    for bad in (0.3, 0.0, -0.1):
        with pytest.raises(ValueError):
            ts.heat_coefficients(bad)


def test_make_kernel_validation(ts):
    """test_stencil_core.cpp:49-79."""
    k = ts.make_kernel(1, "star", 1, [([1], 0.0), ([0], 1.0), ([-1], 0.0)])
    assert [o for o, _ in k.taps()] == [[-1], [0], [1]]  # canonical order
    w25 = [((i, j), 1.0) for i in range(-2, 3) for j in range(-2, 3)]
    assert len(ts.make_kernel(2, "box", 2, w25).taps()) == 25
    with pytest.raises(ValueError):
        ts.make_kernel(1, "star", 1, [([0], 1.0)])
    with pytest.raises(ValueError):
        ts.make_kernel(2, "star", 1, [((0, 0), 1.0), ((-1, 0), .1), ((1, 0), .1), ((0, -1), .1),
                                      ((1, 1), .1)])
    with pytest.raises(ValueError):
        ts.make_kernel(1, "star", 1, [([-1], 0.0), ([0], math.nan), ([1], 0.0)])
    with pytest.raises(ValueError):
        ts.make_kernel(1, "diamond", 1, [([0], 1.0)])
    with pytest.raises(ValueError):
        ts.make_kernel(1, "star", 0, [([0], 1.0)])


def test_table1_point_counts(ts):
    """test_harness.cpp:40-62: point counts and unit weight sums."""
    counts = {"Heat-1D": 3, "Star-1D5P": 5, "Heat-2D": 5, "Star-2D9P": 9, "Box-2D9P": 9,
              "Box-2D25P": 25, "Heat-3D": 7, "Box-3D27P": 27}
    for spec in ts.benchmark_table():
        assert len(spec.kernel.taps()) == counts[spec.name]
        assert spec.kernel.weight_sum == pytest.approx(1.0, abs=1e-12)
    assert "Heat-3D" in ts.benchmark_names()
    with pytest.raises(ValueError):
        ts.find_benchmark("Heat-4D")


def test_line_weights(ts):
    k = ts.find_benchmark("Star-2D9P").kernel
    assert k.line_weights(0, [0, 0]) == [0.08, 0.12, 0.2, 0.12, 0.08]
    assert k.line_weights(1, [1, 0]) == [0.0, 0.0, 0.12, 0.0, 0.0]


def test_grid_validation_and_layout(ts):
    """grid.hpp:29-52 and test_stencil_core.cpp:91-102."""
    with pytest.raises(ValueError):
        ts.Grid([2, 8], [1, 1])
    with pytest.raises(ValueError):
        ts.Grid([6], [4])
    with pytest.raises(ValueError):
        ts.Grid([5, 5], [1, -1])
    g = ts.Grid([4, 5, 7], [1, 2, 3])
    assert [g.stride(a) for a in range(3)] == [(5 + 4) * (7 + 6), 7 + 6, 1]
    assert g.flat(-1, -2, -3) == 0
    assert g.buffer_size() == 6 * 9 * 13
    assert g.parity == 0
    g.flip_parity()
    assert g.parity == 1


def test_grid_numpy_roundtrip(ts):
    """tests/python/test_smoke.py:25-29."""
    field = np.arange(48, dtype=np.float64).reshape(6, 8)
    g = ts.grid_from_numpy(field, halo=[1, 1])
    assert g.extent == [6, 8]
    np.testing.assert_array_equal(g.to_numpy(), field)
    h = ts.grid_from_numpy(field, halo=[2, 1], halo_value=3.5)
    assert h.at(-2, -1) == 3.5 and h.buffer(1)[h.flat(5, 8)] == 3.5
    f = ts.grid_from_numpy(field.astype(np.float32), dtype=np.float32)
    assert isinstance(f, ts.GridF) and f.to_numpy().dtype == np.float32


def test_ttrs_roundtrip_and_golden_header(ts, tmp_path):
    """test_stencil_core.cpp:240-252 and the TTRS layout (grid_io.cpp:34-45)."""
    g = ts.Grid([12, 6], [2, 1])
    ts.fill_random(g, 33)
    g.flip_parity()
    path = str(tmp_path / "roundtrip.ttrs")
    ts.dump_grid(path, g)
    back = ts.load_grid(path)
    assert (back.dims, back.extent, back.halo, back.parity) == (2, [12, 6], [2, 1], 0)
    assert back.buffer(0).tobytes() == g.read_data().tobytes()
    assert back.buffer(1).tobytes() == g.read_data().tobytes()
    golden = ts.load_grid(os.path.join(GOLDEN, "star2d9p_64x64_t12.ttrs"))
    assert os.path.getsize(os.path.join(GOLDEN, "star2d9p_64x64_t12.ttrs")) == 37036
    assert golden.buffer_size() == 68 * 68


def test_plan_tiles_validation(ts):
    """tiling.cpp:48-72 and test_tiling.cpp:52-56, 136-144."""
    p = ts.plan_tiles([12], [6], 3, 1)
    assert (p.upright_tiles, p.inverted_tiles, p.tb) == (2, 2, 3)
    with pytest.raises(ValueError):
        ts.plan_tiles([12], [4], 3, 1)
    with pytest.raises(ValueError):
        ts.plan_tiles([32, 32], [16, 4], 3, 1)
    with pytest.raises(ValueError):
        ts.plan_tiles([12], [6], 0, 1)
    g = ts.Grid([16, 16], [2, 2])
    with pytest.raises(ValueError):  # plan radius 1 vs kernel radius 2
        ts.run_tessellated(g, ts.find_benchmark("Star-2D9P").kernel, 3,
                           ts.plan_tiles([16, 16], [8, 8], 2, 1))
    with pytest.raises(ValueError):  # extent mismatch
        ts.run_tessellated(g, ts.heat_coefficients(0.2), 3, ts.plan_tiles([32, 16], [8, 8], 2, 1))


def test_stencils_per_second(ts):
    """test_stencil_core.cpp:220-238 incl. Table 4's 82.9 / 2.8 GStencil/s."""
    fast = ts.stencils_per_second([9600, 9600], 3_800_000, 4270.9)
    assert fast.stencils_per_second == pytest.approx(8.2e10, rel=0.01)
    slow = ts.stencils_per_second([9600, 9600], 3_800_000, 124_448.5)
    assert slow.stencils_per_second == pytest.approx(2.8e9, rel=0.01)
    r = ts.stencils_per_second([10], 10, 1.0)
    assert (r.stencils_per_second, r.points_per_step) == (100.0, 10)
    for bad in (0.0, -2.0):
        with pytest.raises(ValueError):
            ts.stencils_per_second([10], 10, bad)


def test_max_rel_deviation(ts):
    a = ts.grid_from_numpy(np.full((4, 4), 10.0))
    b = ts.grid_from_numpy(np.full((4, 4), 10.0))
    b.buffer(0)[b.flat(1, 1)] = 12.0
    assert ts.max_rel_deviation(b, a) == pytest.approx(0.2)
    assert ts.max_abs(b) == 12.0
    b.buffer(0)[b.flat(2, 2)] = np.nan
    assert ts.max_rel_deviation(b, a) == math.inf
    with pytest.raises(ValueError):
        ts.max_rel_deviation(a, ts.grid_from_numpy(np.zeros((4, 5))))


def test_gpu_entry_points_fail_loudly_without_a_device(ts):
    """No CPU fallback: without CUDA the sweep raises instead of computing."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    g = ts.Grid([8, 8], [1, 1])
    with pytest.raises(RuntimeError, match="CUDA"):
        ts.naive_run(g, ts.heat_coefficients(0.2), 2)
    assert g.parity == 0


@pytest.mark.parametrize("extent,tile,tb", [([64, 64], [20, 20], 3), ([200, 37], [50, 12], 4),
                                            ([20, 21, 23], [6, 6, 7], 2), ([97], [10], 5),
                                            ([30, 31, 32], [10, 10, 10], 5)])
def test_tile_plan_matches_reference(ts, ref, extent, tile, tb):
    """plan_tiles' phase A / phase B lists (kind, index, wave, in order) and
    count_coverage's (all_ones, min, max) are the reference's
    (tiling.cpp:48-135, module.cpp:180-193)."""
    p = ts.plan_tiles(extent, tile, tb, 1)
    up, inv, cov, tiles = ref.plan_tiles(extent, tile, tb, 1)
    assert (p.upright_tiles, p.inverted_tiles) == (up, inv)
    assert [(t.kind, t.index, t.wave) for t in p.phase_a + p.phase_b] == tiles
    assert ts.count_coverage(p) == cov == (True, 1, 1)
    for t in p.phase_b[:3]:
        for s in range(tb):
            lo, hi = ts.tile_range(p, t, s)
            assert all(0 <= l <= h <= e for l, h, e in zip(lo, hi, extent))
