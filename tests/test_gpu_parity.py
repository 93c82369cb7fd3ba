"""GPU parity: every engine against the CPU oracle (pinned in test_oracle.py)
and the reference's golden fixtures.  EXACT mode must be bitwise equal;
FAST mode within the north star's tolerances (1e-12 fp64, 1e-5 fp32, as
max-rel / L2-rel after N steps)."""
import os

import numpy as np
import pytest

from conftest import (GOLDEN, bitwise_equal_interior, golden_index, load_golden, random_grid)

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}


def both_buffers_equal(a, b):
    return (a.parity == b.parity and
            a.interior_view(0).tobytes() == b.interior_view(0).tobytes() and
            a.interior_view(1).tobytes() == b.interior_view(1).tobytes())


def both_buffers_equal_planes(a, b):
    """both_buffers_equal one axis-0 plane at a time (no full-grid copies)."""
    if a.parity != b.parity:
        return False
    for w in (0, 1):
        x, y = a.interior_view(w), b.interior_view(w)
        if any(x[i].tobytes() != y[i].tobytes() for i in range(x.shape[0])):
            return False
    return True


def halos_equal(a, b):
    mask = np.ones(a.padded(0).shape, bool)
    mask[tuple(slice(h, h + e) for e, h in zip(a.extent, a.halo))] = False
    return all(a.padded(w)[mask].tobytes() == b.padded(w)[mask].tobytes() for w in (0, 1))


@pytest.mark.parametrize("engine", ["auto", "generic"])
@pytest.mark.parametrize("name", sorted(golden_index()))
def test_golden_fixtures(ts, orc, name, engine):
    meta = golden_index()[name]
    cur, prev = load_golden(name)
    k = ts.find_benchmark(meta["benchmark"]).kernel
    g = random_grid(ts, orc, meta["extent"], meta["halo"], meta["seed"], meta["dtype"])
    ts.run_gpu(g, k, meta["steps"], engine=engine)
    assert g.parity == meta["final_parity"]
    assert g.interior_view(g.parity).tobytes() == cur.tobytes()
    assert g.interior_view(1 - g.parity).tobytes() == prev.tobytes()


def test_golden_star2d9p_ttrs(ts, orc):
    golden = ts.load_grid(os.path.join(GOLDEN, "star2d9p_64x64_t12.ttrs"))
    g = random_grid(ts, orc, [64, 64], [2, 2], 42)
    ts.naive_run(g, ts.find_benchmark("Star-2D9P").kernel, 12)
    assert bitwise_equal_interior(g, golden)


@pytest.mark.parametrize("name", ["Heat-2D", "Box-2D9P", "Star-2D9P", "Box-2D25P"])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_fused_2d_bitwise_all_k(ts, orc, name, dt):
    """Every fused step count the engine accepts (1..8; 1..2 for the 25-point
    box), T not a multiple of k, ragged extents (narrower than one strip,
    wider than several), halo wider than r."""
    k = ts.find_benchmark(name).kernel
    rng = np.random.default_rng(7)
    kmax = 2 if name == "Box-2D25P" else 8
    for fused in range(1, kmax + 1):
        for extent in ([int(rng.integers(5, 40)), int(rng.integers(5, 30))],
                       [int(rng.integers(60, 130)), int(rng.integers(100, 300))]):
            halo = [k.radius + int(rng.integers(0, 2)), k.radius + int(rng.integers(0, 3))]
            extent = [max(e, 2 * h + 1) for e, h in zip(extent, halo)]
            steps = int(rng.integers(fused, 3 * fused + 2))
            a = random_grid(ts, orc, extent, halo, fused * 31 + extent[0], dt)
            b = a.copy()
            st = ts.run_gpu(a, k, steps, fused_steps=fused, engine="tuned")
            orc.naive_run(b, k, steps)
            assert st.fused_steps == fused
            assert both_buffers_equal(a, b), (fused, extent, halo, steps)
            assert halos_equal(a, b)


@pytest.mark.parametrize("name", ["Heat-1D", "Star-1D5P"])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_fused_1d_bitwise(ts, orc, name, dt):
    """The 1-D shared-memory engine: fused depths up to 16, segments shorter
    and longer than one CTA's 2048 points, halo wider than r, T not a multiple
    of k — bitwise naive_run, halo untouched."""
    k = ts.find_benchmark(name).kernel
    rng = np.random.default_rng(11)
    for fused in (1, 2, 3, 5, 8, 13, 16):
        for n in (int(rng.integers(5, 60)), 2048, int(rng.integers(2049, 9000))):
            halo = [k.radius + int(rng.integers(0, 3))]
            n = max(n, 2 * halo[0] + 1)
            steps = int(rng.integers(fused, 3 * fused + 2))
            a = random_grid(ts, orc, [n], halo, fused * 7 + n, dt)
            b = a.copy()
            st = ts.run_gpu(a, k, steps, fused_steps=fused, engine="tuned")
            orc.naive_run(b, k, steps)
            assert st.fused_steps == fused and st.engine == "tuned"
            assert both_buffers_equal(a, b), (fused, n, halo, steps)
            assert halos_equal(a, b)


@pytest.mark.parametrize("fused", [1, 2, 3])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_heat3d_tuned_bitwise(ts, orc, dt, fused):
    """tb3d: every fused depth, tiles cut by the grid edge in a1/a2, chunked
    a0, halo wider than r, grids smaller than one tile."""
    k = ts.find_benchmark("Heat-3D").kernel
    for extent, halo, steps in [([17, 13, 35], [1, 1, 1], 5), ([40, 33, 70], [2, 1, 3], 7),
                                ([3, 3, 3], [1, 1, 1], 3), ([130, 70, 131], [1, 1, 1], 4)]:
        a = random_grid(ts, orc, extent, halo, sum(extent), dt)
        b = a.copy()
        st = ts.run_gpu(a, k, steps, fused_steps=fused, engine="tuned")
        orc.naive_run(b, k, steps)
        assert st.engine == "tuned" and st.fused_steps == fused
        assert both_buffers_equal(a, b), (extent, steps)
        assert halos_equal(a, b)


@pytest.mark.parametrize("fused", [1, 2, 3])
def test_heat3d_fast_is_bitwise_for_power_of_two_weights(ts, orc, fused):
    """Heat-3D's weights are 1/4 and 1/8: every product is exact on
    normal-range data, so FAST (one FMA per tap) equals the oracle's mul + add
    bitwise — the property the bench's fast_vs_exact flag reports at full
    size.  Covers boundary-tile warps on interior planes (the column-select
    tier), fill/drain units and a0-boundary planes."""
    k = ts.find_benchmark("Heat-3D").kernel
    for extent, halo, steps in [([130, 70, 131], [1, 1, 1], 6), ([64, 61, 190], [1, 2, 1], 9),
                                ([17, 13, 35], [1, 1, 1], 5)]:
        a = random_grid(ts, orc, extent, halo, 11, "f64")
        b = a.copy()
        ts.run_gpu(a, k, steps, fused_steps=fused, mode="fast", engine="tuned")
        orc.naive_run(b, k, steps)
        assert both_buffers_equal(a, b), (extent, steps)


def test_star7_general_weights_3d(ts, orc):
    """Non-uniform, non-power-of-two 7-point weights (tap order matters)."""
    w = [((-1, 0, 0), 0.11), ((0, -1, 0), 0.13), ((0, 0, -1), 0.17), ((0, 0, 0), 0.19),
         ((0, 0, 1), 0.07), ((0, 1, 0), 0.2), ((1, 0, 0), 0.13)]
    k = ts.make_kernel(3, "star", 1, w)
    for fused in (1, 2, 3):
        a = random_grid(ts, orc, [37, 45, 80], [1, 1, 1], fused)
        b = a.copy()
        ts.run_gpu(a, k, 9, fused_steps=fused)
        orc.naive_run(b, k, 9)
        assert both_buffers_equal(a, b), fused


@pytest.mark.parametrize("name", ["Heat-1D", "Star-1D5P", "Box-2D25P", "Box-3D27P"])
def test_generic_engine_bitwise(ts, orc, name):
    k = ts.find_benchmark(name).kernel
    ext = {1: [301], 2: [37, 41], 3: [11, 19, 23]}[k.dims]
    a = random_grid(ts, orc, ext, [k.radius] * k.dims, 5)
    b = a.copy()
    st = ts.run_gpu(a, k, 6, engine="generic")
    orc.naive_run(b, k, 6)
    assert st.engine == "generic"
    assert both_buffers_equal(a, b)


@pytest.mark.parametrize("fused", [1, 2])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_box27_planesum_bitwise(ts, orc, dt, fused):
    """box3d engine (k=1 and the k=2 two-level plane-sum pipeline): per-plane
    partial sums keep the oracle's tap order; tiles cut by the grid edge,
    chunked a0, halo wider than r, non-zero Dirichlet halo."""
    k = ts.find_benchmark("Box-3D27P").kernel
    for extent, halo, steps in [([11, 19, 23], [1, 1, 1], 4), ([70, 45, 150], [2, 1, 3], 5),
                                ([3, 3, 3], [1, 1, 1], 2), ([40, 66, 130], [1, 1, 1], 3)]:
        a = random_grid(ts, orc, extent, halo, sum(extent), dt)
        a.padded(0)[0] = 2.5  # a non-zero halo plane in both buffers
        a.padded(1)[0] = 2.5
        b = a.copy()
        st = ts.run_gpu(a, k, steps, engine="tuned", fused_steps=fused)
        orc.naive_run(b, k, steps)
        assert st.engine == "tuned" and st.fused_steps == fused
        assert both_buffers_equal(a, b), extent
        assert halos_equal(a, b)


@pytest.mark.parametrize("name", ["Heat-2D", "Box-2D9P", "Heat-3D", "Box-3D27P"])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_fast_mode_within_tolerance(ts, orc, name, dt):
    k = ts.find_benchmark(name).kernel
    ext = [96, 130] if k.dims == 2 else [20, 24, 40]
    a = random_grid(ts, orc, ext, [1] * k.dims, 3, dt)
    b = a.copy()
    ts.run_gpu(a, k, 40, mode="fast")
    orc.naive_run(b, k, 40)
    d = ts.deviation(a, b)
    assert d["max_rel_deviation"] <= TOL[dt] and d["l2_rel_err"] <= TOL[dt], d


def test_step_counts_and_postconditions(ts, orc):
    """T = 0, 1, 2 and odd/even T leave parity and both buffers as naive_run."""
    k = ts.heat_coefficients(0.23)
    for steps in (0, 1, 2, 3, 8, 9):
        a = random_grid(ts, orc, [50, 70], [1, 1], steps)
        b = a.copy()
        ts.naive_run(a, k, steps)
        orc.naive_run(b, k, steps)
        assert both_buffers_equal(a, b), steps
        assert halos_equal(a, b)


def test_nonzero_dirichlet_halo(ts, orc):
    """Halo values other than zero are read, never written, at every fused level."""
    rng = np.random.default_rng(1)
    for name, shape in [("Heat-2D", (45, 67)), ("Box-2D9P", (45, 67)), ("Heat-3D", (9, 14, 40))]:
        k = ts.find_benchmark(name).kernel
        a = ts.grid_from_numpy(rng.random(shape), halo=[2] * len(shape), halo_value=3.5)
        b = a.copy()
        ts.run_gpu(a, k, 7, fused_steps=4)
        orc.naive_run(b, k, 7)
        assert both_buffers_equal(a, b) and halos_equal(a, b)


def test_run_tessellated_drop_in(ts, orc):
    """tests/python/test_smoke.py:49-61 on the GPU path."""
    rng = np.random.default_rng(7)
    field = rng.random((32, 32))
    k = ts.heat_coefficients(0.22)
    a = ts.grid_from_numpy(field, halo=[1, 1])
    b = ts.grid_from_numpy(field, halo=[1, 1])
    plan = ts.plan_tiles([32, 32], [8, 8], 3, 1)
    updates, rounds, trailing = ts.run_tessellated(a, k, 7, plan)
    orc.naive_run(b, k, 7)
    assert updates == 32 * 32 * 7 and (rounds, trailing) == (2, 1)
    assert ts.max_rel_deviation(a, b) <= 1e-12
    assert bitwise_equal_interior(a, b)


def test_device_grid_roundtrip(ts, orc):
    k = ts.find_benchmark("Box-2D9P").kernel
    a = random_grid(ts, orc, [130, 250], [1, 1], 11)
    b = a.copy()
    dg = ts.DeviceGrid(a)
    dg.advance(k, 5, fused_steps=4)
    dg.advance(k, 6, fused_steps=3, keep_previous=True)
    dg.download(a)
    orc.naive_run(b, k, 11)
    assert both_buffers_equal(a, b)


def test_apply_box_on_device(ts, orc):
    import ctypes
    import torch
    from paper_2303_08365_b200 import _abi
    k = ts.find_benchmark("Heat-3D").kernel
    a = random_grid(ts, orc, [12, 10, 20], [1, 1, 1], 2)
    b = a.copy()
    dg = ts.DeviceGrid(a)
    lo = (ctypes.c_int64 * 3)(3, -2, 4)
    hi = (ctypes.c_int64 * 3)(9, 7, 99)
    L = _abi.lib()
    _abi.check(L.tsr_apply_box(ctypes.byref(k.c_struct()), ctypes.byref(dg.desc),
                               ctypes.byref(dg.layout), dg.ptr(0), dg.ptr(1), lo, hi, None,
                               torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    got = a.copy()
    L.tsr_download(ctypes.byref(dg.desc), ctypes.byref(dg.layout), dg.ptr(1),
                   got.buffer(1).ctypes.data, 1, None)
    n = orc.apply_box(b, k, [3, -2, 4], [9, 7, 99], 0)
    assert n == 6 * 7 * 16
    box = (slice(1 + 3, 1 + 9), slice(1, 1 + 7), slice(1 + 4, 1 + 20))
    assert got.padded(1)[box].tobytes() == b.padded(1)[box].tobytes()


@pytest.mark.slow
def test_config1_full_size_bitwise(ts, orc):
    """BASELINE config 1 at full size: Heat-2D 4096^2 fp64, T=100, seed 1."""
    k = ts.find_benchmark("Heat-2D").kernel
    a = ts.Grid([4096, 4096], [1, 1])
    ts.fill_random(a, 1)
    b = a.copy()
    ts.naive_run(a, k, 100)
    orc.naive_run(b, k, 100)
    assert both_buffers_equal(a, b)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_full_shape_properties(ts, orc, cfg):
    """Full BASELINE shapes: tuned engine == generic engine bitwise (exact), and
    the first steps == the oracle; C4's fp32 fast mode within 1e-5."""
    name, ext, dt, steps, fused = {
        "c2": ("Box-2D9P", [16384, 16384], "f64", 8, 4),
        "c3": ("Heat-3D", [512, 512, 512], "f64", 20, 0),
        "c4": ("Box-3D27P", [512, 512, 512], "f32", 6, 0),
    }[cfg]
    k = ts.find_benchmark(name).kernel
    cls = ts.Grid if dt == "f64" else ts.GridF
    a = cls(ext, [1] * len(ext))
    ts.fill_random(a, 1)
    b = a.copy()
    ts.run_gpu(a, k, steps, fused_steps=fused)
    ts.run_gpu(b, k, steps, engine="generic")
    assert both_buffers_equal(a, b)
    c = cls(ext, [1] * len(ext))
    ts.fill_random(c, 1)
    d = c.copy()
    ts.run_gpu(c, k, 2, fused_steps=fused, mode="exact")
    orc.naive_run(d, k, 2)
    assert both_buffers_equal(c, d)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_full_shape_1024(ts, orc, cfg):
    """C4 (Box-3D27P fp32) and C5 (Heat-3D fp64) at their full 1024^3 shape:
    the tuned engine at its default fused depth == the generic engine bitwise
    for k + 1 steps (EXACT), and 2 steps == the oracle bitwise."""
    import gc
    name, dt = {"c4": ("Box-3D27P", "f32"), "c5": ("Heat-3D", "f64")}[cfg]
    k = ts.find_benchmark(name).kernel
    cls = ts.Grid if dt == "f64" else ts.GridF
    ext = [1024, 1024, 1024]
    a = cls(ext, [1, 1, 1])
    ts.fill_random(a, 1)
    b = a.copy()
    st = ts.run_gpu(a, k, 1, mode="exact")
    kf = st.fused_steps
    ts.run_gpu(a, k, kf + 1, fused_steps=kf, mode="exact")
    ts.run_gpu(b, k, kf + 2, engine="generic", mode="exact")
    assert both_buffers_equal_planes(a, b), f"tuned k={kf} != generic"
    del a, b
    gc.collect()
    ts.release_cache()
    c = cls(ext, [1, 1, 1])
    ts.fill_random(c, 1)
    d = c.copy()
    ts.run_gpu(c, k, 2, mode="exact")
    orc.naive_run(d, k, 2)
    assert both_buffers_equal_planes(c, d)
    ts.release_cache()


@pytest.mark.parametrize("name,extent,fused,dt", [
    ("Heat-3D", [90, 40, 70], 3, "f64"),     # tb3d, several a0 chunks
    ("Heat-3D", [50, 33, 41], 2, "f32"),
    ("Box-3D27P", [60, 30, 50], 1, "f32"),   # box3d
    ("Box-3D27P", [60, 30, 50], 2, "f64"),   # box3d two-level
    ("Box-2D9P", [200, 150], 4, "f64"),     # stream2d: the range is along the rows
    ("Heat-2D", [120, 90], 6, "f32"),
    ("Heat-1D", [5000], 8, "f64"),          # stream1d
])
def test_sweep_range_stores_only_its_planes(ts, orc, name, extent, fused, dt):
    """tsr_sweep_range: planes [lo, hi) of axis 0 hold the k-step result
    bitwise, every other cell of the output buffer is left untouched (NaN
    sentinel), for ranges at the low edge, in the middle, at the high edge."""
    import torch
    k = ts.find_benchmark(name).kernel
    g = random_grid(ts, orc, extent, [k.radius] * k.dims, 11, dt)
    ref = g.copy()
    orc.naive_run(ref, k, fused)
    want = ref.interior_view(ref.parity)
    n0 = extent[0]
    for lo, hi in [(0, 7), (n0 // 3, n0 // 3 + 13), (n0 - 5, n0), (0, n0), (4, 4)]:
        dg = ts.DeviceGrid(g, torch.device("cuda", 0))
        dg.buf[1 - dg.cur].fill_(float("nan"))
        dg.sweep_range(k, lo, hi, fused, fused_steps=fused)
        dg.flip(fused)
        got = g.copy()
        dg.download(got)
        cur = got.interior_view(got.parity)
        assert cur[lo:hi].tobytes() == want[lo:hi].tobytes(), (lo, hi)
        assert np.isnan(cur[:lo]).all() and np.isnan(cur[hi:]).all(), (lo, hi)
    with pytest.raises(ValueError):
        dg.sweep_range(k, 0, n0 + 1, fused, fused_steps=fused)
    with pytest.raises(ValueError):
        dg.sweep_range(k, 0, n0, fused + 1, fused_steps=fused)


@pytest.mark.parametrize("name,extent,fused,dt", [
    ("Heat-3D", [40, 36, 70], 3, "f64"),     # tb3d
    ("Box-3D27P", [30, 30, 50], 1, "f32"),   # box3d
    ("Box-3D27P", [30, 30, 50], 2, "f64"),   # box3d two-level
    ("Box-2D9P", [120, 150], 4, "f64"),     # stream2d
    ("Heat-1D", [300], 4, "f64"),           # stream1d
])
def test_sweep_range_mirror(ts, orc, name, extent, fused, dt):
    """tsr_sweep_range_mirror (the fused halo exchange): the stored planes
    land both in `out` and, shifted by `mirror_planes`, in the mirror buffer
    (here a second buffer on the same device); nothing else of the mirror is
    touched."""
    import torch
    k = ts.find_benchmark(name).kernel
    g = random_grid(ts, orc, extent, [k.radius] * k.dims, 5, dt)
    ref = g.copy()
    orc.naive_run(ref, k, fused)
    want = ref.interior_view(ref.parity)
    n0 = extent[0]
    lo, hi, shift = n0 - 3 * k.radius, n0, -(n0 - 3 * k.radius)  # last planes -> first planes
    dg = ts.DeviceGrid(g, torch.device("cuda", 0))
    mirror = ts.DeviceGrid(g, torch.device("cuda", 0), upload=False)
    mirror.buf[0].fill_(float("nan"))
    dg.sweep_range(k, lo, hi, fused, fused_steps=fused, mirror=mirror.ptr(0), mirror_planes=shift)
    dg.flip(fused)
    got = g.copy()
    dg.download(got)
    assert got.interior_view(got.parity)[lo:hi].tobytes() == want[lo:hi].tobytes()
    m = g.copy()
    mirror.cur, mirror.steps_done = 0, 0
    mirror.download(m)
    mi = m.interior_view(m.parity)
    assert mi[:hi - lo].tobytes() == want[lo:hi].tobytes()
    assert np.isnan(mi[hi - lo:]).all()
    with pytest.raises(ValueError):  # mirror aliasing the output buffer
        dg.sweep_range(k, lo, hi, fused, fused_steps=fused, mirror=dg.ptr(1 - dg.cur))


def test_peer_flags_order_a_stream(ts):
    """tsr_peer_signal / tsr_peer_wait on one stream: the wait kernel passes
    once the word reaches the value (wrap-around compare), and work queued
    behind it runs after it."""
    import ctypes
    import torch
    from paper_2303_08365_b200 import _abi
    L = _abi.lib()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _abi.check(L.tsr_peer_signal(ctypes.c_void_p(flag.data_ptr()), 7, s))
    _abi.check(L.tsr_peer_wait(ctypes.c_void_p(flag.data_ptr()), 7, s))
    _abi.check(L.tsr_peer_wait(ctypes.c_void_p(flag.data_ptr()), 0xfffffff0, s))  # 7 is "after" it
    flag.add_(1)
    torch.cuda.synchronize()
    assert int(flag.item()) == 8
    h, off = _abi.ipc_export(flag.data_ptr())
    assert len(h) == 64 and off >= 0


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_reduced_shape_full_steps(ts, orc, cfg):
    """SURVEY §8(d) parity runs: each BASELINE config's kernel, fused depth
    and dtype on a reduced shape for its FULL step count — exact mode bitwise
    against the oracle; C4's fast mode (its bench mode) within 1e-5 max-rel
    and L2-rel as well."""
    name, ext, dt, steps, fused = {
        "c2": ("Box-2D9P", [300, 260], "f64", 100, 4),
        "c3": ("Heat-3D", [40, 44, 48], "f64", 1000, 3),
        "c4": ("Box-3D27P", [36, 40, 44], "f32", 100, 1),
        "c5": ("Heat-3D", [64, 36, 40], "f64", 100, 3),
    }[cfg]
    k = ts.find_benchmark(name).kernel
    a = random_grid(ts, orc, ext, [1] * len(ext), 1, dt)
    ref = a.copy()
    orc.naive_run(ref, k, steps)
    got = a.copy()
    st = ts.run_gpu(got, k, steps, fused_steps=fused, mode="exact")
    assert st.fused_steps == fused
    assert both_buffers_equal(got, ref)
    if cfg == "c2":  # FAST = separable 9-point sums, several fused depths
        for kf in (1, 4, 7):
            fast = a.copy()
            st = ts.run_gpu(fast, k, steps, fused_steps=kf, mode="fast")
            assert st.fused_steps == kf
            d = ts.deviation(fast, ref)
            assert d["max_rel_deviation"] <= TOL["f64"] and d["l2_rel_err"] <= TOL["f64"], (kf, d)
    if cfg == "c4":  # FAST = separable box sums (uniform weights), one and two levels
        for kf in (1, 2):
            fast = a.copy()
            st = ts.run_gpu(fast, k, steps, fused_steps=kf, mode="fast")
            assert st.fused_steps == kf
            d = ts.deviation(fast, ref)
            assert d["max_rel_deviation"] <= TOL["f32"] and d["l2_rel_err"] <= TOL["f32"], (kf, d)


def test_staged_transfers_halo_and_cache_sizes(ts, orc):
    """tsr_run moves each buffer as one contiguous host-layout block and
    relayouts it on the device: the host halo comes back with its own bytes
    (non-zero Dirichlet values, NaN payload included), and a device cache
    sized by a larger earlier grid serves a smaller one."""
    k = ts.find_benchmark("Heat-3D").kernel
    for extent in ([40, 36, 70], [9, 7, 8], [33, 17, 130]):
        g = random_grid(ts, orc, extent, [2, 1, 3], 5)
        for w in (0, 1):
            p = g.padded(w)
            p[1, :, :] = 0.75  # halo planes / columns next to the interior
            p[:, :, -3] = -2.5
            p[-1, 0, 0] = np.float64("nan")
        ref = g.copy()
        ts.run_gpu(g, k, 5)
        orc.naive_run(ref, k, 5)
        assert both_buffers_equal(g, ref)
        assert all(g.padded(w).tobytes() == ref.padded(w).tobytes() for w in (0, 1))


@pytest.mark.parametrize("name", ["Heat-3D", "Box-2D9P", "Heat-1D", "Box-3D27P"])
def test_naive_run_halo_semantics(ts, orc, name):
    """Two buffers with different halo cells: naive_run (naive.hpp:96-100)
    reads each step's halo from that step's read buffer, so odd and even
    steps see different Dirichlet values.  tsr_run uploads both buffers and
    runs one sweep per step: both buffers bitwise equal to the oracle, for
    odd and even T, parity 0 and 1, and a requested fused depth."""
    k = ts.find_benchmark(name).kernel
    extent = {1: [300], 2: [40, 70], 3: [14, 11, 37]}[k.dims]
    for steps, parity, fused in ((5, 0, 0), (4, 1, 3), (1, 0, 0), (7, 1, 0)):
        g = random_grid(ts, orc, extent, [k.radius] * k.dims, 3)
        for w, val in ((0, 0.5), (1, -1.25)):
            p = g.padded(w)
            sl = tuple([0] + [slice(None)] * (k.dims - 1))
            p[sl] = val  # first halo layer of axis 0 differs between buffers
            p[(Ellipsis, -1)] = 2 * val
        if parity:
            g.flip_parity()
        ref = g.copy()
        st = ts.run_gpu(g, k, steps, fused_steps=fused)
        orc.naive_run(ref, k, steps)
        assert st.fused_steps == 1
        assert g.parity == ref.parity
        assert all(g.padded(w).tobytes() == ref.padded(w).tobytes() for w in (0, 1)), steps


@pytest.mark.parametrize("fused", [2, 3, 4])
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_box27_separable_fast_within_tolerance(ts, orc, dt, fused):
    """box3d FAST mode for the uniform 27-point box: the k-level skewed
    pipeline of separable sums, ragged tiles, chunked a0, a non-zero halo
    plane, within the north star's tolerance of the oracle (max-rel and
    L2-rel)."""
    k = ts.find_benchmark("Box-3D27P").kernel
    for extent in ([40, 37, 70], [21, 64, 131], [9, 10, 11], [70, 45, 150]):
        a = random_grid(ts, orc, extent, [1, 1, 1], 3, dt)
        a.padded(0)[0] = 2.5
        a.padded(1)[0] = 2.5
        b = a.copy()
        st = ts.run_gpu(a, k, 13, fused_steps=fused, mode="fast")
        orc.naive_run(b, k, 13)
        assert st.fused_steps == fused
        d = ts.deviation(a, b)
        assert d["max_rel_deviation"] <= TOL[dt] and d["l2_rel_err"] <= TOL[dt], (extent, d)
        assert halos_equal(a, b)


@pytest.mark.parametrize("name,dt,extent,mode,halo", [
    ("Heat-3D", "f64", [200, 40, 70], "exact", None),
    ("Heat-3D", "f64", [131, 33, 65], "fast", None),
    ("Heat-3D", "f64", [150, 21, 40], "exact", [9, 1, 2]),  # halo wider than a chunk's margin
    ("Box-3D27P", "f32", [150, 37, 130], "fast", None),
    ("Box-3D27P", "f64", [97, 20, 33], "exact", None),
    ("Heat-2D", "f64", [300, 90], "exact", None),
    ("Box-2D9P", "f64", [257, 130], "fast", None),
])
@pytest.mark.parametrize("pinned", [False, True])
def test_chunked_round_trip(ts, orc, monkeypatch, name, dt, extent, mode, halo, pinned):
    """tsr_run's chunked round trip (short runs: chunks of the outermost axis
    advanced on windows widened by T*r planes, uploads, windows and downloads
    overlapped) returns exactly what the whole-grid round trip returns, and
    bitwise the oracle in EXACT mode: odd/even T, T = 1, parity 1, a
    non-zero Dirichlet halo plane, chunk counts down to 3; page-locked host
    buffers (direct DMA) and pageable ones (copies staged through pinned
    slots by host threads)."""
    k = ts.find_benchmark(name).kernel

    def grid(steps, parity):
        g = random_grid(ts, orc, extent, halo or [k.radius] * k.dims, 7, dt)
        if pinned:
            pg = type(g)(g.extent, g.halo, pinned=True)
            for w in (0, 1):
                pg.buffer(w)[:] = g.buffer(w)
            g = pg
        for w in (0, 1):
            g.padded(w)[0] = 0.5
        if parity:
            g.flip_parity()
        return g

    for steps, parity in ((5, 0), (4, 1), (1, 0), (2, 1)):
        g, whole = grid(steps, parity), grid(steps, parity)
        monkeypatch.setenv("TSR_RUN_CHUNKED", "1")
        st = ts.run_gpu(g, k, steps, mode=mode)
        monkeypatch.setenv("TSR_RUN_CHUNKED", "0")
        sw = ts.run_gpu(whole, k, steps, mode=mode)
        assert st.fused_steps == sw.fused_steps and st.point_updates == sw.point_updates
        assert st.d2h_bytes < sw.d2h_bytes  # chunked: interior planes only
        assert g.parity == whole.parity
        assert all(g.padded(w).tobytes() == whole.padded(w).tobytes() for w in (0, 1)), steps
        if mode == "exact":
            ref = grid(steps, parity)
            orc.naive_run(ref, k, steps)
            assert all(ref.padded(w).tobytes() == g.padded(w).tobytes() for w in (0, 1))
