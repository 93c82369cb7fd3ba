"""The reference's scheduler API (proj/tests/test_scheduler.cpp restated) and
the multi-slab runtime behind it (tsr_multi_* / tsr_run_multi).

CPU: planning, cost model, CSV, validation.  GPU (-m gpu): slab runs bitwise
against the oracle and against the reference's own run_heterogeneous; on a
one-GPU box every slab shares cuda:0 (the peer stores become local stores,
the event ordering and plane arithmetic are the same), on a multi-GPU box
the `_devices` helper spreads them."""
import os

import numpy as np
import pytest

from conftest import bench_kernel, random_grid


def sim_profile(ts, kind, spm):
    return ts.WorkerProfile(kind=kind, seconds_per_megastencil=spm, iterations=1)


def sim_worker(ts, kind, spm, device=None):
    return ts.WorkerSpec(kind=kind, simulated_seconds_per_megastencil=spm, device=device)


# ---- planning / cost model (test_scheduler.cpp:36-135) --------------------

def test_profiling_with_the_virtual_clock(ts):
    k = ts.heat_coefficients(0.2)
    a, b = ts.profile_workers(sim_worker(ts, "cpu_like", 2.0), sim_worker(ts, "accel_like", 2.0),
                              k, [32, 32], 2)
    assert abs(a.seconds_per_megastencil - b.seconds_per_megastencil) < 1e-12
    c, d = ts.profile_workers(sim_worker(ts, "cpu_like", 3.0), sim_worker(ts, "accel_like", 1.0),
                              k, [32, 32], 1)
    assert d.megastencils_per_second() / c.megastencils_per_second() == pytest.approx(3.0)
    with pytest.raises(ValueError):
        ts.profile_workers(sim_worker(ts, "cpu_like", 1.0), sim_worker(ts, "accel_like", 1.0), k,
                           [32, 32], 0)


def test_partition_planning_and_quantization(ts):
    p = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0), sim_profile(ts, "accel_like", 1.0),
                          [128, 64], 16, 3, 1)
    assert p.ratio == pytest.approx(0.5) and p.boundary == 64 and p.halo_depth == 3
    assert p.bytes_per_exchange == 3 * 64 * 8 * 2
    p = ts.plan_partition(sim_profile(ts, "cpu_like", 3.0), sim_profile(ts, "accel_like", 1.0),
                          [128, 64], 16, 2, 1)
    assert p.ratio == pytest.approx(0.75) and p.boundary == 96
    assert p.first_worker == "accel_like"
    p = ts.plan_partition(sim_profile(ts, "cpu_like", 3.0), sim_profile(ts, "accel_like", 1.0),
                          [80, 64], 16, 2, 1)
    assert p.boundary == 64  # 0.75*80 = 60 snaps toward the faster side
    last = 0.0
    for speed in (1.0, 1.5, 2.0, 3.0, 5.0):
        p = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0 / speed),
                              sim_profile(ts, "accel_like", 1.0), [160, 32], 16, 2, 1)
        assert p.ratio >= last
        last = p.ratio
        assert abs(p.boundary - p.ratio * 160.0) < 16.0 and p.boundary % 16 == 0
    with pytest.raises(ValueError):
        ts.plan_partition(sim_profile(ts, "cpu_like", 1.0), sim_profile(ts, "accel_like", 1.0),
                          [24, 64], 16, 2, 1)


def test_plan_partition_matches_reference_boundary(ts, ref):
    """Equal-rate plans give the reference's boundary (its run_heterogeneous
    shim plans with two equal simulated workers)."""
    for extent, tile, tb in [([128, 64], 16, 3), ([96, 32], 16, 2), ([80, 24], 16, 2)]:
        g = ts.Grid(extent, [1, 1])
        ts.fill_random(g, 1)
        *_, boundary = ref.run_heterogeneous(g, ts.heat_coefficients(0.2), 0, tile, tb)
        p = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0),
                              sim_profile(ts, "accel_like", 1.0), extent, tile, tb, 1)
        assert p.boundary == boundary


def test_communication_cost_model(ts):
    m = ts.CommCostModel(1000.0, 1.0)
    per, batched = ts.comm_cost(m, 10, 100)
    assert per == pytest.approx(11000.0) and batched == pytest.approx(2000.0)
    per, batched = ts.comm_cost(m, 1, 100)
    assert per == batched
    free = ts.CommCostModel(0.0, 2.0)
    per, batched = ts.comm_cost(free, 7, 11)
    assert per == pytest.approx(batched) == pytest.approx(7.0 * 11.0 * 2.0)
    with pytest.raises(ValueError):
        ts.comm_cost(m, 0, 10)
    rng = np.random.default_rng(8)
    for _ in range(200):
        mm = ts.CommCostModel(rng.random() * 1e-3, rng.random() * 1e-8)
        k = 1 + int(rng.integers(64))
        nb = int(rng.integers(100000))
        per, batched = ts.comm_cost(mm, k, nb)
        assert batched <= per + 1e-18
        if k > 1 and mm.alpha > 0.0:
            assert batched < per


def test_dump_comm_log_csv(ts, tmp_path):
    log = ts.CommLog([ts.CommRecord(0, "w0_to_w1", 1536, 1.1536e-05, 0.0),
                      ts.CommRecord(0, "w1_to_w0", 1536, 1.1536e-05, 2.5e-06)], 192)
    path = tmp_path / "comm.csv"
    ts.dump_comm_log(str(path), log)
    lines = path.read_text().splitlines()
    assert lines[0] == "round,direction,bytes,modeled_cost_alpha_beta,wall_seconds"
    assert lines[1] == "0,w0_to_w1,1536,1.1536e-05,0"
    assert lines[2].startswith("0,w1_to_w0,1536,")
    assert log.messages == 2 and log.rounds_and_bytes()[0] == (0, "w0_to_w1", 1536)
    with pytest.raises(RuntimeError):
        ts.dump_comm_log(str(tmp_path / "no" / "such" / "dir.csv"), log)


def test_run_heterogeneous_validates_like_the_reference(ts):
    """run_heterogeneous_impl's argument checks (scheduler.cpp:445-461) fire
    before any device work."""
    k = ts.heat_coefficients(0.23)
    plan = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0), sim_profile(ts, "accel_like", 1.0),
                             [128, 64], 16, 3, 1)
    g = ts.Grid([128, 64], [1, 1])
    w0, w1 = sim_worker(ts, "cpu_like", 1.0), sim_worker(ts, "accel_like", 1.0)
    with pytest.raises(ValueError, match="negative step count"):
        ts.run_heterogeneous(g, k, -1, plan, w0, w1)
    bad = ts.PartitionPlan(**{**plan.__dict__, "radius": 2})
    with pytest.raises(ValueError, match="radius differs"):
        ts.run_heterogeneous(g, k, 3, bad, w0, w1)
    bad = ts.PartitionPlan(**{**plan.__dict__, "halo_depth": 2})
    with pytest.raises(ValueError, match="radius\\*tb"):
        ts.run_heterogeneous(g, k, 3, bad, w0, w1)
    bad = ts.PartitionPlan(**{**plan.__dict__, "boundary": 128})
    with pytest.raises(ValueError, match="boundary outside"):
        ts.run_heterogeneous(g, k, 3, bad, w0, w1)
    bad = ts.PartitionPlan(**{**plan.__dict__, "boundary": 2})
    with pytest.raises(ValueError, match="smaller than the halo depth"):
        ts.run_heterogeneous(g, k, 3, bad, w0, w1)
    log = ts.run_heterogeneous(g, k, 0, plan, w0, w1)  # T = 0 sends nothing
    assert log.messages == 0


def test_fill_random_skip_is_the_global_stream(ts, orc):
    """fill_random(skip=p*cross) of a slab = the global grid's planes from p."""
    glob = ts.Grid([40, 6, 7], [1, 1, 1])
    ts.fill_random(glob, 77)
    for p0, n in [(0, 40), (5, 12), (17, 23)]:
        loc = ts.Grid([n, 6, 7], [1, 1, 1])
        ts.fill_random(loc, 77, skip=p0 * 6 * 7)
        assert loc.interior_view(0).tobytes() == glob.interior_view(0)[p0:p0 + n].tobytes()
    ora = ts.Grid([40, 6, 7], [1, 1, 1])
    orc.fill_random(ora, 77)
    assert ora.interior_view(1).tobytes() == glob.interior_view(1).tobytes()


# ---- slab runs on the GPU ---------------------------------------------------

def _devices(P):
    import torch
    n = torch.cuda.device_count()
    return [i % n for i in range(P)]


CASES = [  # name, extent, steps, fused (0 = engine default), P
    ("Heat-2D", [128, 64], 6, 3, 2),        # test_scheduler.cpp:137-158's shape
    ("Heat-2D", [97, 33], 11, 4, 3),        # ragged slabs, trailing round
    ("Box-2D9P", [90, 130], 9, 4, 3),       # stream2d Q mode
    ("Heat-3D", [70, 40, 67], 7, 3, 2),     # tb3d
    ("Heat-3D", [20, 24, 40], 8, 3, 4),     # thin slabs (own 5 < 2 * depth 6)
    ("Box-3D27P", [40, 30, 50], 4, 1, 2),   # box3d k=1
    ("Box-3D27P", [44, 30, 50], 5, 2, 2),   # box3d k=2
    ("Heat-1D", [300], 7, 3, 3),            # stream1d, 1-D slabs
    ("star3d_r2", [40, 20, 36], 3, 0, 2),   # generic engine (3-D radius 2)
]


def _kernel(ts, name):
    if name == "star3d_r2":
        return ts.star_kernel(3, 2, 0.4, [0.07, 0.03])
    return bench_kernel(ts, name)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["auto", "copy"])
@pytest.mark.parametrize("name,extent,steps,fused,P", CASES)
def test_run_multi_bitwise_oracle(ts, orc, name, extent, steps, fused, P, transport):
    """tsr_run_multi (exact mode) leaves the grid exactly as naive_run does:
    step T in the read buffer, T-1 in the other, parity flipped T times."""
    k = _kernel(ts, name)
    halo = [k.radius] * k.dims
    g = random_grid(ts, orc, extent, halo, 500)
    ref = g.copy()
    st = ts.run_multi(g, k, steps, P, devices=_devices(P), fused_steps=fused,
                      transport=transport)
    orc.naive_run(ref, k, steps)
    assert g.parity == ref.parity
    for w in (0, 1):
        assert g.buffer(w).tobytes() == ref.buffer(w).tobytes(), (name, w)
    assert st.ngpus == P
    rounds = -(-(steps - 1) // st.fused_steps) + 1  # body rounds + the final 1-step round
    assert st.messages == 2 * (P - 1) * rounds
    depth = k.radius * st.fused_steps
    cross = int(np.prod(extent[1:])) if len(extent) > 1 else 1
    assert st.bytes_exchanged == st.messages * depth * cross * 8


@pytest.mark.gpu
@pytest.mark.parametrize("name,extent,steps,P", [("Heat-3D", [64, 20, 40], 9, 3),
                                                  ("Heat-2D", [100, 40], 10, 4),
                                                  ("Box-3D27P", [40, 18, 34], 4, 2)])
def test_run_multi_fast_and_fp32(ts, orc, name, extent, steps, P):
    """FAST mode within 1e-12 (fp64) and fp32 exact mode bitwise."""
    k = bench_kernel(ts, name)
    halo = [k.radius] * k.dims
    g = random_grid(ts, orc, extent, halo, 501)
    ref = g.copy()
    ts.run_multi(g, k, steps, P, devices=_devices(P), mode="fast")
    orc.naive_run(ref, k, steps)
    assert orc.deviation(g, ref)["max_rel_deviation"] <= 1e-12
    gf = random_grid(ts, orc, extent, halo, 502, dtype="f32")
    rf = gf.copy()
    ts.run_multi(gf, k, steps, P, devices=_devices(P))
    orc.naive_run(rf, k, steps)
    assert bitwise(gf, rf)


def bitwise(a, b):
    return a.interior_view(a.parity).tobytes() == b.interior_view(b.parity).tobytes()


@pytest.mark.gpu
def test_run_heterogeneous_equals_oracle_and_reference_log(ts, orc, ref):
    """test_scheduler.cpp:137-158: 128x64 Heat-2D, tb=3, 6 steps: bitwise the
    oracle, 4 messages of 3*64*8 bytes, ghost tally 2*2*(2+1)*64 -- the same
    log the reference's own run_heterogeneous writes."""
    k = ts.heat_coefficients(0.23)
    extent = [128, 64]
    plan = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0), sim_profile(ts, "accel_like", 1.0),
                             extent, 16, 3, 1)
    assert plan.boundary == 64
    g = random_grid(ts, orc, extent, [1, 1], 500)
    want = g.copy()
    mine = g.copy()
    log = ts.run_heterogeneous(g, k, 6, plan, sim_worker(ts, "cpu_like", 1.0, _devices(2)[0]),
                               sim_worker(ts, "accel_like", 1.0, _devices(2)[1]))
    orc.naive_run(want, k, 6)
    assert bitwise(g, want)
    assert log.messages == 4
    assert all(r.bytes == 3 * 64 * 8 and r.modeled_cost_alpha_beta > 0 for r in log.records)
    assert sorted(r.direction for r in log.records) == ["w0_to_w1"] * 2 + ["w1_to_w0"] * 2
    assert log.ghost_recompute_points == 2 * 2 * (2 + 1) * 64
    msgs, ghost, first_bytes, boundary = ref.run_heterogeneous(mine, k, 6, 16, 3)
    assert (msgs, ghost, first_bytes, boundary) == (log.messages, log.ghost_recompute_points,
                                                    log.records[0].bytes, plan.boundary)
    assert bitwise(g, mine)  # the reference's own partitioned run, same bits


@pytest.mark.gpu
@pytest.mark.parametrize("tb", [1, 2, 3])
def test_deep_halo_sufficiency_poisoned(ts, orc, tb):
    """test_scheduler.cpp:208-228: NaN beyond the exchanged ghosts is never read."""
    k = ts.heat_coefficients(0.24)
    extent = [64, 32]
    plan = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0), sim_profile(ts, "accel_like", 1.0),
                             extent, 16, tb, 1)
    g = random_grid(ts, orc, extent, [1, 1], 504)
    want = g.copy()
    ts.run_heterogeneous_instrumented(g, k, 7, plan, sim_worker(ts, "cpu_like", 1.0),
                                      sim_worker(ts, "accel_like", 1.0))
    orc.naive_run(want, k, 7)
    assert np.isfinite(g.interior_view(g.parity)).all()
    assert bitwise(g, want)


@pytest.mark.gpu
def test_message_schedule_across_tb(ts, orc):
    """test_scheduler.cpp:174-191: 2*ceil(T/tb) messages, same physics."""
    k = ts.heat_coefficients(0.22)
    extent = [96, 32]
    want = random_grid(ts, orc, extent, [1, 1], 502)
    orc.naive_run(want, k, 4)
    for tb in (1, 2):
        plan = ts.plan_partition(sim_profile(ts, "cpu_like", 1.0),
                                 sim_profile(ts, "accel_like", 1.0), extent, 16, tb, 1)
        g = random_grid(ts, orc, extent, [1, 1], 502)
        log = ts.run_heterogeneous(g, k, 4, plan, sim_worker(ts, "cpu_like", 1.0),
                                   sim_worker(ts, "accel_like", 1.0), threaded=False)
        assert log.messages == 2 * ((4 + tb - 1) // tb)
        assert bitwise(g, want)


@pytest.mark.gpu
def test_slab_grid_fill_checksums_and_download(ts, orc):
    """SlabGrid.fill_random is fill_random of the global grid; after T steps
    every owned plane's checksum equals the one-device DeviceGrid's, and the
    downloaded grid is bitwise the oracle's."""
    import torch
    k = bench_kernel(ts, "Heat-3D")
    extent, P, steps = [72, 30, 44], 3, 7
    host = ts.Grid(extent, [1, 1, 1])
    ts.fill_random(host, 9)
    want = host.copy()
    with ts.SlabGrid(k, extent, ngpus=P, devices=_devices(P), fused_steps=3) as sg:
        sg.fill_random(9)
        sg.set_logging(True)
        st = sg.advance(steps, keep_previous=True)
        recs = sg.comm_records()
        assert len(recs) == st.messages and all(r.wall_seconds >= 0 for r in recs)
        dg = ts.DeviceGrid(host, torch.device("cuda", 0))
        dg.advance(k, steps, fused_steps=3, keep_previous=True)
        torch.cuda.synchronize()
        assert np.array_equal(sg.plane_checksums(0), dg.plane_checksums(0))
        assert np.array_equal(sg.plane_checksums(1), dg.plane_checksums(1))
        got = ts.Grid(extent, [1, 1, 1])
        sg.download(got)
        info = [sg.slab(i) for i in range(P)]
    assert [s.own_lo for s in info] == [0, 24, 48] and info[1].ghost_lo == 3
    orc.naive_run(want, k, steps)
    assert got.parity == want.parity
    for w in (0, 1):
        assert got.interior_view(w).tobytes() == want.interior_view(w).tobytes()


@pytest.mark.gpu
def test_run_gpu_ngpus_and_errors(ts, orc):
    """tsr_run with opts.ngpus routes to the slab runtime; a slab thinner than
    the halo depth is the reference's invalid_argument."""
    k = bench_kernel(ts, "Heat-3D")
    g = random_grid(ts, orc, [40, 16, 24], [1, 1, 1], 3)
    want = g.copy()
    st = ts.run_gpu(g, k, 5, ngpus=2, fused_steps=2)
    orc.naive_run(want, k, 5)
    assert st.ngpus == 2 and bitwise(g, want)
    with pytest.raises(ValueError, match="smaller than the halo depth"):
        ts.run_multi(random_grid(ts, orc, [8, 16, 24], [1, 1, 1], 3), k, 4, 4,
                     devices=_devices(4), fused_steps=3)
    with pytest.raises(ValueError, match="boundary outside"):
        ts.run_multi(g, k, 2, 2, devices=_devices(2), boundaries=[40])


@pytest.mark.gpu
def test_round_timeline_shows_concurrent_seam_and_interior(ts):
    """Per round and slab the runtime logs the seam passes' interval (seam
    stream) and the interior pass's (second stream); the interior pass of a
    round is issued without waiting for that round's seam passes, so the
    two intervals of a slab overlap in time."""
    k = ts.find_benchmark("Heat-3D").kernel
    with ts.SlabGrid(k, [192, 64, 64], ngpus=2, devices=_devices(2), fused_steps=3,
                     mode="fast") as sg:
        sg.fill_random(1)
        sg.set_logging(True)
        st = sg.advance(18)
        tl = sg.round_timeline()
    assert len(tl) == 2 * 6 and st.rounds == 6
    for e in tl:
        assert e["seam"][0] <= e["seam"][1] and e["interior"][0] <= e["interior"][1]
    assert any(min(e["seam"][1], e["interior"][1]) > max(e["seam"][0], e["interior"][0])
               for e in tl)


@pytest.mark.gpu
@pytest.mark.parametrize("name,extent,dt,fused,P", [
    ("Box-3D27P", [60, 30, 70], "f32", 2, 2),   # C4's bench path: separable k-level pipeline
    ("Box-3D27P", [61, 30, 70], "f32", 3, 3),
    ("Box-2D9P", [130, 150], "f64", 4, 3),      # stream2d separable mode
    ("Heat-3D", [70, 40, 66], "f64", 3, 4),
    # several tiles per axis and several segments per CTA: step tiers differ
    # between the slab and one-device runs, the bits may not (a contracted
    # FMA in one tier once made them differ)
    ("Box-3D27P", [40, 256, 1024], "f32", 3, 2),
    ("Box-2D9P", [700, 2000], "f64", 4, 3),
])
def test_slabs_fast_equal_one_device_fast(ts, orc, name, extent, dt, fused, P):
    """FAST-mode slab runs (seam passes with mirror stores + interior
    ranges) are bitwise the same FAST run on one device: every engine's range
    and mirror path computes each point exactly as its full pass does."""
    k = bench_kernel(ts, name)
    g = random_grid(ts, orc, extent, [1] * k.dims, 77, dt)
    one = g.copy()
    ts.run_multi(g, k, 11, P, devices=_devices(P), fused_steps=fused, mode="fast")
    ts.run_gpu(one, k, 11, fused_steps=fused, mode="fast")
    assert g.parity == one.parity
    for w in (0, 1):
        assert g.interior_view(w).tobytes() == one.interior_view(w).tobytes(), w


@pytest.mark.gpu
def test_run_multi_differing_halos(ts, orc):
    """Two buffers with different halo cells: tsr_run_multi honours naive_run's
    per-step halo (each step reads its read buffer's halo) by running on one
    device, one sweep per step; both buffers bitwise the oracle's."""
    k = _kernel(ts, "Heat-3D")
    g = random_grid(ts, orc, [48, 20, 40], [1, 1, 1], 503)
    g.padded(0)[0] = 0.5
    g.padded(1)[0] = -0.75
    ref = g.copy()
    st = ts.run_multi(g, k, 7, 2, devices=_devices(2))
    orc.naive_run(ref, k, 7)
    assert st.fused_steps == 1 and g.parity == ref.parity
    for w in (0, 1):
        assert g.buffer(w).tobytes() == ref.buffer(w).tobytes(), w


@pytest.mark.gpu
@pytest.mark.parametrize("name,extent,P", [("Heat-3D", [150, 20, 40], 2),
                                           ("Heat-3D", [200, 18, 33], 3),
                                           ("Box-2D9P", [300, 70], 2)])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("per_slab", [False, True])
def test_run_multi_split_round_trip(ts, orc, monkeypatch, name, extent, P, pinned, per_slab):
    """Short runs of tsr_run_multi take the split round trip: every slab's
    planes come from the chunked round trip on its device, the windows
    reading the planes beyond the slab from the host buffers (no exchange),
    after every range's margin planes are up (the barrier; per_slab runs one
    range per slab, each with its own buffers, so the barrier spans several
    ranges on one device).  Both buffers bitwise the oracle's and the slab
    runtime's, odd and even T."""
    k = _kernel(ts, name)
    halo = [k.radius] * k.dims
    monkeypatch.setenv("TSR_RUN_CHUNKED", "1")
    if per_slab:
        monkeypatch.setenv("TSR_SPLIT_PER_SLAB", "1")
    for steps in (5, 4):
        src = random_grid(ts, orc, extent, halo, 504)
        g = src
        if pinned:
            g = ts.Grid(extent, halo, pinned=True)
            for w in (0, 1):
                g.buffer(w)[:] = src.buffer(w)
        ref, slab = src.copy(), src.copy()
        st = ts.run_multi(g, k, steps, P, devices=_devices(P))
        orc.naive_run(ref, k, steps)
        assert st.ngpus == P and st.messages == 0  # no exchange: replicated ghost zones
        assert st.ghost_recompute_points > 0  # the windows' margins, swept twice
        assert st.point_updates == int(np.prod(extent)) * steps
        assert g.parity == ref.parity
        for w in (0, 1):
            assert g.buffer(w).tobytes() == ref.buffer(w).tobytes(), (name, steps, w)
        monkeypatch.setenv("TSR_MULTI_SPLIT", "0")
        st2 = ts.run_multi(slab, k, steps, P, devices=_devices(P))
        monkeypatch.delenv("TSR_MULTI_SPLIT")
        assert st2.messages > 0
        for w in (0, 1):
            assert slab.buffer(w).tobytes() == g.buffer(w).tobytes()
