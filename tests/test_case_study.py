"""Thermal-diffusion case study (proj/src/case_study.cpp:171-290) on the GPU
path: centre series, precision tables and artifacts against the oracle."""
import numpy as np
import pytest


def test_compare_precision_thresholds(ts):
    """case_study.cpp:21-47 semantics: strict '>' against each threshold,
    relative deviation floored at 1e-12."""
    from paper_2303_08365_b200.case_study import compare_precision
    a = ts.grid_from_numpy(np.full((4, 5), 50.0))
    b = ts.grid_from_numpy(np.full((4, 5), 50.0), dtype=np.float32)
    t = compare_precision(a, b)
    assert t.abs_exceed_pct == [0.0, 0.0, 0.0] and t.rel_exceed_pct == [0.0, 0.0, 0.0]
    b.buffer(0)[b.flat(1, 1)] = 50.7   # |d| = 0.7 -> > 0.1, > 0.5 ; rel 1.4% -> > 1%
    b.buffer(0)[b.flat(2, 2)] = 52.0   # |d| = 2.0 -> all abs ; rel 4% -> > 1%, > 3%
    t = compare_precision(a, b)
    assert t.abs_exceed_pct == pytest.approx([10.0, 10.0, 5.0])
    assert t.rel_exceed_pct == pytest.approx([10.0, 5.0, 0.0])
    with pytest.raises(ValueError):
        compare_precision(a, ts.grid_from_numpy(np.zeros((4, 4))))


def test_config_validation(ts):
    from paper_2303_08365_b200.case_study import (CaseStudyConfig, apply_full_scale,
                                                  case_study_heat)
    cfg = CaseStudyConfig()
    apply_full_scale(cfg)
    assert (cfg.extent, cfg.steps, cfg.checkpoints) == (9600, 3_800_000, [1_000_000, 2_000_000, 3_800_000])
    with pytest.raises(ValueError):
        case_study_heat(CaseStudyConfig(extent=8))
    with pytest.raises(ValueError):
        case_study_heat(CaseStudyConfig(steps=100, checkpoints=[101]))
    with pytest.raises(ValueError):
        case_study_heat(CaseStudyConfig(steps=100, checkpoints=[30], sample_every=25))


def test_initial_plate_is_the_references(ts, ref, tmp_path):
    """The initial field (case_study.cpp:193-207, std::exp in double) is
    bit-identical to the reference's: its case_study_heat with 0 steps dumps
    the untouched plate as final.ttrs."""
    from paper_2303_08365_b200.case_study import CaseStudyConfig, _init
    for n, sigma in [(96, 0.0), (101, 7.5)]:
        out = tmp_path / f"ref{n}"
        ref.case_study_heat(str(out), n, 0, [], 25, sigma=sigma)
        g = ts.Grid([n, n], [1, 1])
        _init(g, CaseStudyConfig(extent=n), sigma if sigma > 0 else n / 8.0)
        ts.dump_grid(str(tmp_path / f"ours{n}.ttrs"), g)
        assert (tmp_path / f"ours{n}.ttrs").read_bytes() == (out / "final.ttrs").read_bytes()
        assert g.buffer(0).tobytes() == g.buffer(1).tobytes()
        f = ts.GridF([n, n], [1, 1])
        _init(f, CaseStudyConfig(extent=n), sigma if sigma > 0 else n / 8.0)
        assert f.buffer(0).tobytes() == g.buffer(0).astype(np.float32).tobytes()


def _check_against_reference(ts, ref, cfg, tmp_path, threads=1):
    from paper_2303_08365_b200.case_study import case_study_heat
    res = case_study_heat(cfg, str(tmp_path / "ours"))
    want = ref.case_study_heat(str(tmp_path / "ref"), cfg.extent, cfg.steps, cfg.checkpoints,
                               cfg.sample_every, mu=cfg.mu, path="tessellate", threads=threads)
    assert res["series_steps"] == want["series_steps"]
    assert res["center_series"] == want["center_series"]  # bitwise
    assert res["final_center"] == want["final_center"]
    assert res["checkpoint_steps"] == want["checkpoint_steps"]
    for got, (wa, wr) in zip(res["checkpoint_errors"], want["checkpoint_errors"]):
        assert got.abs_exceed_pct == wa and got.rel_exceed_pct == wr
    ours, theirs = tmp_path / "ours", tmp_path / "ref"
    assert (ours / "final.ttrs").read_bytes() == (theirs / "final.ttrs").read_bytes()
    for name in ("center_series.csv", "error_table.csv"):
        assert (ours / name).read_text() == (theirs / name).read_text(), name
    return res


@pytest.mark.gpu
def test_small_study_matches_reference(ts, ref, tmp_path):
    """case_study_heat on the GPU against the reference's own case_study_heat
    (tessellate path): centre series, exceedance tables, final.ttrs and the
    two CSVs, all identical."""
    from paper_2303_08365_b200.case_study import CaseStudyConfig
    cfg = CaseStudyConfig(extent=96, steps=300, checkpoints=[100, 300], sample_every=50)
    _check_against_reference(ts, ref, cfg, tmp_path)
    # final step off the checkpoint list: final.ttrs is still written
    cfg = CaseStudyConfig(extent=64, steps=130, checkpoints=[50], sample_every=25)
    _check_against_reference(ts, ref, cfg, tmp_path / "b")


@pytest.mark.gpu
@pytest.mark.slow
def test_desk_scale_study_matches_reference(ts, ref, tmp_path):
    """The reference's default desk-scale study (480 x 480, 9500 steps,
    checkpoints 1000/5000/9500), identical end to end."""
    import os
    from paper_2303_08365_b200.case_study import CaseStudyConfig
    res = _check_against_reference(ts, ref, CaseStudyConfig(), tmp_path,
                                   threads=os.cpu_count() or 1)
    assert len(res["center_series"]) == 9500 // 25 + 1


@pytest.mark.gpu
def test_snapshot_and_resume_reproduce_the_run(ts, tmp_path):
    """TTRS snapshots of the device fields every 150 steps; resuming from the
    step-150 snapshots reproduces the rest of the uninterrupted run exactly:
    centre series, checkpoint table and final.ttrs (grid_io.cpp:34-68)."""
    import shutil
    from paper_2303_08365_b200.case_study import CaseStudyConfig, case_study_heat
    cfg = CaseStudyConfig(extent=96, steps=300, checkpoints=[100, 300], sample_every=50,
                          snapshot_every=150)
    full = case_study_heat(cfg, str(tmp_path / "full"))
    assert (tmp_path / "full" / "snapshot_150_fp64.ttrs").exists()
    (tmp_path / "resumed").mkdir()
    for name in ("snapshot_150_fp64.ttrs", "snapshot_150_fp32.ttrs"):
        shutil.copy(tmp_path / "full" / name, tmp_path / "resumed" / name)
    part = case_study_heat(cfg, str(tmp_path / "resumed"), resume_step=150)
    k = full["series_steps"].index(150)
    assert part["series_steps"] == full["series_steps"][k:]
    assert part["center_series"] == full["center_series"][k:]
    assert part["checkpoint_steps"] == [300]
    got, want = part["checkpoint_errors"][0], full["checkpoint_errors"][-1]
    assert got.abs_exceed_pct == want.abs_exceed_pct and got.rel_exceed_pct == want.rel_exceed_pct
    assert ((tmp_path / "resumed" / "final.ttrs").read_bytes() ==
            (tmp_path / "full" / "final.ttrs").read_bytes())
    # a snapshot is the device state itself: resuming it and snapshotting again is identity
    dg = ts.DeviceGrid.resume(str(tmp_path / "full" / "snapshot_300_fp32.ttrs"), dtype="f32")
    dg.snapshot(str(tmp_path / "again.ttrs"))
    assert ((tmp_path / "again.ttrs").read_bytes() ==
            (tmp_path / "full" / "snapshot_300_fp32.ttrs").read_bytes())
