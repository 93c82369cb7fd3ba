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


@pytest.mark.gpu
def test_small_study_matches_oracle(ts, orc, tmp_path):
    from paper_2303_08365_b200.case_study import (CaseStudyConfig, _init, case_study_heat,
                                                  compare_precision)
    cfg = CaseStudyConfig(extent=96, steps=300, checkpoints=[100, 300], sample_every=50)
    res = case_study_heat(cfg, str(tmp_path))
    k = ts.heat_coefficients(cfg.mu)
    g64, g32 = ts.Grid([96, 96], [1, 1]), ts.GridF([96, 96], [1, 1])
    _init(g64, cfg, 96 / 8.0)
    _init(g32, cfg, 96 / 8.0)
    centers, tables = [g64.at(48, 48)], []
    for done in range(50, 301, 50):
        orc.naive_run(g64, k, 50)
        orc.naive_run(g32, k, 50)
        centers.append(g64.at(48, 48))
        if done in (100, 300):
            tables.append(compare_precision(g64, g32))
    assert res["series_steps"] == list(range(0, 301, 50))
    assert res["center_series"] == [float(c) for c in centers]  # bitwise
    assert res["checkpoint_steps"] == [100, 300]
    for got, want in zip(res["checkpoint_errors"], tables):
        assert got.abs_exceed_pct == want.abs_exceed_pct
        assert got.rel_exceed_pct == want.rel_exceed_pct
    final = ts.load_grid(str(tmp_path / "final.ttrs"))
    assert final.to_numpy().tobytes() == g64.to_numpy().tobytes()
    assert (tmp_path / "center_series.csv").read_text().startswith("step,center_celsius")
