"""The operator CLI (proj/tools/bench.cpp:71-129 rebuilt on argparse) and the
case-study config parser (proj/src/case_study.cpp:74-116)."""
import io

import pytest


def test_list_matches_benchmark_table(ts):
    from paper_2303_08365_b200.cli import main
    out = io.StringIO()
    assert main(["list"], out) == 0
    lines = out.getvalue().splitlines()
    assert lines[0].split() == ["name", "pts", "radius", "extent", "T", "blocking"]
    assert len(lines) == 1 + len(ts.benchmark_table())
    # bench.cpp:69-81 rows: Heat-3D is 7 taps, radius 1, 1024^3, T=1000, 20^3 x 10
    row = next(l for l in lines if l.startswith("Heat-3D")).split()
    assert row == ["Heat-3D", "7", "1", "1024x1024x1024", "1000", "20x20x20x10"]


def test_errors_exit_1(capsys):
    from paper_2303_08365_b200.cli import main
    assert main(["run", "--name", "No-Such"], io.StringIO()) == 1
    assert "error:" in capsys.readouterr().err
    assert main(["run", "--path", "warp"], io.StringIO()) == 1
    with pytest.raises(SystemExit):
        main(["run", "--scale", "huge"], io.StringIO())


def test_cpu_only_paths_report_unsupported(ts):
    """vector/mm are the reference's CPU simulators: rows say so."""
    from paper_2303_08365_b200.cli import main
    out = io.StringIO()
    assert main(["run", "--name", "Heat-2D,Heat-3D", "--path", "mm"], out) == 0
    rows = out.getvalue().splitlines()
    assert len(rows) == 3 and all(",unsupported," in r for r in rows[1:])


def test_parse_case_config(tmp_path):
    from paper_2303_08365_b200.case_study import parse_case_config
    p = tmp_path / "c.cfg"
    p.write_text("# plate\nextent = 96  # cells\nsteps=300\ncheckpoints = 100, 300\n"
                 "sample_every = 50\nmu = 0.2\npath = tessellate\nthreads = 4\n")
    cfg = parse_case_config(str(p))
    assert (cfg.extent, cfg.steps, cfg.checkpoints, cfg.sample_every, cfg.mu) == \
        (96, 300, [100, 300], 50, 0.2)
    p.write_text("full = true\n")
    cfg = parse_case_config(str(p))
    assert (cfg.extent, cfg.steps, cfg.checkpoints) == \
        (9600, 3_800_000, [1_000_000, 2_000_000, 3_800_000])
    p.write_text("extent 96\n")
    with pytest.raises(RuntimeError, match="line 1: expected key = value"):
        parse_case_config(str(p))
    p.write_text("\nwidth = 3\n")
    with pytest.raises(RuntimeError, match="line 2: unknown key 'width'"):
        parse_case_config(str(p))
    p.write_text("mu = 0.3\n")  # unstable CFL number (kernel.cpp:118-128)
    with pytest.raises(ValueError):
        parse_case_config(str(p))
    with pytest.raises(RuntimeError, match="cannot open config"):
        parse_case_config(str(tmp_path / "missing.cfg"))


@pytest.mark.gpu
def test_run_rows_verify_on_gpu(ts, tmp_path):
    from paper_2303_08365_b200.cli import main
    out = io.StringIO()
    rep = tmp_path / "r.csv"
    assert main(["run", "--name", "Heat-2D,Heat-3D,Box-3D27P", "--steps", "12",
                 "--out", str(rep)], out) == 0
    rows = out.getvalue().splitlines()
    assert len(rows) == 4 and all(",pass," in r for r in rows[1:])
    assert rep.read_text().splitlines() == rows


@pytest.mark.gpu
def test_case_study_cli(ts, tmp_path):
    from paper_2303_08365_b200.cli import main
    cfgf = tmp_path / "c.cfg"
    cfgf.write_text("extent = 64\nsteps = 200\ncheckpoints = 100, 200\nsample_every = 50\n")
    out = io.StringIO()
    assert main(["case-study", "--config", str(cfgf), "--out", str(tmp_path / "o")], out) == 0
    text = out.getvalue()
    assert text.startswith("final center temperature: ")
    assert "T=100  abs>0.1C:" in text and "T=200  abs>0.1C:" in text
    assert (tmp_path / "o" / "final.ttrs").exists()
